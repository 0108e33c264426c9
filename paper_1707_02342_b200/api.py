"""Host-side mirror of the reference controller API over the C ABI.

The reference (C++, /root/reference/proj) exposes its hot path as free
functions over a value-type ``ControllerState`` plus a ``RolloutSystem``
callback triple (proj/include/mppi/controller.hpp:18-90).  Here the state and
the data-described system live on the device behind one handle; the names,
argument meaning and error behaviour follow the reference:

=============================  =============================================
reference                      here
=============================  =============================================
``make_controller_state``      ``Controller(...)`` (controller.cpp:37-53)
``make_vehicle_system``        ``Controller.set_mlp`` / ``set_costmap``
``sample_perturbations``       ``Controller.sample_perturbations`` (sampler.cpp:5-39)
``rollout_batch``              ``Controller.rollout_batch`` (controller.cpp:55-109)
``compute_weights``/``it_weights``  ``Controller.compute_weights`` (weights.cpp:8-25)
``update_plan``                ``Controller.update_plan`` (controller.cpp:118-131)
``mpc_step``                   ``Controller.mpc_step`` (controller.cpp:133-148)
``optimize_to_convergence``    ``Controller.optimize_to_convergence`` (controller.cpp:150-164)
``sg_coefficients``            ``sg_coefficients`` (smoothing.cpp:5-33)
=============================  =============================================

``std::invalid_argument`` surfaces as :class:`InvalidArgument` (a
``ValueError``), ``std::runtime_error`` as ``RuntimeError``.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (DeviceError, DomainError, InvalidArgument, MppiError, NonFiniteCost, Unsupported, check, dptr)

__all__ = [
    "SamplingParams", "ControlBounds", "CostParams", "SGFilter", "WeightResult", "MlpWeights",
    "CostMap", "Controller", "sg_coefficients", "device_count", "fp32_peak_tflops",
    "MppiError", "InvalidArgument", "NonFiniteCost", "DeviceError", "Unsupported",
]


@dataclass
class SamplingParams:
    """SamplingParams (types.hpp:92-123).  ``sigma_diag`` holds variances."""
    samples: int = 1200
    horizon_steps: int = 80
    dt: float = 0.025
    sigma_diag: Sequence[float] = (0.0306, 0.0506)
    lambda_: float = 12.5
    gamma: float = 0.1
    explore_fraction: float = 0.01
    seed: int = 0


@dataclass
class ControlBounds:
    """ControlBounds (dynamics.hpp:12-29); default [-1, 1]^2."""
    lower: Sequence[float] = (-1.0, -1.0)
    upper: Sequence[float] = (1.0, 1.0)


@dataclass
class CostParams:
    """CostParams (costs.hpp:46-64) + the BASELINE crash term (mppi_gpu.h)."""
    alpha_track: float = 100.0
    alpha_speed: float = 4.25
    alpha_stab: float = 10.0
    v_des: float = 6.0
    impulse: float = 10000.0
    decay: float = 0.9
    boundary_threshold: float = 0.99
    slip_limit: float = 0.75
    crash_penalty: float = 0.0
    crash_threshold: float = 1.0
    roll_limit: float = math.inf

    @staticmethod
    def baseline() -> "CostParams":
        """BASELINE.json cost: 200 h + (v_x - 6)^2 + 10000 [h > 1 or |roll| > 0.6]."""
        return CostParams(alpha_track=200.0, alpha_speed=1.0, alpha_stab=0.0, v_des=6.0,
                          impulse=0.0, decay=1.0, boundary_threshold=1.0, slip_limit=0.75,
                          crash_penalty=10000.0, crash_threshold=1.0, roll_limit=0.6)


@dataclass
class SGFilter:
    """SGFilter (smoothing.hpp:9-13)."""
    window: int = 9
    degree: int = 3


@dataclass
class WeightResult:
    """WeightResult (weights.hpp:9-17)."""
    weights: np.ndarray
    rho: float
    normalizer: float


@dataclass
class MlpWeights:
    """MlpWeights (dynamics.hpp:110-119), row-major, H in {32, 64}."""
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    w3: np.ndarray
    b3: np.ndarray

    @property
    def hidden(self) -> int:
        return int(self.b1.shape[0])

    @staticmethod
    def zeros(hidden: int = 32) -> "MlpWeights":
        H = hidden
        return MlpWeights(np.zeros((H, 6)), np.zeros(H), np.zeros((H, H)), np.zeros(H),
                          np.zeros((4, H)), np.zeros(4))

    @staticmethod
    def xavier(hidden: int = 32, seed: int = 0, out_scale: float = 0.1) -> "MlpWeights":
        """Seeded Xavier-uniform weights, output layer scaled (BASELINE configs)."""
        w = MlpWeights.zeros(hidden)
        check(_lib.load().mppi_workload_mlp_xavier(
            hidden, seed, out_scale, dptr(w.w1), dptr(w.b1), dptr(w.w2), dptr(w.b2), dptr(w.w3), dptr(w.b3)))
        return w

    def save(self, path: str) -> None:
        """save_mlp text format (dynamics.cpp:297-307), header ``6 H H 4``."""
        H = self.hidden
        with open(path, "w") as f:
            f.write(f"6 {H} {H} 4\n")
            for m in (self.w1, self.b1.reshape(-1, 1), self.w2, self.b2.reshape(-1, 1), self.w3,
                      self.b3.reshape(-1, 1)):
                for row in np.atleast_2d(m):
                    f.write(" ".join(repr(float(v)) for v in row) + "\n")

    @staticmethod
    def load(path: str, allowed_hidden: Sequence[int] = (32, 64)) -> "MlpWeights":
        """load_mlp (dynamics.cpp:276-295); the reference accepts only 6 32 32 4."""
        try:
            with open(path) as f:
                tok = f.read().split()
        except OSError as e:
            raise RuntimeError(f"cannot open file: {path}") from e
        if len(tok) < 4:
            raise RuntimeError("load_mlp: missing layer-size header")
        sizes = [int(t) for t in tok[:4]]
        if sizes[0] != 6 or sizes[3] != 4 or sizes[1] != sizes[2] or sizes[1] not in allowed_hidden:
            raise RuntimeError("load_mlp: layer sizes must be 6 H H 4 with H in %s" % (list(allowed_hidden),))
        H = sizes[1]
        vals = np.array([float(t) for t in tok[4:]])
        n = [H * 6, H, H * H, H, 4 * H, 4]
        if vals.size < sum(n):
            raise RuntimeError("load_mlp: truncated weights")
        parts, o = [], 0
        for c in n:
            parts.append(vals[o:o + c])
            o += c
        return MlpWeights(parts[0].reshape(H, 6), parts[1], parts[2].reshape(H, H), parts[3],
                          parts[4].reshape(4, H), parts[5])


@dataclass
class CostMap:
    """CostMap (costs.hpp:11-38): row-major values[iy, ix], (x0, y0) = centre of cell (0, 0)."""
    values: np.ndarray
    x0: float = 0.0
    y0: float = 0.0
    resolution: float = 1.0

    @property
    def width(self) -> int:
        return int(self.values.shape[1])

    @property
    def height(self) -> int:
        return int(self.values.shape[0])

    @staticmethod
    def ellipse(width: int = 2000, height: int = 2000, x0: float = -50.0, y0: float = -50.0,
                resolution: float = 0.05, semi_a: float = 40.0, semi_b: float = 25.0,
                half_width: float = 3.0) -> "CostMap":
        """BASELINE track: min(|distance to the centreline ellipse| / half_width, 2.5)."""
        v = np.zeros((height, width), dtype=np.float32)
        check(_lib.load().mppi_workload_ellipse_costmap(
            width, height, x0, y0, resolution, semi_a, semi_b, half_width,
            v.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
        return CostMap(v, x0, y0, resolution)

    def save(self, path: str) -> None:
        """save_costmap text format (costs.cpp:140-151)."""
        with open(path, "w") as f:
            f.write(f"{self.width} {self.height} {self.x0!r} {self.y0!r} {self.resolution!r}\n")
            for row in self.values:
                f.write(" ".join(repr(float(v)) for v in row) + "\n")

    @staticmethod
    def load(path: str) -> "CostMap":
        """load_costmap (costs.cpp:118-138)."""
        try:
            with open(path) as f:
                tok = f.read().split()
        except OSError as e:
            raise RuntimeError(f"cannot open map file: {path}") from e
        if len(tok) < 5:
            raise RuntimeError(f"map file: bad header in {path}")
        w, h = int(tok[0]), int(tok[1])
        if w < 2 or h < 2:
            raise RuntimeError(f"map file: grid must be at least 2x2 in {path}")
        vals = np.array([float(t) for t in tok[5:5 + w * h]])
        if vals.size != w * h:
            raise RuntimeError(f"map file: truncated grid in {path}")
        v = vals.reshape(h, w)
        if not np.all(np.isfinite(v)) or np.any(np.abs(v) > 2.5):
            raise InvalidArgument(_lib.MPPI_ERR_INVALID_ARGUMENT, "CostMap: values must be finite and within +-2.5")
        return CostMap(v, float(tok[2]), float(tok[3]), float(tok[4]))


def initial_states(n: int, seed: int, semi_a: float = 40.0, semi_b: float = 25.0, uniform_arc: bool = True,
                   vx_range=(3.0, 8.0), noise_std: float = 0.05) -> np.ndarray:
    """BASELINE initial states on the track centreline (n x 7)."""
    out = np.zeros((n, 7))
    check(_lib.load().mppi_workload_initial_states(n, seed, semi_a, semi_b, int(uniform_arc), vx_range[0],
                                                    vx_range[1], noise_std, dptr(out)))
    return out


def sg_coefficients(window: int, degree: int) -> np.ndarray:
    """sg_coefficients (smoothing.cpp:5-33)."""
    out = np.zeros(max(window, 1))
    check(_lib.load().mppi_sg_coefficients(window, degree, dptr(out)))
    return out


@dataclass
class BicycleParams:
    """BicycleParams (dynamics.hpp:42-62): the truth plant and the
    "vehicle_bicycle" rollout system."""
    mass: float = 22.0
    yaw_inertia: float = 1.8
    a: float = 0.45
    b: float = 0.35
    stiffness: float = 180.0
    mu: float = 0.65
    load: float = 107.9
    steer_scale: float = 0.35
    force_scale: float = 35.0

    def c(self) -> "_lib.BicycleParamsC":
        return _lib.BicycleParamsC(*[float(getattr(self, f)) for f in BicycleParams.__dataclass_fields__])


def brush_tire_force(alpha: float, u_F: float, p: BicycleParams = BicycleParams()) -> float:
    """brush_tire_force (dynamics.cpp:23-43) on the host (DomainError outside the friction circle)."""
    out = ctypes.c_double()
    pc = p.c()
    check(_lib.load().mppi_brush_tire_force(alpha, u_F, ctypes.byref(pc), ctypes.byref(out)))
    return out.value


def step_bicycle_truth(x, v, dt: float, p: BicycleParams = BicycleParams()) -> np.ndarray:
    """step_bicycle_truth (dynamics.cpp:51-81) on the host; v is the applied input."""
    xa = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(7))
    va = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(2))
    out = np.zeros(7)
    pc = p.c()
    check(_lib.load().mppi_bicycle_step(ctypes.byref(pc), dptr(xa), dptr(va), dt, dptr(out)))
    return out


@dataclass
class Disturbance:
    """Disturbance (simulator.hpp:10-16)."""
    time_s: float = 0.0
    dv_x: float = 0.0
    dv_y: float = 0.0
    dtheta_dot: float = 0.0


@dataclass
class SimConfig:
    """The closed-loop parts of SimConfig (simulator.hpp:72-88); sampling,
    bounds, costs, SG and the weight rule live in the controller."""
    episode_s: float = 30.0
    exec_noise: bool = True
    exec_noise_diag: Optional[Sequence[float]] = None    # variances; None = sampling covariance
    estimate_noise_std: Optional[Sequence[float]] = None  # 7 std devs; None = exact state feedback
    plant: BicycleParams = field(default_factory=BicycleParams)
    start_state: Sequence[float] = (0.0,) * 7
    disturbances: Sequence[Disturbance] = ()


@dataclass
class EpisodeTrace:
    """EpisodeTrace (simulator.hpp:26-32) as arrays, one row per step."""
    time: np.ndarray
    state: np.ndarray       # n x 7
    commanded: np.ndarray   # n x 2
    realized: np.ndarray    # n x 2
    cost: np.ndarray
    map_h: np.ndarray
    dt: float
    seed: int
    aborted: bool


TRACE_HEADER = ("time_s,p_x,p_y,theta,roll,v_x,v_y,theta_dot,steer_cmd,throttle_cmd,"
                "steer_real,throttle_real,cost,map_h")


def save_trace(trace: EpisodeTrace, path: str) -> None:
    """save_trace (simulator.cpp:180-200): the documented columns, %.17g."""
    with open(path, "w") as f:
        f.write(TRACE_HEADER + "\n")
        for i in range(len(trace.time)):
            row = [trace.time[i], *trace.state[i], *trace.commanded[i], *trace.realized[i], trace.cost[i],
                   trace.map_h[i]]
            f.write(",".join("%.17g" % float(v) for v in row) + "\n")


def simulate_episode(ctrl: "Controller", sim: SimConfig) -> EpisodeTrace:
    """simulate_episode (simulator.cpp:102-177) over a single-controller handle:
    mpc_step on the device every period, the bicycle truth plant on the host."""
    c = _lib.SimConfigC()
    _lib.load().mppi_sim_config_init(ctypes.byref(c))
    c.episode_s = sim.episode_s
    c.exec_noise = int(bool(sim.exec_noise))
    if sim.exec_noise_diag is not None:
        c.has_exec_noise_diag = 1
        c.exec_noise_diag[0], c.exec_noise_diag[1] = (float(v) for v in sim.exec_noise_diag)
    if sim.estimate_noise_std is not None:
        if len(sim.estimate_noise_std) != 7:
            raise InvalidArgument(_lib.MPPI_ERR_INVALID_ARGUMENT, "estimate_noise_std needs 7 entries")
        c.has_estimate_noise = 1
        for i, v in enumerate(sim.estimate_noise_std):
            c.estimate_noise_std[i] = float(v)
    c.plant = sim.plant.c()
    for i, v in enumerate(sim.start_state):
        c.start_state[i] = float(v)
    dist = (_lib.DisturbanceC * max(1, len(sim.disturbances)))(
        *[_lib.DisturbanceC(d.time_s, d.dv_x, d.dv_y, d.dtheta_dot) for d in sim.disturbances])
    c.n_disturbances = len(sim.disturbances)
    c.disturbances = ctypes.cast(dist, ctypes.POINTER(_lib.DisturbanceC))
    steps = int(round(sim.episode_s / ctrl.params.dt)) + 1
    recs = (_lib.SimRecordC * steps)()
    n, ab = ctypes.c_int(), ctypes.c_int()
    check(_lib.load().mppi_sim_episode(ctrl._h, ctypes.byref(c), recs, steps, ctypes.byref(n), ctypes.byref(ab)))
    arr = np.ctypeslib.as_array(ctypes.cast(recs, ctypes.POINTER(ctypes.c_double)), shape=(steps, 14))[:n.value]
    return EpisodeTrace(arr[:, 0].copy(), arr[:, 1:8].copy(), arr[:, 8:10].copy(), arr[:, 10:12].copy(),
                        arr[:, 12].copy(), arr[:, 13].copy(), ctrl.params.dt, int(ctrl.params.seed), bool(ab.value))


def device_count() -> int:
    return int(_lib.load().mppi_gpu_device_count())


def pipe_peaks(device: int = 0):
    """Measured mma.sync f16 peak (TFLOP/s) and MUFU ex2 peak (G lane-ops/s)."""
    t, m = ctypes.c_double(), ctypes.c_double()
    check(_lib.load().mppi_gpu_pipe_peak_probe(device, ctypes.byref(t), ctypes.byref(m)))
    return t.value, m.value


def fp32_peak_tflops(device: int = 0):
    """Measured FP32 FMA peak (TFLOP/s) and the device max SM clock (MHz)."""
    t, mhz = ctypes.c_double(), ctypes.c_double()
    check(_lib.load().mppi_gpu_fp32_peak_probe(device, ctypes.byref(t), ctypes.byref(mhz)))
    return t.value, mhz.value


_NOISE = {"injected": _lib.NOISE_INJECTED, "ref_splitmix": _lib.NOISE_REF_SPLITMIX, "philox": _lib.NOISE_PHILOX}
_PREC = {"fp32": _lib.FP32, "fp64": _lib.FP64}
_SYSTEM = {"vehicle_mlp": _lib.SYSTEM_VEHICLE_MLP, "quadratic": _lib.SYSTEM_QUADRATIC,
           "vehicle_bicycle": _lib.SYSTEM_VEHICLE_BICYCLE,
           "vehicle_basis": _lib.SYSTEM_VEHICLE_BASIS}


SHARD_KEYS = ("rank", "world_size", "chunks", "groups", "chunk_lo", "chunk_hi", "group_lo", "group_hi")


def shard_plan(samples: int, chunk_samples: int, rank: int, world_size: int) -> dict:
    """The sample partition of mppi_gpu_set_comm as a pure host function (no
    device): chunks of ``chunk_samples``, fixed groups, this rank's ranges."""
    v = (ctypes.c_int32 * 8)()
    check(_lib.load().mppi_gpu_shard_plan(samples, chunk_samples, rank, world_size, v))
    return dict(zip(SHARD_KEYS, list(v)))


def make_config(params: SamplingParams, bounds: ControlBounds = ControlBounds(),
                sg: Optional[SGFilter] = SGFilter(), cost: CostParams = CostParams(), *,
                system: str = "vehicle_mlp", hidden: int = 32, precision: str = "fp32",
                noise: str = "philox", n_controllers: int = 1, device: int = 0,
                with_terminal: bool = True, quad_cost_scale: float = 1.0, weight_rule: str = "it",
                cem_delta: float = 0.8, controller_offset: int = 0) -> _lib.ConfigC:
    """mppi_gpu_config from the reference's parameter objects; ``weight_rule``
    "it" (it_weights) or "cem" (cem_weights with ``cem_delta``, the
    WeightRuleConfig of controller.hpp:32-37)."""
    cfg = _lib.ConfigC()
    _lib.load().mppi_gpu_config_init(ctypes.byref(cfg))
    sig = list(params.sigma_diag)
    if len(sig) != 2:
        raise InvalidArgument(_lib.MPPI_ERR_INVALID_ARGUMENT, "the device path has m = 2 controls")
    cfg.samples = params.samples
    cfg.horizon_steps = params.horizon_steps
    cfg.dt = params.dt
    cfg.sigma_diag[0], cfg.sigma_diag[1] = sig
    cfg.lambda_ = params.lambda_
    cfg.gamma = params.gamma
    cfg.explore_fraction = params.explore_fraction
    cfg.seed = params.seed
    cfg.bounds_lower[0], cfg.bounds_lower[1] = bounds.lower
    cfg.bounds_upper[0], cfg.bounds_upper[1] = bounds.upper
    cfg.sg_window = sg.window if sg is not None else 0
    cfg.sg_degree = sg.degree if sg is not None else 0
    cfg.with_terminal = int(with_terminal)
    cfg.noise_mode = _NOISE[noise]
    cfg.precision = _PREC[precision]
    cfg.system = _SYSTEM[system]
    cfg.mlp_hidden = hidden
    cfg.n_controllers = n_controllers
    cfg.device = device
    cfg.quad_cost_scale = quad_cost_scale
    cfg.weight_rule = {"it": _lib.WEIGHT_IT, "cem": _lib.WEIGHT_CEM}[weight_rule]
    cfg.cem_delta = cem_delta
    cfg.controller_offset = controller_offset
    for f in CostParams.__dataclass_fields__:
        setattr(cfg.cost, f, float(getattr(cost, f)))
    return cfg


class Controller:
    """ControllerState + device rollout system (one handle, one CUDA stream).

    ``n_controllers > 1`` makes an independent-controller fleet: per-controller
    arrays carry a leading controller dimension.
    """

    def __init__(self, params: SamplingParams, bounds: ControlBounds = ControlBounds(),
                 sg: Optional[SGFilter] = SGFilter(), cost: CostParams = CostParams(), **kw):
        self.params = params
        self.bounds = bounds
        self.sg = sg
        self.cost = cost
        self.config = make_config(params, bounds, sg, cost, **kw)
        self.n_controllers = int(self.config.n_controllers)
        self.state_dim = 2 if self.config.system == _lib.SYSTEM_QUADRATIC else 7
        self.T = int(params.horizon_steps)
        self.K = int(params.samples)
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        check(self._lib.mppi_gpu_create(ctypes.byref(self.config), ctypes.byref(h)))
        self._h = h
        # per-call host buffers of the hot path (mpc_step / compute_control),
        # allocated once with their ctypes pointers: the per-step host cost is
        # then one copy in, the C call and one copy out
        self._xbuf = np.zeros(self.n_controllers * self.state_dim)
        self._ubuf = np.zeros((self.n_controllers, 2))
        self._xptr, self._uptr = dptr(self._xbuf), dptr(self._ubuf)

    # -- lifetime -----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            self._lib.mppi_gpu_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- model / cost data --------------------------------------------------
    def set_mlp(self, w: MlpWeights) -> None:
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (w.w1, w.b1, w.w2, w.b2, w.w3, w.b3)]
        check(self._lib.mppi_gpu_set_dynamics_mlp(self._h, w.hidden, *[dptr(a) for a in arrs]))

    def set_bicycle(self, p: BicycleParams = BicycleParams()) -> None:
        """BicycleTruthModel as the controller's model ("vehicle_bicycle" system)."""
        pc = p.c()
        check(self._lib.mppi_gpu_set_dynamics_bicycle(self._h, ctypes.byref(pc)))

    def set_basis(self, theta) -> None:
        """BasisFunctionModel Theta (dynamics.hpp:75-82): 25 x 4, coeffs(b, o)."""
        t = np.ascontiguousarray(theta, dtype=np.float64).reshape(25, 4)
        check(self._lib.mppi_gpu_set_dynamics_basis(self._h, dptr(t)))

    def set_costmap(self, m: CostMap, controller: int = -1) -> None:
        v = m.values
        if v.dtype == np.float32:
            v = np.ascontiguousarray(v)
            check(self._lib.mppi_gpu_set_costmap_f32(self._h, controller, v.ctypes.data_as(
                ctypes.POINTER(ctypes.c_float)), m.width, m.height, m.x0, m.y0, m.resolution))
        else:
            v = np.ascontiguousarray(v, dtype=np.float64)
            check(self._lib.mppi_gpu_set_costmap(self._h, controller, dptr(v), m.width, m.height, m.x0, m.y0,
                                                 m.resolution))

    def perturb_fleet_costmaps(self, sigma: float, seed: int) -> None:
        check(self._lib.mppi_gpu_perturb_fleet_costmaps(self._h, sigma, seed))

    def get_costmap(self, like: "CostMap", controller: int = 0) -> "CostMap":
        """Controller ``controller``'s device map (geometry of ``like``)."""
        v = np.zeros(like.values.shape, dtype=np.float32)
        check(self._lib.mppi_gpu_get_costmap_f32(self._h, controller, v.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
        return CostMap(v, like.x0, like.y0, like.resolution)

    # -- ControllerState ----------------------------------------------------
    def get_plan(self, controller: int = 0) -> np.ndarray:
        U = np.zeros((self.T, 2))
        check(self._lib.mppi_gpu_get_plan(self._h, controller, dptr(U)))
        return U

    def set_plan(self, U, controller: int = 0) -> None:
        U = np.ascontiguousarray(np.asarray(U, dtype=np.float64).reshape(self.T, 2))
        check(self._lib.mppi_gpu_set_plan(self._h, controller, dptr(U)))

    plan = property(get_plan, set_plan)

    def get_iteration(self, controller: int = 0) -> int:
        it = ctypes.c_uint64()
        check(self._lib.mppi_gpu_get_iteration(self._h, controller, ctypes.byref(it)))
        return int(it.value)

    def set_iteration(self, value: int, controller: int = 0) -> None:
        check(self._lib.mppi_gpu_set_iteration(self._h, controller, value))

    iteration = property(get_iteration, set_iteration)

    def set_seed(self, seed: int, controller: int = 0) -> None:
        check(self._lib.mppi_gpu_set_seed(self._h, controller, seed))

    def set_noise(self, eps: np.ndarray) -> None:
        """INJECTED mode: the batch (K x 2 x T, reference layout) of the next rollout."""
        e = np.ascontiguousarray(eps, dtype=np.float64).reshape(-1)
        if e.size != self.K * 2 * self.T:
            raise InvalidArgument(_lib.MPPI_ERR_INVALID_ARGUMENT, "eps must have K*2*T entries")
        check(self._lib.mppi_gpu_set_noise(self._h, dptr(e)))

    def _x(self, x0) -> np.ndarray:
        x = np.ascontiguousarray(np.asarray(x0, dtype=np.float64).reshape(-1))
        if x.size != self.n_controllers * self.state_dim:
            raise InvalidArgument(_lib.MPPI_ERR_INVALID_ARGUMENT, "x0 dimension mismatch")
        return x

    # -- hot path -----------------------------------------------------------
    def _stage_x(self, x0) -> None:
        x = np.asarray(x0, dtype=np.float64)
        if x.size != self._xbuf.size:
            raise InvalidArgument(_lib.MPPI_ERR_INVALID_ARGUMENT, "x0 dimension mismatch")
        self._xbuf[:] = x.reshape(-1)

    def mpc_step(self, x0) -> np.ndarray:
        """mpc_step (controller.cpp:133-148): returns clamp(U'[0]) and slides."""
        self._stage_x(x0)
        check(self._lib.mppi_gpu_step(self._h, self._xptr, self._uptr))
        return self._ubuf[0].copy() if self.n_controllers == 1 else self._ubuf.copy()

    def compute_control(self, x0) -> np.ndarray:
        self._stage_x(x0)
        check(self._lib.mppi_gpu_compute_control(self._h, self._xptr, self._uptr))
        return self._ubuf[0].copy() if self.n_controllers == 1 else self._ubuf.copy()

    def slide(self) -> None:
        check(self._lib.mppi_gpu_slide(self._h))

    def optimize_to_convergence(self, x0, iterations: int) -> np.ndarray:
        check(self._lib.mppi_gpu_optimize(self._h, dptr(self._x(x0)), iterations))
        return self.get_plan()

    def closed_loop(self, x_init, iterations: int, traces: bool = True):
        """Receding-horizon loop with the device plant; returns (u_trace, x_trace)."""
        C = self.n_controllers
        u = np.zeros((iterations, C, 2)) if traces else None
        x = np.zeros((iterations + 1, C, self.state_dim)) if traces else None
        check(self._lib.mppi_gpu_closed_loop(self._h, dptr(self._x(x_init)), iterations, dptr(u), dptr(x)))
        return u, x

    def closed_loop_timed(self, x_init, iterations: int, flush_l2_bytes: int = 0, per_iteration: bool = False):
        """Device-timed receding-horizon loop: total ms, or (total ms, per-iteration
        ms array) with ``per_iteration`` (flush mode only)."""
        ms = ctypes.c_double()
        it = np.zeros(iterations) if per_iteration else None
        check(self._lib.mppi_gpu_closed_loop_timed(self._h, dptr(self._x(x_init)), iterations, flush_l2_bytes,
                                                   ctypes.byref(ms), dptr(it)))
        return (ms.value, it) if per_iteration else ms.value

    # -- parity entry points ------------------------------------------------
    def sample_perturbations(self, iteration: int):
        """sample_perturbations (sampler.cpp:5-39): (eps K x 2 x T, flags K)."""
        eps = np.zeros((self.K, 2, self.T))
        flags = np.zeros(self.K, dtype=np.uint8)
        check(self._lib.mppi_gpu_sample_perturbations(self._h, iteration, dptr(eps),
                                                      flags.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
        return eps, flags

    def rollout_batch(self, x0, eps: Optional[np.ndarray] = None, return_batch: bool = False):
        """rollout_batch (controller.cpp:55-109) on the current plan and iteration."""
        costs = np.zeros(self.K)
        e_in = None if eps is None else np.ascontiguousarray(eps, dtype=np.float64).reshape(-1)
        if e_in is not None and e_in.size != self.K * 2 * self.T:
            raise InvalidArgument(_lib.MPPI_ERR_INVALID_ARGUMENT, "eps must have K*2*T entries")
        stored = np.zeros((self.K, 2, self.T)) if return_batch else None
        check(self._lib.mppi_gpu_rollout_costs(self._h, dptr(self._x(x0)), dptr(e_in), dptr(costs), dptr(stored)))
        return (costs, stored) if return_batch else costs

    def compute_weights(self, costs) -> WeightResult:
        """compute_weights (controller.cpp:111-116): it_weights (weights.cpp:8-25) or cem_weights (:27-53)."""
        c = np.ascontiguousarray(costs, dtype=np.float64)
        if c.size != self.K:
            raise InvalidArgument(_lib.MPPI_ERR_INVALID_ARGUMENT, "costs must have K entries")
        w = np.zeros(self.K)
        rho, eta = ctypes.c_double(), ctypes.c_double()
        check(self._lib.mppi_gpu_weights(self._h, dptr(c), dptr(w), ctypes.byref(rho), ctypes.byref(eta)))
        return WeightResult(w, rho.value, eta.value)

    def update_plan(self, weights) -> np.ndarray:
        """update_plan (controller.cpp:118-131) with the last rollout batch; returns U'."""
        w = np.ascontiguousarray(getattr(weights, "weights", weights), dtype=np.float64)
        if w.size != self.K:
            raise InvalidArgument(_lib.MPPI_ERR_INVALID_ARGUMENT, "update_plan: weight/sample count mismatch")
        check(self._lib.mppi_gpu_update_plan(self._h, dptr(w)))
        return self.get_plan()

    def rollout_states(self, x0, sample: int) -> np.ndarray:
        out = np.zeros((self.T + 1, self.state_dim))
        check(self._lib.mppi_gpu_rollout_states(self._h, dptr(self._x(x0)), sample, dptr(out)))
        return out

    # -- multi-GPU ----------------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        check(_lib.load().mppi_gpu_nccl_unique_id(buf))
        return bytes(buf)

    def set_comm(self, rank: int, world_size: int, unique_id: Optional[bytes]) -> None:
        """NCCL sample sharding: this handle is rank ``rank`` of ``world_size``
        (mppi_gpu_set_comm; the group rows are all-gathered every iteration)."""
        buf = None
        if unique_id is not None:
            buf = (ctypes.c_uint8 * 128)(*unique_id)
        check(self._lib.mppi_gpu_set_comm(self._h, rank, world_size, buf))

    @staticmethod
    def set_comm_local(ctrls: Sequence["Controller"]) -> None:
        """In-process sample sharding: ``ctrls[r]`` becomes rank r (one handle
        per GPU of this process, or several on one GPU); the exchange is a
        device-to-device copy of the group rows (mppi_gpu_set_comm_local)."""
        hs = (ctypes.c_void_p * len(ctrls))(*[c._h.value for c in ctrls])
        check(_lib.load().mppi_gpu_set_comm_local(hs, len(ctrls)))

    @staticmethod
    def step_local(ctrls: Sequence["Controller"], x0) -> np.ndarray:
        """mpc_step of a controller sharded with set_comm_local; returns every
        rank's u0 (n x 2, identical rows)."""
        x = np.ascontiguousarray(np.asarray(x0, dtype=np.float64).reshape(-1))
        u = np.zeros((len(ctrls), 2))
        hs = (ctypes.c_void_p * len(ctrls))(*[c._h.value for c in ctrls])
        check(_lib.load().mppi_gpu_step_local(hs, len(ctrls), dptr(x), dptr(u)))
        return u

    @property
    def shard_info(self) -> dict:
        """{rank, world_size, chunks, groups, chunk_lo, chunk_hi, group_lo, group_hi}."""
        v = (ctypes.c_int32 * 8)()
        check(self._lib.mppi_gpu_shard_info(self._h, v))
        return dict(zip(SHARD_KEYS, list(v)))

    def profile_read_exchange(self, reset: bool = True):
        """(ms, count) of the group-row exchange over the profiled closed-loop iterations."""
        ms, n = ctypes.c_double(), ctypes.c_uint64()
        check(self._lib.mppi_gpu_profile_read_exchange(self._h, ctypes.byref(ms), ctypes.byref(n), int(reset)))
        return ms.value, int(n.value)

    # -- instrumentation ----------------------------------------------------
    @property
    def stream(self) -> int:
        s = ctypes.c_void_p()
        check(self._lib.mppi_gpu_get_stream(self._h, ctypes.byref(s)))
        return int(s.value or 0)

    @property
    def launch_count(self) -> int:
        n = ctypes.c_uint64()
        check(self._lib.mppi_gpu_launch_count(self._h, ctypes.byref(n)))
        return int(n.value)

    def profile(self, enable: bool) -> None:
        check(self._lib.mppi_gpu_profile_enable(self._h, int(enable)))

    def profile_read(self, reset: bool = True):
        ms, n = ctypes.c_double(), ctypes.c_uint64()
        check(self._lib.mppi_gpu_profile_read(self._h, ctypes.byref(ms), ctypes.byref(n), int(reset)))
        return ms.value, int(n.value)

    @property
    def kernel_variant(self) -> str:
        buf = ctypes.create_string_buffer(256)
        check(self._lib.mppi_gpu_kernel_variant(self._h, buf, 256))
        return buf.value.decode()
