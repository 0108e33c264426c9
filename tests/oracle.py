"""ctypes wrapper of oracle/build/liboracle.so — TEST INFRASTRUCTURE ONLY.

The oracle is the CPU restatement of the reference hot path
(oracle/mppi_oracle.cpp).  Tests use it as the checker; it is never part of
the product path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_uint8, c_uint32, c_uint64, c_void_p

import numpy as np

from paper_1707_02342_b200 import _lib as plib
from paper_1707_02342_b200.api import make_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "build", "liboracle.so")
_d = POINTER(c_double)

_SIG = {
    "oracle_last_error": (c_char_p, []),
    "oracle_set_mlp_order": (None, [c_int]),
    "oracle_splitmix64": (c_uint64, [c_uint64]),
    "oracle_counter_hash": (c_uint64, [c_uint64] * 6),
    "oracle_counter_normal": (c_double, [c_uint64] * 5 + [c_int]),
    "oracle_philox4x32_10": (None, [POINTER(c_uint32), POINTER(c_uint32), POINTER(c_uint32)]),
    "oracle_sample_perturbations": (c_int, [c_int, c_int, c_int, _d, c_double, c_uint64, c_uint64, c_int, _d,
                                            POINTER(c_uint8)]),
    "oracle_sg_coefficients": (c_int, [c_int, c_int, _d]),
    "oracle_sg_smooth": (c_int, [_d, c_int, c_int, _d, c_int, _d]),
    "oracle_it_weights": (c_int, [_d, c_int, c_double, _d, _d, _d]),
    "oracle_cem_weights": (c_int, [_d, c_int, c_double, _d, _d, _d]),
    "oracle_it_weights_f32": (c_int, [POINTER(c_float), c_int, c_float, POINTER(c_float), POINTER(c_float),
                                      POINTER(c_float)]),
    "oracle_mlp_forward": (c_int, [c_int, _d, _d, _d, _d, _d, _d, _d, _d]),
    "oracle_advance_split": (c_int, [_d, _d, c_double, _d]),
    "oracle_clamp_controls": (c_int, [_d, _d, _d, c_int, _d]),
    "oracle_costmap_lookup": (c_int, [_d, c_int, c_int, c_double, c_double, c_double, c_double, c_double, _d]),
    "oracle_state_cost": (c_int, [_d, c_int, _d, c_int, c_int, c_double, c_double, c_double,
                                  POINTER(plib.CostParamsC), _d]),
    "oracle_side_slip": (c_double, [c_double, c_double]),
    "oracle_create": (c_int, [POINTER(plib.ConfigC), POINTER(c_void_p)]),
    "oracle_destroy": (None, [c_void_p]),
    "oracle_set_mlp": (c_int, [c_void_p, c_int, _d, _d, _d, _d, _d, _d]),
    "oracle_set_costmap": (c_int, [c_void_p, _d, c_int, c_int, c_double, c_double, c_double]),
    "oracle_set_theta": (c_int, [c_void_p, _d]),
    "oracle_set_bicycle": (c_int, [c_void_p, _d]),
    "oracle_brush_tire_force": (c_int, [c_double, c_double, _d, _d]),
    "oracle_step_bicycle": (c_int, [_d, _d, c_double, _d, _d]),
    "oracle_eval_basis": (c_int, [_d, _d, _d]),
    "oracle_step_basis": (c_int, [_d, _d, c_double, _d, _d]),
    "oracle_set_costmap_f32": (c_int, [c_void_p, POINTER(c_float), c_int, c_int, c_double, c_double, c_double]),
    "oracle_set_plan": (c_int, [c_void_p, _d]),
    "oracle_get_plan": (c_int, [c_void_p, _d]),
    "oracle_set_iteration": (c_int, [c_void_p, c_uint64]),
    "oracle_get_iteration": (c_int, [c_void_p, POINTER(c_uint64)]),
    "oracle_set_noise": (c_int, [c_void_p, _d]),
    "oracle_rollout_costs": (c_int, [c_void_p, _d, _d, _d, _d, c_int]),
    "oracle_weights": (c_int, [c_void_p, _d, _d, _d, _d]),
    "oracle_update_plan": (c_int, [c_void_p, _d]),
    "oracle_rollout_states": (c_int, [c_void_p, _d, c_int, _d]),
    "oracle_mpc_step": (c_int, [c_void_p, _d, _d, c_int]),
    "oracle_optimize": (c_int, [c_void_p, _d, c_int, c_int]),
    "oracle_vehicle_step": (c_int, [c_void_p, _d, _d, _d]),
}

_lib = None


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class OracleInvalidArgument(OracleError, ValueError):
    pass


def build() -> None:
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(
                os.path.join(ORACLE_DIR, "mppi_oracle.cpp")):
            build()
        lib = ctypes.CDLL(ORACLE_SO)
        for n, (r, a) in _SIG.items():
            f = getattr(lib, n)
            f.restype = r
            f.argtypes = a
        _lib = lib
    return _lib


def chk(code):
    if code:
        msg = load().oracle_last_error().decode()
        if code in (plib.MPPI_ERR_INVALID_ARGUMENT, plib.MPPI_ERR_NONFINITE):
            raise OracleInvalidArgument(code, msg)
        raise OracleError(code, msg)


def p(a):
    return None if a is None else a.ctypes.data_as(_d)


def splitmix64(x):
    return int(load().oracle_splitmix64(x))


def counter_normal(seed, stream, it, k, t, c):
    return float(load().oracle_counter_normal(seed, stream, it, k, t, c))


def philox(ctr, key):
    c = (c_uint32 * 4)(*ctr)
    k = (c_uint32 * 2)(*key)
    o = (c_uint32 * 4)()
    load().oracle_philox4x32_10(c, k, o)
    return list(o)


def sample_perturbations(K, T, sigma_diag, explore_fraction, seed, iteration, mode=plib.NOISE_REF_SPLITMIX):
    m = len(sigma_diag)
    sig = np.asarray(sigma_diag, dtype=np.float64)
    eps = np.zeros((K, m, T))
    flags = np.zeros(K, dtype=np.uint8)
    chk(load().oracle_sample_perturbations(K, T, m, p(sig), explore_fraction, seed, iteration, mode, p(eps),
                                           flags.ctypes.data_as(POINTER(c_uint8))))
    return eps, flags


def sg_coefficients(window, degree):
    out = np.zeros(max(window, 1))
    chk(load().oracle_sg_coefficients(window, degree, p(out)))
    return out


def sg_smooth(seq, coeffs):
    seq = np.ascontiguousarray(np.atleast_2d(np.asarray(seq, dtype=np.float64).T).T)
    n, m = seq.shape
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    out = np.zeros_like(seq)
    chk(load().oracle_sg_smooth(p(seq), n, m, p(c), c.size, p(out)))
    return out


def it_weights(costs, lam):
    c = np.ascontiguousarray(costs, dtype=np.float64)
    w = np.zeros(c.size)
    rho, eta = c_double(), c_double()
    chk(load().oracle_it_weights(p(c), c.size, lam, p(w), ctypes.byref(rho), ctypes.byref(eta)))
    return w, rho.value, eta.value


def cem_weights(costs, delta):
    """cem_weights (weights.cpp:27-53) of the restatement: (weights, rho, normalizer)."""
    c = np.ascontiguousarray(costs, dtype=np.float64)
    w = np.zeros(len(c))
    rho, eta = c_double(), c_double()
    chk(load().oracle_cem_weights(p(c), len(c), delta, p(w), ctypes.byref(rho), ctypes.byref(eta)))
    return w, rho.value, eta.value


def mlp_forward(w, x_d, v):
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (w.w1, w.b1, w.w2, w.b2, w.w3, w.b3)]
    inp = np.array(list(x_d) + list(v), dtype=np.float64)
    out = np.zeros(4)
    chk(load().oracle_mlp_forward(w.hidden, *[p(a) for a in arrs], p(inp), p(out)))
    return out


def advance_split(x, d, dt):
    x = np.asarray(x, dtype=np.float64)
    d = np.asarray(d, dtype=np.float64)
    out = np.zeros(7)
    chk(load().oracle_advance_split(p(x), p(d), dt, p(out)))
    return out


def clamp_controls(v, lo, hi):
    v, lo, hi = (np.asarray(a, dtype=np.float64) for a in (v, lo, hi))
    out = np.zeros(v.size)
    chk(load().oracle_clamp_controls(p(v), p(lo), p(hi), v.size, p(out)))
    return out


def costmap_lookup(values, x0, y0, res, px, py):
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = c_double()
    chk(load().oracle_costmap_lookup(p(v), v.shape[1], v.shape[0], x0, y0, res, px, py, ctypes.byref(out)))
    return out.value


def state_cost(x, t, values, x0, y0, res, cost):
    v = np.ascontiguousarray(values, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    cp = plib.CostParamsC()
    for f in cost.__dataclass_fields__:
        setattr(cp, f, float(getattr(cost, f)))
    out = c_double()
    chk(load().oracle_state_cost(p(x), t, p(v), v.shape[1], v.shape[0], x0, y0, res, ctypes.byref(cp),
                                 ctypes.byref(out)))
    return out.value


class OracleController:
    """Oracle mirror of paper_1707_02342_b200.Controller (same config)."""

    def __init__(self, params, bounds=None, sg=None, cost=None, **kw):
        from paper_1707_02342_b200.api import ControlBounds, CostParams, SGFilter
        bounds = bounds if bounds is not None else ControlBounds()
        cost = cost if cost is not None else CostParams()
        sg = SGFilter() if sg == "default" else sg
        kw.setdefault("noise", "ref_splitmix")
        kw.setdefault("precision", "fp64")
        self.cfg = make_config(params, bounds, sg, cost, **kw)
        self.K, self.T = params.samples, params.horizon_steps
        self.state_dim = 2 if kw.get("system") == "quadratic" else 7
        h = c_void_p()
        chk(load().oracle_create(ctypes.byref(self.cfg), ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            load().oracle_destroy(self.h)

    def set_mlp(self, w):
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (w.w1, w.b1, w.w2, w.b2, w.w3, w.b3)]
        chk(load().oracle_set_mlp(self.h, w.hidden, *[p(a) for a in arrs]))

    def set_bicycle(self, params=None):
        from paper_1707_02342_b200.api import BicycleParams
        b = params or BicycleParams()
        v = np.array([getattr(b, f) for f in BicycleParams.__dataclass_fields__], dtype=np.float64)
        chk(load().oracle_set_bicycle(self.h, p(v)))

    def set_basis(self, theta):
        t = np.ascontiguousarray(theta, dtype=np.float64).reshape(25, 4)
        chk(load().oracle_set_theta(self.h, p(t)))

    def set_costmap(self, m):
        v = np.ascontiguousarray(m.values, dtype=np.float64)
        chk(load().oracle_set_costmap(self.h, p(v), m.width, m.height, m.x0, m.y0, m.resolution))

    def get_plan(self):
        U = np.zeros((self.T, 2))
        chk(load().oracle_get_plan(self.h, p(U)))
        return U

    def set_plan(self, U):
        U = np.ascontiguousarray(np.asarray(U, dtype=np.float64).reshape(self.T, 2))
        chk(load().oracle_set_plan(self.h, p(U)))

    plan = property(get_plan, set_plan)

    @property
    def iteration(self):
        it = c_uint64()
        chk(load().oracle_get_iteration(self.h, ctypes.byref(it)))
        return int(it.value)

    @iteration.setter
    def iteration(self, v):
        chk(load().oracle_set_iteration(self.h, v))

    def set_noise(self, eps):
        e = np.ascontiguousarray(eps, dtype=np.float64)
        chk(load().oracle_set_noise(self.h, p(e)))

    def rollout_batch(self, x0, eps=None, threads=1, return_batch=False):
        costs = np.zeros(self.K)
        x = np.ascontiguousarray(x0, dtype=np.float64)
        e = None if eps is None else np.ascontiguousarray(eps, dtype=np.float64)
        stored = np.zeros((self.K, 2, self.T)) if return_batch else None
        chk(load().oracle_rollout_costs(self.h, p(x), p(e), p(costs), p(stored), threads))
        return (costs, stored) if return_batch else costs

    def compute_weights(self, costs):
        c = np.ascontiguousarray(costs, dtype=np.float64)
        w = np.zeros(self.K)
        rho, eta = c_double(), c_double()
        chk(load().oracle_weights(self.h, p(c), p(w), ctypes.byref(rho), ctypes.byref(eta)))
        from paper_1707_02342_b200.api import WeightResult
        return WeightResult(w, rho.value, eta.value)

    def update_plan(self, w):
        w = np.ascontiguousarray(getattr(w, "weights", w), dtype=np.float64)
        chk(load().oracle_update_plan(self.h, p(w)))
        return self.get_plan()

    def rollout_states(self, x0, sample):
        out = np.zeros((self.T + 1, self.state_dim))
        x = np.ascontiguousarray(x0, dtype=np.float64)
        chk(load().oracle_rollout_states(self.h, p(x), sample, p(out)))
        return out

    def mpc_step(self, x0, threads=1):
        u = np.zeros(2)
        x = np.ascontiguousarray(x0, dtype=np.float64)
        chk(load().oracle_mpc_step(self.h, p(x), p(u), threads))
        return u

    def optimize_to_convergence(self, x0, iterations, threads=1):
        x = np.ascontiguousarray(x0, dtype=np.float64)
        chk(load().oracle_optimize(self.h, p(x), iterations, threads))
        return self.get_plan()

    def vehicle_step(self, x, u):
        out = np.zeros(7)
        chk(load().oracle_vehicle_step(self.h, p(np.ascontiguousarray(x, dtype=np.float64)),
                                       p(np.ascontiguousarray(u, dtype=np.float64)), p(out)))
        return out


def side_slip(vx, vy):
    return float(load().oracle_side_slip(vx, vy))


def eval_basis(x_d, v):
    """eval_basis (dynamics.cpp:83-133) of the restatement, double."""
    phi = np.zeros(25)
    load().oracle_eval_basis(p(np.ascontiguousarray(x_d, dtype=np.float64)),
                             p(np.ascontiguousarray(v, dtype=np.float64)), p(phi))
    return phi


def step_basis(x, v, dt, theta):
    """step_basis_model (dynamics.cpp:152-157) of the restatement, double."""
    out = np.zeros(7)
    chk(load().oracle_step_basis(p(np.ascontiguousarray(x, dtype=np.float64)),
                                 p(np.ascontiguousarray(v, dtype=np.float64)), dt,
                                 p(np.ascontiguousarray(theta, dtype=np.float64).reshape(100)), p(out)))
    return out


# ---------------------------------------------------------------- LQ oracle
def _require_psd(M, what):
    """require_psd (verification.cpp): symmetric and positive semidefinite."""
    M = np.asarray(M, dtype=np.float64)
    if not np.allclose(M, M.T, rtol=0.0, atol=1e-12) or np.linalg.eigvalsh(0.5 * (M + M.T)).min() < -1e-12:
        raise OracleInvalidArgument(-1, f"{what} must be symmetric positive semidefinite")
    return M


def riccati_plan(A, B, Q, Qf, R, T, x0):
    """riccati_plan (verification.cpp:72-99): backward Riccati recursion
    K_t = (R + B'PB)^-1 B'PA, P <- Q + A'P(A - B K_t) from P = Qf, then the
    forward rollout u_t = -K_t x_t.  Returns the T x m plan."""
    A, B = np.asarray(A, dtype=np.float64), np.asarray(B, dtype=np.float64)
    Q, Qf, R = _require_psd(Q, "riccati_plan: Q"), _require_psd(Qf, "riccati_plan: Qf"), _require_psd(R, "riccati_plan: R")
    if np.linalg.eigvalsh(R).min() <= 0.0:
        raise OracleInvalidArgument(-1, "riccati_plan: R must be positive definite")
    gains = [None] * T
    P = Qf
    for t in range(T - 1, -1, -1):
        BtP = B.T @ P
        gains[t] = np.linalg.solve(R + BtP @ B, BtP @ A)
        P = Q + A.T @ P @ (A - B @ gains[t])
    plan = np.zeros((T, B.shape[1]))
    x = np.asarray(x0, dtype=np.float64)
    for t in range(T):
        u = -gains[t] @ x
        plan[t] = u
        x = A @ x + B @ u
    return plan


def lqr_oracle(A, B, Q, Qf, sigma_diag, lam, T, x0):
    """lqr_oracle (verification.cpp:101-108): the running cost lands on the
    post-step states, so x_T carries Q + Qf; the sampling optimizer's control
    penalty with gamma = lambda is R = (lambda / 2) Sigma^-1."""
    if not lam > 0.0:
        raise OracleInvalidArgument(-1, "LQInstance: lambda must be > 0")
    sig = np.asarray(sigma_diag, dtype=np.float64)
    if sig.min() <= 0.0:
        raise OracleInvalidArgument(-1, "LQInstance: sigma entries must be > 0")
    R = np.diag(lam / 2.0 / sig)
    return riccati_plan(A, B, Q, np.asarray(Q) + np.asarray(Qf), R, T, x0)
