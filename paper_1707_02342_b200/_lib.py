"""ctypes binding of the C ABI in include/mppi_gpu.h (libmppi_gpu.so).

The library is the product: there is no Python or CPU fallback.  Importing
this module only loads the shared object (which works on a CPU-only host);
every compute entry point then needs a CUDA device and fails loudly with
:class:`DeviceError` when none is usable.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_size_t, c_uint8, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libmppi_gpu.so")

# status codes (mppi_gpu.h)
MPPI_OK = 0
MPPI_ERR_INVALID_ARGUMENT = 1
MPPI_ERR_NONFINITE = 2
MPPI_ERR_RUNTIME = 3
MPPI_ERR_CUDA = 4
MPPI_ERR_NCCL = 5
MPPI_ERR_UNSUPPORTED = 6
MPPI_ERR_DOMAIN = 7

NOISE_INJECTED, NOISE_REF_SPLITMIX, NOISE_PHILOX = 0, 1, 2
FP32, FP64 = 0, 1
SYSTEM_VEHICLE_MLP, SYSTEM_QUADRATIC, SYSTEM_VEHICLE_BASIS, SYSTEM_VEHICLE_BICYCLE = 0, 1, 2, 3
WEIGHT_IT, WEIGHT_CEM = 0, 1


class MppiError(Exception):
    """Base class; ``code`` is the MPPI_* status."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class InvalidArgument(MppiError, ValueError):
    """std::invalid_argument in the reference (types.hpp:105-122 and friends)."""


class NonFiniteCost(InvalidArgument):
    """it_weights' "non-finite cost" (weights.cpp:12)."""


class DeviceError(MppiError, RuntimeError):
    """CUDA / NCCL failure, or no usable device (no CPU fallback exists)."""


class Unsupported(MppiError, NotImplementedError):
    pass


class MppiRuntimeError(MppiError, RuntimeError):
    """std::runtime_error in the reference."""


class DomainError(MppiError, ArithmeticError):
    """std::domain_error in the reference (brush_tire_force, dynamics.cpp:25-27)."""


_ERRORS = {
    MPPI_ERR_INVALID_ARGUMENT: InvalidArgument,
    MPPI_ERR_NONFINITE: NonFiniteCost,
    MPPI_ERR_RUNTIME: MppiRuntimeError,
    MPPI_ERR_CUDA: DeviceError,
    MPPI_ERR_NCCL: DeviceError,
    MPPI_ERR_UNSUPPORTED: Unsupported,
    MPPI_ERR_DOMAIN: DomainError,
}


class CostParamsC(ctypes.Structure):
    _fields_ = [(n, c_double) for n in (
        "alpha_track", "alpha_speed", "alpha_stab", "v_des", "impulse", "decay",
        "boundary_threshold", "slip_limit", "crash_penalty", "crash_threshold", "roll_limit")]


class ConfigC(ctypes.Structure):
    _fields_ = [
        ("samples", c_int32),
        ("horizon_steps", c_int32),
        ("dt", c_double),
        ("sigma_diag", c_double * 2),
        ("lambda_", c_double),
        ("gamma", c_double),
        ("explore_fraction", c_double),
        ("seed", c_uint64),
        ("bounds_lower", c_double * 2),
        ("bounds_upper", c_double * 2),
        ("sg_window", c_int32),
        ("sg_degree", c_int32),
        ("weight_rule", c_int32),
        ("cem_delta", c_double),
        ("with_terminal", c_int32),
        ("noise_mode", c_int32),
        ("precision", c_int32),
        ("system", c_int32),
        ("mlp_hidden", c_int32),
        ("n_controllers", c_int32),
        ("device", c_int32),
        ("quad_cost_scale", c_double),
        ("cost", CostParamsC),
        ("controller_offset", c_int32),
    ]


class BicycleParamsC(ctypes.Structure):
    _fields_ = [(n, c_double) for n in (
        "mass", "yaw_inertia", "a", "b", "stiffness", "mu", "load", "steer_scale", "force_scale")]


class DisturbanceC(ctypes.Structure):
    _fields_ = [("time_s", c_double), ("dv_x", c_double), ("dv_y", c_double), ("dtheta_dot", c_double)]


class SimConfigC(ctypes.Structure):
    _fields_ = [
        ("episode_s", c_double),
        ("exec_noise", c_int32),
        ("has_exec_noise_diag", c_int32),
        ("exec_noise_diag", c_double * 2),
        ("has_estimate_noise", c_int32),
        ("estimate_noise_std", c_double * 7),
        ("plant", BicycleParamsC),
        ("start_state", c_double * 7),
        ("n_disturbances", c_int32),
        ("disturbances", POINTER(DisturbanceC)),
    ]


class SimRecordC(ctypes.Structure):
    _fields_ = [("time", c_double), ("state", c_double * 7), ("commanded", c_double * 2),
                ("realized", c_double * 2), ("cost", c_double), ("map_h", c_double)]


_P = POINTER
_d = _P(c_double)
_SIGNATURES = {
    "mppi_gpu_abi_version": (c_int, []),
    "mppi_gpu_config_sizeof": (c_size_t, []),
    "mppi_gpu_last_error": (c_char_p, []),
    "mppi_gpu_config_init": (None, [_P(ConfigC)]),
    "mppi_gpu_device_count": (c_int, []),
    "mppi_gpu_create": (c_int, [_P(ConfigC), _P(c_void_p)]),
    "mppi_gpu_destroy": (c_int, [c_void_p]),
    "mppi_gpu_set_dynamics_mlp": (c_int, [c_void_p, c_int, _d, _d, _d, _d, _d, _d]),
    "mppi_gpu_set_dynamics_basis": (c_int, [c_void_p, _d]),
    "mppi_gpu_set_dynamics_bicycle": (c_int, [c_void_p, _P(BicycleParamsC)]),
    "mppi_bicycle_params_init": (None, [_P(BicycleParamsC)]),
    "mppi_brush_tire_force": (c_int, [c_double, c_double, _P(BicycleParamsC), _d]),
    "mppi_bicycle_step": (c_int, [_P(BicycleParamsC), _d, _d, c_double, _d]),
    "mppi_sim_config_init": (None, [_P(SimConfigC)]),
    "mppi_sim_episode": (c_int, [c_void_p, _P(SimConfigC), _P(SimRecordC), c_int, _P(c_int), _P(c_int)]),
    "mppi_gpu_set_costmap": (c_int, [c_void_p, c_int, _d, c_int, c_int, c_double, c_double, c_double]),
    "mppi_gpu_set_costmap_f32": (c_int, [c_void_p, c_int, _P(c_float), c_int, c_int, c_double, c_double, c_double]),
    "mppi_gpu_perturb_fleet_costmaps": (c_int, [c_void_p, c_double, c_uint64]),
    "mppi_gpu_get_costmap_f32": (c_int, [c_void_p, c_int, _P(c_float)]),
    "mppi_gpu_set_plan": (c_int, [c_void_p, c_int, _d]),
    "mppi_gpu_get_plan": (c_int, [c_void_p, c_int, _d]),
    "mppi_gpu_set_iteration": (c_int, [c_void_p, c_int, c_uint64]),
    "mppi_gpu_get_iteration": (c_int, [c_void_p, c_int, _P(c_uint64)]),
    "mppi_gpu_set_seed": (c_int, [c_void_p, c_int, c_uint64]),
    "mppi_gpu_set_noise": (c_int, [c_void_p, _d]),
    "mppi_gpu_compute_control": (c_int, [c_void_p, _d, _d]),
    "mppi_gpu_slide": (c_int, [c_void_p]),
    "mppi_gpu_step": (c_int, [c_void_p, _d, _d]),
    "mppi_gpu_optimize": (c_int, [c_void_p, _d, c_int]),
    "mppi_gpu_closed_loop": (c_int, [c_void_p, _d, c_int, _d, _d]),
    "mppi_gpu_closed_loop_timed": (c_int, [c_void_p, _d, c_int, c_uint64, _d, _d]),
    "mppi_gpu_sample_perturbations": (c_int, [c_void_p, c_uint64, _d, _P(c_uint8)]),
    "mppi_gpu_rollout_costs": (c_int, [c_void_p, _d, _d, _d, _d]),
    "mppi_gpu_weights": (c_int, [c_void_p, _d, _d, _d, _d]),
    "mppi_gpu_update_plan": (c_int, [c_void_p, _d]),
    "mppi_gpu_rollout_states": (c_int, [c_void_p, _d, c_int, _d]),
    "mppi_gpu_nccl_unique_id": (c_int, [_P(c_uint8)]),
    "mppi_gpu_set_comm": (c_int, [c_void_p, c_int, c_int, _P(c_uint8)]),
    "mppi_gpu_set_comm_local": (c_int, [_P(c_void_p), c_int]),
    "mppi_gpu_step_local": (c_int, [_P(c_void_p), c_int, _d, _d]),
    "mppi_gpu_shard_info": (c_int, [c_void_p, _P(c_int32)]),
    "mppi_gpu_shard_plan": (c_int, [c_int, c_int, c_int, c_int, _P(c_int32)]),
    "mppi_gpu_profile_read_exchange": (c_int, [c_void_p, _d, _P(c_uint64), c_int]),
    "mppi_gpu_get_stream": (c_int, [c_void_p, _P(c_void_p)]),
    "mppi_gpu_launch_count": (c_int, [c_void_p, _P(c_uint64)]),
    "mppi_gpu_profile_enable": (c_int, [c_void_p, c_int]),
    "mppi_gpu_profile_read": (c_int, [c_void_p, _d, _P(c_uint64), c_int]),
    "mppi_gpu_kernel_variant": (c_int, [c_void_p, ctypes.c_char_p, c_int]),
    "mppi_gpu_fp32_peak_probe": (c_int, [c_int, _d, _d]),
    "mppi_gpu_pipe_peak_probe": (c_int, [c_int, _d, _d]),
    "mppi_workload_mlp_xavier": (c_int, [c_int, c_uint64, c_double, _d, _d, _d, _d, _d, _d]),
    "mppi_workload_ellipse_costmap": (c_int, [c_int, c_int, c_double, c_double, c_double, c_double,
                                              c_double, c_double, _P(c_float)]),
    "mppi_workload_initial_states": (c_int, [c_int, c_uint64, c_double, c_double, c_int, c_double,
                                             c_double, c_double, _d]),
    "mppi_sg_coefficients": (c_int, [c_int, c_int, _d]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libmppi_gpu.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA library is not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'` or `make -C paper_1707_02342_b200`)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.mppi_gpu_config_sizeof() != ctypes.sizeof(ConfigC):
        raise ImportError("mppi_gpu_config layout mismatch between mppi_gpu.h and the ctypes binding")
    _lib = lib
    return lib


def check(code: int) -> None:
    if code == MPPI_OK:
        return
    msg = load().mppi_gpu_last_error()
    msg = msg.decode() if msg else ""
    raise _ERRORS.get(code, MppiError)(code, msg)


def dptr(a):
    """double* of a C-contiguous float64 numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(_d)
