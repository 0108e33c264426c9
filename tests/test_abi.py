"""CPU checks of the C-ABI library: it loads, exports every symbol the header
declares, its config layout matches the bindings, and the host-side pieces
(SG kernel, workload generators, error mapping) behave.  No device compute."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
from paper_1707_02342_b200 import _lib, api, workload

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mppi_gpu.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b((?:mppi_gpu|mppi_workload|mppi_sg|mppi_sim|mppi_bicycle|mppi_brush)_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 40
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b[TW] (\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        assert hasattr(lib, s)
    # the ctypes binding covers the whole header
    assert set(syms) <= set(_lib._SIGNATURES), set(syms) - set(_lib._SIGNATURES)


def test_config_layout_and_defaults():
    lib = _lib.load()
    assert lib.mppi_gpu_config_sizeof() == ctypes.sizeof(_lib.ConfigC)
    assert lib.mppi_gpu_abi_version() == 2
    cfg = _lib.ConfigC()
    lib.mppi_gpu_config_init(ctypes.byref(cfg))
    # SamplingParams{} (types.hpp:92-101), SGFilter{9,3}, CostParams{} (costs.hpp:46-54)
    assert (cfg.samples, cfg.horizon_steps, cfg.dt, cfg.lambda_, cfg.gamma) == (1200, 80, 0.025, 12.5, 0.1)
    assert list(cfg.sigma_diag) == [0.0306, 0.0506] and cfg.explore_fraction == 0.01
    assert (cfg.sg_window, cfg.sg_degree) == (9, 3)
    assert (cfg.cost.alpha_track, cfg.cost.alpha_speed, cfg.cost.alpha_stab) == (100.0, 4.25, 10.0)
    assert (cfg.cost.impulse, cfg.cost.decay, cfg.cost.boundary_threshold, cfg.cost.slip_limit) == \
        (10000.0, 0.9, 0.99, 0.75)


def test_sg_coefficients_match_oracle():
    for window in (3, 5, 7, 9, 11, 21):
        for degree in range(window):
            assert np.allclose(api.sg_coefficients(window, degree), oracle.sg_coefficients(window, degree),
                               rtol=0, atol=1e-13)
    assert np.allclose(api.sg_coefficients(9, 2) * 231, [-21, 14, 39, 54, 59, 54, 39, 14, -21], atol=1e-10)
    with pytest.raises(ValueError):
        api.sg_coefficients(4, 2)


def test_workload_generators():
    m = workload.track_map()
    assert m.values.shape == (2000, 2000) and m.values.dtype == np.float32
    assert m.values.min() >= 0 and m.values.max() == pytest.approx(2.5)
    # centreline points of the 40 x 25 ellipse have h ~ 0, boundaries h ~ 1
    for phi in np.linspace(0, 2 * np.pi, 13):
        px, py = 40 * np.cos(phi), 25 * np.sin(phi)
        assert oracle.costmap_lookup(m.values.astype(np.float64), -50, -50, 0.05, px, py) < 0.02
    assert oracle.costmap_lookup(m.values.astype(np.float64), -50, -50, 0.05, 43.0, 0.0) == pytest.approx(1.0,
                                                                                                          abs=0.02)
    a = api.MlpWeights.xavier(32, 5)
    b = api.MlpWeights.xavier(32, 5)
    assert np.array_equal(a.w2, b.w2) and np.abs(a.w1).max() <= np.sqrt(6 / 38)
    assert np.abs(a.w3).max() <= 0.1 * np.sqrt(6 / 36) and np.all(a.b1 == 0)
    x = api.initial_states(64, 3)
    assert x.shape == (64, 7) and np.all((x[:, 4] >= 3) & (x[:, 4] <= 8))
    r = (x[:, 0] / 40) ** 2 + (x[:, 1] / 25) ** 2
    assert np.allclose(r, 1.0, atol=1e-3)
    assert abs(x[:, 3].std() - 0.05) < 0.02


def test_mlp_and_costmap_file_round_trip(tmp_path):
    w = api.MlpWeights.xavier(64, 1)
    w.save(str(tmp_path / "w.txt"))
    back = api.MlpWeights.load(str(tmp_path / "w.txt"))
    assert back.hidden == 64 and np.array_equal(back.w2, w.w2)
    m = api.CostMap(np.random.default_rng(0).uniform(0, 2.5, (3, 4)), -1.0, 2.0, 0.5)
    m.save(str(tmp_path / "m.txt"))
    mb = api.CostMap.load(str(tmp_path / "m.txt"))
    assert np.array_equal(mb.values, m.values) and (mb.x0, mb.y0, mb.resolution) == (-1.0, 2.0, 0.5)
    with pytest.raises(RuntimeError):
        api.CostMap.load(str(tmp_path / "missing.txt"))


@pytest.mark.skipif(api.device_count() > 0, reason="checks the no-device error path")
def test_no_cpu_fallback_without_device():
    with pytest.raises(api.DeviceError):
        api.Controller(api.SamplingParams())


def test_invalid_config_is_rejected_before_device_use():
    # validation is reported as InvalidArgument even when no device exists
    lib = _lib.load()
    cfg = api.make_config(api.SamplingParams(samples=0))
    h = ctypes.c_void_p()
    code = lib.mppi_gpu_create(ctypes.byref(cfg), ctypes.byref(h))
    assert code == _lib.MPPI_ERR_INVALID_ARGUMENT
    assert b"samples" in lib.mppi_gpu_last_error()


def build_binding_check(tmp_dir):
    """g++ the header-only C++ binding (include/mppi_gpu.hpp) against the library."""
    exe = os.path.join(tmp_dir, "binding_check")
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "binding_check.cpp"), "-L", libdir, "-lmppi_gpu",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    return exe


@pytest.mark.skipif(api.device_count() > 0, reason="checks the no-device error path")
def test_cpp_binding_exception_mapping(tmp_path):
    out = subprocess.run([build_binding_check(str(tmp_path))], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "invalid_argument mapping ok" in out.stdout and "no-device runtime_error ok" in out.stdout


@pytest.mark.gpu
def test_cpp_binding_on_device(tmp_path):
    out = subprocess.run([build_binding_check(str(tmp_path))], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "device binding ok" in out.stdout and "size checks ok" in out.stdout
