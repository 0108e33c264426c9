"""The reference's config / weight-file formats on the host side (SURVEY
§8(f) row 4): the "sampling" JSON (config.cpp:26-70), the hot-path sections of
an experiment JSON (config.cpp:139-248) with its validation (config.cpp:113-137),
and the Theta file (dynamics.cpp:230-254)."""
import json
import os

import numpy as np
import pytest

from paper_1707_02342_b200 import config, workload
from paper_1707_02342_b200.api import InvalidArgument, MlpWeights, SamplingParams

REF_CONFIG = "/root/reference/proj/configs/oval_it.json"

EXPERIMENT = {
    "sampling": {"lambda": 6.66, "gamma": 0.666, "sigma_diag": [0.09, 0.1225], "horizon_steps": 50, "dt": 0.02,
                 "samples": 2048, "seed": 11},
    "controller": {"weight_rule": "cem", "delta": 0.75, "sg_window": 9, "sg_degree": 2,
                   "bounds_lower": [-0.8, -1.0], "bounds_upper": [0.8, 1.0], "model": "basis",
                   "theta_file": "theta.txt", "terminal_cost": False},
    "costs": {"alpha_track": 200.0, "alpha_speed": 1.0, "alpha_stab": 0.0, "v_des_mps": 6.0, "impulse": 50.0,
              "decay": 1.0, "boundary_threshold": 1.0},
    "sim": {"episode_s": 10.0},
}


def test_sampling_json_round_trip_and_defaults():
    p = SamplingParams(samples=1920, horizon_steps=100, dt=0.02, sigma_diag=(0.09, 0.1225), lambda_=6.66,
                       gamma=0.666, explore_fraction=0.02, seed=7)
    base = np.random.default_rng(0).normal(size=(100, 2))
    q, b = config.sampling_params_from_json(config.sampling_params_to_json(p, base))
    assert q == p and np.array_equal(b, base)
    j = json.loads(config.sampling_params_to_json(p))
    del j["explore_fraction"], j["seed"]
    q, b = config.sampling_params_from_json(json.dumps(j))
    assert q.explore_fraction == 0.01 and q.seed == 0 and b is None  # config.cpp:56-57
    del j["dt"]
    with pytest.raises(InvalidArgument):
        config.sampling_params_from_json(json.dumps(j))
    j = json.loads(config.sampling_params_to_json(p))
    j["lambda"] = 0.0
    with pytest.raises(InvalidArgument):
        config.sampling_params_from_json(json.dumps(j))


def test_experiment_sections_and_validation(tmp_path):
    spec = config.experiment_from_json(json.dumps(EXPERIMENT), str(tmp_path))
    assert spec.params.samples == 2048 and spec.params.explore_fraction == 0.01
    assert spec.weight_rule == "cem" and spec.delta == 0.75 and spec.with_terminal is False
    assert (spec.sg.window, spec.sg.degree) == (9, 2)
    assert spec.bounds.lower == (-0.8, -1.0) and spec.cost.alpha_track == 200.0 and spec.cost.impulse == 50.0
    assert spec.cost.slip_limit == 0.75  # CostParams default (costs.hpp:46-54)
    assert spec.theta_file == os.path.join(str(tmp_path), "theta.txt")
    for key, val in (("gamma", 7.0),):
        bad = json.loads(json.dumps(EXPERIMENT))
        bad["sampling"][key] = val
        with pytest.raises(InvalidArgument, match="gamma"):
            config.experiment_from_json(json.dumps(bad))
    bad = json.loads(json.dumps(EXPERIMENT))
    bad["controller"]["sg_window"] = 8
    with pytest.raises(InvalidArgument, match="sg_window"):
        config.experiment_from_json(json.dumps(bad))
    bad = json.loads(json.dumps(EXPERIMENT))
    del bad["controller"]["theta_file"]
    with pytest.raises(InvalidArgument, match="weights file"):
        config.experiment_from_json(json.dumps(bad))
    bad = json.loads(json.dumps(EXPERIMENT))
    bad["controller"]["weight_rule"] = "pi"
    with pytest.raises(InvalidArgument, match="weight_rule"):
        config.experiment_from_json(json.dumps(bad))
    bad = json.loads(json.dumps(EXPERIMENT))
    bad["controller"]["sg_window"] = 0
    assert config.experiment_from_json(json.dumps(bad)).sg is None


@pytest.mark.skipif(not os.path.exists(REF_CONFIG), reason="reference tree not mounted")
def test_reference_experiment_file_parses():
    spec = config.load_experiment(REF_CONFIG)
    assert spec.params.samples == 512 and spec.params.lambda_ == 12.5 and spec.params.horizon_steps == 80
    assert spec.params.sigma_diag == (0.0306, 0.0506) and (spec.sg.window, spec.sg.degree) == (9, 3)
    assert spec.model == "truth" and spec.weight_rule == "it" and spec.cost.v_des == 6.0


def test_theta_file_round_trip(tmp_path):
    th = workload.basis_theta()
    config.save_theta(th, str(tmp_path / "t.txt"))
    assert np.array_equal(config.load_theta(str(tmp_path / "t.txt")), th)
    (tmp_path / "short.txt").write_text("1 2 3\n")
    with pytest.raises(RuntimeError, match="25x4"):
        config.load_theta(str(tmp_path / "short.txt"))
    (tmp_path / "nan.txt").write_text(" ".join(["nan"] + ["0"] * 99))
    with pytest.raises(RuntimeError, match="non-finite"):
        config.load_theta(str(tmp_path / "nan.txt"))


@pytest.mark.gpu
def test_experiment_drives_device_controller(tmp_path):
    config.save_theta(workload.basis_theta(), str(tmp_path / "theta.txt"))
    path = tmp_path / "exp.json"
    path.write_text(json.dumps(EXPERIMENT))
    spec = config.load_experiment(str(path))
    ctl = spec.controller()
    ctl.set_costmap(workload.track_map())
    u = ctl.mpc_step(workload.make("c0").x0[0])
    assert np.all(np.isfinite(u)) and np.all(np.abs(u) <= 1.0) and ctl.iteration == 1
    exp = json.loads(json.dumps(EXPERIMENT))
    exp["controller"].update(model="mlp", mlp_file="net.txt", weight_rule="it")
    MlpWeights.xavier(32, 3, 0.1).save(str(tmp_path / "net.txt"))
    path.write_text(json.dumps(exp))
    ctl = config.load_experiment(str(path)).controller()
    ctl.set_costmap(workload.track_map())
    assert np.all(np.isfinite(ctl.mpc_step(workload.make("c0").x0[0])))
