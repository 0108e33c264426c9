"""The reference's file and config formats on the host side,
so its experiment files and weight files drive the B200 controller unchanged.

* ``sampling_params_from_json`` / ``sampling_params_to_json``: the
  ``"sampling"`` object (config.cpp:26-70): lambda, gamma, sigma_diag (variances),
  horizon_steps, dt, samples, explore_fraction (default 0.01), seed (default 0),
  optional base_mean (T x m rows, the initial plan).
* ``load_experiment``: the controller-relevant part of an ExperimentConfig JSON
  (config.cpp:139-248): "sampling", "controller" (weight_rule it|cem, delta,
  sg_window, sg_degree, bounds_lower/upper, model, theta_file, mlp_file,
  terminal_cost) and "costs" (alpha_track, alpha_speed, alpha_stab, v_des_mps,
  impulse, decay, boundary_threshold, slip_limit_rad), with the reference's
  validation (config.cpp:113-137).  The simulator, vehicle-truth, map
  generator and run sections are outside the hot path and are ignored.
* ``load_theta`` / ``save_theta``: the basis-model coefficient file (25 rows of
  4, dynamics.cpp:230-254).  The MLP and costmap files are ``MlpWeights.load /
  save`` and ``CostMap.load / save`` (api.py).
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .api import (ControlBounds, Controller, CostMap, CostParams, InvalidArgument, MlpWeights, SamplingParams,
                  SGFilter)


def _invalid(msg: str) -> InvalidArgument:
    return InvalidArgument(_lib.MPPI_ERR_INVALID_ARGUMENT, msg)


def _sampling_from_obj(j: dict):
    try:
        p = SamplingParams(samples=int(j["samples"]), horizon_steps=int(j["horizon_steps"]), dt=float(j["dt"]),
                           sigma_diag=tuple(float(v) for v in j["sigma_diag"]), lambda_=float(j["lambda"]),
                           gamma=float(j["gamma"]), explore_fraction=float(j.get("explore_fraction", 0.01)),
                           seed=int(j.get("seed", 0)))
    except KeyError as e:  # json::at throws on a missing key
        raise _invalid(f"sampling: missing key {e.args[0]!r}") from None
    base = None
    if "base_mean" in j:
        base = np.array(j["base_mean"], dtype=np.float64)
        if base.ndim != 2 or base.shape[1] != len(p.sigma_diag):
            raise _invalid("sampling: base_mean must be T x m rows")
    _validate_sampling(p, base)
    return p, base


def _validate_sampling(p: SamplingParams, base) -> None:
    """SamplingParams::validate (types.hpp:105-122)."""
    if p.samples < 1 or p.horizon_steps < 1:
        raise _invalid("SamplingParams: samples and horizon_steps must be >= 1")
    if not p.dt > 0:
        raise _invalid("SamplingParams: dt must be > 0")
    if any(not (s > 0 and np.isfinite(s)) for s in p.sigma_diag):
        raise _invalid("SamplingParams: sigma_diag entries must be finite and > 0")
    if not p.lambda_ > 0:
        raise _invalid("SamplingParams: lambda must be > 0")
    if not p.gamma >= 0:
        raise _invalid("SamplingParams: gamma must be >= 0")
    if not 0.0 <= p.explore_fraction < 1.0:
        raise _invalid("SamplingParams: explore_fraction must be in [0, 1)")
    if base is not None and base.shape[0] != p.horizon_steps:
        raise _invalid("SamplingParams: base_mean must have horizon_steps rows")


def sampling_params_from_json(text: str):
    """sampling_params_from_json (config.cpp:84-86): (SamplingParams, base_mean or None)."""
    return _sampling_from_obj(json.loads(text))


def sampling_params_to_json(p: SamplingParams, base_mean=None) -> str:
    """sampling_params_to_json (config.cpp:80-82), same keys and layout."""
    j = {"lambda": p.lambda_, "gamma": p.gamma, "sigma_diag": list(p.sigma_diag), "horizon_steps": p.horizon_steps,
         "dt": p.dt, "samples": p.samples, "explore_fraction": p.explore_fraction, "seed": p.seed}
    if base_mean is not None:
        j["base_mean"] = np.asarray(base_mean, dtype=np.float64).tolist()
    return json.dumps(j, indent=2) + "\n"


@dataclass
class ExperimentSpec:
    """The hot-path part of ExperimentConfig (config.hpp)."""
    params: SamplingParams
    bounds: ControlBounds
    sg: Optional[SGFilter]
    cost: CostParams
    weight_rule: str = "it"
    delta: float = 0.8
    with_terminal: bool = True
    model: str = "truth"
    theta_file: str = ""
    mlp_file: str = ""
    base_mean: Optional[np.ndarray] = None

    def controller(self, **kw) -> Controller:
        """make_controller_state + make_vehicle_system on the device.  The learned
        controller models load their weight files (relative to the config's
        directory); the reference's "truth" controller model (the bicycle
        plant) is not a device model."""
        if self.model == "basis":
            c = Controller(self.params, self.bounds, self.sg, self.cost, system="vehicle_basis",
                           weight_rule=self.weight_rule, cem_delta=self.delta, with_terminal=self.with_terminal, **kw)
            c.set_basis(load_theta(self.theta_file))
        elif self.model == "mlp":
            w = MlpWeights.load(self.mlp_file)
            c = Controller(self.params, self.bounds, self.sg, self.cost, hidden=w.hidden,
                           weight_rule=self.weight_rule, cem_delta=self.delta, with_terminal=self.with_terminal, **kw)
            c.set_mlp(w)
        else:
            raise _invalid(f"controller model {self.model!r} has no device implementation (basis, mlp)")
        if self.base_mean is not None:
            c.set_plan(self.base_mean)
        return c


def experiment_from_json(text: str, base_dir: str = ".") -> ExperimentSpec:
    """experiment_config_from_json (config.cpp:139-248), hot-path sections, with
    ExperimentConfig::validate's checks on them (config.cpp:113-137)."""
    j = json.loads(text)
    if "sampling" not in j:
        raise _invalid("config: missing 'sampling'")
    params, base = _sampling_from_obj(j["sampling"])
    spec = ExperimentSpec(params=params, bounds=ControlBounds(), sg=SGFilter(9, 3), cost=CostParams(), base_mean=base)
    c = j.get("controller", {})
    spec.weight_rule = c.get("weight_rule", "it")
    if spec.weight_rule not in ("it", "cem"):
        raise _invalid(f"weight_rule must be 'it' or 'cem', got: {spec.weight_rule}")
    spec.delta = float(c.get("delta", 0.8))
    window, degree = int(c.get("sg_window", 9)), int(c.get("sg_degree", 3))
    if window != 0 and (window < 3 or window % 2 == 0 or degree >= window):
        raise _invalid("config: sg_window must be 0 (off) or odd with degree < window")
    spec.sg = SGFilter(window, degree) if window != 0 else None
    if "bounds_lower" in c:
        spec.bounds = ControlBounds(tuple(c["bounds_lower"]), tuple(c["bounds_upper"]))
    spec.model = c.get("model", "truth")
    spec.theta_file = os.path.join(base_dir, c["theta_file"]) if c.get("theta_file") else ""
    spec.mlp_file = os.path.join(base_dir, c["mlp_file"]) if c.get("mlp_file") else ""
    spec.with_terminal = bool(c.get("terminal_cost", True))
    k = j.get("costs", {})
    d = CostParams()
    spec.cost = CostParams(alpha_track=k.get("alpha_track", d.alpha_track), alpha_speed=k.get("alpha_speed", d.alpha_speed),
                           alpha_stab=k.get("alpha_stab", d.alpha_stab), v_des=k.get("v_des_mps", d.v_des),
                           impulse=k.get("impulse", d.impulse), decay=k.get("decay", d.decay),
                           boundary_threshold=k.get("boundary_threshold", d.boundary_threshold),
                           slip_limit=k.get("slip_limit_rad", d.slip_limit))
    if params.gamma > params.lambda_:
        raise _invalid("config: gamma must satisfy 0 <= gamma <= lambda (base mixing in [0, 1])")
    if (spec.model == "basis" and not spec.theta_file) or (spec.model == "mlp" and not spec.mlp_file):
        raise _invalid("config: learned controller models need a weights file")
    return spec


def load_experiment(path: str) -> ExperimentSpec:
    """load_experiment_config (config.cpp:333-335)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError as e:
        raise RuntimeError(f"cannot open config file: {path}") from e
    return experiment_from_json(text, os.path.dirname(os.path.abspath(path)))


def load_theta(path: str) -> np.ndarray:
    """load_theta (dynamics.cpp:230-244): 25 x 4 whitespace-separated values."""
    try:
        with open(path) as f:
            tok = f.read().split()
    except OSError as e:
        raise RuntimeError(f"cannot open file: {path}") from e
    if len(tok) < 100:
        raise RuntimeError(f"load_theta: expected 25x4 values in {path}")
    th = np.array([float(t) for t in tok[:100]]).reshape(25, 4)
    if not np.all(np.isfinite(th)):
        raise RuntimeError(f"load_theta: non-finite entry in {path}")
    return th


def save_theta(theta, path: str) -> None:
    """save_theta (dynamics.cpp:246-254): one basis row per line, %.17g."""
    th = np.asarray(theta, dtype=np.float64).reshape(25, 4)
    with open(path, "w") as f:
        for row in th:
            f.write(" ".join(repr(float(v)) for v in row) + "\n")


__all__ = ["sampling_params_from_json", "sampling_params_to_json", "ExperimentSpec", "experiment_from_json",
           "load_experiment", "load_theta", "save_theta", "CostMap"]
