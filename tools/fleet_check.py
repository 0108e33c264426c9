#!/usr/bin/env python3
"""Per-sample-step cost of a fleet (C controllers x K samples) against one
controller with C*K samples, same kernel variant, closed loop with L2 flush."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_02342_b200 import workload  # noqa: E402
from paper_1707_02342_b200.api import Controller  # noqa: E402


def run(C, K, perturb, steps=10):
    w = workload.make("c3", samples=K, controllers=C)
    c = Controller(w.params, w.bounds, w.sg, w.cost, hidden=32, precision="fp32", noise="philox", n_controllers=C)
    c.set_mlp(w.mlp)
    c.set_costmap(w.costmap)
    if perturb and C > 1:
        c.perturb_fleet_costmaps(0.02, 7)
    x = w.x0 if C > 1 else w.x0[0]
    c.closed_loop_timed(x, 3, 256 << 20)
    c.profile_read(reset=True)
    ms = c.closed_loop_timed(x, steps, 256 << 20)
    c.profile(True)  # K1 durations: the event-bracketed graph, a separate pass
    c.profile_read(reset=True)
    c.closed_loop_timed(x, min(steps, 30), 256 << 20)
    k1, n = c.profile_read(reset=True)
    c.profile(False)
    u, xt = c.closed_loop(x, 2, traces=True)
    print(json.dumps({"C": C, "K": K, "perturb": perturb, "ms_per_iter": ms / steps, "k1_ms": k1 / max(n, 1),
                      "Gsteps_per_s": C * K * 100 / (ms / steps * 1e-3) / 1e9, "kernel": c.kernel_variant,
                      "x_finite": bool((xt == xt).all()), "u0": u[-1][0].tolist()}), flush=True)


for C, K, p in ((1, 262144, False), (128, 2048, False), (128, 2048, True), (512, 2048, True)):
    run(C, K, p)
