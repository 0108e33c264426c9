#!/usr/bin/env python3
"""Small runs of every device kernel family for the device-checks build
(tools/gpu_device_checks.sh; compute-sanitizer is closed on the GPU pool):
the sample-split and warp-pair K1s (c0 shape), the
single-warp K1 with eps' on chip and regenerated (MT=1 / MT=2), the tcgen05 K1 (one- and two-tile CTAs), the H=64 K1,
the FFMA2 and generic K1, fp64, the group merge, the tail (closed loop with
the device plant), a local 2-rank shard, the CEM rule, the bicycle model and
the parity kernels.  Short horizons keep the sanitizer run in minutes."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_02342_b200 import workload  # noqa: E402
from paper_1707_02342_b200.api import Controller, CostParams  # noqa: E402


def run(cfg, K, T, steps=2, **kw):
    w = workload.make(cfg, samples=K, horizon_steps=T)
    c = Controller(w.params, w.bounds, w.sg, w.cost, hidden=w.hidden, precision=kw.pop("precision", "fp32"),
                   noise=kw.pop("noise", "philox"), **kw)
    if kw.get("system") == "vehicle_bicycle":
        c.set_bicycle()
    else:
        c.set_mlp(w.mlp)
    c.set_costmap(w.costmap)
    for _ in range(steps):
        c.mpc_step(w.x0[0])
    c.closed_loop(w.x0[0], 2)
    print("ok", cfg, K, T, c.kernel_variant[:60], flush=True)
    return c, w


run("c0", 1920, 20)                                   # sample-split K1 (the c0 default)
run("c0", 1000, 21)                                   # sample-split K1, ragged last chunk, odd T
os.environ["MPPI_TC_SPLIT"] = "0"
os.environ["MPPI_TC_PAIR"] = "1"
run("c0", 1920, 20)                                   # warp-pair K1 (opt-in), one wave
del os.environ["MPPI_TC_PAIR"]
run("c0", 1920, 20)                                   # single-warp K1, predicated stage stores
del os.environ["MPPI_TC_SPLIT"]
run("c1", 4096, 20)                                   # MT=1, eps' on chip
os.environ["MPPI_TC_STORE"] = "0"
run("c1", 4096, 21)                                   # MT=1, regenerated eps', odd T
del os.environ["MPPI_TC_STORE"]
os.environ["MPPI_KERNEL"] = "mma"
run("c4", 40000, 10, steps=1)                         # MT=2 (mma.sync forced: tcgen05 is the default here)
del os.environ["MPPI_KERNEL"]
run("c4", 40000, 10, steps=1)                         # tcgen05 / TMEM K1
run("c2", 2048, 12)                                   # H=64
os.environ["MPPI_KERNEL"] = "umma"
run("c2", 2001, 12)                                   # tcgen05 K1 at H=64, ragged last tile
os.environ["MPPI_UMMA_TPC2"] = "1"
run("c2", 1800, 12)                                   # two-tile CTAs, a half-empty last CTA (15 tiles)
del os.environ["MPPI_UMMA_TPC2"]
del os.environ["MPPI_KERNEL"]
os.environ["MPPI_KERNEL"] = "ws"
run("c1", 2048, 12)                                   # FFMA2 K1
del os.environ["MPPI_KERNEL"]
run("c0", 600, 12, precision="fp64", noise="ref_splitmix")   # generic fp64
run("c0", 500, 12, system="vehicle_bicycle", precision="fp64")
c, w = run("c0", 700, 16, noise="ref_splitmix")
costs = c.rollout_batch(w.x0[0])
c.rollout_states(w.x0[0], 3)
c.update_plan(c.compute_weights(costs).weights)
wc = workload.make("c0", samples=600, horizon_steps=12)
cem = Controller(wc.params, wc.bounds, wc.sg, wc.cost, precision="fp32", weight_rule="cem")
cem.set_mlp(wc.mlp)
cem.set_costmap(wc.costmap)
cem.mpc_step(wc.x0[0])
wl = workload.make("c1", samples=3000, horizon_steps=12)
ranks = []
for _ in range(2):
    r = Controller(wl.params, wl.bounds, wl.sg, wl.cost, precision="fp32", noise="philox")
    r.set_mlp(wl.mlp)
    r.set_costmap(wl.costmap)
    ranks.append(r)
Controller.set_comm_local(ranks)
Controller.step_local(ranks, wl.x0[0])
wf = workload.make("c3", samples=256, horizon_steps=10, controllers=3)
f = Controller(wf.params, wf.bounds, wf.sg, wf.cost, precision="fp32", n_controllers=3)
f.set_mlp(wf.mlp)
f.set_costmap(wf.costmap)
f.perturb_fleet_costmaps(0.02, 5)
f.closed_loop(wf.x0, 2)
print("all ok")
