#!/usr/bin/env python3
"""Small closed-loop run for ncu captures: python tools/ncu_target.py CFG K [iters]
(kernel variant via MPPI_KERNEL / MPPI_WS_L / MPPI_WS_SMEM_W)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_02342_b200 import workload  # noqa: E402
from paper_1707_02342_b200.api import Controller  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
K = (int(sys.argv[2]) or None) if len(sys.argv) > 2 else None
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = workload.make(cfg, samples=K)
c = Controller(w.params, w.bounds, w.sg, w.cost, hidden=w.hidden, precision="fp32", noise="philox")
c.set_mlp(w.mlp)
c.set_costmap(w.costmap)
c.closed_loop(w.x0[0], iters, traces=False)
print("ok", c.kernel_variant)
