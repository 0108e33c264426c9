#!/usr/bin/env python3
"""Accuracy study of the fp32 K1 variants against the oracle.

For each variant (chosen by env in a fresh process: MPPI_KERNEL, MPPI_TC_PAIR,
MPPI_TC_W3_SHIFT) and workload (c0, c1): `iters` receding-horizon
iterations, the device and the oracle on the same plan and state every
iteration (reference splitmix64 noise), reporting per iteration the max |dU| of
the updated plan against
  * the float restatement (ascending-order MLP dot products, the default),
  * the float restatement with DESCENDING dot products — not a device
    comparison: the spread between the two oracle orders is the rounding
    envelope of a valid fp32 evaluation,
  * the double restatement (the reference arithmetic),
plus the per-sample cost relative errors against the float restatement.
One JSON line per (variant, workload)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(cfg, iters):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    import numpy as np
    import oracle
    from paper_1707_02342_b200 import workload
    from paper_1707_02342_b200.api import Controller
    oracle.load()
    w = workload.make(cfg)
    thr = os.cpu_count() or 1
    g = Controller(w.params, w.bounds, w.sg, w.cost, hidden=w.hidden, precision="fp32", noise="ref_splitmix")
    o32 = oracle.OracleController(w.params, w.bounds, w.sg, w.cost, hidden=w.hidden, precision="fp32",
                                  noise="ref_splitmix")
    o64 = oracle.OracleController(w.params, w.bounds, w.sg, w.cost, hidden=w.hidden, precision="fp64",
                                  noise="ref_splitmix")
    for c in (g, o32, o64):
        c.set_mlp(w.mlp)
        c.set_costmap(w.costmap)
    x = w.x0[0].copy()
    rows = []
    for it in range(iters):
        U, n = o64.plan, o64.iteration
        for c in (g, o32):
            c.plan = U
            c.iteration = n
        # costs on this plan (the batch the update uses)
        dc = g.rollout_batch(x)
        oc = o32.rollout_batch(x, threads=thr)
        rel = np.abs(dc - oc) / np.maximum(np.abs(oc), 1e-30)
        for c in (g, o32):
            c.plan = U
            c.iteration = n
        g.mpc_step(x)
        o32.mpc_step(x, threads=thr)
        p_dev, p_f = g.plan, o32.plan
        oracle.load().oracle_set_mlp_order(1)
        o32.plan = U
        o32.iteration = n
        o32.mpc_step(x, threads=thr)
        p_rev = o32.plan
        oracle.load().oracle_set_mlp_order(0)
        u = o64.mpc_step(x, threads=thr)
        p_d = o64.plan
        rows.append({"it": it, "dev_vs_f32": float(np.abs(p_dev - p_f).max()),
                     "f32_rev_vs_f32": float(np.abs(p_rev - p_f).max()),
                     "dev_vs_f64": float(np.abs(p_dev - p_d).max()), "f32_vs_f64": float(np.abs(p_f - p_d).max()),
                     "cost_rel_p50": float(np.median(rel)), "cost_rel_p99": float(np.quantile(rel, 0.99)),
                     "cost_rel_max": float(rel.max()), "cost_jumps": int((np.abs(dc - oc) > 5000).sum())})
        x = o64.vehicle_step(x, u)
    agg = {k: max(r[k] for r in rows) for k in ("dev_vs_f32", "f32_rev_vs_f32", "dev_vs_f64", "f32_vs_f64",
                                                 "cost_rel_p99")}
    print(json.dumps({"cfg": cfg, "kernel": g.kernel_variant, "max": agg, "per_iteration": rows}), flush=True)


VARIANTS = [{}, {"MPPI_TC_W3_SHIFT": "0"}, {"MPPI_TC_PAIR": "1", "MPPI_TC_SPLIT": "0"}, {"MPPI_KERNEL": "ws"}]

if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "one":
        one(sys.argv[2], int(sys.argv[3]))
        sys.exit(0)
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c0", "c1"]
    for env in VARIANTS:
        for cfg in cfgs:
            e = dict(os.environ)
            for k in ("MPPI_KERNEL", "MPPI_TC_PAIR", "MPPI_TC_SPLIT", "MPPI_TC_W3_SHIFT"):
                e.pop(k, None)
            e.update(env)
            r = subprocess.run([sys.executable, __file__, "one", cfg, "6" if cfg == "c0" else "3"], env=e,
                               capture_output=True, text=True)
            print(json.dumps({"env": env, "result": json.loads(r.stdout.strip().splitlines()[-1])
                              if r.returncode == 0 else r.stderr[-1500:]}), flush=True)
