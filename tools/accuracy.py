#!/usr/bin/env python3
"""Accuracy study of the fp32 K1 variants against the float / double oracle
(c0 workload): per-sample cost rel error (injected reference noise) and the
max |dU| of mpc_step over 5 receding-horizon iterations.  One JSON line per
variant; the variant is chosen by env (MPPI_KERNEL, MPPI_TC_MT,
MPPI_TC_PRODUCTS) in a fresh process per run."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one():
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    import numpy as np
    import oracle
    from paper_1707_02342_b200 import workload
    from paper_1707_02342_b200.api import Controller
    w = workload.make("c0")
    out = {}
    for noise in ("ref_splitmix", "philox"):
        for oprec in ("fp32", "fp64"):
            g = Controller(w.params, w.bounds, w.sg, w.cost, hidden=32, precision="fp32", noise=noise)
            o = oracle.OracleController(w.params, w.bounds, w.sg, w.cost, hidden=32, precision=oprec, noise=noise)
            o32 = oracle.OracleController(w.params, w.bounds, w.sg, w.cost, hidden=32, precision="fp32", noise=noise)
            for c in (g, o, o32):
                c.set_mlp(w.mlp)
                c.set_costmap(w.costmap)
            x = w.x0[0].copy()
            worst = worst32 = 0.0
            for it in range(5):
                g.mpc_step(x)
                o32.plan = o.plan
                o32.iteration = o.iteration
                o32.mpc_step(x, threads=os.cpu_count() or 1)
                uo = o.mpc_step(x, threads=os.cpu_count() or 1)
                worst = max(worst, float(np.max(np.abs(g.plan - o.plan))))
                worst32 = max(worst32, float(np.max(np.abs(o32.plan - o.plan))))
                g.plan = o.plan
                x = o.vehicle_step(x, uo)
            out[f"plan_max_abs_{noise}_vs_{oprec}_oracle"] = worst
            if oprec == "fp64":
                out[f"float_oracle_vs_double_oracle_{noise}"] = worst32
    eps, _ = oracle.sample_perturbations(w.params.samples, w.params.horizon_steps, w.params.sigma_diag,
                                         w.params.explore_fraction, w.params.seed, 0)
    U = np.random.default_rng(2).uniform(-0.3, 0.3, (w.params.horizon_steps, 2))
    res = {}
    for prec in ("fp32", "fp64"):
        g = Controller(w.params, w.bounds, w.sg, w.cost, hidden=32, precision="fp32", noise="injected")
        o = oracle.OracleController(w.params, w.bounds, w.sg, w.cost, hidden=32, precision=prec, noise="injected")
        for c in (g, o):
            c.set_mlp(w.mlp)
            c.set_costmap(w.costmap)
            c.plan = U
        dc = g.rollout_batch(w.x0[0], eps)
        oc = o.rollout_batch(w.x0[0], eps, threads=os.cpu_count() or 1)
        rel = np.abs(dc - oc) / np.maximum(np.abs(oc), 1e-30)
        res[prec] = {"frac_within_1e-5": float((rel <= 1e-5).mean()), "median_rel": float(np.median(rel)),
                     "p99_rel": float(np.quantile(rel, 0.99)), "big_jumps": int((np.abs(dc - oc) > 5000).sum())}
        out["kernel"] = g.kernel_variant
    out["costs_vs_oracle"] = res
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
        sys.exit(0)
    for env in ({"MPPI_KERNEL": "ws"}, {"MPPI_TC_MT": "1"}, {"MPPI_TC_MT": "2"}):
        e = dict(os.environ)
        for k in ("MPPI_KERNEL", "MPPI_TC_MT", "MPPI_TC_PRODUCTS"):
            e.pop(k, None)
        e.update(env)
        r = subprocess.run([sys.executable, __file__, "one"], env=e, capture_output=True, text=True)
        print(json.dumps(env), r.stdout.strip() or r.stderr[-2000:], flush=True)
