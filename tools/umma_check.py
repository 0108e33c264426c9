#!/usr/bin/env python3
"""A/B of the tcgen05 K1 (MPPI_KERNEL=umma) against the mma.sync K1 and the
float restatement: per-sample costs (rtol 1e-5), mpc_step plans, then timing."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def costs(kernel, K, T, noise="ref_splitmix"):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    import numpy as np
    from paper_1707_02342_b200 import workload
    from paper_1707_02342_b200.api import Controller
    if kernel:
        os.environ["MPPI_KERNEL"] = kernel
    w = workload.make("c1", samples=K, horizon_steps=T)
    g = Controller(w.params, w.bounds, w.sg, w.cost, hidden=32, precision="fp32", noise=noise)
    g.set_mlp(w.mlp)
    g.set_costmap(w.costmap)
    g.plan = np.random.default_rng(3).uniform(-0.4, 0.4, (T, 2))
    c = g.rollout_batch(w.x0[0])
    u = [g.mpc_step(w.x0[0]).tolist() for _ in range(3)]
    return {"variant": g.kernel_variant, "costs": c.tolist(), "plan": g.plan.tolist(), "u": u}


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        print(json.dumps(costs(sys.argv[2] if sys.argv[2] != "-" else None, int(sys.argv[3]), int(sys.argv[4]))))
        sys.exit(0)
    import numpy as np
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    for K, T in ((1024, 20), (4096, 100), (20000, 37)):
        res = {}
        for kern in ("umma", "-"):
            out = subprocess.run([sys.executable, __file__, "one", kern, str(K), str(T)], capture_output=True,
                                 text=True, timeout=240)
            if out.returncode != 0:
                print(kern, K, T, "FAILED", out.stderr[-1500:], flush=True)
                sys.exit(1)
            res[kern] = json.loads(out.stdout.strip().splitlines()[-1])
        a, b = np.array(res["umma"]["costs"]), np.array(res["-"]["costs"])
        rel = np.abs(a - b) / np.abs(b)
        pa, pb = np.array(res["umma"]["plan"]), np.array(res["-"]["plan"])
        print(json.dumps({"K": K, "T": T, "umma": res["umma"]["variant"][:40], "frac_rel_1e-5": float((rel <= 1e-5).mean()),
                          "max_rel": float(rel.max()), "jumps": int((np.abs(a - b) > 5000).sum()),
                          "plan_max_abs": float(np.abs(pa - pb).max())}), flush=True)
