#!/usr/bin/env python3
"""Kernel-variant sweep: device ms per IT-MPPI iteration (closed loop, L2
flushed between iterations) for each K1 variant, on the BASELINE configs."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(cfg, K, variant, L, steps=30, sw=1):
    if variant != "env":  # "env": keep the caller's MPPI_* selection
        for v in ("MPPI_KERNEL", "MPPI_WS_L", "MPPI_WS_SMEM_W", "MPPI_TC_MT"):
            os.environ.pop(v, None)
    if variant == "env":
        pass
    elif variant == "generic":
        os.environ["MPPI_KERNEL"] = "generic"
    elif variant == "tc":
        if L:
            os.environ["MPPI_TC_MT"] = str(L)
    else:
        os.environ["MPPI_KERNEL"] = "ws"
        if L:
            os.environ["MPPI_WS_L"] = str(L)
        os.environ["MPPI_WS_SMEM_W"] = str(sw)
    from paper_1707_02342_b200 import workload
    from paper_1707_02342_b200.api import Controller
    w = workload.make(cfg, samples=K)
    c = Controller(w.params, w.bounds, w.sg, w.cost, hidden=w.hidden, precision="fp32", noise="philox")
    c.set_mlp(w.mlp)
    c.set_costmap(w.costmap)
    c.closed_loop_timed(w.x0[0], 5, 256 << 20)
    c.profile_read(reset=True)
    ms = c.closed_loop_timed(w.x0[0], steps, 256 << 20)
    c.profile(True)  # K1 durations: the event-bracketed graph, a separate pass
    c.profile_read(reset=True)
    c.closed_loop_timed(w.x0[0], min(steps, 30), 256 << 20)
    k1_ms, n = c.profile_read(reset=True)
    c.profile(False)
    k1 = k1_ms / max(n, 1)
    T = w.params.horizon_steps
    fl = K * T * workload.flops_per_sample_step(w.hidden)
    out = {"cfg": cfg, "K": K, "T": T, "H": w.hidden, "variant": c.kernel_variant, "ms_per_iter": ms / steps,
           "k1_ms": k1, "k1_tflops": fl / (k1 * 1e-3) / 1e12 if k1 > 0 else None,
           "Gsteps_per_s": K * T / (ms / steps * 1e-3) / 1e9}
    print(json.dumps(out), flush=True)
    c.close()


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    cases = []
    if which == "tail":
        for cfg, K in (("c1", 16384), ("c0", 1920), ("c4", 262144)):
            for tail in ("off", "split", "fused"):
                os.environ["MPPI_TAIL"] = tail
                r = subprocess.run([sys.executable, __file__, "one", cfg, str(K), "tc", "0"], capture_output=True,
                                   text=True, env=dict(os.environ))
                print(tail, r.stdout.strip() or r.stderr[-500:], flush=True)
        sys.exit(0)
    if which == "envs":
        # python tools/sweep.py envs '[["c1",16384,{"MPPI_TC_STORE":"0"}], ...]'
        for cfg, K, env in json.loads(sys.argv[2]):
            e = dict(os.environ)
            e.update(env)
            r = subprocess.run([sys.executable, __file__, "one", cfg, str(K), "env", "0"], capture_output=True,
                               text=True, env=e)
            print(json.dumps(env), r.stdout.strip() or r.stderr[-500:], flush=True)
        sys.exit(0)
    if which == "one":
        run(sys.argv[2], int(sys.argv[3]), sys.argv[4], int(sys.argv[5]), steps=30)
        sys.exit(0)
    if which == "tc":
        for cfg, K in (("c1", 16384), ("c0", 1920), ("c4", 262144), ("c4", 1048576)):
            for variant, L in (("tc", 1), ("tc", 2), ("ws", 0)):
                run(cfg, K, variant, L, steps=10 if K >= 262144 else 30)
        sys.exit(0)
    for cfg, K in (("c1", 16384), ("c0", 1920), ("c2", 65536), ("c4", 262144)):
        for variant, L, sw in (("generic", 0, 0), ("ws", 1, 0), ("ws", 1, 1), ("ws", 2, 1), ("ws", 4, 1),
                               ("ws", 8, 1), ("ws", 2, 0), ("ws", 4, 0)):
            if cfg == "c2" and variant == "ws" and L == 1:
                continue
            if K >= 262144 and variant == "generic":
                continue
            cases.append((cfg, K, variant, L, sw))
    for cfg, K, variant, L, sw in cases:
        if which != "all" and cfg != which:
            continue
        try:
            run(cfg, K, variant, L, steps=10 if K >= 262144 else 30, sw=sw)
        except Exception as e:  # keep sweeping
            print(json.dumps({"cfg": cfg, "K": K, "variant": variant, "L": L, "error": str(e)}), flush=True)
