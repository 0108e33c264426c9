#!/usr/bin/env python3
"""Benchmark of the B200 IT-MPPI hot path (one IT-MPPI iteration = one step).

Workload (BASELINE.json configs[1], "c1"): K = 16384 samples, T = 100, 6-32-32-4
tanh MLP vehicle, 2000 x 2000 elliptical-track costmap, receding horizon with
the device plant; all inputs synthetic from a seed (workload.py).  With
``--gpus N`` the samples of the controller are sharded over N ranks, one
process per GPU (bench.py launches them itself through torch.distributed.run
unless it already runs under torchrun): one NCCL all-gather of the fixed group
rows per iteration (group.cuh).  ``value`` is whole-job sample-timesteps/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl ours|reference]

``--impl reference`` times the reference's own algorithm on the host cores:
oracle/build/mppi_ref_bench, the double-precision restatement of
controller.cpp:55-148 with the reference sampler and its std::thread chunks
(the reference itself cannot be built here: Eigen3 is absent).  That arm
imports nothing from the product package and loads no CUDA library.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))

METRIC = "MPPI iteration latency (ms) and rollout sample-timesteps/sec at 1/2/4/8 B200"
UNIT = "sample-timesteps/s"
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2
REF_BENCH = os.path.join(ROOT, "oracle", "build", "mppi_ref_bench")
SEED = 1707_02342

# BASELINE.json configs as plain data (the same table as
# paper_1707_02342_b200/workload.py CONFIGS, checked by
# tests/test_bench_contract.py): the reference arm reads this copy so that it
# imports nothing from the product package.
BENCH_CONFIGS = {
    "c0": dict(samples=1920, horizon_steps=100, hidden=32, controllers=1),
    "c1": dict(samples=16384, horizon_steps=100, hidden=32, controllers=1),
    "c2": dict(samples=65536, horizon_steps=150, hidden=64, controllers=1),
    "c3": dict(samples=2048, horizon_steps=100, hidden=32, controllers=512),
    "c4": dict(samples=1024, horizon_steps=100, hidden=32, controllers=1),
}
SAMPLING = dict(dt=0.02, sigma0=0.3 ** 2, sigma1=0.35 ** 2, lambda_=6.66, gamma=0.1 * 6.66, explore=0.01,
                sg_window=9, sg_degree=2)
# CostParams.baseline(): 200 h + (v_x - 6)^2 + 10000 [h > 1 or |roll| > 0.6]
BASELINE_COST = (200.0, 1.0, 0.0, 6.0, 0.0, 1.0, 1.0, 0.75, 10000.0, 1.0, 0.6)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c1", choices=sorted(BENCH_CONFIGS))
    ap.add_argument("--samples", type=int, default=None, help="override K (c4 sweep)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def workload_shape(args):
    c = dict(BENCH_CONFIGS[args.config])
    if args.samples is not None:
        c["samples"] = args.samples
    return c


def config_dict(args, world):
    """The `config` object of both arms (same keys and values)."""
    c = workload_shape(args)
    K, T, H, C = c["samples"], c["horizon_steps"], c["hidden"], c["controllers"]
    fleet = C > 1
    return {"workload": f"{args.config}: IT-MPPI iteration, K={K}, T={T}, H={H}, MLP vehicle, receding horizon"
                        + (f", fleet of {C} controllers (perturbed maps)" if fleet else ""),
            "samples": K, "horizon": T, "hidden": H, "controllers": C,
            "parallelism": (f"{C // world} independent controllers per GPU on {world} GPU(s), no communication"
                            if fleet else f"samples sharded over {world} GPU(s)"),
            "l2": "flushed between timed iterations (256 MiB memset, excluded from timing)"}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------------- CPU arm ---
def ref_bench(shape, threads, steps, warmup):
    """Run oracle/build/mppi_ref_bench (reference algorithm, fp64, host cores)."""
    if not os.path.exists(REF_BENCH):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
    s = SAMPLING
    cmd = [REF_BENCH, "--samples", str(shape["samples"]), "--horizon", str(shape["horizon_steps"]),
           "--hidden", str(shape["hidden"]), "--threads", ",".join(str(t) for t in threads), "--steps", str(steps),
           "--warmup", str(warmup), "--dt", repr(s["dt"]), "--lambda", repr(s["lambda_"]), "--gamma",
           repr(s["gamma"]), "--sigma0", repr(s["sigma0"]), "--sigma1", repr(s["sigma1"]), "--explore",
           repr(s["explore"]), "--seed", str(SEED), "--sg-window", str(s["sg_window"]), "--sg-degree",
           str(s["sg_degree"]), "--cost", ",".join(repr(v) for v in BASELINE_COST)]
    out = subprocess.run(cmd, check=True, capture_output=True, text=True)
    return json.loads(out.stdout)


def cpu_sample_text(shape, run):
    fleet = shape["controllers"] > 1
    return (f"{run['steps']} timed mpc_step calls after {run['warmup']} warm-up calls (steady_clock, median; "
            f"acceptance.cpp:381-389) on the FULL K={shape['samples']}, T={shape['horizon_steps']}, "
            f"H={shape['hidden']}"
            + (" (one controller of the fleet: the CPU runs controllers one after another)" if fleet else "")
            + f", fp64, reference splitmix64 noise, {run['threads']} std::threads per call; reference algorithm "
              "restated in oracle/mppi_oracle.cpp (the reference needs Eigen3, absent)")


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    shape = workload_shape(args)
    threads = cpu_threads()
    res = ref_bench(shape, [threads], args.steps, args.warmup)
    run = res["runs"][0]
    K, T = shape["samples"], shape["horizon_steps"]
    value = K * T / (run["median_ms"] * 1e-3)
    ms = sorted(run["ms"])
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": run["median_ms"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Xavier MLP, 2000x2000 ellipse map, "
                                                          "reference splitmix64 noise)",
            "impl": "reference", "config": config_dict(args, world),
            "latency_ms": {"p50": float(np.percentile(ms, 50)), "p99": float(np.percentile(ms, 99)),
                           "mean": float(np.mean(ms))},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": run["threads"], "kind": "port",
                             "sample": cpu_sample_text(shape, run)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU arm -----
class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML every few ms during the
    timed region (nvidia-smi itself is too slow for a sub-second region; it
    is the fallback)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, device, period_s=0.002):
        self.device = device
        self.period = period_s
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None
            self.max_mhz = None

    def _sample(self):
        if self._nvml is not None:
            n = self._nvml
            sm = n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)
            mask = n.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            return sm, mask
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        a = [x.strip() for x in out.stdout.strip().split(",")]
        self.max_mhz = float(a[1])
        return float(a[0]), 0

    def _run(self):
        while True:
            try:
                self.rows.append(self._sample())
            except Exception:
                pass
            if self._stop.wait(self.period):
                break

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["clock sampling unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows]
        reasons = sorted({name for _, m in self.rows for name, bit in self.REASONS.items() if m & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self._nvml else "nvidia-smi"}


def load_ncu_summary():
    """Per-launch DRAM bytes and XU (SFU) warp-instructions of K1 from the
    committed ncu --set full capture (profiles/ncu_rollout_summary.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_rollout_summary.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


def spawn_ranks(args):
    """--gpus N outside torchrun: launch N ranks of this script (one process per GPU)."""
    import socket
    import torch
    n_dev = torch.cuda.device_count()
    if n_dev < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} needs {args.gpus} GPUs, {n_dev} visible"}),
              flush=True)
        sys.exit(2)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.run(cmd).returncode)


def run_ours(args):
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        spawn_ranks(args)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch with torchrun "
                         f"--nproc-per-node {args.gpus}, or without torchrun to let bench.py spawn the ranks)")
    import torch
    sys.path.insert(0, ROOT)
    from paper_1707_02342_b200 import workload
    from paper_1707_02342_b200.api import Controller, fp32_peak_tflops, pipe_peaks

    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist

    shape = workload_shape(args)
    w = workload.make(args.config, samples=args.samples)
    assert (w.params.samples, w.params.horizon_steps, w.hidden, w.controllers) == (
        shape["samples"], shape["horizon_steps"], shape["hidden"], shape["controllers"])
    fleet = w.controllers > 1
    # fleet (c3): the independent controllers are split over the ranks, no
    # communicator, seeds and map perturbations keyed by the global controller
    # index; otherwise the samples of one controller are sharded
    if fleet and w.controllers % world:
        raise SystemExit(f"bench.py: {w.controllers} controllers do not split over {world} GPUs")
    C = w.controllers // world if fleet else 1
    ctrl = Controller(w.params, w.bounds, w.sg, w.cost, hidden=w.hidden, precision="fp32", noise="philox",
                      device=local, n_controllers=C, system=w.system, controller_offset=rank * C if fleet else 0)
    ctrl.set_mlp(w.mlp)
    ctrl.set_costmap(w.costmap)
    if fleet:
        ctrl.perturb_fleet_costmaps(0.02, workload.SEED)  # per-controller N(0, 0.02^2) map noise
    elif world > 1:
        obj = [Controller.nccl_unique_id() if rank == 0 else None]
        pg.broadcast_object_list(obj, src=0)
        ctrl.set_comm(rank, world, obj[0])
    K, T = w.params.samples, w.params.horizon_steps
    x0 = w.x0[rank * C:(rank + 1) * C] if fleet else w.x0[0]
    stream = torch.cuda.ExternalStream(ctrl.stream)

    def barrier():
        torch.cuda.synchronize()
        if pg:
            pg.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(values):
        t = torch.tensor(values, dtype=torch.float64, device="cuda")
        if pg:
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return t.cpu().numpy()

    # warm-up (graphs captured, clocks up)
    ctrl.closed_loop_timed(x0, max(3, args.warmup), L2_FLUSH_BYTES)
    barrier()
    n_launch0 = ctrl.launch_count
    with ClockSampler(local) as clocks:
        ms, iter_ms = ctrl.closed_loop_timed(x0, args.steps, L2_FLUSH_BYTES, per_iteration=True)
    barrier()
    launches = ctrl.launch_count - n_launch0
    # K1's own launch duration (roofline) and the exchange time: a separate pass
    # of the iteration graph with event nodes around K1 and the all-gather (not
    # in the timed region: those nodes cut the programmatic-launch edges)
    ctrl.profile(True)
    ctrl.profile_read(reset=True)
    ctrl.profile_read_exchange(reset=True)
    ctrl.closed_loop_timed(x0, min(args.steps, 50), L2_FLUSH_BYTES)
    k1_ms, k1_n = ctrl.profile_read(reset=True)
    x_ms, x_n = ctrl.profile_read_exchange(reset=True)
    ctrl.profile(False)
    red = max_over_ranks([ms, k1_ms / max(k1_n, 1), x_ms / max(x_n, 1)] + list(iter_ms))
    ms_max, k1_avg_ms, x_avg_ms, iters_max = float(red[0]), float(red[1]), float(red[2]), red[3:]
    ms_per_step = ms_max / args.steps
    units_per_step = (C * world if fleet else 1) * K * T  # sample-steps of the whole job per iteration
    value = units_per_step * args.steps / (ms_max * 1e-3)

    # end to end through the public API: host x0 -> H2D, step, D2H u0, every step
    e2e = None
    if not args.no_e2e:
        x = np.array(x0, dtype=np.float64).reshape(C, 7)
        for _ in range(3):
            ctrl.mpc_step(x)
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        dt = w.params.dt
        for _ in range(args.steps):
            u = np.asarray(ctrl.mpc_step(x)).reshape(C, 2)
            # host plant (outside the controller): kinematic pose update, the
            # executed throttle nudges v_x (scalar math for one controller)
            if C == 1:
                r = x[0]
                px, py, th, vx, vy, thd = float(r[0]), float(r[1]), float(r[2]), float(r[4]), float(r[5]), float(r[6])
                c, s_ = math.cos(th), math.sin(th)
                r[0], r[1], r[2] = px + (c * vx - s_ * vy) * dt, py + (s_ * vx + c * vy) * dt, th + thd * dt
                r[4] = vx + 0.5 * float(u[0, 1]) * dt
            else:
                px, py, th, vx, vy = x[:, 0].copy(), x[:, 1].copy(), x[:, 2].copy(), x[:, 4].copy(), x[:, 5].copy()
                x[:, 0] = px + (np.cos(th) * vx - np.sin(th) * vy) * dt
                x[:, 1] = py + (np.sin(th) * vx + np.cos(th) * vy) * dt
                x[:, 2] = th + x[:, 6] * dt
                x[:, 4] = vx + 0.5 * u[:, 1] * dt
        ev1.record(stream)
        ev1.synchronize()
        e_ms = float(max_over_ranks([ev0.elapsed_time(ev1)])[0])
        e2e = {"value": units_per_step * args.steps / (e_ms * 1e-3), "unit": UNIT, "ms_per_step": e_ms / args.steps,
               "h2d_bytes_per_step": C * 8 * 4, "d2h_bytes_per_step": C * 96,
               "path": "Controller.mpc_step -> mppi_gpu_step (C ABI): graph replay whose first kernel reads x0 "
                       "from pinned host memory (H2D over PCIe), status D2H written to pinned host memory by the "
                       "tail kernel; the host waits on its sequence word"}

    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return

    # ---- roofline of K1: FP32 (the north star's), tensor (mma f16x3) and SFU ceilings
    flop_unit = workload.flops_per_sample_step(w.hidden)
    info = ctrl.shard_info
    chunk = max(1, -(-K // info["chunks"]))
    k_local = K * C if fleet else min(K, (info["chunk_hi"] - info["chunk_lo"]) * chunk)
    k1_flops = k_local * T * flop_unit
    peak, _ = fp32_peak_tflops(local)
    hmma_tflops, mufu_gops = pipe_peaks(local)
    achieved = k1_flops / (k1_avg_ms * 1e-3) / 1e12 if k1_avg_ms > 0 else None
    ncu = load_ncu_summary()
    same_shape = ncu.get("samples") == K and ncu.get("horizon") == T and ncu.get("hidden") == w.hidden and not fleet \
        and world == 1
    xu_per_ss = ncu.get("xu_warp_inst_per_launch", 0) * 32 / (ncu["samples"] * ncu["horizon"]) \
        if ncu.get("xu_warp_inst_per_launch") else None
    sfu_frac = (xu_per_ss * k_local * T / (k1_avg_ms * 1e-3) / (mufu_gops * 1e9)) \
        if (xu_per_ss and k1_avg_ms > 0 and mufu_gops > 0) else None
    tensor_peak = hmma_tflops / 3.0  # three fp16 products (hi*hi + hi*lo + lo*hi) per fp32 MAC
    tc05_peak = measured_bf16_tflops()
    tc05_peak = tc05_peak / 3.0 if tc05_peak else None
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        shape1 = dict(shape)
        res = ref_bench(shape1, [1, cpu_threads()], 7, 2)
        runs = {r["threads"]: r for r in res["runs"]}
        allc = runs[cpu_threads()]
        one = runs[1]
        cpu = {"value": allc["sample_steps_per_s"], "unit": UNIT, "cores": allc["threads"], "kind": "port",
               "sample": cpu_sample_text(shape1, allc), "ms_per_step": allc["median_ms"],
               "single_thread": {"value": one["sample_steps_per_s"], "cores": 1, "ms_per_step": one["median_ms"]}}
    it = np.asarray(iters_max)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        # the total work (K samples of one controller, or the 512-controller
        # fleet) is fixed and split over the GPUs
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded Xavier MLP, 2000x2000 ellipse map, Philox noise)",
        "config": dict(config_dict(args, world), kernel=ctrl.kernel_variant),
        "latency_ms": {"p50": float(np.percentile(it, 50)), "p99": float(np.percentile(it, 99)),
                       "mean": float(it.mean()), "max": float(it.max()),
                       "note": "per-iteration CUDA-event intervals of the timed loop, max over ranks"},
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if (achieved and peak) else None,
                     "traffic": ncu.get("dram_bytes_per_launch") if same_shape else None,
                     "kernel": ctrl.kernel_variant.split("<")[0] + " (K1)", "k1_ms_per_launch": k1_avg_ms,
                     "k1_share_of_step": k1_avg_ms / ms_per_step if ms_per_step else None,
                     "flop_per_launch": k1_flops, "flop_per_sample_step": flop_unit,
                     "peak_source": "measured FFMA/FFMA2 probe on this GPU (mppi_gpu_fp32_peak_probe); "
                                    "MEASURED_PEAKS.json has no FP32 CUDA-core figure",
                     "ceilings": {
                         "tensor_mma_f16x3": {"peak_tflops": tensor_peak, "frac": achieved / tensor_peak
                                              if (achieved and tensor_peak) else None,
                                              "note": "measured mma.sync m16n8k16 f16 peak / 3 (the fp16x3 split)"},
                         "tensor_tcgen05_f16x3": {"peak_tflops": tc05_peak, "frac": achieved / tc05_peak
                                                  if (achieved and tc05_peak) else None,
                                                  "note": "MEASURED_PEAKS.json dense bf16 (cuBLAS, tcgen05) / 3 "
                                                          "(the fp16x3 split); the ceiling of rollout_umma_kernel"},
                         "sfu": {"peak_gops": mufu_gops, "xu_lane_ops_per_sample_step": xu_per_ss, "frac": sfu_frac,
                                 "note": "XU instructions per sample-step from the ncu capture x K1 units / K1 time "
                                         "vs the measured MUFU ex2 peak"},
                     },
                     "traffic_source": ncu.get("source") if same_shape else None},
        "exchange_ms_per_iteration": x_avg_ms if world > 1 else 0.0,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks.summary(),
        "iteration_latency_ms": ms_per_step,
    }
    print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


def measured_bf16_tflops():
    """Dense bf16 tensor peak of this pool's B200s (driver-written
    MEASURED_PEAKS.json, cuBLAS = tcgen05 kind::f16 rate), or None."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
