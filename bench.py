#!/usr/bin/env python3
"""Benchmark of the B200 IT-MPPI hot path (one IT-MPPI iteration = one step).

Workload (BASELINE.json configs[1], "c1"): K = 16384 samples, T = 100, 6-32-32-4
tanh MLP vehicle, 2000 x 2000 elliptical-track costmap, receding horizon with
the device plant; all inputs synthetic from a seed (see
paper_1707_02342_b200/workload.py).  Samples shard over the ranks of a
torchrun launch (one NCCL all-gather of per-chunk softmin partials per
iteration); ``value`` is whole-job sample-timesteps/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl ours|reference]

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
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MPPI iteration latency (ms) and rollout sample-timesteps/sec at 1/2/4/8 B200"
UNIT = "sample-timesteps/s"
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c1")
    ap.add_argument("--samples", type=int, default=None, help="override K (c4 sweep)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


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


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_cpu(w, steps, warmup, sample_k):
    """The reference CPU path (oracle restatement: double, splitmix noise, std::thread
    chunks per call, serial sampling/weights/update) on a bounded sample of the workload."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle  # test infrastructure; the CPU arm only
    from paper_1707_02342_b200.api import SamplingParams
    p = SamplingParams(**{**w.params.__dict__, "samples": sample_k})
    o = oracle.OracleController(p, w.bounds, w.sg, w.cost, hidden=w.hidden, precision="fp64", noise="ref_splitmix",
                                system=w.system)
    if w.theta is not None:
        o.set_basis(w.theta)
    else:
        o.set_mlp(w.mlp)
    o.set_costmap(w.costmap)
    threads = cpu_threads()
    x = w.x0[0].copy()
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        u = o.mpc_step(x, threads=threads)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
        x = o.vehicle_step(x, u)
    med = statistics.median(times)
    return {"value": sample_k * w.params.horizon_steps / med, "unit": UNIT, "cores": threads, "kind": "port",
            "ms_per_step": med * 1e3, "total_s": sum(times),
            "sample": f"{len(times)} mpc_step calls on {sample_k} of the {w.params.samples} samples, "
                      f"T={w.params.horizon_steps}, fp64, reference splitmix noise, {threads} std::threads"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1707_02342_b200 import workload
    w = workload.make(args.config, samples=args.samples)
    sample_k = min(w.params.samples, 2048)
    steps = max(1, min(args.steps, 60))
    warm = max(1, min(args.warmup, 3))
    cb = reference_cpu(w, steps, warm, sample_k)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
            "warmup": warm, "ms_per_step": cb["ms_per_step"] * (w.params.samples / sample_k),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{args.config}: K={w.params.samples}, T={w.params.horizon_steps}, H={w.hidden}",
                       "parallelism": f"{cb['cores']} CPU threads"},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def load_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_rollout_summary.json")
    try:
        d = json.load(open(p))
        return d.get("dram_bytes_per_launch"), d.get("source")
    except Exception:
        return None, None


def run_ours(args):
    import torch
    from paper_1707_02342_b200 import workload
    from paper_1707_02342_b200.api import Controller, fp32_peak_tflops

    rank, world, local = dist_env()
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist

    w = workload.make(args.config, samples=args.samples)
    fleet = w.controllers > 1
    # fleet (c3): the independent controllers are split over the ranks, no
    # communicator; otherwise the samples of one controller are sharded
    C = max(1, w.controllers // world) if fleet else 1
    ctrl = Controller(w.params, w.bounds, w.sg, w.cost, hidden=w.hidden, precision="fp32", noise="philox",
                      device=local, n_controllers=C, system=w.system)
    if w.theta is not None:
        ctrl.set_basis(w.theta)
    else:
        ctrl.set_mlp(w.mlp)
    ctrl.set_costmap(w.costmap)
    if fleet:
        ctrl.perturb_fleet_costmaps(0.02, workload.SEED + rank)  # per-controller N(0, 0.02^2) map noise
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

    # warm-up (graphs captured, clocks up)
    ctrl.closed_loop_timed(x0, max(3, args.warmup), L2_FLUSH_BYTES)
    ctrl.profile_read(reset=True)
    barrier()
    n_launch0 = ctrl.launch_count
    with ClockSampler(local) as clocks:
        ms = ctrl.closed_loop_timed(x0, args.steps, L2_FLUSH_BYTES)
    barrier()
    launches = ctrl.launch_count - n_launch0
    # K1's own launch duration (roofline): a separate pass of the iteration
    # graph that brackets K1 with event nodes (not in the timed region: those
    # nodes would cut the tail's programmatic-launch edge to K1)
    ctrl.profile(True)
    ctrl.profile_read(reset=True)
    ctrl.closed_loop_timed(x0, min(args.steps, 50), L2_FLUSH_BYTES)
    k1_ms, k1_n = ctrl.profile_read(reset=True)
    ctrl.profile(False)
    t = torch.tensor([ms, k1_ms / max(k1_n, 1)], dtype=torch.float64, device="cuda")
    if pg:
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
    ms_max, k1_avg_ms = float(t[0]), float(t[1])
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
        e_ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device="cuda")
        if pg:
            pg.all_reduce(e_ms, op=pg.ReduceOp.MAX)
        e_ms = float(e_ms[0])
        e2e = {"value": units_per_step * args.steps / (e_ms * 1e-3), "unit": UNIT, "ms_per_step": e_ms / args.steps,
               "h2d_bytes_per_step": C * 8 * 4, "d2h_bytes_per_step": C * 96,
               "path": "Controller.mpc_step -> mppi_gpu_step (C ABI): x0 pinned H2D, graph replay, status D2H (written to pinned host memory by the tail kernel)"}

    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return

    # algorithmic FLOPs per sample-step: the MLP GEMVs, or Theta^T phi (25 x 4) of the basis model
    flop_unit = 2 * 25 * 4 if w.theta is not None else workload.flops_per_sample_step(w.hidden)
    k_local = K * C if fleet else (K // world if world > 1 else K)
    k1_flops = k_local * T * flop_unit
    peak, clk = fp32_peak_tflops(local)
    achieved = k1_flops / (k1_avg_ms * 1e-3) / 1e12 if k1_avg_ms > 0 else None
    traffic, traffic_src = load_traffic()
    cpu = None
    if not args.no_cpu_baseline and world == 1 and not fleet:
        cb = reference_cpu(w, steps=3, warmup=1, sample_k=min(K, 2048))
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        # the total work (K samples of one controller, or the 512-controller
        # fleet) is fixed and split over the GPUs
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded Xavier MLP, 2000x2000 ellipse map, Philox noise)",
        "config": {"workload": f"{args.config}: IT-MPPI iteration, K={K}, T={T}, "
                               + ("basis-function vehicle (reference acceptance #10 shape), "
                                  if w.theta is not None else f"H={w.hidden}, MLP vehicle, ") +
                               f"receding horizon with device plant"
                               + (f", fleet of {C * world} controllers (perturbed maps)" if fleet else ""),
                   "samples": K, "horizon": T, "hidden": w.hidden, "controllers": C * world,
                   "parallelism": (f"{C} independent controllers per GPU on {world} GPU(s), no communication"
                                   if fleet else f"samples sharded over {world} GPU(s)"),
                   "l2": "flushed between timed iterations (256 MiB memset, excluded from timing)",
                   "kernel": ctrl.kernel_variant},
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if (achieved and peak) else None, "traffic": traffic,
                     "kernel": "rollout_kernel (K1)", "k1_ms_per_launch": k1_avg_ms,
                     "k1_share_of_step": k1_avg_ms / ms_per_step if ms_per_step else None,
                     "flop_per_launch": k1_flops, "flop_per_sample_step": flop_unit,
                     "peak_source": "measured FFMA/FFMA2 probe on this GPU (mppi_gpu_fp32_peak_probe); "
                                    "MEASURED_PEAKS.json has no FP32 CUDA-core figure",
                     "traffic_source": traffic_src},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks.summary(),
        "iteration_latency_ms": ms_per_step,
    }
    print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
