#!/bin/bash
# One A/B pass on the GPU box: optional GPU tests, then the config sweep —
# env-variable variants inside CFGS (tools/sweep.py envs), library builds
# named on the command line (lib/<v>/libmppi_gpu.so, via gpu_libvariants.sh).
# Usage (from the repo root, under gpurun):
#   CFGS='[["c0",1920,{}],["c0",1920,{"MPPI_TC_SPLIT":"0"}]]' TESTS='split_kernel' bash tools/gpu_ab.sh [variant ...]
# Build a library variant first, e.g.
#   make -C paper_1707_02342_b200 BUILD=build_v LIB=lib/v/libmppi_gpu.so NVFLAGS="... -DMPPI_SPLIT_MINB=7"
mkdir -p gpurun_out
CFGS=${CFGS:-'[["c0",1920,{}],["c1",16384,{}]]'}
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$TESTS" > gpurun_out/ab_test.log 2>&1
  echo "rc=$?" >> gpurun_out/ab_test.log
  tail -2 gpurun_out/ab_test.log
fi
if [ $# -gt 0 ]; then
  rm -f gpurun_out/libvariants.log
  CFGS="$CFGS" bash tools/gpu_libvariants.sh "$@"
else
  timeout 1200 python tools/sweep.py envs "$CFGS" > gpurun_out/ab_sweep.jsonl 2>&1
  python3 - <<'PY'
import json
for l in open("gpurun_out/ab_sweep.jsonl"):
    try:
        env = l[:l.index("{", 2)].strip(); d = json.loads(l[l.index("{", 2):])
        print(env, d["cfg"], d["K"], "iter %.1f us  K1 %.1f us" % (d["ms_per_iter"] * 1e3, d["k1_ms"] * 1e3), d["variant"][:40])
    except Exception:
        print(l[:160].rstrip())
PY
fi
