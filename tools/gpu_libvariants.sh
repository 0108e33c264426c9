#!/bin/bash
# Sweep configs over alternative library builds (paper_1707_02342_b200/lib/<v>/libmppi_gpu.so),
# swapping each in for the default one on the (scratch) GPU-box copy of the repo.
# Usage: CFGS='[["c1",16384,{}]]' bash tools/gpu_libvariants.sh v1 v2 ...  (default build = "default")
mkdir -p gpurun_out
L=paper_1707_02342_b200/lib
cp $L/libmppi_gpu.so /tmp/libmppi_gpu_default.so
CFGS=${CFGS:-'[["c1",16384,{}],["c0",1920,{}],["c4",262144,{}],["c2",65536,{}]]'}
for rep in 1 2; do
for v in default "$@"; do
  if [ "$v" = default ]; then cp /tmp/libmppi_gpu_default.so $L/libmppi_gpu.so; else cp $L/$v/libmppi_gpu.so $L/libmppi_gpu.so; fi
  echo "== $v" >> gpurun_out/libvariants.log
  timeout 300 python tools/sweep.py envs "$CFGS" >> gpurun_out/libvariants.log 2>&1
done
done
cp /tmp/libmppi_gpu_default.so $L/libmppi_gpu.so
python3 - <<'PY'
import json
cur = None
for line in open("gpurun_out/libvariants.log"):
    if line.startswith("== "):
        cur = line[3:].strip(); continue
    try:
        d = json.loads(line[line.index("{", 2):])
        print(f"{cur:10s} {d['cfg']} K={d['K']:8d} iter {d['ms_per_iter']*1e3:9.2f} us  K1 {d['k1_ms']*1e3:9.2f} us")
    except Exception:
        pass
PY
