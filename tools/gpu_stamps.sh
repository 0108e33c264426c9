#!/bin/bash
# Iteration timeline from the %globaltimer stamps build (lib/st, -DMPPI_STAMPS):
# K1 end -> group merge -> tail phases, printed by the tail each iteration.
mkdir -p gpurun_out
L=paper_1707_02342_b200/lib
cp $L/libmppi_gpu.so /tmp/libmppi_gpu_default.so
cp $L/st/libmppi_gpu.so $L/libmppi_gpu.so
for cfg in "c1 16384" "c0 1920"; do
  set -- $cfg
  echo "== $1" >> gpurun_out/stamps.log
  timeout 300 python tools/ncu_target.py $1 $2 40 2>&1 | grep STAMPS | tail -20 >> gpurun_out/stamps.log
done
cp /tmp/libmppi_gpu_default.so $L/libmppi_gpu.so
python3 - <<'PY'
import re, statistics
cur=None; rows={}
for l in open("gpurun_out/stamps.log"):
    if l.startswith("=="): cur=l[3:].strip(); rows[cur]=[]; continue
    v = [int(x) for x in re.findall(r"(-?\d+)", l.split("STAMPS")[1])]
    if all(0 <= x < 10**8 for x in v): rows[cur].append(v)
for k,v in rows.items():
    names=["k1_end->tail_start","rho_loads","scales","elements","sg_plan","plant","status"]
    print(k, {n: statistics.median([r[i] for r in v]) for i,n in enumerate(names)})
PY
