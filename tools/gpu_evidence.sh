#!/bin/bash
# Round evidence for profiles/: the bench line, the ncu launch list of the same
# bench command, one ncu --set full capture of K1 at the bench config.
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launch_$TAG.log 2>&1
bash tools/gpu_ncu_full.sh $TAG c1 0
python tools/sweep.py envs '[["c0",1920,{}],["c1",16384,{}],["c2",65536,{}],["c4",1024,{}],["c4",4096,{}],["c4",65536,{}],["c4",262144,{}],["c4",1048576,{}]]' > gpurun_out/sweep_$TAG.jsonl 2>&1
cat gpurun_out/bench_$TAG.json
