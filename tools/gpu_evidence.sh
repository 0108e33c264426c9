#!/bin/bash
# Round evidence for profiles/<TAG>/: bench lines (c1 with the CPU baseline,
# the reference arm, c0/c2/c3), the ncu launch list of the c1 bench command,
# one ncu --set full capture each of K1, the group merge and the tail at c1,
# of the sample-split K1 at c0,
# of the tcgen05 K1 at c2 (H = 64) and K = 262144 (H = 32) with the mma.sync
# K1 beside them, the config sweep and the accuracy study.
# Usage: bash tools/gpu_evidence.sh TAG
TAG=${1:-r02d}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/nvsmi.txt 2>&1
nproc > $O/nproc.txt
timeout 900 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref_c1.json 2> $O/bench_ref_c1.err
for c in c0 c2 c3; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/ncu_launches_bench_c1.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
  > $O/ncu_launch.log 2>&1
for k in rollout group_merge tail_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o $O/ncu_full_${k}_c1 -f python tools/ncu_target.py c1 0 4 > $O/ncu_full_$k.log 2>&1
  ncu -i $O/ncu_full_${k}_c1.ncu-rep --page raw --csv > $O/ncu_full_${k}_c1_raw.csv 2>&1
  ncu -i $O/ncu_full_${k}_c1.ncu-rep --page details --csv > $O/ncu_full_${k}_c1_details.csv 2>&1
done
ncu -i $O/ncu_full_rollout_c1.ncu-rep --page source --csv --print-source sass > $O/ncu_full_rollout_c1_source.csv 2>&1
bash tools/gpu_ncu_full.sh $TAG c0 0 rollout_tc_split > /dev/null 2>&1
bash tools/gpu_ncu_full.sh $TAG c2 0 rollout_umma > /dev/null 2>&1
bash tools/gpu_ncu_full.sh $TAG c4 262144 rollout_umma > /dev/null 2>&1
MPPI_KERNEL=mma bash tools/gpu_ncu_full.sh $TAG c2 0 rollout_tc > /dev/null 2>&1
MPPI_KERNEL=mma bash tools/gpu_ncu_full.sh $TAG c4 262144 rollout_tc > /dev/null 2>&1
timeout 900 python tools/sweep.py envs '[["c0",1920,{}],["c1",16384,{}],["c2",65536,{}],["c4",1024,{}],["c4",4096,{}],["c4",8192,{}],["c4",16384,{}],["c4",32768,{}],["c4",65536,{}],["c4",262144,{}],["c4",1048576,{}],["c2",65536,{"MPPI_KERNEL":"mma"}],["c4",32768,{"MPPI_KERNEL":"mma"}],["c4",262144,{"MPPI_KERNEL":"mma"}],["c4",1048576,{"MPPI_KERNEL":"mma"}]]' > $O/sweep_configs.jsonl 2>&1
timeout 1200 python tools/accuracy.py c0,c1 > $O/accuracy.jsonl 2>&1
rm -f $O/*.ncu-rep.tmp
cat $O/bench_c1.json | cut -c1-600
