mkdir -p gpurun_out/umma
export MPPI_KERNEL=umma
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rollout_umma -s 2 -c 1 -o gpurun_out/umma/k1_262k -f python tools/ncu_target.py c4 262144 4 > gpurun_out/umma/ncu.log 2>&1
ncu -i gpurun_out/umma/k1_262k.ncu-rep --page raw --csv > gpurun_out/umma/raw.csv 2>&1
ncu -i gpurun_out/umma/k1_262k.ncu-rep --page source --csv --print-source sass > gpurun_out/umma/source.csv 2>&1
ncu -i gpurun_out/umma/k1_262k.ncu-rep --page details --csv > gpurun_out/umma/details.csv 2>&1
tail -2 gpurun_out/umma/ncu.log
