#!/bin/bash
# A/B of the two-tile tcgen05 CTAs at H = 64 (MPPI_UMMA_TPC2) + bit-identity tests.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "two_tile" > gpurun_out/tpc2_test.log 2>&1; echo "rc=$?" >> gpurun_out/tpc2_test.log
timeout 900 python tools/sweep.py envs '[["c2",65536,{"MPPI_UMMA_TPC2":"0"}],["c2",65536,{}],["c2",65536,{"MPPI_UMMA_TPC2":"0"}],["c2",65536,{}],["c2",131072,{}],["c2",32768,{}],["c2",81920,{}],["c2",81920,{"MPPI_UMMA_TPC2":"1"}]]' > gpurun_out/tpc2_sweep.jsonl 2>&1
tail -3 gpurun_out/tpc2_test.log; python3 -c "
import json
for l in open('gpurun_out/tpc2_sweep.jsonl'):
    try:
        e=l[:l.index('{',2)]; d=json.loads(l[l.index('{',2):]); print(e.strip(), d['cfg'], d['K'], 'iter %.1f us K1 %.1f us' % (d['ms_per_iter']*1e3, d['k1_ms']*1e3))
    except Exception as x: print(l[:200])
"
