"""bench.py contract checks that need no GPU.

* The reference arm's copy of the BASELINE configs (bench.BENCH_CONFIGS,
  SAMPLING, BASELINE_COST) equals the product's workload table, so both arms
  time the same workload.
* The reference arm (`bench.py --impl reference`) imports nothing from the
  product package and maps no CUDA library of the repo: it runs the reference
  algorithm (oracle/build/mppi_ref_bench) on the host cores.
"""
import json
import os
import subprocess
import sys

import pytest

import bench
from paper_1707_02342_b200 import workload
from paper_1707_02342_b200.api import CostParams

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "c4"])
def test_reference_arm_config_matches_workload(name):
    w = workload.make(name)
    b = bench.BENCH_CONFIGS[name]
    assert (b["samples"], b["horizon_steps"], b["hidden"], b["controllers"]) == (
        w.params.samples, w.params.horizon_steps, w.hidden, w.controllers)
    s = bench.SAMPLING
    p = w.params
    assert (s["dt"], s["sigma0"], s["sigma1"], s["lambda_"], s["gamma"], s["explore"]) == (
        p.dt, p.sigma_diag[0], p.sigma_diag[1], p.lambda_, p.gamma, p.explore_fraction)
    assert (s["sg_window"], s["sg_degree"]) == (w.sg.window, w.sg.degree)
    assert bench.SEED == p.seed == workload.SEED
    c = CostParams.baseline()
    assert tuple(getattr(c, f) for f in CostParams.__dataclass_fields__) == bench.BASELINE_COST


_PROBE = r"""
import json, runpy, sys
sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c0', '--samples', '64', '--steps', '2', '--warmup', '1']
runpy.run_path(sys.argv_path if hasattr(sys, 'argv_path') else 'bench.py', run_name='__main__')
mods = sorted(m for m in sys.modules if m.startswith('paper_1707_02342_b200') or m == 'torch')
maps = open('/proc/self/maps').read()
print(json.dumps({'mods': mods, 'libmppi_gpu': 'libmppi_gpu' in maps, 'libcuda': 'libcuda.so' in maps}))
"""


def test_reference_arm_loads_no_product_code():
    out = subprocess.run([sys.executable, "-c", _PROBE], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    line = json.loads(lines[0])
    probe = json.loads(lines[-1])
    assert probe["mods"] == [] and not probe["libmppi_gpu"] and not probe["libcuda"], probe
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "port"
    assert line["steps"] == 2 and line["warmup"] == 1 and line["value"] > 0
    assert line["config"] == bench.config_dict(type("A", (), {"config": "c0", "samples": 64})(), 1)
    assert line["e2e"]["h2d_bytes_per_step"] == 0
