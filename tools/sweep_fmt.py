#!/usr/bin/env python3
"""Compact view of tools/sweep.py output lines (stdin): env, config, K, iteration / K1 us, G sample-steps/s."""
import json
import sys

for line in sys.stdin:
    try:
        i = line.index("{", 2) if line.startswith("{") and not line.startswith('{"cfg"') else line.index("{")
        env = line[:i].strip()
        d = json.loads(line[i:])
        print(f"{env:40s} {d['cfg']} K={d['K']:8d} iter {d['ms_per_iter'] * 1e3:9.2f} us  K1 {d['k1_ms'] * 1e3:9.2f} us"
              f"  {d['Gsteps_per_s']:6.2f} G/s")
    except Exception:
        print(line.rstrip()[:300])
