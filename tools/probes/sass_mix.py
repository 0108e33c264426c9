#!/usr/bin/env python3
"""Opcode histogram of the first `for` loop body that contains HMMA in a cubin
(the unrolled step pair of the tensor-core rollout).  Usage: sass_mix.py CUBIN"""
import collections, re, subprocess, sys

sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
ins = []
for ln in sass.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
# the step-pair loop: the backward branch whose body holds the most HMMAs
best = None
for i, (addr, s) in enumerate(ins):
    m = re.search(r"BRA (?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", s)
    if not m or not m.group(1):
        continue
    tgt = int(m.group(1), 16)
    if tgt >= addr:
        continue
    body = [x for x in ins if tgt <= x[0] <= addr]
    n = sum("HMMA" in x[1] for x in body)
    if best is None or n > best[0]:
        best = (n, body)
body = best[1] if best else ins
ops = collections.Counter()
for _, s in body:
    s = s.split(None, 1)[1] if s.startswith("@") else s
    ops[s.split()[0]] += 1
print(f"loop body: {len(body)} instructions, {best[0] if best else 0} HMMA")
for o, c in ops.most_common(30):
    print(f"  {o:26s} {c}")
