#!/usr/bin/env python3
"""Summarise an `ncu --page source --csv --print-source sass` export: executed
instructions per opcode and the warp-stall samples per reason (where the time
goes), for the kernel of one capture.  Usage: ncu_sass_summary.py FILE [top]"""
import collections
import csv
import io
import sys


def load(path):
    txt = open(path).read()
    i = txt.index('"Address"')
    return list(csv.DictReader(io.StringIO(txt[i:])))


def main():
    rows = load(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    by_op = collections.Counter()
    stalls = collections.Counter()
    total = 0
    for r in rows:
        src = r["Source"].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        n = int(r["Instructions Executed"] or 0)
        by_op[op] += n
        total += n
        for k, v in r.items():
            if k.startswith("stall_") and "Not Issued" not in k and v:
                stalls[k] += int(v)
    print(f"executed warp instructions: {total}")
    for op, n in by_op.most_common(top):
        print(f"  {op:10s} {n:12d} {100.0 * n / total:6.2f}%")
    s = sum(stalls.values())
    print(f"stall samples: {s}")
    for k, v in stalls.most_common(12):
        print(f"  {k:24s} {v:9d} {100.0 * v / s:6.2f}%")


if __name__ == "__main__":
    main()
