#!/usr/bin/env python3
"""Attribute ncu per-instruction execution counts and stall samples to CUDA
source lines: aligns an `ncu --page source --csv --print-source sass` export
(one kernel, instructions in address order) with `nvdisasm -g -c` of the same
cubin function (which carries `//## File ..., line N` markers).
Usage: ncu_by_line.py NCU_SOURCE_CSV NVDISASM_FILE FUNCTION_MANGLED [top]"""
import collections
import csv
import io
import re
import sys


def sass_lines(path, fn):
    out, cur, inside = [], None, False
    for ln in open(path):
        if ln.startswith("//-----") and ".text." in ln:
            inside = (".text." + fn + " ") in ln or ln.rstrip().endswith(".text." + fn + " --------------------------")
            inside = fn in ln
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            out.append((cur, m.group(2).strip()))
    return out


def main():
    txt = open(sys.argv[1]).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"Address"'):])))
    sl = sass_lines(sys.argv[2], sys.argv[3])
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    if len(sl) != len(rows):
        print(f"warning: {len(sl)} disassembled vs {len(rows)} profiled instructions")
    ex, st = collections.Counter(), collections.Counter()
    for (line, _), r in zip(sl, rows):
        ex[line] += int(r["Instructions Executed"] or 0)
        st[line] += int(r["Warp Stall Sampling (All Samples)"] or 0)
    tot, tots = sum(ex.values()), sum(st.values())
    print(f"{'line':28s} {'executed':>12s} {'%':>6s} {'stall%':>7s}")
    for line, n in ex.most_common(top):
        print(f"{str(line):28s} {n:12d} {100 * n / tot:6.2f} {100 * st[line] / max(tots, 1):7.2f}")


if __name__ == "__main__":
    main()
