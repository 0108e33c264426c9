#!/usr/bin/env python3
"""Pick the roofline-relevant metrics out of an `ncu --page raw --csv` export
(one kernel): DRAM bytes, duration, pipe utilisation.  Prints JSON."""
import csv
import io
import json
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]


def main():
    txt = open(sys.argv[1]).read()
    rows = list(csv.reader(io.StringIO(txt[txt.index('"ID"'):])))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")]}
    for j, h in enumerate(hdr):
        if h in WANT:
            v = vals[j].replace(",", "")
            try:
                v = float(v)
            except ValueError:
                pass
            out[h] = {"value": v, "unit": units[j]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
