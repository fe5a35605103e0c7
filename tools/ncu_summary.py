"""Per-kernel summary of an ncu --set full report (the lines profiles/ keeps):
duration, throughputs, occupancy, registers, shared memory, issue activity.

  python tools/ncu_summary.py report.ncu-rep [header line ...]
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEEP = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block",
        "Issue Slots Busy", "Executed Ipc Active", "Warp Cycles Per Issued Instruction",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Mem Busy", "Max Bandwidth", "Executed Instructions"]


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ii, ki, mi, ui, vi = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"),
                          h.index("Metric Unit"), h.index("Metric Value"))
    kern = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi or not r[mi]:
            continue
        d = kern.setdefault(int(r[ii]), {"name": r[ki], "m": {}})
        d["m"].setdefault(r[mi], (r[vi], r[ui]))
    for line in sys.argv[2:]:
        print("# " + line)
    print()
    for i, d in kern.items():
        m = re.search(r"(k_[a-z0-9_]+(<[^>]*>)?)", d["name"])
        print(f"[{i}] {m.group(1) if m else d['name'][:60]}")
        for k in KEEP:
            if k in d["m"]:
                v, u = d["m"][k]
                print(f"    {k:36s} {v} {u}".rstrip())
        print()


if __name__ == "__main__":
    main()
