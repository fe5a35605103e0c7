"""Aggregates an ncu CSV launch list (metrics gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum) of ONE rtg_process_tile call
into per-stage duration and DRAM traffic, and writes profiles/traffic.json
(per-launch DRAM bytes per stage, consumed by bench.py's roofline.traffic).

Stages are recovered from the deterministic launch order of the pipeline
(csrc/rtg_abi.cu pipeline()): each stage starts at a known first kernel.

  python tools/stage_traffic.py launches.csv [out.json]
"""
import collections
import csv
import json
import re
import sys

STARTS = [  # (stage, first kernel of the stage, kernel that must precede it)
    ("colordeconv", "k_colordeconv_tma", None),
    ("recon", "k_ccl_tile", None),
    ("fill_holes", "k_ccl_tile_fb", None),
    ("area", "k_fb_tree", None),
    ("edt", "k_edt_rowdist", None),
    ("markers", "k_hmax_init", None),
    ("watershed", "k_ws_arrows", None),
    ("label", "k_ccl_tile", "k_ws_separate"),
    ("features", "k_feat_list", None),
]


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("ID"))
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        m = re.search(r"(k_[a-z0-9_]+)", r[ki])
        d = launches.setdefault(int(r[ii]), {"name": m.group(1) if m else r[ki][:40]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    return list(launches.values())


def split_stages(launches):
    """Assigns the LAST complete pipeline pass of the list to stages."""
    starts = [i for i, l in enumerate(launches) if l["name"].startswith("k_colordeconv")]
    seq = launches[starts[-1]:] if starts else launches
    out, si, seen = [], -1, set()
    for l in seq:
        if si + 1 < len(STARTS):
            _, first, after = STARTS[si + 1]
            if l["name"] == first and (after is None or after in seen):
                si += 1
        seen.add(l["name"])
        out.append((STARTS[max(si, 0)][0], l))
    return out


def main():
    if sys.argv[1] == "--kernels":  # per-launch listing of the last pass
        for st, l in split_stages(load(sys.argv[2])):
            dram = l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
            print(f"{st:12s} {l['name']:28s} {l.get('gpu__time_duration.sum', 0.0) / 1e3:8.1f} us"
                  f" {dram / 1e6:8.1f} MB")
        return
    launches = load(sys.argv[1])
    staged = split_stages(launches)
    agg = collections.OrderedDict()
    for st, l in staged:
        a = agg.setdefault(st, {"launches": 0, "ns": 0.0, "dram_bytes": 0.0})
        a["launches"] += 1
        a["ns"] += l.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["ns"] for a in agg.values())
    print(f"{'stage':12s} {'launches':>8s} {'us':>9s} {'share':>6s} {'DRAM MB':>9s} {'GB/s':>8s}")
    for st, a in agg.items():
        gbs = a["dram_bytes"] / a["ns"] if a["ns"] else 0.0
        print(f"{st:12s} {a['launches']:8d} {a['ns'] / 1e3:9.1f} {100 * a['ns'] / tot:5.1f}% "
              f"{a['dram_bytes'] / 1e6:9.1f} {gbs:8.1f}")
    print(f"{'total':12s} {sum(a['launches'] for a in agg.values()):8d} {tot / 1e3:9.1f}")
    if len(sys.argv) > 2:
        traffic = {st: int(a["dram_bytes"]) for st, a in agg.items()}
        json.dump(traffic, open(sys.argv[2], "w"), indent=1)


if __name__ == "__main__":
    main()
