"""Per-source-line hot spots of one kernel from an ncu --set full report
captured with --import-source on (the binaries carry -lineinfo):
warp instructions executed and warp-stall samples summed over the SASS of
each CUDA line.

  python tools/src_hot.py report.ncu-rep KERNEL_REGEX [launch_index] [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "-k", "regex:" + kern, "--launch-skip", str(skip),
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, line, src = "?", None, ""
    agg = {}
    ii = si = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            ii = r.index("Instructions Executed")
            si = r.index("Warp Stall Sampling (All Samples)")
            continue
        if ii is None or len(r) <= ii:
            continue
        if r[0]:  # a CUDA line; its SASS rows follow
            line, src = int(r[0]), r[1].strip()
            continue
        key = (fname, line)
        a = agg.setdefault(key, [0, 0, src])
        try:
            a[0] += int(r[ii])
            a[1] += int(r[si])
        except ValueError:
            pass
    tot_i = sum(v[0] for v in agg.values()) or 1
    tot_s = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {tot_i / 1e6:.2f} M, stall samples {tot_s}")
    for (f, ln), (ni, ns, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * ni / tot_i:5.1f}% inst {100 * ns / tot_s:5.1f}% stall  {f}:{ln}  {s[:90]}")


if __name__ == "__main__":
    main()
