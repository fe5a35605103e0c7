"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
per-kernel totals for the launches after --skip (warm-up), descending."""
import collections, csv, re, sys
path = sys.argv[1]
skip_frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, ii = h.index('Kernel Name'), h.index('Metric Value'), h.index('ID')
per = []
for r in rows[hi + 1:]:
    if len(r) <= vi or ('Metric Name' in h and r[h.index('Metric Name')] != 'gpu__time_duration.sum'):
        continue
    k = r[ki]
    m = re.search(r'(k_[a-z0-9_]+)', k)
    name = m.group(1) if m else k[:40]
    if name == 'k_iwpp':
        t = re.search(r'k_iwpp<([^,]+), (\d+), [^>]*?(PlainMask|ComplementMask)', k)
        name += f"<{t.group(1).replace('unsigned ', 'u')},{t.group(2)},{t.group(3)[:5]}>" if t else ''
    per.append((int(r[ii]), name, float(r[vi].replace(',', ''))))
per = per[int(len(per) * skip_frac):]
tot = collections.OrderedDict(); cnt = collections.Counter()
for _, n, t in per:
    tot[n] = tot.get(n, 0) + t; cnt[n] += 1
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:36s} {cnt[k]:4d} {v / 1e3:9.1f} us {100 * v / s:5.1f}%")
print(f"total {s / 1e3:.1f} us over {len(per)} launches")
