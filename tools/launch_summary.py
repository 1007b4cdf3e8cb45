"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list into kernel shares."""
import collections
import csv
import sys

path, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].replace('void ', '')
    v = float(r[vi].replace(',', ''))
    v = v / 1e3 if r[ui] in ('ns', 'nsecond') else (v * 1e3 if r[ui] in ('ms', 'msecond') else v)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(title)
print(f"{'kernel':45s} {'launches':>8s} {'total_us':>12s} {'share':>7s} {'mean_us':>10s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:45]:45s} {cnt[k]:8d} {tot[k]:12.1f} {tot[k] / T * 100:6.2f}% {tot[k] / cnt[k]:10.1f}")
