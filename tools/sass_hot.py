"""Summarise an ncu report's SASS page: samples grouped by (exec count, avg threads) regions + stall mix."""
import csv, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; idx = {k: i for i, k in enumerate(h)}; data = rows[2:]
def f(r, k):
    try: return float(r[idx[k]].replace(',', ''))
    except Exception: return 0.0
tot = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in data)
g = defaultdict(lambda: [0, 0, defaultdict(int)])
for r in data:
    key = (int(f(r, 'Instructions Executed')), round(f(r, 'Avg. Threads Executed')))
    g[key][0] += f(r, 'Warp Stall Sampling (All Samples)'); g[key][1] += 1
    src = r[idx['Source']].split()
    op = src[1] if src and src[0].startswith('@') and len(src) > 1 else (src[0] if src else '')
    g[key][2][op.split('.')[0]] += 1
for k, v in sorted(g.items(), key=lambda x: -x[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 10]:
    ops = ','.join(f"{a}:{b}" for a, b in sorted(v[2].items(), key=lambda x: -x[1])[:6])
    print(f"exec={k[0]:>10} thr={k[1]:>3} samples={v[0]/tot*100:5.1f}% ninstr={v[1]:4d} {ops}")
stalls = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
agg = {k: sum(f(r, k) for r in data) for k in stalls}
print({k[6:]: round(v / tot * 100, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]})
