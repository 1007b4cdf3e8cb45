"""Summarise an ncu --set full report: duration, stall reasons, shared-memory
wavefronts/conflicts, instruction mix and the hottest source lines.
Usage: ncu_summary.py report.ncu-rep [kernel-regex]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
filt = ["-k", f"regex:{sys.argv[2]}"] if len(sys.argv) > 2 else []


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *filt, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
m = dict(zip(h, v))
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]
for k in want:
    print(f"{k:70s} {m.get(k)}")
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(m[k]) for k in h
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and m[k] not in ("", "0")}
tot = sum(st.values())
print("stalls:", ", ".join(f"{k} {100 * x / tot:.1f}%" for k, x in sorted(st.items(), key=lambda kv: -kv[1])[:10]))
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
hdr, cur, lines, ops = None, None, [], Counter()
for r in src:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        try:
            lines.append((float(r[4] or 0), cur, r[0], r[1].strip()[:90]))
        except ValueError:
            pass
    elif r[2].startswith("0x"):
        op = r[3].split()
        if op:
            o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
            try:
                ops[o] += int(r[7])
            except ValueError:
                pass
t2 = sum(ops.values())
print("inst mix:", ", ".join(f"{o} {100 * c / t2:.1f}%" for o, c in ops.most_common(14)))
ts = sum(x[0] for x in lines)
print("hot lines (stall samples):")
for x in sorted(lines, reverse=True)[:18]:
    print(f"  {100 * x[0] / ts:5.1f}% {x[1]}:{x[2]} {x[3]}")
