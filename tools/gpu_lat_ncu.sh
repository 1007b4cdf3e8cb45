#!/bin/bash
# ncu launch list of the latency-mode M2L (batch 1) kernels
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:m2l --csv --log-file gpurun_out/lat_ncu.csv python tools/lat_m2l.py exact > gpurun_out/lat_ncu.log 2>&1
echo rc=$?
python - <<'PY'
import csv
rows=list(csv.DictReader(l for l in open("gpurun_out/lat_ncu.csv") if not l.startswith("==")))
seen={}
for r in rows[:60]:
    k=(r["ID"], r["Kernel Name"][:40])
    seen.setdefault(k,{})[r["Metric Name"]]=r["Metric Value"]
for k,v in list(seen.items())[:24]:
    print(k, v)
PY
