"""Per-kernel key-metric listing of ncu --set full reports, in the format of
profiles/r*_*_ncu_full.txt (bench.py reads the M2L DRAM traffic from it).
Usage: ncu_full_txt.py report.ncu-rep [report2 ...] > profiles/rXX_..._ncu_full.txt"""
import csv
import io
import subprocess
import sys

KEYS = ["launch__grid_size", "launch__block_size", "launch__registers_per_thread", "gpu__time_duration.sum",
        "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        m = dict(zip(h, v))
        unit = dict(zip(h, u))
        print(f"== ncu --set full: {rep}")
        print(f"  {'Kernel Name':75s} {m.get('Kernel Name', '')} ")
        for k in KEYS:
            if k in m:
                print(f"  {k:75s} {m[k]} {unit.get(k, '')}")
        try:
            fp = sum(float(m[k]) for k in KEYS[8:11])
            sms = 148
            print(f"  -> FP64 thread-instr per elapsed cycle (chip) = {fp:.1f} of {sms * 64} peak "
                  f"({sms} SM x 64) = {100 * fp / (sms * 64):.1f}%")
        except (KeyError, ValueError):
            pass
