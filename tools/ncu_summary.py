"""Summarise an ncu --set full report into a committed text record:
launch config, duration, FP64 pipe / DP instruction counts, DRAM traffic,
occupancy, stall mix and the hottest SASS regions."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]
keys = ['Kernel Name', 'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread',
        'gpu__time_duration.sum', 'sm__cycles_elapsed.avg.per_second', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed',
        'smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed',
        'smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'smsp__sass_inst_executed_op_shared_ld.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']
for r in rows[2:]:
    d = dict(zip(h, r))
    print('== ncu --set full:', rep)
    for k in keys:
        if k in d:
            u = units[h.index(k)]
            print(f'  {k:75s} {d[k]} {u}')
    try:
        dp = sum(float(d[k]) for k in keys[9:12])
        print(f'  -> FP64 thread-instr per elapsed cycle (chip) = {dp:.1f} of 9472 peak (148 SM x 64) = {dp/9472*100:.1f}%')
    except Exception:
        pass
print()
sys.argv = ['sass_hot', rep, '10']
exec(open(__file__.replace('ncu_summary.py', 'sass_hot.py')).read())
