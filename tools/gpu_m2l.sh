#!/bin/bash
# GPU session: gpu tests, bench, then ncu --set full on the M2L kernel only
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} 2>&1 | tail -5
timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value', d['value'], 'ms/step', d['ms_per_step'], 'e2e', d['e2e']['value'])
print({k:(round(v['mean_ms'],4), round(v['subgrids_per_s'])) for k,v in d['per_kernel'].items()})
print('roofline', d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['frac_issue'], 'clocks', d.get('clocks'))
print('cpu', d.get('cpu_baseline',{}).get('value'))
"
if [ -n "$PROF" ]; then
python tools/prof_kernels.py gravity ${PROF_LEVEL:-3} > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${PROF_K:-m2l_kernel}" -s 1 -c 1 \
     -o gpurun_out/${PROF} -f python tools/prof_kernels.py gravity ${PROF_LEVEL:-3} > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
fi
