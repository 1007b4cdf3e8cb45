# ad-hoc A/B session (edited per experiment): GPU tests, then the default
# bench with P2P beside M2L (side stream) and serial (SG_P2P_OVERLAP=0)
python -m pytest tests -m gpu -q > gpurun_out/tests_ab.log 2>&1; tail -3 gpurun_out/tests_ab.log
for i in 1 2; do
python bench.py --no-cpu 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('overlap', b['value'], b['ms_per_step'], b['e2e']['value'], b['per_kernel']['p2p']['mean_ms'], b['per_kernel']['m2l']['mean_ms'])"
SG_P2P_OVERLAP=0 python bench.py --no-cpu 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('serial', b['value'], b['ms_per_step'], b['e2e']['value'], b['per_kernel']['p2p']['mean_ms'], b['per_kernel']['m2l']['mean_ms'])"
done
