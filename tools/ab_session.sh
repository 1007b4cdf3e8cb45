set -x
python -m pytest tests -m gpu -q -x > gpurun_out/tests_k8.log 2>&1; tail -3 gpurun_out/tests_k8.log
python tools/p2p_time.py 4 40
SG_P2P_NO_K8=1 python tools/p2p_time.py 4 40
python tools/p2p_time.py 3 40
SG_P2P_NO_K8=1 python tools/p2p_time.py 3 40
cp paper_2210_06439_b200/libsg.so /tmp/orig.so
cp paper_2210_06439_b200/libsg_nt4.so paper_2210_06439_b200/libsg.so; python tools/p2p_time.py 4 40
cp /tmp/orig.so paper_2210_06439_b200/libsg.so
python tools/ab_hydro.py 4 10
cp paper_2210_06439_b200/libsg_sel0.so paper_2210_06439_b200/libsg.so; python tools/ab_hydro.py 4 10
cp /tmp/orig.so paper_2210_06439_b200/libsg.so; python tools/ab_hydro.py 4 10
