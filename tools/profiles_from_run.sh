#!/bin/bash
# Turn a tools/gpu_round.sh run's gpurun_out/ artefacts (TAG=rXX) into the
# tracked text records under profiles/.  Usage: tools/profiles_from_run.sh rXX
T=${1:?tag}
python tools/ncu_full_txt.py gpurun_out/prof_m2l_$T.ncu-rep > profiles/${T}_m2l_L4_ncu_full.txt
python tools/ncu_full_txt.py gpurun_out/prof_hydro_$T.ncu-rep > profiles/${T}_hydro_L4_ncu_full.txt
python tools/ncu_summary.py gpurun_out/prof_m2l_$T.ncu-rep p2p_ > profiles/${T}_p2p_L4_ncu_summary.txt
python tools/ncu_summary.py gpurun_out/prof_m2l_$T.ncu-rep m2l_pair > profiles/${T}_m2l_pair_L4_ncu_summary.txt
python tools/ncu_summary.py gpurun_out/prof_m2lfma_$T.ncu-rep > profiles/${T}_m2l_fma_mirror_L4_ncu_summary.txt
python tools/ncu_summary.py gpurun_out/prof_hydro_$T.ncu-rep hydro_dedup > profiles/${T}_hydro_dedup_L4_ncu_summary.txt
python tools/launch_summary.py gpurun_out/launches_$T.csv "$T bench.py --no-cpu, L=4" > profiles/${T}_launches_summary.txt
gzip -c gpurun_out/launches_$T.csv > profiles/${T}_launches.csv.gz
cp gpurun_out/bench_$T.json profiles/${T}_bench.json
for f in dropin_$T:dropin_latency bench_ref_$T:bench_reference_arm p2p_time_$T:p2p_time time_kernels_$T:time_kernels; do
  [ -f gpurun_out/${f%%:*}.json ] && cp gpurun_out/${f%%:*}.json profiles/${T}_${f##*:}.json
done
