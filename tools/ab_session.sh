# ad-hoc A/B session (edited per experiment): P2P double-buffered (4 CTAs/SM,
# 4 targets per pass) vs single-buffer TMA kernel (8 CTAs/SM, 2 per pass),
# then the bounds-checked build over the GPU suite
for i in 1 2; do
python tools/p2p_time.py 4 40
SG_P2P_TMA_SINGLE=1 python tools/p2p_time.py 4 40
done
bash tools/debug_bounds.sh
