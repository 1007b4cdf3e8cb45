#!/bin/bash
# The paper-style figures (plots.py, the reference frontend's three SVGs) from
# REAL runs on the GPU box: the reference harness itself (baseline/_ref, numba,
# CPU backends scalar / emulated8 over 1..16 threads, after a JIT warm-up run)
# and this repo's driver (backend "cuda": the B200 kernels) on the same
# scenarios, plus a reference legacy-hydro run for the hydro comparison.
# Output: gpurun_out/figures/{simd_speedup,node_scaling,hydro_compare}.svg + CSVs.
set -e
OUT=gpurun_out/figures
mkdir -p $OUT
export NUMBA_CACHE_DIR=/tmp/sg_numba_cache
L=${L:-2}
REF="env PYTHONPATH=baseline/_ref python -m simdgrid.cli --max-level $L --stop-step 1 --disable-output"
rm -f $OUT/*.csv
$REF --scenario rotating-star-proxy --sweep 1xscalar,emulated8 --csv /tmp/warm.csv   # JIT warm-up
$REF --scenario blast --sweep 1xscalar,emulated8 --hydro-kernel legacy --csv /tmp/warm.csv
$REF --scenario rotating-star-proxy --sweep 1,2,4,8,16xscalar,emulated8 --csv $OUT/sweep.csv
$REF --scenario blast --sweep 1,16xscalar,emulated8 --csv $OUT/sweep.csv
$REF --scenario blast --sweep 1,16xscalar --hydro-kernel legacy --csv $OUT/legacy.csv
python - <<PY
from paper_2210_06439_b200 import driver as D
for name in ("rotating-star-proxy", "blast"):
    cfg = D.ScenarioConfig(name, max_level=$L, stop_step=1)
    D.run_scenario(cfg)  # warm-up (module load, first launches)
    D.sweep(cfg, [1, 16] if name == "blast" else [1, 2, 4, 8, 16], ["scalar"], "$OUT/sweep.csv")
PY
python -m paper_2210_06439_b200.plots --filename $OUT/sweep.csv --simd-key cuda --outdir $OUT \
    --legacy-files $OUT/legacy.csv
