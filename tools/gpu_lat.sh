#!/bin/bash
# GPU parity tests + M2L batch-size latency sweep (outputs -> gpurun_out/)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python tools/lat_m2l.py exact 2>&1 | tail -3
timeout 300 python tools/lat_m2l.py fma 2>&1 | tail -3
