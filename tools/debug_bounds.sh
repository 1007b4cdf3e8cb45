#!/bin/bash
# Bounds-checked run (the compute-sanitizer stand-in; the sanitizer is closed
# on this pool): swap in libsg_debug.so (device asserts on leaf boxes and
# shared-memory indices, SG_DEBUG_BOUNDS), run the GPU suite and the
# sanitize cases, restore the release library.
set -u
make -s -C paper_2210_06439_b200/csrc debug
cp paper_2210_06439_b200/libsg.so /tmp/libsg_release.so
cp paper_2210_06439_b200/libsg_debug.so paper_2210_06439_b200/libsg.so
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/sanitize_cases.py 2>&1 | tail -3
cp /tmp/libsg_release.so paper_2210_06439_b200/libsg.so
