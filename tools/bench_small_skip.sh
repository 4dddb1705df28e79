#!/bin/bash
# Where does a pivot step of the small-node kernel spend its ~1000 cycles?  Profile builds of the
# column-cyclic schedule with pieces removed (results are wrong on purpose: timing only):
# BRI_SN_SKIP bit 1 = no pivot search, 2 = no reciprocal, 4 = no trailing updates.
set -e
cd "$(dirname "$0")/../paper_1612_00001_b200/csrc"
for skip in 0 1 2 3 4 7; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -DBRI_SMALL_PROFILE -DBRI_SN_SKIP=$skip -c small.cu -o /tmp/small_skip$skip.o
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a ../../tools/bench_small_prof.cu /tmp/small_skip$skip.o -o /tmp/bench_small_skip$skip
  echo "== BRI_SN_SKIP=$skip"
  if nvidia-smi > /dev/null 2>&1; then timeout 60 /tmp/bench_small_skip$skip 64 64 | grep -E "mode=0 dominant cyclic|mode=0 pivoting cyclic"; fi
done
