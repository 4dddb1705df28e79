#!/bin/bash
# build + run the small-node kernel micro-benchmark with the clock64 phase split
set -e
cd "$(dirname "$0")/../paper_1612_00001_b200/csrc"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -DBRI_SMALL_PROFILE -c small.cu -o /tmp/small_prof.o
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a ../../tools/bench_small_prof.cu /tmp/small_prof.o -o /tmp/bench_small_prof
cp /tmp/bench_small_prof ../../tools/bench_small_prof 2>/dev/null || true
if nvidia-smi > /dev/null 2>&1; then for n in 64 32 96; do timeout 60 /tmp/bench_small_prof $n 64; done; fi
