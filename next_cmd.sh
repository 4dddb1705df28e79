timeout 900 bash tools/bench_small_skip.sh > gpurun_out/s5_small_skip.txt 2>&1
