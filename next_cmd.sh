timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s5_b3_div2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py::test_config4_singular_pivot_matches_reference tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -p no:cacheprovider -rf > gpurun_out/s5_cfg4b.log 2>&1; echo rc=$? >> gpurun_out/s5_cfg4b.log
timeout 300 bash tools/bench_small.sh > gpurun_out/s5_small_bench3.txt 2>&1
