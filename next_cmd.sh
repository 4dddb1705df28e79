python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_regressions.py tests/test_gpu_configs.py::test_config3_full_inverse_true_size -q -p no:cacheprovider --durations=10 -rf > gpurun_out/s5_sub1.log 2>&1; echo rc=$? >> gpurun_out/s5_sub1.log
python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s5_b2_split.log 2>&1
BRI_EXT_SPLIT=0 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s5_b2_nosplit.log 2>&1
python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s5_b3_dinv.log 2>&1
python tools/timeline.py --config 2 --out gpurun_out/s5_tl2b.json > gpurun_out/s5_tl2b.txt 2>&1
