python -m pytest tests/test_gpu_engine.py tests/test_gpu_api.py tests/test_gpu_kernels.py tests/test_gpu_regressions.py -q -p no:cacheprovider -rf > gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b8.log 2>&1
BRI_DEFER_LASWP=0 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b8_nodefer.log 2>&1
for v in lo256 leaf256 leaf1024 st5 st3; do BRI_LIB=build/$v/libbri_b200.so python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b8_$v.log 2>&1; done
python tools/run_config.py --config 1 --reps 50 --oracle-targets 16 > gpurun_out/cfg1f.log 2>&1
