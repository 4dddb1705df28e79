BRI_TRSM_BN64=2 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -p no:cacheprovider -x -rf > gpurun_out/s5_bn64_tests.log 2>&1; echo rc=$? >> gpurun_out/s5_bn64_tests.log
for rep in 1 2; do
for w in 1 0; do
BRI_TRSM_BN64=$w timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s5_bn64_${w}_r$rep.log 2>&1
done; done
