set -u
O=gpurun_out/s6f; mkdir -p $O
BRI_TRSM_DENSE=1 timeout 600 python tools/hash_config.py --config 3 >> $O/hash.txt 2>$O/hash_err.txt
BRI_TRSM_DENSE=1 timeout 600 python tools/hash_config.py --config 2 >> $O/hash.txt 2>>$O/hash_err.txt
for r in 1 2; do
  for v in 0 1; do
    BRI_TRSM_DENSE=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/cfg3_dense${v}_$r.json 2> $O/cfg3_dense${v}_$r.err
  done
done
BRI_TRSM_DENSE=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -k "not config5" > $O/tests_dense.log 2>&1; echo rc=$? >> $O/tests_dense.log
echo done
