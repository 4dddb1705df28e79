set -u
O=gpurun_out/s6e; mkdir -p $O
BRI_PANEL_2CTA=1 timeout 600 python tools/hash_config.py --config 3 >> $O/hash.txt 2>$O/hash_err.txt
BRI_PANEL_2CTA=1 timeout 600 python tools/hash_config.py --config 2 >> $O/hash.txt 2>>$O/hash_err.txt
for r in 1 2; do
  for v in 0 1; do
    BRI_PANEL_2CTA=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/cfg3_2cta${v}_$r.json 2> $O/cfg3_2cta${v}_$r.err
  done
done
BRI_PANEL_2CTA=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -k "getrf or invert or config3 or config4" > $O/tests_2cta.log 2>&1; echo rc=$? >> $O/tests_2cta.log
echo done
