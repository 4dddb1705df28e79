set -u
O=gpurun_out/s6d; mkdir -p $O
V=$PWD/tools/var
timeout 600 python tools/hash_config.py --config 3 >> $O/hash.txt 2>$O/hash_err.txt
timeout 600 python tools/hash_config.py --config 2 >> $O/hash.txt 2>>$O/hash_err.txt
for r in 1 2; do
  for v in default leaf256 outer256 leaf256o256; do
    if [ $v = default ]; then unset BRI_LIB; else export BRI_LIB=$V/libbri_$v.so; fi
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/cfg3_${v}_$r.json 2> $O/cfg3_${v}_$r.err
  done
done
export BRI_LIB=$V/libbri_leaf256.so
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -k "config3 or config4" > $O/tests_leaf256.log 2>&1; echo rc=$? >> $O/tests_leaf256.log
export BRI_LIB=$V/libbri_leaf256o256.so
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -k "config3 or config4" > $O/tests_leaf256o256.log 2>&1; echo rc=$? >> $O/tests_leaf256o256.log
unset BRI_LIB
echo done
