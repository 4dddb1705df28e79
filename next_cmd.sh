set -u
O=gpurun_out/s6a; mkdir -p $O
V=$PWD/tools/var
# bit identity across fragment maps (configs 1-3)
for c in 1 2 3; do
  timeout 600 python tools/hash_config.py --config $c >> $O/hash.txt 2>$O/hash_err_$c.txt
  BRI_LIB=$V/libbri_noperm.so timeout 600 python tools/hash_config.py --config $c >> $O/hash.txt 2>>$O/hash_err_$c.txt
done
# kernel + api parity
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py -m gpu -q -p no:cacheprovider -x > $O/tests_kernels.log 2>&1; echo rc=$? >> $O/tests_kernels.log
# A/B/C config 3, interleaved twice
for r in 1 2; do
  for v in default noperm trsmonly; do
    if [ $v = default ]; then unset BRI_LIB; else export BRI_LIB=$V/libbri_$v.so; fi
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/cfg3_${v}_$r.json 2> $O/cfg3_${v}_$r.err
  done
done
unset BRI_LIB
for v in default noperm; do
  if [ $v = default ]; then unset BRI_LIB; else export BRI_LIB=$V/libbri_$v.so; fi
  timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > $O/cfg2_$v.json 2> $O/cfg2_$v.err
  timeout 600 python tools/gemm_level_probe.py --b 1024 --count 148 > $O/gemm_probe_$v.json 2>&1
  timeout 600 python tools/gemm_level_probe.py --b 1024 --count 444 --shape 1024,1024,128 > $O/gemm_probe128_$v.json 2>&1
done
echo done
