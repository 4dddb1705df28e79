set -u
O=gpurun_out/s6b; mkdir -p $O
for c in 2 3; do timeout 600 python tools/hash_config.py --config $c >> $O/hash.txt 2>$O/hash_err_$c.txt; done
BRI_GEMM_N64_MAXK=100000 timeout 600 python tools/hash_config.py --config 3 >> $O/hash.txt 2>>$O/hash_err_3.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -x > $O/tests_kernels.log 2>&1; echo rc=$? >> $O/tests_kernels.log
for k in 0 256 100000; do
  export BRI_GEMM_N64_MAXK=$k
  for shape in 1024,1024,128 896,768,128 1024,1024,256 512,1024,512 1024,1024,1024; do
    cnt=444; [ $shape = 1024,1024,1024 ] && cnt=148
    timeout 300 python tools/gemm_level_probe.py --b 1024 --count $cnt --shape $shape >> $O/probe_maxk$k.txt 2>&1
  done
done
for r in 1 2; do
  for k in 0 256 512 100000; do
    export BRI_GEMM_N64_MAXK=$k
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/cfg3_maxk${k}_$r.json 2> $O/cfg3_maxk${k}_$r.err
  done
done
for k in 0 256; do
  export BRI_GEMM_N64_MAXK=$k
  timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > $O/cfg2_maxk$k.json 2> $O/cfg2_maxk$k.err
done
echo done
