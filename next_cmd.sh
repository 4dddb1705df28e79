for rep in 1 2; do
for e in 1 0; do
BRI_PDL_EARLY=$e BRI_EXT_SPLIT=$e timeout 600 python bench.py --config 2 --b 8192 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5_b8192_e${e}_r$rep.log 2>&1
BRI_PDL_EARLY=$e BRI_EXT_SPLIT=$e timeout 600 python bench.py --config 2 --b 2048 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s5_b2048_e${e}_r$rep.log 2>&1
done; done
