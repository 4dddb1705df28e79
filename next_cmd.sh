for rep in 1 2; do
for cfg in "132 80 2" "160 88 2" "160 96 3" "150 80 2" "132 80 3" "180 100 4"; do
set -- $cfg
BRI_CAP_A=$1 BRI_CAP_HI=$2 BRI_CAP_LAG=$3 timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s5_cap_$1_$2_$3_r$rep.log 2>&1
done; done
