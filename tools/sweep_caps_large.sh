# LU concurrency caps at large block orders (one node + inversion, config-5 matrix):
#   bash tools/sweep_caps_large.sh 20480 > gpurun_out/caps_20480.jsonl
B=${1:-20480}
for env in "" "BRI_CAP_ROWS=4096" "BRI_CAP_ROWS=6144" "BRI_CAP_ROWS=8192" "BRI_CAP_ROWS=12288" \
           "BRI_TRAIL_CAP=0 BRI_FOLD_CAP=0" "BRI_TRAIL_CAP=112 BRI_FOLD_CAP=24" "BRI_TRAIL_CAP=128 BRI_FOLD_CAP=0"; do
  env $env timeout 300 python tools/node_time.py --b $B --reps 3
done
