#!/bin/bash
# Round-end evidence on one B200 (one gpurun call): GPU test suite, bench lines (ours + reference
# arm, configs 3 / 1 / 2), the ncu launch list of one config-3 step and `ncu --set full` captures of
# the top kernels.  Each ncu pass runs only after the same command exited 0 without ncu.
set -u
OUT=${OUT:-gpurun_out/final}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=12 > $OUT/gputest.log 2>&1; echo "rc=$?" >> $OUT/gputest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_cfg3.json 2> $OUT/bench_cfg3.err; echo "rc=$?" >> $OUT/bench_cfg3.err
( time timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/ref_cfg3.json ) 2> $OUT/ref_cfg3.err
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 > $OUT/bench_cfg1.json 2> $OUT/bench_cfg1.err
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
for c in 1 2 3; do timeout 600 python tools/hash_config.py --config $c >> $OUT/hashes.txt 2>> $OUT/hashes.err; done
timeout 600 python tools/timeline.py --config 3 --out $OUT/timeline_cfg3.json > $OUT/timeline_cfg3.txt 2>&1
timeout 600 python tools/timeline.py --config 2 --out $OUT/timeline_cfg2.json > $OUT/timeline_cfg2.txt 2>&1
python tools/chain_gaps.py $OUT/timeline_cfg2.json > $OUT/chain_cfg2.txt 2>&1
# launch list: one config-3 step (cold-cache, serialised: compare shares, not absolutes)
python tools/profile_step.py --config 3 --warmup 1 --steps 1 > /dev/null 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $OUT/launches_cfg3.csv python tools/profile_step.py --config 3 --warmup 1 --steps 1 > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_cfg3.csv > $OUT/launch_summary_cfg3.txt 2>&1
# full captures of the top kernels
python tools/gemm_level_probe.py --b 1024 --count 148 > $OUT/gemm_probe.json 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 2 -c 1 \
    -o $OUT/ncu_gemm_level -f python tools/gemm_level_probe.py --b 1024 --count 148 > $OUT/ncu_gemm.log 2>&1
for spec in "trsm_kernel:40" "lu_panel_kernel:200" "laswp_kernel:40" "dinv_kernel:40"; do
  name=${spec%%:*}; skip=${spec##*:}
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"$name" \
    -s $skip -c 1 -o $OUT/ncu_${name}_cfg3 -f python tools/profile_step.py --config 3 --warmup 1 --steps 1 \
    > $OUT/ncu_${name}.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:small_node_kernel -s 2 -c 1 -o $OUT/ncu_small_node_cfg1 -f \
  python tools/profile_step.py --config 1 --warmup 1 --steps 1 > $OUT/ncu_small.log 2>&1
python tools/ncu_summary.py $OUT/ncu_*.ncu-rep > $OUT/kernels_ncu.json 2> $OUT/kernels_ncu.err
# config 5 at true size with the final build (bounded schedule, ~7 min), Neumann check and hash
timeout 1500 python tools/run_config5.py --terms 2 --out $OUT/config5.json > $OUT/config5.log 2>&1
echo done
