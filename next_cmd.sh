mkdir -p gpurun_out/g2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g2/smoke.log 2>&1; echo rc=$? >> gpurun_out/g2/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -rf --durations=5 > gpurun_out/g2/gputest.log 2>&1; echo rc=$? >> gpurun_out/g2/gputest.log
( time python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/g2/ref_default.json ) 2> gpurun_out/g2/ref_default.err
( time python bench.py > gpurun_out/g2/bench_default.json ) 2> gpurun_out/g2/bench_default.err
