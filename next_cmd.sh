mkdir -p gpurun_out/g1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1/smoke.log 2>&1; echo rc=$? >> gpurun_out/g1/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x --timeout 900 > gpurun_out/g1/gputest.log 2>&1; echo rc=$? >> gpurun_out/g1/gputest.log
python bench.py > gpurun_out/g1/bench_cfg3.json 2> gpurun_out/g1/bench_cfg3.err
python bench.py --config 1 > gpurun_out/g1/bench_cfg1.json 2> gpurun_out/g1/bench_cfg1.err
