# GPU tests + bench line + launch list of the bench command (one gpurun call)
python __graft_entry__.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x 2>&1 | tail -5 > gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --frames 16384 --no-e2e --no-extras --no-cpu > gpurun_out/bench_under_ncu.json 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
