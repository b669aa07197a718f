# round-2 re-entry check: full GPU suite + default bench at HEAD
python __graft_entry__.py > /dev/null
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf 2>&1 | tail -15 > gpurun_out/gpu_tests_check.log
tail -4 gpurun_out/gpu_tests_check.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err
tail -2 gpurun_out/bench_check.err; cut -c1-600 gpurun_out/bench_check.json
