# round-2 closing evidence: GPU suite, smoke, default bench (final round-2 code: histogram fixed-depth instantiations 3-11)
python __graft_entry__.py > /dev/null
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf 2>&1 | tail -15 > gpurun_out/gpu_tests_final.log
tail -3 gpurun_out/gpu_tests_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -2 gpurun_out/bench_final.err; cut -c1-200 gpurun_out/bench_final.json
