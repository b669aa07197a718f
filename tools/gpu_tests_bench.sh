# GPU tests + bench + launch list (one gpurun call)
python __graft_entry__.py
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf -x 2>&1 | tail -40 > gpurun_out/gpu_tests.log
tail -30 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
