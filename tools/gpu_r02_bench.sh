# new GPU tests + full bench + multi-GPU launch check + config X smoke
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -q -p no:cacheprovider -rf tests/test_gpu_dist.py \
  "tests/test_gpu_sweep_route.py::test_sweep_records_a_matches_oracle" 2>&1 | tail -15 > gpurun_out/gpu_tests_new.log
tail -8 gpurun_out/gpu_tests_new.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
tail -3 gpurun_out/bench_r02a.err
timeout 300 python bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --no-extras --no-cpu > gpurun_out/bench_g2.out 2>&1; echo "gpus2 rc=$?" >> gpurun_out/bench_g2.out
tail -2 gpurun_out/bench_g2.out
timeout 900 python bench.py --workload x --x-streams 2 --x-hours 2 > gpurun_out/bench_x.json 2> gpurun_out/bench_x.err
tail -3 gpurun_out/bench_x.err; cat gpurun_out/bench_x.json
