# round-2 final evidence (after the balanced sweep evaluation): GPU suite, smoke, default bench, launch list, config X at full size, torchrun 1 rank
python __graft_entry__.py > /dev/null
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf 2>&1 | tail -15 > gpurun_out/gpu_tests_final.log
tail -3 gpurun_out/gpu_tests_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -2 gpurun_out/bench_final.err; cut -c1-200 gpurun_out/bench_final.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-extras --no-cpu > gpurun_out/launches_final.log 2>&1
echo "launch list rc=$?"
timeout 1200 python bench.py --workload x --x-streams 8 --x-hours 24 --no-cpu > gpurun_out/bench_x_full.json 2> gpurun_out/bench_x_full.err
echo "x rc=$?"; cut -c1-300 gpurun_out/bench_x_full.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --frames 27000 --no-extras --no-cpu --no-e2e > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err
echo "torchrun rc=$?"; grep -i "nranks" gpurun_out/bench_torchrun1.err | head -2
