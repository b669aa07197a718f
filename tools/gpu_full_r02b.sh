# full GPU suite + bench + torchrun/NCCL path at one rank + config X (2 streams x 1 h)
python __graft_entry__.py > /dev/null
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf 2>&1 | tail -15 > gpurun_out/gpu_tests_full.log
tail -4 gpurun_out/gpu_tests_full.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
tail -2 gpurun_out/bench_r02c.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --frames 27000 --no-extras --no-cpu --no-e2e > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err
grep -i "nranks\|NCCL version" gpurun_out/bench_torchrun1.err | head -5; cat gpurun_out/bench_torchrun1.json | cut -c1-300
timeout 900 python bench.py --workload x --x-streams 2 --x-hours 1 > gpurun_out/bench_x2.json 2> gpurun_out/bench_x2.err
cut -c1-400 gpurun_out/bench_x2.json
