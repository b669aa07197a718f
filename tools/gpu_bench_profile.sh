set -x
python __graft_entry__.py
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_1.json 2> gpurun_out/bench_1.err
tail -5 gpurun_out/bench_1.err
cat gpurun_out/bench_1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_1.csv python bench.py --steps 2 --warmup 1 --frames 16384 --no-e2e --no-extras --no-cpu > gpurun_out/bench_ncu_list.json 2>&1
tail -3 gpurun_out/bench_ncu_list.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dd_downsample -s 2 -c 1 -o gpurun_out/prof_dd python bench.py --steps 1 --warmup 1 --frames 16384 --no-e2e --no-extras --no-cpu > gpurun_out/ncu_full_dd.log 2>&1
tail -5 gpurun_out/ncu_full_dd.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:convN -s 1 -c 1 -o gpurun_out/prof_convN python bench.py --steps 1 --warmup 1 --frames 16384 --no-e2e --no-extras --no-cpu > gpurun_out/ncu_full_conv.log 2>&1
tail -3 gpurun_out/ncu_full_conv.log
ls -la gpurun_out
