# round-2 evidence at HEAD: full GPU suite, default bench, bench launch list, dd_kernel + fused CNN full captures
python __graft_entry__.py > /dev/null
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf 2>&1 | tail -15 > gpurun_out/gpu_tests_final.log
tail -3 gpurun_out/gpu_tests_final.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -2 gpurun_out/bench_final.err; cut -c1-300 gpurun_out/bench_final.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-extras --no-cpu > gpurun_out/launches_final.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dd_kernel -s 1 -c 1 -o gpurun_out/prof_dd_r02 python bench.py --steps 1 --warmup 1 --frames 16384 --no-e2e --no-extras --no-cpu > gpurun_out/ncu_dd_r02.log 2>&1
echo "dd full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv12_fused -s 1 -c 1 -o gpurun_out/prof_conv12_r02 python tools/prof_cnn.py 2 32 32 32768 1 > gpurun_out/ncu_conv12_r02.log 2>&1
echo "conv12 full rc=$?"
ls -la gpurun_out | tail -12
