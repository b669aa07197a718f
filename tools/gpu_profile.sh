# ncu evidence for profiles/: launch list of the bench command + full captures of the top kernels
python __graft_entry__.py
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --frames 16384 --no-e2e --no-extras --no-cpu > gpurun_out/bench_under_ncu.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dd_kernel -s 2 -c 1 -o gpurun_out/prof_dd python bench.py --steps 1 --warmup 1 --frames 16384 --no-e2e --no-extras --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv12 -c 1 -o gpurun_out/prof_fused python tools/prof_cnn.py 2 32 32 8192 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:convt -c 1 -o gpurun_out/prof_convt python tools/prof_cnn.py 2 64 32 8192 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^(ns::)?convg_kernel' -c 1 -o gpurun_out/prof_convg python tools/prof_cnn.py 4 64 32 8192 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_hist -c 1 -o gpurun_out/prof_sweep python tools/prof_sweep.py 100000000 > /dev/null 2>&1
for c in "2 32" "2 64" "4 32" "4 64"; do set -- $c; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnn_launches_L$1C$2.csv python tools/prof_cnn.py $1 $2 32 8192 1 > /dev/null 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/next_launches.csv python tools/prof_next.py > /dev/null 2>&1
ls -la gpurun_out | head -40
