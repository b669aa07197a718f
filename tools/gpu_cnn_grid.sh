# CNN: parity tests, then per-arch throughput and launch lists of the C=64 nets + L4C32
python __graft_entry__.py
timeout 900 python -m pytest tests/test_gpu_cnn.py -q --timeout 120 -p no:cacheprovider -rf -x 2>&1 | tail -3
for L in 2 4; do for C in 32 64; do timeout 300 python tools/prof_cnn.py $L $C 32 65536 3; done; done
for cfg in "2 64" "4 32" "4 64"; do
  set -- $cfg
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnn_launches_L$1C$2.csv python tools/prof_cnn.py $1 $2 32 8192 1 > /dev/null 2>&1
done
[ -n "$NCU_FULL" ] && timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:^(ns::)?convg_kernel' -s 1 -c 1 -o gpurun_out/prof_convg python tools/prof_cnn.py 2 64 32 8192 1 > /dev/null 2>&1
ls gpurun_out | head -30
