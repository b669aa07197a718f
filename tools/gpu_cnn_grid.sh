# CNN: parity tests, then per-arch throughput and a launch list of the 4-layer C=64 net
python __graft_entry__.py
timeout 900 python -m pytest tests/test_gpu_cnn.py -q --timeout 120 -p no:cacheprovider -rf -x 2>&1 | tail -8
for L in 2 4; do for C in 32 64; do timeout 300 python tools/prof_cnn.py $L $C 32 65536 3; done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnn_launches.csv python tools/prof_cnn.py 4 64 32 16384 1 > /dev/null 2>&1
python tools/ncu_summary.py --launches gpurun_out/cnn_launches.csv
