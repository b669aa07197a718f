# training: parity tests + throughput A/B (graph replay on/off)
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -q -p no:cacheprovider -rf -x tests/test_gpu_gemm.py tests/test_gpu_train.py 2>&1 | tail -3
for cfg in "NOSCOPE_TRAIN_GRAPH=0" "NOSCOPE_TRAIN_GRAPH=1" "NOSCOPE_TRAIN_GRAPH=0" "NOSCOPE_TRAIN_GRAPH=1"; do
  echo "$cfg $(env $cfg timeout 300 python tools/time_train.py 2>&1 | tail -1 | cut -c1-90)"
done
