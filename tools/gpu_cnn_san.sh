# CNN TMEM plans: CNN-using GPU tests, grid timing, compute-sanitizer memcheck + synccheck
python __graft_entry__.py > /dev/null
timeout 1800 python -m pytest -q -p no:cacheprovider -rf tests/test_gpu_cnn.py tests/test_gpu_cascade.py tests/test_gpu_overlap.py tests/test_gpu_cbo.py tests/test_gpu_eval.py tests/test_gpu_edge.py 2>&1 | tail -2
for a in "2 32 32" "2 32 128" "4 32 32" "4 32 128" "2 64 32" "2 64 128" "4 64 32" "4 64 128" "2 16 32" "4 16 32"; do timeout 300 python tools/prof_cnn.py $a 65536 5; done
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_$tool.log
done
