# GPU parity suite (changed areas first, then everything) + smoke
python __graft_entry__.py > /dev/null
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rf \
  tests/test_gpu_fit.py tests/test_gpu_train.py tests/test_gpu_cbo.py tests/test_gpu_sweep_route.py \
  tests/test_gpu_dd.py tests/test_gpu_cnn.py 2>&1 | tail -40 > gpurun_out/gpu_tests_changed.log
tail -30 gpurun_out/gpu_tests_changed.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
