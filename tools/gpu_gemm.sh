python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -q -p no:cacheprovider -rf -x tests/test_gpu_gemm.py tests/test_gpu_train.py 2>&1 | tail -25
