# fixed-depth histogram instantiations: sweep parity + 1e9-record timing (depth 7)
python __graft_entry__.py > /dev/null
timeout 1200 python -m pytest -q -p no:cacheprovider -rf tests/test_gpu_sweep_route.py tests/test_gpu_cbo.py tests/test_gpu_dist.py --timeout 900 2>&1 | tail -3
timeout 300 python tools/prof_sweep.py 1000000000 2>&1 | tail -1
