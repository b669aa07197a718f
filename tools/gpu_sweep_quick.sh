python __graft_entry__.py
timeout 600 python -m pytest tests/test_gpu_sweep_route.py -q --timeout 300 -p no:cacheprovider -rf -x 2>&1 | tail -3
python tools/prof_sweep.py 100000000
python tools/prof_sweep.py 1000000
