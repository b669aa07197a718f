# compaction with grid-interleaved phase 1: parity + timing
python __graft_entry__.py > /dev/null
timeout 1200 python -m pytest -x -q -p no:cacheprovider -rf tests/test_gpu_sweep_route.py tests/test_gpu_dd.py tests/test_gpu_cascade.py tests/test_gpu_edge.py 2>&1 | tail -2
timeout 300 python tools/prof_scan.py 0.0 0.15 0.5 2>&1 | grep -v "^$"
