python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -q -p no:cacheprovider -rf -x tests/test_gpu_sweep_route.py 2>&1 | tail -3
timeout 300 python tools/prof_sweep.py 1000000000 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_hist -c 1 -o gpurun_out/prof_sweep python tools/prof_sweep.py 100000000 > /dev/null 2>&1
ls gpurun_out/prof_sweep*
