# compaction / routing: parity tests, timing, ncu captures
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -q -p no:cacheprovider -rf tests/test_gpu_sweep_route.py tests/test_gpu_cascade.py tests/test_gpu_dist.py 2>&1 | tail -8 > gpurun_out/gpu_tests_scan.log
tail -5 gpurun_out/gpu_tests_scan.log
timeout 300 python tools/prof_scan.py 2>&1 | tee gpurun_out/prof_scan.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:compact_fired -s 1 -c 1 -o gpurun_out/prof_compact python tools/prof_scan.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_kernel -s 1 -c 1 -o gpurun_out/prof_route python tools/prof_scan.py > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
