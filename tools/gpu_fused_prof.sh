python __graft_entry__.py
timeout 120 ./tools/umma_bench
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:conv12' -c 1 -o gpurun_out/prof_fused3 python tools/prof_cnn.py 2 32 32 8192 1 > /dev/null 2>&1
ls gpurun_out | grep fused3
