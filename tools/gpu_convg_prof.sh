# generic conv layer: parity tests + one full ncu capture of the conv2 layer of L2C64
python __graft_entry__.py
timeout 900 python -m pytest tests/test_gpu_cnn.py -q --timeout 120 -p no:cacheprovider -rf -x > gpurun_out/cnn_tests.txt 2>&1; tail -3 gpurun_out/cnn_tests.txt
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:^(ns::)?convg_kernel' -s 1 -c 1 -o gpurun_out/prof_convg python tools/prof_cnn.py 2 64 32 8192 1 > /dev/null 2>&1
ls gpurun_out
