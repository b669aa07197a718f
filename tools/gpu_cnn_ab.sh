# fused CNN kernel: parity tests, timing of the C=32 archs, ncu capture of conv12_fused
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -q -p no:cacheprovider -rf -x tests/test_gpu_cnn.py tests/test_gpu_cascade.py 2>&1 | tail -4
for a in "2 32 32" "4 32 32" "2 64 32" "2 16 32"; do timeout 300 python tools/prof_cnn.py $a 65536 5 2>&1 | tail -1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv12 -s 2 -c 1 -o gpurun_out/prof_fused python tools/prof_cnn.py 2 32 32 32768 3 > /dev/null 2>&1
ls gpurun_out/prof_fused*
