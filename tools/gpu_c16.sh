python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -q -p no:cacheprovider -rf tests/test_gpu_cnn.py 2>&1 | tail -8 > gpurun_out/gpu_tests_cnn.log
tail -5 gpurun_out/gpu_tests_cnn.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smem_atomic_bw tools/smem_atomic_bw.cu && /tmp/smem_atomic_bw | tee gpurun_out/smem_atomic_bw.txt
timeout 300 python tools/prof_cnn.py 2 16 32 65536 3 2>&1 | tail -3
