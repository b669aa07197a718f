# fused CNN with the skewed image layout: parity + grid timing + ncu wavefronts
python __graft_entry__.py > /dev/null
timeout 1200 python -m pytest -x -q -p no:cacheprovider -rf tests/test_gpu_cnn.py tests/test_gpu_cascade.py 2>&1 | tail -2
for a in "2 32 32" "2 16 32" "2 64 32" "4 32 32"; do timeout 300 python tools/prof_cnn.py $a 65536 5; done
for a in "2 32 32" "2 16 32"; do timeout 300 python tools/prof_cnn.py $a 65536 5; done
timeout 600 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:conv12_fused -c 1 python tools/prof_cnn.py 2 32 32 32768 1 2>&1 | grep -E "conv12|wavefronts|conflicts|duration|tensor" | head
