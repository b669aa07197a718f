# ncu tensor-pipe activity of every kernel of each CNN-grid arch (65,536 frames, one call),
# time-weighted per arch (tools/tensor_weighted.py)
python __graft_entry__.py > /dev/null
for a in "2 32 32" "2 32 128" "2 64 32" "2 64 128" "4 32 32" "4 32 128" "4 64 32" "4 64 128" "2 16 32" "4 16 32"; do
  set -- $a
  timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/tensor_L$1C$2D$3.csv python tools/prof_cnn.py $1 $2 $3 65536 1 > /dev/null 2>&1
done
ls gpurun_out/tensor_*.csv | wc -l
