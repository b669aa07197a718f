# tensor-pipe evidence after the TMEM-plan changes: per-arch time-weighted (non-realtime counter)
# + one --set full capture of the fused C = 32 kernel (realtime counter)
bash tools/gpu_cnn_tensor.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv12_fused -s 1 -c 1 -o gpurun_out/prof_conv12_r02b python tools/prof_cnn.py 2 32 32 32768 1 > gpurun_out/ncu_conv12_r02b.log 2>&1
echo "conv12 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv12_fused -s 1 -c 1 -o gpurun_out/prof_conv12c64_r02b python tools/prof_cnn.py 2 64 32 32768 1 > gpurun_out/ncu_conv12c64_r02b.log 2>&1
echo "conv12 c64 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:convt -s 1 -c 1 -o gpurun_out/prof_convt_r02b python tools/prof_cnn.py 2 64 32 16384 1 > gpurun_out/ncu_convt_r02b.log 2>&1
echo "convt rc=$?"
