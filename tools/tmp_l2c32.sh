python __graft_entry__.py
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnn_launches_L2C32.csv python tools/prof_cnn.py 2 32 32 8192 1 > /dev/null 2>&1
for k in 254; do NOSCOPE_LIB=build/libnoscope_exp$k.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnn_launches_L2C32_exp$k.csv python tools/prof_cnn.py 2 32 32 8192 1 > /dev/null 2>&1; done
