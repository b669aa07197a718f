python __graft_entry__.py > /dev/null
for k in 256 64 32 16 8; do echo "ks<=$k $(NOSCOPE_GEMM_KSPLIT_MAX=$k timeout 300 python tools/time_train.py 2>&1 | tail -1 | cut -c1-80)"; done
