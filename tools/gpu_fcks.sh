python __graft_entry__.py > /dev/null
for r in 1 2; do for cfg in "4 2304" "8 1152" "16 576"; do set -- $cfg
  echo "ks<=$1 $(NOSCOPE_FC_KSPLIT_MAX=$1 NOSCOPE_FC_KGRAN=$2 timeout 300 python tools/prof_cnn.py 2 32 32 65536 5) $(NOSCOPE_FC_KSPLIT_MAX=$1 NOSCOPE_FC_KGRAN=$2 timeout 300 python tools/prof_cnn.py 2 32 32 16384 5) $(NOSCOPE_FC_KSPLIT_MAX=$1 NOSCOPE_FC_KGRAN=$2 timeout 300 python tools/prof_cnn.py 2 32 32 256 20)"
done; done
