# NS_EXP variants (tools/exp_fused.sh builds) on the C = 16 fused kernel
python __graft_entry__.py > /dev/null
for k in 0 16 8 24 32 64 96 6 1 2 0; do echo "EXP=$k $(NOSCOPE_LIB=build/libnoscope_exp$k.so timeout 300 python tools/prof_cnn.py 2 16 32 65536 5)"; done
