# second builder set for C = 16 / 64: parity + A/B
python __graft_entry__.py > /dev/null
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_cnn.py tests/test_gpu_overlap.py 2>&1 | tail -1
for r in 1 2; do for a in "2 16 32" "4 16 32" "2 64 32" "4 64 32"; do echo "b2 $(timeout 300 python tools/prof_cnn.py $a 65536 3)"; echo "b1 $(NOSCOPE_LIB=build/libnoscope_b1.so timeout 300 python tools/prof_cnn.py $a 65536 3)"; done; done
