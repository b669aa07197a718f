# C = 64 conv1-only: N = 64 MMAs (wide) vs two N = 32 halves
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_cnn.py 2>&1 | tail -1
for r in 1 2; do for a in "2 64 32" "4 64 32"; do echo "asmem $(timeout 300 python tools/prof_cnn.py $a 65536 3)"; echo "atmem1 $(NOSCOPE_LIB=build/libnoscope_c64narrow.so timeout 300 python tools/prof_cnn.py $a 65536 3)"; done; done
