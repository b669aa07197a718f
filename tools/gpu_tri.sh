# C = 32: 1 conv1 group + 4 conv2 accumulators issued as triples vs 2 groups + 2 accumulators
python __graft_entry__.py > /dev/null
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_cnn.py tests/test_gpu_overlap.py 2>&1 | tail -1
for r in 1 2; do for a in "2 32 32" "4 32 32"; do echo "tri $(timeout 300 python tools/prof_cnn.py $a 65536 5)"; echo "pairs $(NOSCOPE_LIB=build/libnoscope_notri.so timeout 300 python tools/prof_cnn.py $a 65536 5)"; done; done
