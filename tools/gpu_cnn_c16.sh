# C = 16 conv1 4-chain issue: parity + timing
python __graft_entry__.py > /dev/null
timeout 1200 python -m pytest -x -q -p no:cacheprovider -rf tests/test_gpu_cnn.py tests/test_gpu_overlap.py 2>&1 | tail -2
for a in "2 16 32" "4 16 32" "2 32 32" "2 16 32" "4 16 32" "2 32 32"; do timeout 300 python tools/prof_cnn.py $a 65536 5; done
