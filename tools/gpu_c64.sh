# C = 64 conv1-only kernel: 8 chains (both halves interleaved) vs the previous build
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_cnn.py 2>&1 | tail -1
for r in 1 2; do for a in "2 64 32" "4 64 32"; do echo "now $(timeout 300 python tools/prof_cnn.py $a 65536 3)"; done; done
