# C = 32 with 8 A slots + 2 conv2 accumulators vs 4 A slots + 3 (build/libnoscope_c32a4.so)
python __graft_entry__.py > /dev/null
timeout 1200 python -m pytest -x -q -p no:cacheprovider -rf tests/test_gpu_cnn.py 2>&1 | tail -2
for r in 1 2; do
  for a in "2 32 32" "4 32 32" "2 32 128"; do echo "A8 $(timeout 300 python tools/prof_cnn.py $a 65536 5)"; echo "A4 $(NOSCOPE_LIB=build/libnoscope_c32a4.so timeout 300 python tools/prof_cnn.py $a 65536 5)"; done
done
