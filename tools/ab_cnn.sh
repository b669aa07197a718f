# A/B of two library builds on the CNN (L2C32D32 and L4C32D32, 65,536 frames)
python __graft_entry__.py > /dev/null
NOSCOPE_LIB=build/libnoscope_new.so timeout 600 python -m pytest tests/test_gpu_cnn.py -q -x -p no:cacheprovider 2>&1 | tail -1
for r in 1 2 3; do for v in base new; do
  echo -n "$v "; NOSCOPE_LIB=build/libnoscope_$v.so timeout 300 python tools/prof_cnn.py 2 32 32 65536 3
done; done
