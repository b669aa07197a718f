# C = 32 fused-kernel TMEM plans (NS_C32_CFG): parity of each + timing
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -x -q -p no:cacheprovider -rf tests/test_gpu_cnn.py -k "fused or L2 or full" 2>&1 | tail -1
for c in 2 3; do NOSCOPE_LIB=build/libnoscope_cfg$c.so timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_cnn.py 2>&1 | tail -1; done
for r in 1 2; do
  echo "cfg1 $(timeout 300 python tools/prof_cnn.py 2 32 32 65536 5)"
  for c in 0 2 3; do echo "cfg$c $(NOSCOPE_LIB=build/libnoscope_cfg$c.so timeout 300 python tools/prof_cnn.py 2 32 32 65536 5)"; done
done
