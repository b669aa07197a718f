# sweep histogram launch shapes (threads per CTA x records per thread)
python __graft_entry__.py > /dev/null
for r in 1 2; do
  echo "512x8 (product) $(timeout 300 python tools/prof_sweep.py 1000000000 | tail -1)"
  for v in 1024_4 1024_2 1024_5 1024_6; do echo "$v $(NOSCOPE_LIB=build/libnoscope_h$v.so timeout 300 python tools/prof_sweep.py 1000000000 | tail -1)"; done
done
