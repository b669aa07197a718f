# A/B of two builds on the tiny cascade and the CNN grid archs (same box)
python __graft_entry__.py > /dev/null
for r in 1 2; do
  for v in base new; do
    echo "== $v"
    NOSCOPE_LIB=build/libnoscope_$v.so python tools/prof_tiny.py | tail -1
    for a in "2 32 32" "2 32 128" "4 32 128" "4 64 128"; do NOSCOPE_LIB=build/libnoscope_$v.so python tools/prof_cnn.py $a 65536 5 | tail -1; done
  done
done
