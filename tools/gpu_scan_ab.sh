# compaction / routing launch shapes (threads per CTA, CTAs per SM)
python __graft_entry__.py > /dev/null
for r in 1 2; do
  echo "512x3/2 (product)"; timeout 300 python tools/prof_scan.py 0.15 2>&1 | grep -v "^$"
  for v in 1024_1_1 768_2_1 896_2_1 640_2_1; do echo "$v"; NOSCOPE_LIB=build/libnoscope_m$v.so timeout 300 python tools/prof_scan.py 0.15 2>&1 | grep -v "^$"; done
done
