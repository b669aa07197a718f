# histogram launch shapes with the vector record loads (threads x records per thread)
for i in 1 2; do
echo "== 1024x4"; timeout 300 python tools/prof_sweep.py 1000000000 2>&1 | tail -1
for v in 1024x8 512x8 512x4; do echo "== $v"; NOSCOPE_LIB=$PWD/tools/libnoscope_h$v.so timeout 300 python tools/prof_sweep.py 1000000000 2>&1 | tail -1; done
done
