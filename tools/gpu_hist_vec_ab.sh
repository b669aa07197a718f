# A/B of the histogram's vector record loads vs the previous build (tools/libnoscope_old.so)
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -q -p no:cacheprovider -rf -x tests/test_gpu_sweep_route.py tests/test_gpu_cbo.py tests/test_gpu_dist.py --timeout 600 2>&1 | tail -3
for i in 1 2; do
echo "== new"; timeout 300 python tools/prof_sweep.py 1000000000 2>&1 | tail -1
echo "== old"; NOSCOPE_LIB=$PWD/tools/libnoscope_old.so timeout 300 python tools/prof_sweep.py 1000000000 2>&1 | tail -1
done
