# A/B of the sweep's balanced phase-2 evaluation vs HEAD (tools/libnoscope_old.so)
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -q -p no:cacheprovider -rf -x tests/test_gpu_sweep_route.py tests/test_gpu_cbo.py tests/test_gpu_dist.py --timeout 600 2>&1 | tail -3
for i in 1 2; do
echo "== new"; timeout 300 python tools/time_sweep_p2.py 2>&1 | tail -3
echo "== old"; NOSCOPE_LIB=$PWD/tools/libnoscope_old.so timeout 300 python tools/time_sweep_p2.py 2>&1 | tail -3
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_eval.json 2> gpurun_out/bench_eval.err
cut -c1-200 gpurun_out/bench_eval.json
