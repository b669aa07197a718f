# dd_kernel with the spare ring stages given to the busiest groups: parity + A/B
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -x -q -p no:cacheprovider -rf tests/test_gpu_dd.py tests/test_gpu_fullsize.py tests/test_gpu_cascade.py tests/test_gpu_edge.py 2>&1 | tail -2
for cfg in "NOSCOPE_DD_EVEN=1" "NOSCOPE_DD_X=0" "NOSCOPE_DD_EVEN=1" "NOSCOPE_DD_X=0"; do
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-extras --no-cpu > gpurun_out/ring_bench.json 2> gpurun_out/ring_bench.err
  echo "$cfg $(python -c "import json;d=json.load(open('gpurun_out/ring_bench.json'));print(d['value'], d['ms_per_step'], d['stage_ms']['dd_kernel'], d['roofline']['frac'], d['clocks']['sm_mhz'])")"
done
