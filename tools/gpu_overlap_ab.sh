# does plain ALU work on the side SMs slow dd_kernel?
python __graft_entry__.py > /dev/null
for cfg in "NOSCOPE_SIDE_EXP=64" "NOSCOPE_SIDE_EXP=2" "NOSCOPE_SIDE_EXP=64"; do
  env $cfg NOSCOPE_DD_TRACE=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-extras --no-cpu > gpurun_out/ovl_bench.json 2> gpurun_out/ovl_bench.err
  echo "$cfg $(python -c "import json;d=json.load(open('gpurun_out/ovl_bench.json'));print(d['value'], d['ms_per_step'], d['stage_ms']['dd_kernel'], d['stage_ms']['dd_tail'], d['clocks']['sm_mhz'])")"
  grep DDTRACE gpurun_out/ovl_bench.err | tail -1 | cut -c1-700
done
