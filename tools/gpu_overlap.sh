# overlapped cascade (opt-in): parity vs serial vs oracle; bench A/B; default-path regression
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -x -q -p no:cacheprovider -rf tests/test_gpu_overlap.py tests/test_gpu_cascade.py tests/test_gpu_edge.py tests/test_gpu_cnn.py 2>&1 | tail -5
for cfg in "NOSCOPE_OVERLAP=0" "NOSCOPE_OVERLAP=1"; do
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-extras --no-cpu > gpurun_out/ovl_bench.json 2> gpurun_out/ovl_bench.err
  echo "$cfg $(python -c "import json;d=json.load(open('gpurun_out/ovl_bench.json'));print(d['value'], d['ms_per_step'], d['stage_ms'], d['clocks'])")"
done
