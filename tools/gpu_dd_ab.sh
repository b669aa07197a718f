# dd_kernel parity + geometry A/B (NG worker groups, CTAs per SM) on the headline bench
python __graft_entry__.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_dd.py tests/test_gpu_fullsize.py tests/test_gpu_cascade.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -5
DD_CFGS=${DD_CFGS:-"2,1 3,1 4,1"}
for r in 1 2; do
  for cfg in $DD_CFGS; do
    set -- ${cfg/,/ }
    NOSCOPE_DD_NG=$1 NOSCOPE_DD_CPS=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-extras --no-cpu 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NG=$1 CPS=$2', d['value'], d['stage_ms']['dd_kernel'], d['roofline']['frac'])"
  done
done
