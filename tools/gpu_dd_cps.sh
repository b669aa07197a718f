# dd_kernel: CTAs per SM / worker groups A/B (NOSCOPE_DD_CPS, NOSCOPE_DD_NG)
python __graft_entry__.py > /dev/null
for cfg in "1 4" "2 4" "2 3" "2 2" "1 4"; do
  set -- $cfg
  NOSCOPE_DD_CPS=$1 NOSCOPE_DD_NG=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-extras --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cps', $1, 'ng', $2, d['stage_ms']['dd_kernel'], d['ms_per_step'])"
done
