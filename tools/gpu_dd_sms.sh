# dd_kernel time vs the number of SMs it runs on (overlap headroom experiment)
python __graft_entry__.py > /dev/null
for n in 148 140 132 124 116; do
  NOSCOPE_DD_SMS=$n timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-extras --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, d['stage_ms']['dd_kernel'], d['ms_per_step'])"
done
