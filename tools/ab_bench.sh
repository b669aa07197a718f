# A/B of two library builds on the headline bench (same box, alternating runs)
python __graft_entry__.py > /dev/null
for r in 1 2 3; do
  for v in base new; do
    NOSCOPE_LIB=build/libnoscope_$v.so timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-extras --no-cpu 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['stage_ms']['dd_kernel'], d['roofline']['frac'])"
  done
done
