# A/B: base build (NG=4) vs new build at NG=4 and NG=5 (same box, alternating)
python __graft_entry__.py > /dev/null
for r in 1 2; do
  for v in "base 4" "new 4" "new 5"; do
    set -- $v
    NOSCOPE_DD_NG=$2 NOSCOPE_LIB=build/libnoscope_$1.so timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-extras --no-cpu 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 NG=$2', d['value'], d['stage_ms']['dd_kernel'])"
  done
done
