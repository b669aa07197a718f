# full GPU suite + smoke + sanitizers + bench (one call)
python __graft_entry__.py > /dev/null
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf 2>&1 | tail -15 > gpurun_out/gpu_tests_full.log
tail -4 gpurun_out/gpu_tests_full.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err
tail -2 gpurun_out/bench_r02b.err
