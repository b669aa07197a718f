# one CNN chunk for fused L = 2 archs: CNN/cascade tests + bench
python __graft_entry__.py > /dev/null
timeout 1800 python -m pytest -q -p no:cacheprovider -rf tests/test_gpu_cnn.py tests/test_gpu_cascade.py tests/test_gpu_fullsize.py tests/test_gpu_overlap.py tests/test_gpu_edge.py 2>&1 | tail -2
for r in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-extras --no-cpu > gpurun_out/chunk_bench.json 2> gpurun_out/chunk_bench.err
python -c "import json;d=json.load(open('gpurun_out/chunk_bench.json'));print(d['value'], d['ms_per_step'], d['stage_ms'], d['gpu_launches'])"
done
