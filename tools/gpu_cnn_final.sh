# fused CNN TMEM plan: CNN-using GPU tests + CNN grid timing + bench
python __graft_entry__.py > /dev/null
timeout 1800 python -m pytest -q -p no:cacheprovider -rf tests/test_gpu_cnn.py tests/test_gpu_cascade.py tests/test_gpu_fullsize.py tests/test_gpu_overlap.py tests/test_gpu_cbo.py tests/test_gpu_eval.py tests/test_gpu_dist.py tests/test_gpu_edge.py tests/test_gpu_train.py 2>&1 | tail -3
for a in "2 32 32" "2 32 128" "4 32 32" "2 16 32" "4 16 32" "2 64 32" "4 64 32"; do timeout 300 python tools/prof_cnn.py $a 65536 5; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-extras --no-cpu > gpurun_out/cnnf_bench.json 2> gpurun_out/cnnf_bench.err
python -c "import json;d=json.load(open('gpurun_out/cnnf_bench.json'));print(d['value'], d['ms_per_step'], d['stage_ms'], d['cnn'])"
