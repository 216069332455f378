python -c "import __graft_entry__; __graft_entry__.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tokens.py tests/test_gpu_readme_example.py -q -x --timeout 900 > gpurun_out/h_t.log 2>&1; tail -n 2 gpurun_out/h_t.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-a2a > gpurun_out/h1.log 2>&1; grep '^{' gpurun_out/h1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N1', d['value'], d['stages_ms']['dispatch'], d['stages_ms']['update_kernel'], d['stages_ms']['host_wait_counts'])"
done
