python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "modes or full_size or single or fuzz or repeated or invalid or capacity" > gpurun_out/rs_tests.log 2>&1; tail -n 2 gpurun_out/rs_tests.log
timeout 900 python bench.py --config qwen3-fine --no-cpu-baseline --no-e2e > gpurun_out/rs_q.log 2>&1
grep '^{' gpurun_out/rs_q.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('qwen3', d['value'], d['roofline']['frac'], d['step_roofline']['frac'], d['stages_ms']['update_kernel'], d['stages_ms']['dispatch'], d['step_ms_dist']['median'], d['gpu_launches'], json.dumps({k: v for k, v in d['stages_ms'].items() if k.startswith('host')}))"
B="python bench.py --config qwen3-fine --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-a2a"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/rs_q_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_hist|k_scan|k_scatter" -s 12 -c 3 -o gpurun_out/rs_q_disp -f $B > /dev/null 2>&1
