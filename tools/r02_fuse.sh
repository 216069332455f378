python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tokens.py tests/test_gpu_readme_example.py -q -x --timeout 900 > gpurun_out/fu_tests.log 2>&1; tail -n 2 gpurun_out/fu_tests.log
for cfg in gpt-small qwen3-fine; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/fu_$cfg.log 2>&1
  grep '^{' gpurun_out/fu_$cfg.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['roofline']['frac'], d['step_roofline']['frac'], d['stages_ms']['update_kernel'], d['stages_ms']['dispatch'], d['step_ms_dist']['median'], d['gpu_launches'])"
done
B="python bench.py --config gpt-small --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-a2a"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/fu_g_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_hist|k_scatter" -s 8 -c 2 -o gpurun_out/fu_g_disp -f $B > /dev/null 2>&1
