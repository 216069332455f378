python -c "import __graft_entry__; __graft_entry__.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "repeated or invalid or tiny or capacity or full_size" > gpurun_out/d_t.log 2>&1; tail -n 2 gpurun_out/d_t.log
for cfg in qwen3-fine gpt-small; do
timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-a2a > gpurun_out/d1.log 2>&1; grep '^{' gpurun_out/d1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['step_roofline']['frac'], json.dumps({k: v for k, v in d['stages_ms'].items() if k != 'note'}))"
done
B="python bench.py --config qwen3-fine --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-a2a"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_hist|k_scan|k_scatter" -s 9 -c 3 -o gpurun_out/q_disp -f $B > gpurun_out/q_ncu.log 2>&1; tail -n 1 gpurun_out/q_ncu.log
