python -c "import __graft_entry__; __graft_entry__.build()"
B="python bench.py --config qwen3-fine --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-a2a"
timeout 600 $B > gpurun_out/q1.log 2>&1; grep '^{' gpurun_out/q1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['step_roofline']['frac'], json.dumps({k: v for k, v in d['stages_ms'].items() if k != 'note'}))"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_hist|k_scan|k_scatter" -s 9 -c 3 -o gpurun_out/q_disp -f $B > gpurun_out/q_ncu.log 2>&1; tail -n 1 gpurun_out/q_ncu.log
