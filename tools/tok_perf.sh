python -c "import __graft_entry__; __graft_entry__.build()"
timeout 900 python -m pytest tests/test_gpu_tokens.py -q -x --timeout 600 > gpurun_out/tok1.log 2>&1; tail -n 2 gpurun_out/tok1.log
for cfg in gpt-small qwen3-fine gpt-small; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $cfg > gpurun_out/ab.log 2>&1; grep '^{' gpurun_out/ab.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); a=d['token_a2a']; print('$cfg', a.get('rows_per_slot'), a.get('dispatch_ms'), a.get('dispatch_roofline',{}).get('frac'), a.get('combine_ms'), a.get('combine_roofline',{}).get('frac'), a.get('skipped'))"
done
