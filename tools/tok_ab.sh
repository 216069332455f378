python -c "import __graft_entry__; __graft_entry__.build()"
for cfg in qwen3-fine gpt-small; do for u in 2 4 2 4; do
MOE_COMB_U=$u timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $cfg > gpurun_out/ab.log 2>&1; grep '^{' gpurun_out/ab.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); a=d['token_a2a']; print('$cfg U=$u', a.get('rows_per_slot'), a.get('dispatch_ms'), a.get('combine_ms'), a.get('combine_roofline',{}).get('frac'), a.get('skipped'))"
done; done
