# 1 GPU: HBM ceilings by read/write mix, and the token dispatch with streaming stores (A/B).
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
mkdir -p gpurun_out
python tools/hbm_mix.py > gpurun_out/tc_hbm_mix.json 2>&1; cat gpurun_out/tc_hbm_mix.json
for cfg in qwen3-fine gpt-small; do
  for m in plain cs; do
    if [ $m = cs ]; then export MOE_TOK_STORE_CS=1; else unset MOE_TOK_STORE_CS; fi
    timeout 400 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tc_${m}_$cfg.log 2>&1
    grep '^{' gpurun_out/tc_${m}_$cfg.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); t=d['token_a2a']; print('$m $cfg', d['value'], t['dispatch_ms'], t['dispatch_roofline']['frac'], t['combine_ms'], t['combine_roofline']['frac'])" || tail -n 3 gpurun_out/tc_${m}_$cfg.log
  done
done
MOE_TOK_STORE_CS=1 timeout 600 python -m pytest tests/test_gpu_tokens.py -q -x > gpurun_out/tc_tests.log 2>&1; tail -n 2 gpurun_out/tc_tests.log
