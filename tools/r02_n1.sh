# 1-GPU: default bench lines (with cpu_baseline), early-launch A/B, reference arm wall time.
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
mkdir -p gpurun_out
T=${1:-n1}
for mode in default early; do
  if [ $mode = early ]; then export MOE_EARLY_UPDATE=1; fi
  for cfg in qwen3-fine gpt-small; do
    extra="--no-cpu-baseline"; if [ $mode = default ] && [ $cfg = qwen3-fine ]; then extra=""; fi
    timeout 900 python bench.py --config $cfg $extra > gpurun_out/${T}_${mode}_$cfg.log 2>&1
    grep '^{' gpurun_out/${T}_${mode}_$cfg.log > gpurun_out/${T}_${mode}_$cfg.json
    python -c "import json; d=json.load(open('gpurun_out/${T}_${mode}_$cfg.json')); a=d.get('token_a2a') or {}; c=d.get('cpu_baseline') or {}; print('$mode $cfg', d['value'], d['roofline']['frac'], d['step_roofline']['frac'], d['stages_ms']['update_kernel'], d['stages_ms']['dispatch'], d['step_ms_dist']['median'], (a.get('dispatch_roofline') or {}).get('frac'), (a.get('combine_roofline') or {}).get('frac'), d['e2e']['value'], c.get('value'), c.get('cores'), json.dumps(c.get('stages_ms')))" || tail -n 5 gpurun_out/${T}_${mode}_$cfg.log
  done
  unset MOE_EARLY_UPDATE
done
s=$(date +%s.%N)
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_ref.log 2>&1
e=$(date +%s.%N)
python -c "print('reference arm wall', $e - $s)"
tail -n 1 gpurun_out/${T}_ref.log | cut -c1-600
