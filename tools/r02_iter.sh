# Round-2 iteration on 1 GPU: build, full GPU suite, Qwen3 + GPT-small bench lines, launch list
# and --set full captures of the dispatch kernels and k_update_tma at Qwen3 scale.
# usage: bash tools/r02_iter.sh TAG [notests]
T=${1:-it}
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
if [ "$2" != "notests" ]; then
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/${T}_tests.log 2>&1; tail -n 3 gpurun_out/${T}_tests.log
fi
for cfg in qwen3-fine gpt-small; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/${T}_bench_$cfg.log 2>&1
  grep '^{' gpurun_out/${T}_bench_$cfg.log > gpurun_out/${T}_bench_$cfg.json
  python -c "import json; d=json.load(open('gpurun_out/${T}_bench_$cfg.json')); a=d.get('token_a2a') or {}; print('$cfg', d['value'], d['roofline']['frac'], d['step_roofline']['frac'], json.dumps({k: v for k, v in d['stages_ms'].items() if k != 'note'}), (a.get('dispatch_roofline') or {}).get('frac'), (a.get('combine_roofline') or {}).get('frac'), a.get('skipped'))"
done
B="python bench.py --config qwen3-fine --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-a2a"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_q_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_hist|k_scan|k_scatter" -s 12 -c 3 -o gpurun_out/${T}_q_disp -f $B > /dev/null 2>&1
B="python bench.py --config gpt-small --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/${T}_g_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_hist|k_scan|k_scatter" -s 12 -c 3 -o gpurun_out/${T}_g_disp -f $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_tok" -c 2 -o gpurun_out/${T}_g_tok -f $B > /dev/null 2>&1
ls gpurun_out | grep $T
