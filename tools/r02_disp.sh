# 1-GPU dispatch iteration: parity tests touching the dispatch, bench lines, dispatch ncu.
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
mkdir -p gpurun_out
T=${1:-d}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tokens.py -q -x --timeout 900 -k "tiny or odd or capacity or fuzz or repeated or invalid or full_size or edge or token or medium" > gpurun_out/${T}_tests.log 2>&1; tail -n 2 gpurun_out/${T}_tests.log
for cfg in qwen3-fine gpt-small; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/${T}_$cfg.log 2>&1
  grep '^{' gpurun_out/${T}_$cfg.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['roofline']['frac'], d['step_roofline']['frac'], d['stages_ms']['update_kernel'], d['stages_ms']['dispatch'], d['step_ms_dist']['median'])"
  c=$( [ $cfg = qwen3-fine ] && echo q || echo g )
  B="python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-a2a"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_${c}_launches.csv $B > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_hist|k_scan|k_scatter" -s 12 -c 3 -o gpurun_out/${T}_${c}_disp -f $B > /dev/null 2>&1
done
