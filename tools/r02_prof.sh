# 1-GPU ncu captures for profiles/r02: launch lists (the bench command) and --set full of the
# dispatch kernels, k_update_tma and the token kernels at Qwen3 and GPT-small scale.
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
mkdir -p gpurun_out
T=${1:-pf}
for cfg in qwen3-fine gpt-small; do
  c=$( [ $cfg = qwen3-fine ] && echo q || echo g )
  B="python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/${T}_${c}_launches.csv $B > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_hist|k_scan|k_scatter" -s 12 -c 3 -o gpurun_out/${T}_${c}_disp -f $B > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_update_tma" -s 4 -c 1 -o gpurun_out/${T}_${c}_update -f $B > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_tok" -s 2 -c 2 -o gpurun_out/${T}_${c}_tok -f $B > /dev/null 2>&1
done
ls -la gpurun_out | grep $T
