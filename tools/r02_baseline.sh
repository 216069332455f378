# Round-2 baseline on 1 GPU at the required N=1 config (qwen3-fine): GPU tests, bench line,
# ncu launch list, --set full captures of k_update_tma and the three dispatch kernels.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.build()"
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/b_tests.log 2>&1; tail -n 3 gpurun_out/b_tests.log
timeout 900 python bench.py --config qwen3-fine --no-cpu-baseline > gpurun_out/b_bench_q.log 2>&1; grep '^{' gpurun_out/b_bench_q.log > gpurun_out/b_bench_q.json; tail -c 600 gpurun_out/b_bench_q.json
B="python bench.py --config qwen3-fine --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-a2a"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/q_launches.csv $B > gpurun_out/q_launch.log 2>&1; tail -n 2 gpurun_out/q_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_update_tma" -s 4 -c 1 -o gpurun_out/q_update -f $B > gpurun_out/q_ncu_u.log 2>&1; tail -n 1 gpurun_out/q_ncu_u.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_hist|k_scan|k_scatter" -s 12 -c 3 -o gpurun_out/q_disp -f $B > gpurun_out/q_ncu_d.log 2>&1; tail -n 1 gpurun_out/q_ncu_d.log
