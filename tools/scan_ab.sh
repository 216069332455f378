python -c "import __graft_entry__; __graft_entry__.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "tiny or single or split or capacity or full_size" > gpurun_out/s_t.log 2>&1; tail -n 1 gpurun_out/s_t.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-a2a > gpurun_out/s1.log 2>&1; grep '^{' gpurun_out/s1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N1', d['value'], d['stages_ms']['dispatch'], d['stages_ms']['update_kernel'])"
done
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-a2a"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s_launches.csv $B > /dev/null 2>&1; grep -E "k_hist|k_scan|k_scatter" gpurun_out/s_launches.csv | tail -n 3 | cut -c1-160
