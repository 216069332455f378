# full GPU suite + smoke + default bench + ncu launch list + captures (N=1)
python -c "import __graft_entry__; __graft_entry__.build()"
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/ck_tests.log 2>&1; tail -n 3 gpurun_out/ck_tests.log
timeout 900 python -c "import __graft_entry__; __graft_entry__.smoke()" 2>&1 | tail -n 1
timeout 900 python bench.py > gpurun_out/ck_bench.log 2>&1; grep '^{' gpurun_out/ck_bench.log > gpurun_out/ck_bench.json; python -c "import json; d=json.load(open('gpurun_out/ck_bench.json')); print(d['value'], d['roofline']['frac'], d['step_roofline']['frac'], d['cpu_baseline']['value'], d['e2e']['value'])"
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ck_launches.csv $B > gpurun_out/ck_ncu1.log 2>&1; tail -n 1 gpurun_out/ck_ncu1.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update_tma -s 3 -c 1 -o gpurun_out/ck_update -f $B > gpurun_out/ck_ncu2.log 2>&1; tail -n 1 gpurun_out/ck_ncu2.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_hist|k_scan|k_scatter" -s 9 -c 3 -o gpurun_out/ck_dispatch -f $B > gpurun_out/ck_ncu3.log 2>&1; tail -n 1 gpurun_out/ck_ncu3.log
