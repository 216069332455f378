python -c "import __graft_entry__; __graft_entry__.build()"
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/fc_tests.log 2>&1; tail -n 2 gpurun_out/fc_tests.log
timeout 900 python -c "import __graft_entry__; __graft_entry__.smoke()" 2>&1 | tail -n 1
timeout 900 python bench.py > gpurun_out/fc_bench.log 2>&1; grep '^{' gpurun_out/fc_bench.log > gpurun_out/fc_bench.json; python -c "import json; d=json.load(open('gpurun_out/fc_bench.json')); print(d['value'], d['roofline']['frac'], d['step_roofline']['frac'], d['cpu_baseline']['value'], d['e2e']['value'], d['gpu_launches'], json.dumps(d['clocks']))"
