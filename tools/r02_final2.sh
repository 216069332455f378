# End of round 2, final code, 2-GPU box (files land in gpurun_out/fin2_*): the whole GPU suite
# (1-GPU tests + torchrun G=2; G=4/8 cases skip), smoke(), the driver's default bench line at
# N=1 (+ cpu_baseline) and N=2.
T=fin2
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 600 python -c "import __graft_entry__; __graft_entry__.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -n 1 gpurun_out/${T}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 900 > gpurun_out/${T}_tests.log 2>&1; tail -n 2 gpurun_out/${T}_tests.log
summ() { python -c "import json; d=json.load(open('$1')); a=d.get('token_a2a') or {}; c=d.get('cpu_baseline') or {}; print('$2', d['value'], d['roofline']['bound'], d['roofline']['frac'], d['step_roofline']['frac'], d['stages_ms']['update_kernel'], d['stages_ms']['dispatch'], d['step_ms_dist']['median'], d['step_ms_dist']['max'], (a.get('dispatch_roofline') or {}).get('frac'), (a.get('combine_roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), c.get('value'), d['gpu_launches'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))" || tail -n 3 ${1%.json}.log; }
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_n1.log 2>&1; grep '^{' gpurun_out/${T}_n1.log > gpurun_out/${T}_n1.json; summ gpurun_out/${T}_n1.json "default N=1"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/${T}_n2.log 2>&1; grep '^{' gpurun_out/${T}_n2.log > gpurun_out/${T}_n2.json; summ gpurun_out/${T}_n2.json "default N=2"
