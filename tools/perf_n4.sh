# dedup parity (virtual + real) and N=1/N=4 bench lines after an update-stage change
set -x
python -c "import __graft_entry__; __graft_entry__.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "dedup or split or host_state" > gpurun_out/p_t.log 2>&1; tail -n 3 gpurun_out/p_t.log
timeout 900 python -m pytest tests/test_multi_gpu.py -q -x --timeout 600 -k "dedup" > gpurun_out/p_t2.log 2>&1; tail -n 3 gpurun_out/p_t2.log
for cfg in gpt-small mixtral; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --config $cfg > gpurun_out/p_b4_$cfg.log 2>&1; grep '^{' gpurun_out/p_b4_$cfg.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['n_gpus'], d['value'], d['roofline']['frac'], d['step_roofline']['frac'], json.dumps({k: v for k, v in d['stages_ms'].items() if k != 'note'}), json.dumps(d.get('token_a2a')))"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29662 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-a2a --config $cfg > gpurun_out/p_b2_$cfg.log 2>&1; grep '^{' gpurun_out/p_b2_$cfg.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['n_gpus'], d['value'], d['roofline']['frac'], d['step_roofline']['frac'], json.dumps({k: v for k, v in d['stages_ms'].items() if k != 'note'}), json.dumps(d.get('token_a2a')))"
done
