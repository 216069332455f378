# host-stage timing check + N=4 numbers for the other workloads
python -c "import __graft_entry__; __graft_entry__.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "split or tiny_configs" > gpurun_out/r_t.log 2>&1; tail -n 1 gpurun_out/r_t.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-a2a > gpurun_out/r1.log 2>&1; grep '^{' gpurun_out/r1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('gpt-small 1', d['value'], json.dumps({k: v for k, v in d['stages_ms'].items() if k != 'note'}))"
for cfg in qwen3-fine stress gpt-small; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-a2a --config $cfg > gpurun_out/r4.log 2>&1; grep '^{' gpurun_out/r4.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg 4', d['value'], d['roofline']['bound'], d['roofline']['frac'], d['step_roofline']['frac'], json.dumps({k: v for k, v in d['stages_ms'].items() if k != 'note'}))"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29692 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-a2a --dedup off --config $cfg > gpurun_out/r4p.log 2>&1; grep '^{' gpurun_out/r4p.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg 4 plain', d['value'], d['roofline']['bound'], d['roofline']['frac'], d['step_roofline']['frac'])"
done
for cfg in qwen3-fine stress; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-a2a --config $cfg > gpurun_out/r1.log 2>&1; grep '^{' gpurun_out/r1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg 1', d['value'], d['roofline']['frac'], d['step_roofline']['frac'], json.dumps({k: v for k, v in d['stages_ms'].items() if k != 'note'}))"
done
