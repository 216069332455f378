python -c "import __graft_entry__; __graft_entry__.build()"
timeout 1200 python -m pytest tests/test_multi_gpu.py -q -x --timeout 900 -k "dedup" > gpurun_out/pf_t.log 2>&1; tail -n 1 gpurun_out/pf_t.log
for cfg in gpt-small mixtral gpt-small; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-a2a --config $cfg > gpurun_out/pf4.log 2>&1; grep '^{' gpurun_out/pf4.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg 4', d['value'], json.dumps({k: v for k, v in d['stages_ms'].items() if k in ('dispatch','update_kernel','presum','replicate')}))"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29742 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-a2a > gpurun_out/pf2.log 2>&1; grep '^{' gpurun_out/pf2.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('gpt-small 2', d['value'])"
