python -c "import __graft_entry__; __graft_entry__.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "dedup" > gpurun_out/l_t.log 2>&1; tail -n 1 gpurun_out/l_t.log
timeout 900 python -m pytest tests/test_multi_gpu.py -q -x --timeout 600 -k "lazy" > gpurun_out/l_t2.log 2>&1; tail -n 1 gpurun_out/l_t2.log
for cfg in gpt-small mixtral; do for lz in on off; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-a2a --config $cfg --lazy $lz > gpurun_out/l4.log 2>&1; grep '^{' gpurun_out/l4.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg 4 lazy=$lz', d['value'], d['step_roofline']['frac'], json.dumps({k: v for k, v in d['stages_ms'].items() if k not in ('note',)}))"
done; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29702 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-a2a > gpurun_out/l2.log 2>&1; grep '^{' gpurun_out/l2.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('gpt-small 2 lazy', d['value'], d['step_roofline']['frac'])"
