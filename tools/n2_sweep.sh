python -c "import __graft_entry__; __graft_entry__.build()"
for cfg in qwen3-fine stress mixtral; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29791 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-a2a --config $cfg > gpurun_out/n2.log 2>&1; grep '^{' gpurun_out/n2.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg 2', d['value'], d['roofline']['bound'], d['roofline']['frac'], d['step_roofline']['frac'])"
done
