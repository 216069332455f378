python -c "import __graft_entry__; __graft_entry__.build()"
for sl in 12 16 12 16; do
MOE_GRAD_SLOTS=$sl timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-a2a > gpurun_out/rg1.log 2>&1; grep '^{' gpurun_out/rg1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N1 slots=$sl', d['value'], d['stages_ms']['update_kernel'])"
MOE_GRAD_SLOTS=$sl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29723 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-a2a --config mixtral > gpurun_out/rg4m.log 2>&1; grep '^{' gpurun_out/rg4m.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N4 mixtral slots=$sl', d['value'], d['stages_ms']['update_kernel'])"
MOE_GRAD_SLOTS=$sl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29724 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-a2a > gpurun_out/rg4.log 2>&1; grep '^{' gpurun_out/rg4.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N4 slots=$sl', d['value'], d['stages_ms']['update_kernel'])"
done
