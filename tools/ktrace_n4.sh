python -c "import __graft_entry__; __graft_entry__.build()"
MOE_KTRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 bench.py --gpus 4 --steps 6 --warmup 3 --no-e2e --no-a2a > gpurun_out/kt4.log 2>&1
grep KTRACE gpurun_out/kt4.log | tail -n 16
MOE_KTRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 4 --steps 3 --warmup 3 --no-e2e --no-a2a --config mixtral > gpurun_out/kt4m.log 2>&1
grep KTRACE gpurun_out/kt4m.log | tail -n 8
