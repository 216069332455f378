# row f3 measurement: bench lines with token_a2a at N=1 and N=4, then ncu launch list at N=1
set -x
python -c "import __graft_entry__; __graft_entry__.build()"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/f3_b1.log 2>&1; grep '^{' gpurun_out/f3_b1.log | tail -n 1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config mixtral --no-e2e > gpurun_out/f3_b1m.log 2>&1; grep '^{' gpurun_out/f3_b1m.log | tail -n 1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/f3_b4.log 2>&1; grep '^{' gpurun_out/f3_b4.log | tail -n 1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 4 --steps 5 --warmup 3 --config mixtral --no-e2e > gpurun_out/f3_b4m.log 2>&1; grep '^{' gpurun_out/f3_b4m.log | tail -n 1
tail -n 5 gpurun_out/f3_b4.log
