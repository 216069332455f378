set -x
python -c "import __graft_entry__; __graft_entry__.build()"
timeout 900 python -m pytest tests/test_gpu_tokens.py -q -x --timeout 600 > gpurun_out/tok1.log 2>&1; tail -n 3 gpurun_out/tok1.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f3_b1.log 2>&1; grep '^{' gpurun_out/f3_b1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps(d['token_a2a']))"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/f3_b4.log 2>&1; grep '^{' gpurun_out/f3_b4.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps(d['token_a2a']))"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29642 bench.py --gpus 4 --steps 5 --warmup 3 --config mixtral --no-e2e > gpurun_out/f3_b4m.log 2>&1; grep '^{' gpurun_out/f3_b4m.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps(d['token_a2a']))"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tok -c 2 -o gpurun_out/tok_n1 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_tok.log 2>&1; tail -n 3 gpurun_out/ncu_tok.log
