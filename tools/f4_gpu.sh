set -x
python -c "import __graft_entry__; __graft_entry__.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "host_state" > gpurun_out/f4_t.log 2>&1; tail -n 15 gpurun_out/f4_t.log
MOE_UPDATE_KERNEL=ldg timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "host_state_is and medium-1" > gpurun_out/f4_t2.log 2>&1; tail -n 3 gpurun_out/f4_t2.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-a2a --host-state > gpurun_out/f4_b1.log 2>&1; grep '^{' gpurun_out/f4_b1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['roofline']), json.dumps(d['stages_ms']))"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-a2a --host-state > gpurun_out/f4_b4.log 2>&1; grep '^{' gpurun_out/f4_b4.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['roofline']), json.dumps(d['stages_ms']))"
tail -n 4 gpurun_out/f4_b4.log
