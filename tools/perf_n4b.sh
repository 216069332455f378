set -x
python -c "import __graft_entry__; __graft_entry__.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "dedup or split or host_state or medium" > gpurun_out/p_t.log 2>&1; tail -n 3 gpurun_out/p_t.log
timeout 900 python -m pytest tests/test_multi_gpu.py -q -x --timeout 600 -k "dedup" > gpurun_out/p_t2.log 2>&1; tail -n 3 gpurun_out/p_t2.log
for cfg in gpt-small mixtral; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-a2a --config $cfg > gpurun_out/p_b4_$cfg.log 2>&1; grep '^{' gpurun_out/p_b4_$cfg.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['roofline']['frac'], json.dumps(d['step_roofline']), json.dumps(d['stages_ms']))"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29662 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-a2a --config $cfg > gpurun_out/p_b2_$cfg.log 2>&1; grep '^{' gpurun_out/p_b2_$cfg.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['roofline']['frac'], json.dumps(d['step_roofline']), json.dumps(d['stages_ms']))"
done
MOE_KTRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 --log-dir gpurun_out/ktl --redirects 1 bench.py --gpus 4 --steps 4 --warmup 3 --no-e2e --no-a2a > /dev/null 2>&1
for f in $(find gpurun_out/ktl -name "stdout.log" | sort); do echo $f; grep KTRACE $f | tail -n 3; done
