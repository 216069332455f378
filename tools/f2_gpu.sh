set -x
python -c "import __graft_entry__; __graft_entry__.build()"
python -m pytest tests/test_multi_gpu.py -q -x --timeout 900 -k "cf" > gpurun_out/f2_mgpu.log 2>&1; tail -3 gpurun_out/f2_mgpu.log
python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "policy_drops" > gpurun_out/f2_pol.log 2>&1; tail -3 gpurun_out/f2_pol.log
for pol in "--policy alg1" "--policy static" "--policy alg1 --interval 10"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --steps 20 --warmup 5 --config gpt-small $pol --no-e2e 2>&1 | grep '^{' >> gpurun_out/f2_bench4.jsonl
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --steps 10 --warmup 3 --config mixtral $pol --no-e2e 2>&1 | grep '^{' >> gpurun_out/f2_bench4.jsonl
done
timeout 900 python tests/policy_study.py --iters 2000 --out gpurun_out/policy_study.json > gpurun_out/policy_study.log 2>&1; tail -20 gpurun_out/policy_study.log
