# 4-GPU check of the early update launch: the GPU parity tests that exercise it, the torchrun
# G=2/4 parity cases, N=1/2/4 Qwen3 + GPT-small bench lines, MOE_TIMELINE at N=4.
T=${1:-m}
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_multi_gpu.py -q -rA -x --timeout 900 > gpurun_out/${T}_tests.log 2>&1; tail -n 2 gpurun_out/${T}_tests.log
for cfg in qwen3-fine gpt-small; do
  for n in 1 2 4; do
    if [ $n = 1 ]; then
      timeout 900 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/${T}_b${n}_$cfg.log 2>&1
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2975$n bench.py --gpus $n --config $cfg > gpurun_out/${T}_b${n}_$cfg.log 2>&1
    fi
    grep '^{' gpurun_out/${T}_b${n}_$cfg.log > gpurun_out/${T}_b${n}_$cfg.json
    python -c "import json; d=json.load(open('gpurun_out/${T}_b${n}_$cfg.json')); a=d.get('token_a2a') or {}; print('$cfg', $n, d['value'], d['roofline']['bound'], d['roofline']['frac'], d['step_roofline']['frac'], json.dumps({k: v for k, v in d['stages_ms'].items() if k != 'note'}), (a.get('dispatch_roofline') or {}).get('frac'), (a.get('combine_roofline') or {}).get('frac'), json.dumps(d['step_ms_dist']))" || tail -n 5 gpurun_out/${T}_b${n}_$cfg.log
  done
done
for cfg in qwen3-fine gpt-small; do
rm -rf gpurun_out/${T}_tl
MOE_TIMELINE=1 MOE_KTRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29672 --log-dir gpurun_out/${T}_tl --redirects 3 bench.py --gpus 4 --config $cfg --steps 6 --warmup 3 --no-e2e --no-a2a > /dev/null 2>&1
for f in $(find gpurun_out/${T}_tl -name "std*.log" | sort); do grep "TIMELINE\|KTRACE" $f | tail -n 8; done > gpurun_out/${T}_timeline_n4_$cfg.txt
done
rm -rf gpurun_out/${T}_tl
head -n 40 gpurun_out/${T}_timeline_n4_qwen3-fine.txt
