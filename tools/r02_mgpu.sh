# Round-2 check on a 4-GPU box: the whole GPU suite (1-GPU tests + torchrun G=2/4 parity),
# N=1/2/4 bench lines for Qwen3 and GPT-small, a KTRACE log at N=4, dispatch launch list.
# usage: bash tools/r02_mgpu.sh TAG
T=${1:-m}
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${T}_tests.log 2>&1; tail -n 4 gpurun_out/${T}_tests.log
for cfg in qwen3-fine gpt-small; do
  for n in 1 2 4; do
    if [ $n = 1 ]; then
      timeout 900 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/${T}_b${n}_$cfg.log 2>&1
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2975$n bench.py --gpus $n --config $cfg > gpurun_out/${T}_b${n}_$cfg.log 2>&1
    fi
    grep '^{' gpurun_out/${T}_b${n}_$cfg.log > gpurun_out/${T}_b${n}_$cfg.json
    python -c "import json; d=json.load(open('gpurun_out/${T}_b${n}_$cfg.json')); a=d.get('token_a2a') or {}; print('$cfg', $n, d['value'], d['roofline']['bound'], d['roofline']['frac'], d['step_roofline']['frac'], json.dumps({k: v for k, v in d['stages_ms'].items() if k != 'note'}), (a.get('dispatch_roofline') or {}).get('frac'), (a.get('combine_roofline') or {}).get('frac'), json.dumps(d['step_ms_dist']))"
  done
done
rm -rf gpurun_out/${T}_ktl
MOE_KTRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 --log-dir gpurun_out/${T}_ktl --redirects 1 bench.py --gpus 4 --steps 6 --warmup 3 --no-e2e --no-a2a > /dev/null 2>&1
for f in $(find gpurun_out/${T}_ktl -name "stdout.log" | sort); do grep KTRACE $f | tail -n 4; done > gpurun_out/${T}_ktrace_n4_qwen3.txt
cat gpurun_out/${T}_ktrace_n4_qwen3.txt
rm -rf gpurun_out/${T}_ktl
B="python bench.py --config qwen3-fine --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-a2a"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_q_launches.csv $B > /dev/null 2>&1
B="python bench.py --config gpt-small --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-a2a"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_g_launches.csv $B > /dev/null 2>&1
