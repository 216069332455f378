# End-of-round-2 evidence on a 4-GPU box (files land in gpurun_out/fin_*):
#   full GPU suite (1-GPU tests + torchrun G=2/4) with per-test results, smoke(),
#   the driver's default bench line at N=1 (+ cpu_baseline) and N=2/4, GPT-small / stress
#   lines, row f4 (host state) at N=1/4, the reference arm at N=1, TIMELINE + KTRACE at N=4.
T=fin
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 3000 python -m pytest tests -m gpu -q -rA --timeout 900 > gpurun_out/${T}_tests.log 2>&1; tail -n 2 gpurun_out/${T}_tests.log
timeout 600 python -c "import __graft_entry__; __graft_entry__.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -n 1 gpurun_out/${T}_smoke.log
summ() { python -c "import json; d=json.load(open('$1')); a=d.get('token_a2a') or {}; c=d.get('cpu_baseline') or {}; print('$2', d['value'], d['roofline']['bound'], d['roofline']['frac'], d['step_roofline']['frac'], d['stages_ms']['update_kernel'], d['stages_ms']['dispatch'], d['step_ms_dist']['median'], d['step_ms_dist']['max'], (a.get('dispatch_roofline') or {}).get('frac'), (a.get('combine_roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), c.get('value'), d['gpu_launches'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))" || tail -n 3 ${1%.json}.log; }
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_n1.log 2>&1; grep '^{' gpurun_out/${T}_n1.log > gpurun_out/${T}_n1.json; summ gpurun_out/${T}_n1.json "default N=1"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2981$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/${T}_n$n.log 2>&1; grep '^{' gpurun_out/${T}_n$n.log > gpurun_out/${T}_n$n.json; summ gpurun_out/${T}_n$n.json "default N=$n"
done
for cfg in gpt-small stress; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/${T}_${cfg}_n1.log 2>&1; grep '^{' gpurun_out/${T}_${cfg}_n1.log > gpurun_out/${T}_${cfg}_n1.json; summ gpurun_out/${T}_${cfg}_n1.json "$cfg N=1"
  for n in 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2982$n bench.py --gpus $n --config $cfg > gpurun_out/${T}_${cfg}_n$n.log 2>&1; grep '^{' gpurun_out/${T}_${cfg}_n$n.log > gpurun_out/${T}_${cfg}_n$n.json; summ gpurun_out/${T}_${cfg}_n$n.json "$cfg N=$n"
  done
done
timeout 900 python bench.py --config gpt-small --host-state --no-cpu-baseline --no-a2a > gpurun_out/${T}_hs_n1.log 2>&1; grep '^{' gpurun_out/${T}_hs_n1.log > gpurun_out/${T}_hs_n1.json; summ gpurun_out/${T}_hs_n1.json "host-state gpt-small N=1"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29834 bench.py --gpus 4 --config gpt-small --host-state --no-a2a > gpurun_out/${T}_hs_n4.log 2>&1; grep '^{' gpurun_out/${T}_hs_n4.log > gpurun_out/${T}_hs_n4.json; summ gpurun_out/${T}_hs_n4.json "host-state gpt-small N=4"
s=$(date +%s.%N)
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_ref.log 2>&1
e=$(date +%s.%N); python -c "print('reference arm wall s', round($e - $s, 1))"
grep '^{' gpurun_out/${T}_ref.log > gpurun_out/${T}_ref.json; python -c "import json; d=json.load(open('gpurun_out/${T}_ref.json')); print('reference', d['value'], d['cpu_baseline']['cores'], d.get('timed_region_s'), d.get('wall_s'))"
rm -rf gpurun_out/${T}_tl
MOE_TIMELINE=1 MOE_KTRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29835 --log-dir gpurun_out/${T}_tl --redirects 3 bench.py --gpus 4 --steps 8 --warmup 3 --no-e2e --no-a2a > /dev/null 2>&1
for f in $(find gpurun_out/${T}_tl -name "std*.log" | sort); do grep "TIMELINE\|KTRACE" $f | tail -n 12; done > gpurun_out/${T}_timeline_n4_qwen3.txt
rm -rf gpurun_out/${T}_tl
echo done
