# A/B on 4 GPUs: early update launch and presum grid; N=2/4; Qwen3 + GPT-small; timelines.
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
mkdir -p gpurun_out
run() {  # mode cfg n
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $3 --master-addr 127.0.0.1 --master-port 2976$3 bench.py --gpus $3 --config $2 --no-a2a --no-e2e > gpurun_out/ab_$1_$2_$3.log 2>&1
  grep '^{' gpurun_out/ab_$1_$2_$3.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('$1 $2 $3', d['value'], d['step_roofline']['frac'], d['roofline']['frac'], json.dumps(d['step_ms_dist']['median']), s['update_kernel'], s['presum'], s['dispatch'], json.dumps((d.get('nvlink_counters') or {}).get('per_rank', [None])[0]))" || tail -n 3 gpurun_out/ab_$1_$2_$3.log
}
for n in 4 2; do for cfg in gpt-small qwen3-fine; do
  unset MOE_NO_EARLY MOE_PRESUM_GRID; run default $cfg $n
  export MOE_PRESUM_GRID=items; run peritem $cfg $n; unset MOE_PRESUM_GRID
  export MOE_NO_EARLY=1; run noearly $cfg $n; unset MOE_NO_EARLY
done; done
for cfg in gpt-small qwen3-fine; do
rm -rf gpurun_out/ab_tl
MOE_TIMELINE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29773 --log-dir gpurun_out/ab_tl --redirects 3 bench.py --gpus 4 --config $cfg --steps 8 --warmup 3 --no-e2e --no-a2a > /dev/null 2>&1
for f in $(find gpurun_out/ab_tl -name "std*.log" | sort); do grep "TIMELINE" $f | sed -n 5,12p; done > gpurun_out/ab_timeline_$cfg.txt
done
rm -rf gpurun_out/ab_tl
cat gpurun_out/ab_timeline_gpt-small.txt | head -16
