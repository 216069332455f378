# A/B on 4 GPUs: de-dup pre-sum concurrent with the dispatch (default) vs after it.
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
mkdir -p gpurun_out
run() {  # mode cfg n
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $3 --master-addr 127.0.0.1 --master-port 2976$3 bench.py --gpus $3 --config $2 --no-a2a --no-e2e > gpurun_out/ab2_$1_$2_$3.log 2>&1
  grep '^{' gpurun_out/ab2_$1_$2_$3.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('$1 $2 $3', d['value'], d['step_roofline']['frac'], d['roofline']['frac'], json.dumps(d['step_ms_dist']['median']), s['update_kernel'], s['presum'], s['dispatch'], s['update_stage'], json.dumps((d.get('nvlink_counters') or {}).get('per_rank', [None])[0]))" || tail -n 3 gpurun_out/ab2_$1_$2_$3.log
}
for n in 4 2; do for cfg in gpt-small qwen3-fine stress; do
  unset MOE_PRESUM_SERIAL; run concurrent $cfg $n
  export MOE_PRESUM_SERIAL=1; run serial $cfg $n; unset MOE_PRESUM_SERIAL
done; done
for mode in concurrent serial; do
if [ $mode = serial ]; then export MOE_PRESUM_SERIAL=1; fi
rm -rf gpurun_out/ab_tl
MOE_TIMELINE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29773 --log-dir gpurun_out/ab_tl --redirects 3 bench.py --gpus 4 --config qwen3-fine --steps 8 --warmup 3 --no-e2e --no-a2a > /dev/null 2>&1
for f in $(find gpurun_out/ab_tl -name "std*.log" | sort); do grep "TIMELINE" $f | sed -n 5,8p; done > gpurun_out/ab2_timeline_$mode.txt
unset MOE_PRESUM_SERIAL
done
rm -rf gpurun_out/ab_tl
head -4 gpurun_out/ab2_timeline_concurrent.txt; head -4 gpurun_out/ab2_timeline_serial.txt
