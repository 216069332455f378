# N=2 stall hunt: step-time distributions with and without the early update launch, host phases
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
mkdir -p gpurun_out
for mode in early noearly; do
  if [ $mode = noearly ]; then export MOE_NO_EARLY=1; else unset MOE_NO_EARLY; fi
  for cfg in gpt-small qwen3-fine; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29752 bench.py --gpus 2 --config $cfg --no-a2a --no-e2e > gpurun_out/st_${mode}_$cfg.log 2>&1
    grep '^{' gpurun_out/st_${mode}_$cfg.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$mode $cfg', d['value'], json.dumps(d['step_ms_dist']), d['stages_ms']['update_kernel'])"
  done
done
unset MOE_NO_EARLY
rm -rf gpurun_out/st_tl
MOE_TIMELINE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29753 --log-dir gpurun_out/st_tl --redirects 3 bench.py --gpus 2 --config gpt-small --steps 8 --warmup 3 --no-e2e --no-a2a > /dev/null 2>&1
for f in $(find gpurun_out/st_tl -name "std*.log" | sort); do grep "TIMELINE\|HOSTSTEP" $f | head -n 60; done > gpurun_out/st_timeline.txt
rm -rf gpurun_out/st_tl
grep -n "rank 0" gpurun_out/st_timeline.txt | head -50
for cfg in qwen3-fine gpt-small; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-a2a --no-e2e > gpurun_out/st_n1_$cfg.log 2>&1
  grep '^{' gpurun_out/st_n1_$cfg.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('n1 $cfg', d['value'], d['roofline']['frac'], json.dumps(d['step_ms_dist']), d['stages_ms']['update_kernel'])"
done
