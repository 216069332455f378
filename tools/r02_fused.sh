# 4 GPUs: validate the fused de-dup pre-sum (HEAD default) and A/B it against the separate pre-sum.
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.smoke()" > gpurun_out/fu_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "dedup or edge or zero_token or early or fuzz" > gpurun_out/fu_tests1.log 2>&1; tail -n 2 gpurun_out/fu_tests1.log
timeout 1200 python -m pytest tests/test_multi_gpu.py -q -rA -x --timeout 600 > gpurun_out/fu_tests2.log 2>&1; tail -n 3 gpurun_out/fu_tests2.log
run() {  # mode cfg n
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $3 --master-addr 127.0.0.1 --master-port 2986$3 bench.py --gpus $3 --config $2 --no-a2a --no-e2e > gpurun_out/fu_$1_$2_$3.log 2>&1
  grep '^{' gpurun_out/fu_$1_$2_$3.log > gpurun_out/fu_$1_$2_$3.json
  python -c "import sys,json; d=json.load(open('gpurun_out/fu_$1_$2_$3.json')); s=d['stages_ms']; print('$1 $2 $3', d['value'], d['step_roofline']['frac'], d['roofline']['frac'], d['step_ms_dist'], s)" || tail -n 3 gpurun_out/fu_$1_$2_$3.log
}
for cfg in qwen3-fine gpt-small stress; do
  unset MOE_PRESUM_SEPARATE; run fused $cfg 4
  export MOE_PRESUM_SEPARATE=1; run separate $cfg 4; unset MOE_PRESUM_SEPARATE
done
unset MOE_PRESUM_SEPARATE; run fused qwen3-fine 2
export MOE_PRESUM_SEPARATE=1; run separate qwen3-fine 2; unset MOE_PRESUM_SEPARATE
rm -rf gpurun_out/fu_tl
MOE_TIMELINE=1 MOE_KTRACE=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29873 --log-dir gpurun_out/fu_tl --redirects 3 bench.py --gpus 4 --config gpt-small --steps 8 --warmup 3 --no-e2e --no-a2a > /dev/null 2>&1
for f in $(find gpurun_out/fu_tl -name "std*.log" | sort); do grep "TIMELINE\|KTRACE" $f | tail -n 8; done > gpurun_out/fu_timeline_n4_gpt-small.txt
rm -rf gpurun_out/fu_tl
head -20 gpurun_out/fu_timeline_n4_gpt-small.txt
