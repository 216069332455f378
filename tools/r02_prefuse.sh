# 4 GPUs: the de-dup pre-sum fused into the update kernel -- parity (virtual + torchrun) and A/B.
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "dedup or edge or fuzz or early or host_state or interval" > gpurun_out/pf2_tests1.log 2>&1; tail -n 2 gpurun_out/pf2_tests1.log
timeout 1800 python -m pytest tests/test_multi_gpu.py -q -rA -x --timeout 900 > gpurun_out/pf2_tests2.log 2>&1; tail -n 3 gpurun_out/pf2_tests2.log
run() {  # mode cfg n
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $3 --master-addr 127.0.0.1 --master-port 2986$3 bench.py --gpus $3 --config $2 --no-a2a --no-e2e > gpurun_out/pf2_$1_$2_$3.log 2>&1
  grep '^{' gpurun_out/pf2_$1_$2_$3.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('$1 $2 $3', d['value'], d['step_roofline']['frac'], d['roofline']['frac'], d['step_ms_dist']['median'], d['step_ms_dist']['max'], s['update_kernel'], s['presum'], s['dispatch'])" || tail -n 3 gpurun_out/pf2_$1_$2_$3.log
}
for n in 4 2; do for cfg in qwen3-fine gpt-small stress; do
  unset MOE_PRESUM_SEPARATE; run fused $cfg $n
  export MOE_PRESUM_SEPARATE=1; run separate $cfg $n; unset MOE_PRESUM_SEPARATE
done; done
rm -rf gpurun_out/pf2_tl
MOE_TIMELINE=1 MOE_KTRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29873 --log-dir gpurun_out/pf2_tl --redirects 3 bench.py --gpus 4 --steps 8 --warmup 3 --no-e2e --no-a2a > /dev/null 2>&1
for f in $(find gpurun_out/pf2_tl -name "std*.log" | sort); do grep "TIMELINE\|KTRACE" $f | tail -n 8; done > gpurun_out/pf2_timeline_n4_qwen3.txt
rm -rf gpurun_out/pf2_tl
head -16 gpurun_out/pf2_timeline_n4_qwen3.txt
