# 2 GPUs: the bulk-copy de-dup pre-sum over NVLink -- torchrun G=2 de-dup parity cases and the
# Qwen3 / GPT-small N=2 bench A/B against the register-staged kernel (MOE_PRESUM_KERNEL=ldg).
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 600 python -m pytest tests/test_multi_gpu.py -q -rA --timeout 300 -k "dedup and (2-medium or 2-tiny)" > gpurun_out/pt2_tests.log 2>&1; tail -n 2 gpurun_out/pt2_tests.log
run() {  # mode cfg
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29872 bench.py --gpus 2 --config $2 --steps 20 --warmup 5 --no-a2a --no-e2e > gpurun_out/pt2_$1_$2.log 2>&1
  grep '^{' gpurun_out/pt2_$1_$2.log > gpurun_out/pt2_$1_$2.json
  python -c "import json; d=json.load(open('gpurun_out/pt2_$1_$2.json')); s=d['stages_ms']; print('$1 $2', d['value'], d['step_roofline']['frac'], s['presum'], s['update_kernel'], d['step_ms_dist']['median'])" || tail -n 3 gpurun_out/pt2_$1_$2.log
}
for cfg in qwen3-fine gpt-small; do
  unset MOE_PRESUM_KERNEL; run tma $cfg
  export MOE_PRESUM_KERNEL=ldg; run ldg $cfg; unset MOE_PRESUM_KERNEL
done
