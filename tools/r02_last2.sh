# 2 GPUs, final code: torchrun G=2 de-dup parity (real-mode k_presum_tma + byte-weighted
# k_replicate) and the N=2 default bench line (Qwen3) and GPT-small.
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 120 python -m pytest tests/test_multi_gpu.py -q -rA --timeout 100 -k "dedup and (2-medium or 2-tiny)" > gpurun_out/l2_tests.log 2>&1; tail -n 1 gpurun_out/l2_tests.log
for cfg in qwen3-fine gpt-small; do
  timeout 100 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29873 bench.py --gpus 2 --config $cfg --steps 20 --warmup 5 --no-a2a --no-e2e > gpurun_out/l2_$cfg.log 2>&1
  grep '^{' gpurun_out/l2_$cfg.log > gpurun_out/l2_$cfg.json
  python -c "import json; d=json.load(open('gpurun_out/l2_$cfg.json')); s=d['stages_ms']; print('$cfg', d['value'], d['step_roofline']['frac'], s['presum'], s['replicate'], s['update_kernel'])" || tail -n 3 gpurun_out/l2_$cfg.log
done
