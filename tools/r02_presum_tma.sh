# 1 GPU: the bulk-copy de-dup pre-sum -- parity (virtual de-dup / fuzz / edge subsets) and its
# A/B against the register-staged kernel in virtual mode.
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 300 python tools/presum_ab.py gpt-small 4 > gpurun_out/pt_gpt.log 2>&1; tail -n 9 gpurun_out/pt_gpt.log
timeout 300 python tools/presum_ab.py qwen3-fine 4 8 > gpurun_out/pt_qwen3.log 2>&1; tail -n 9 gpurun_out/pt_qwen3.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "dedup or fuzz or edge or zero_token or fused" > gpurun_out/pt_tests.log 2>&1; tail -n 3 gpurun_out/pt_tests.log
