# 1 GPU: k_replicate's byte-weighted grid -- parity (virtual de-dup subsets) and the virtual-mode
# A/B (tools/presum_ab.py: the "ldg" arm also runs the old 2-D replicate grid).
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 300 python tools/presum_ab.py gpt-small 4 > gpurun_out/rp_gpt.log 2>&1; tail -n 5 gpurun_out/rp_gpt.log
timeout 300 python tools/presum_ab.py stress 4 8 > gpurun_out/rp_stress.log 2>&1; tail -n 5 gpurun_out/rp_stress.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "dedup or fuzz or edge_values" > gpurun_out/rp_tests.log 2>&1; tail -n 2 gpurun_out/rp_tests.log
