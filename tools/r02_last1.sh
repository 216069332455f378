# 1 GPU, final code: the parity cases the de-dup subsets did not select (host state, early
# launch, every-element, capacity/policies, split calls) and smoke().
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 230 python -m pytest tests/test_gpu_parity.py -q -x --timeout 200 -k "host_state or early or medium_every or capacity or split_calls" > gpurun_out/l1_tests.log 2>&1; tail -n 2 gpurun_out/l1_tests.log
timeout 60 python -c "import __graft_entry__; __graft_entry__.smoke()" 2>&1 | tail -n 1
