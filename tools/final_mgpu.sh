python -c "import __graft_entry__; __graft_entry__.build()"
timeout 2400 python -m pytest tests/test_multi_gpu.py -q --timeout 900 > gpurun_out/fm_t.log 2>&1; tail -n 3 gpurun_out/fm_t.log
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2973$n bench.py --gpus $n > gpurun_out/fm_b$n.log 2>&1; grep '^{' gpurun_out/fm_b$n.log > gpurun_out/fm_b$n.json; python -c "import json; d=json.load(open('gpurun_out/fm_b$n.json')); print($n, d['value'], d['roofline']['bound'], d['roofline']['frac'], d['step_roofline']['frac'], d['e2e']['value'], d['e2e']['router_inputs_only']['value'], json.dumps(d['step_ms_dist']))"
done
