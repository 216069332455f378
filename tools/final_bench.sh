# default bench lines at N=1,2,4 (the driver's command), saved as gpurun_out/fb_n{N}.json
python -c "import __graft_entry__; __graft_entry__.build()"
timeout 900 python bench.py > gpurun_out/fb1.log 2>&1; grep '^{' gpurun_out/fb1.log > gpurun_out/fb_n1.json
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2977$n bench.py --gpus $n > gpurun_out/fb$n.log 2>&1; grep '^{' gpurun_out/fb$n.log > gpurun_out/fb_n$n.json
done
for n in 1 2 4; do python -c "import json; d=json.load(open('gpurun_out/fb_n$n.json')); print($n, d['value'], d['roofline']['bound'], d['roofline']['frac'], d['step_roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['clocks']['reasons'])"; done
