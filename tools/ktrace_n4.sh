# N=4 run with MOE_KTRACE=1: per-phase timestamps of the update kernel, one log per rank
python -c "import __graft_entry__; __graft_entry__.build()"
rm -rf gpurun_out/ktl
MOE_KTRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 --log-dir gpurun_out/ktl --redirects 1 bench.py --gpus 4 --steps 6 --warmup 3 --no-e2e --no-a2a > /dev/null 2>&1
for f in $(find gpurun_out/ktl -name "stdout.log" | sort); do grep KTRACE $f | tail -n 4; done
