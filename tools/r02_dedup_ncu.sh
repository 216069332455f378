# 1 GPU: the de-dup update stage in virtual mode (GPT-small, G = 4 on one device) -- algorithmic
# bytes summed over the virtual GPUs vs ncu --set full DRAM bytes of k_presum, k_update_tma and
# k_replicate (the same command first runs without ncu and must exit 0).
mkdir -p gpurun_out
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 300 python tools/dedup_traffic.py gpt-small 4 > gpurun_out/dd_plain.log 2>&1 || { tail -n 20 gpurun_out/dd_plain.log; exit 1; }
tail -n 1 gpurun_out/dd_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_presum|k_update_tma|k_replicate" --launch-skip 6 -c 3 -f -o gpurun_out/dedup_virtual_g4_gpt_small python tools/dedup_traffic.py gpt-small 4 > gpurun_out/dd_ncu.log 2>&1; echo ncu rc=$?
tail -n 3 gpurun_out/dd_ncu.log
ncu -i gpurun_out/dedup_virtual_g4_gpt_small.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum > gpurun_out/dd_raw.csv 2>&1; cat gpurun_out/dd_raw.csv | cut -c1-400 | head -8
