# NVLink/NVLS probe on a 2-GPU box: sweep (plain), then ncu NVLink counters of one
# push and one multicast launch (single process; never under torchrun)
M=gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 python scripts/nvlink_probe.py > gpurun_out/nvl_probe_n2.jsonl 2> gpurun_out/nvl_probe_n2.err; echo "probe rc=$?"
timeout 200 python scripts/nvlink_probe.py --once mc --gb 2 > gpurun_out/plain_mc.log 2>&1 && \
timeout 400 ncu --metrics $M --clock-control none -k regex:k_multicast --csv --log-file gpurun_out/ncu_nvl_mc.csv python scripts/nvlink_probe.py --once mc --gb 2 > gpurun_out/ncu_mc.log 2>&1; echo "ncu mc rc=$?"
