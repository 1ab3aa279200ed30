M=gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 300 python scripts/nvlink_probe.py --ctas 48 --unrolls 8 > gpurun_out/nvl_probe3_n2.jsonl 2>&1; echo "probe rc=$?"
grep copy_panels gpurun_out/nvl_probe3_n2.jsonl
timeout 200 python scripts/nvlink_probe.py --once panels --nctas 128 > gpurun_out/plain_panels.log 2>&1 && \
timeout 400 ncu --metrics $M --clock-control none -k regex:k_copy_panels --csv --log-file gpurun_out/ncu_nvl_panels.csv python scripts/nvlink_probe.py --once panels --nctas 128 > gpurun_out/ncu_panels.log 2>&1; echo "ncu rc=$?"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29741"
timeout 1500 $TR bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2c.json 2> gpurun_out/bench_n2c.err; echo "bench rc=$?"
tail -4 gpurun_out/bench_n2c.err
