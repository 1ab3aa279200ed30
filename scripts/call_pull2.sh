# pull engine on 2 GPUs: probe + ncu of one pulled hop, the GPU suite, the default N=2 bench
timeout 300 python scripts/nvlink_probe.py --once pull --gb 2 --nctas 64 > gpurun_out/pull_once.log 2>&1; echo "pull once rc=$?"; tail -1 gpurun_out/pull_once.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum \
  --clock-control none -k regex:k_push_tiles --csv --log-file gpurun_out/ncu_nvlink_pull_n2.csv \
  python scripts/nvlink_probe.py --once pull --gb 2 --nctas 64 > gpurun_out/ncu_pull.log 2>&1; echo "ncu rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -rs -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_n2_pull.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu_n2_pull.log | tail -5
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 1200 $TR --master-port 29801 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2_pull.json 2> gpurun_out/bench_n2_pull.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_n2_pull.json').read().strip().splitlines()[-1]); print(d['value'], d['per_dest_GBps'], d['e2e']['value'], d['bit_exact'], d['roofline']['mover'], d['roofline']['frac'], d['roofline'].get('traffic_source'))
lp=d.get('live_pair') or {}; print(lp.get('avg_latency_ms'))"
