timeout 1500 python -m pytest tests -m gpu -q -rs -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_n2b.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_gpu_n2b.log | tail -3
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29751"
timeout 1500 $TR bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2d.json 2> gpurun_out/bench_n2d.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_n2d.json').read().strip().splitlines()[-1])
print(d['value'], d['per_dest_GBps'], d['roofline']['mover'], d['roofline']['frac'], d['e2e']['value'], d['live_pair']['avg_latency_ms'])"
