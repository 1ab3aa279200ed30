# pull engine on 4 GPUs: the GPU suite, N=4 bench (+ reference arm), 13B TP=2
timeout 1800 python -m pytest tests -m gpu -q -rs -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_n4_pull.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu_n4_pull.log | tail -5
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1500 $TR --master-port 29811 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_n4_pull.json 2> gpurun_out/bench_n4_pull.err; echo "bench rc=$?"
timeout 900 $TR --master-port 29812 bench.py --gpus 4 --tp 2 --arch llama2-13b --steps 5 --warmup 3 --no-c3 --no-coop > gpurun_out/bench_n4_pull_13b.json 2> gpurun_out/bench_n4_pull_13b.err; echo "bench 13b rc=$?"
for f in bench_n4_pull bench_n4_pull_13b; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['per_dest_GBps'],1), round(d['e2e']['value'],1), d['bit_exact'], d['roofline']['mover'], round(d['roofline']['frac'],3))
lp=d.get('live_pair') or {}; print(lp.get('avg_latency_ms'))"; done
