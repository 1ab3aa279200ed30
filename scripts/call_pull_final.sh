# pull rule (source -> leaf hops only): GPU suite on 2 GPUs, N=2 bench, N=2 13B? (no: 4 GPUs for TP groups)
timeout 1800 python -m pytest tests -m gpu -q -rs -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_n2_pullf.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu_n2_pullf.log | tail -5
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 1200 $TR --master-port 29841 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2_pullf.json 2> gpurun_out/bench_n2_pullf.err; echo "bench rc=$?"
timeout 600 $TR --master-port 29842 bench.py --impl reference --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2_pullf_ref.json 2> gpurun_out/bench_n2_pullf_ref.err; echo "ref rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_n2_pullf.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['per_dest_GBps'],1), round(d['e2e']['value'],1), d['bit_exact'], d['roofline']['mover'], round(d['roofline']['frac'],3), d['roofline'].get('traffic'), d['clocks'])
lp=d.get('live_pair') or {}; print(lp.get('avg_latency_ms'))"
