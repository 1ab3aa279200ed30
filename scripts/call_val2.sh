timeout 1800 python -m pytest tests -m gpu -q -rs -p no:cacheprovider --timeout 600 > gpurun_out/pytest_val2.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/pytest_val2.log | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 1200 $TR --master-port 29861 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_val2.json 2> gpurun_out/bench_val2.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_val2.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['per_dest_GBps'],1), r['frac'], r.get('protocol_bound_GBps'), r.get('frac_of_protocol_bound'), r['traffic_source'][:60], d['gpu_launches'])"
