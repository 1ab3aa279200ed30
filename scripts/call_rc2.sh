timeout 900 python -m pytest tests/test_realclock_gpu.py tests/test_multigpu.py -q -rs -p no:cacheprovider --timeout 600 2>&1 | grep -E "^FAILED|passed|failed" | head -3
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 1500 $TR --master-port 29931 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_rc2.json 2> gpurun_out/bench_rc2.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_rc2.json').read().strip().splitlines()[-1])
rc=d.get('c3_realclock') or {}
print(round(d['per_dest_GBps'],1))
for k,v in rc.items():
    if isinstance(v, dict) and 'p99_ttft_ms' in str(v):
        print(k, {kk: (round(vv,1) if isinstance(vv,(int,float)) else vv) for kk,vv in v.items() if 'ttft' in kk or 'tbt' in kk})
print(json.dumps(rc)[:1500])
PY
