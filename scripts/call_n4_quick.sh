TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29771 bench.py --gpus 4 --steps 5 --warmup 3 --no-c3 --no-coop --no-live --no-realclock > gpurun_out/bench_n4g.json 2> gpurun_out/bench_n4g.err; echo "bench rc=$?"
timeout 900 $TR --master-port 29772 bench.py --gpus 4 --tp 2 --arch llama2-13b --steps 3 --warmup 3 --no-c3 --no-coop --no-cpu --no-stripe > gpurun_out/bench_n4g_13b_nostripe.json 2> gpurun_out/bench_n4g_13b_nostripe.err; echo "bench 13b rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/bench_n4g.json", "gpurun_out/bench_n4g_13b_nostripe.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["per_dest_GBps"], d["roofline"]["mover"], d["e2e"]["value"], d["e2e"].get("last_layer_ms_by_gpu"))
PY
