TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
X="--steps 3 --warmup 3 --no-c3 --no-coop --no-realclock --no-cpu"
p=29870
for eng in ce pull ce pull; do
  p=$((p+1))
  timeout 900 $TR --master-port $p bench.py --gpus 2 $X --live-engine $eng > gpurun_out/lp.json 2> gpurun_out/lp.err
  echo -n "live-engine $eng rc=$? "; python -c "
import json; d=json.loads(open('gpurun_out/lp.json').read().strip().splitlines()[-1]); lp=d['live_pair']; a=lp['avg_latency_ms']; print({k: round(v,1) for k,v in a.items()}, 'weights', round(lp.get('weights_load_ms',0),2))"
done 2>&1 | tee gpurun_out/live_pull.log
