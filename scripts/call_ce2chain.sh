# all-copy-engine chain (ENGINE_CE2; relay gates ahead on their own stream) vs auto on 4 GPUs
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
X="--steps 5 --warmup 3 --no-c3 --no-coop --no-live --no-realclock --no-cpu"
p=29890
for cfg in "--engine auto" "--engine ce2" "--engine ce2 --ce2-tiles 64" "--engine ce2 --ce2-tiles 32" "--engine ce2 --ce2-tiles 256"; do
  p=$((p+1))
  timeout 600 $TR --master-port $p bench.py --gpus 4 $X $cfg > gpurun_out/ce2c.json 2> gpurun_out/ce2c.err
  echo -n "$cfg rc=$? "; python -c "
import json; d=json.loads(open('gpurun_out/ce2c.json').read().strip().splitlines()[-1]); print(round(d['per_dest_GBps'],1), 'e2e', round(d['e2e']['value'],1), d['bit_exact'], round(d['first_layer_ms'],2))"
done 2>&1 | tee gpurun_out/ce2chain_gated.log
