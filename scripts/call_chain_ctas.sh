TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
X="--steps 5 --warmup 3 --no-c3 --no-coop --no-live --no-realclock --no-cpu"
p=29850
for cfg in "--nctas 48" "--nctas 96" "--nctas 148" "--nctas 32" "--engine vec256 --nctas 96" "--tile-kib 512" "--tile-kib 2048"; do
  p=$((p+1))
  timeout 600 $TR --master-port $p bench.py --gpus 4 $X $cfg > gpurun_out/cc.json 2> gpurun_out/cc.err
  echo -n "$cfg rc=$? "; python -c "
import json; d=json.loads(open('gpurun_out/cc.json').read().strip().splitlines()[-1]); print(round(d['per_dest_GBps'],1), d['bit_exact'], round(d['first_layer_ms'],2))"
done 2>&1 | tee gpurun_out/chain_ctas.log
