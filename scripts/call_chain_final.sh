TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
X="--steps 5 --warmup 3 --no-c3 --no-coop --no-live --no-realclock --no-cpu"
p=29910
for cfg in "--engine auto" "--engine auto --ce2-tiles 512" "--engine auto --fanout nvls" "--engine auto --no-group"; do
  p=$((p+1))
  timeout 600 $TR --master-port $p bench.py --gpus 4 $X $cfg > gpurun_out/cf.json 2> gpurun_out/cf.err
  echo -n "$cfg rc=$? "; python -c "
import json; d=json.loads(open('gpurun_out/cf.json').read().strip().splitlines()[-1]); print(round(d['per_dest_GBps'],1), d['bit_exact'], round(d['first_layer_ms'],2), d['config']['fanout'], d['roofline']['mover'][:40])"
done 2>&1 | tee gpurun_out/chain_final.log
