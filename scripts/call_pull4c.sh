TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
X="--steps 5 --warmup 3 --no-c3 --no-coop --no-live --no-realclock --no-cpu"
p=29830
for cfg in "--engine auto" "--engine vector" "--engine auto --nctas 96" "--engine auto --no-group"; do
  p=$((p+1))
  timeout 600 $TR --master-port $p bench.py --gpus 4 $X $cfg > gpurun_out/p4.json 2> gpurun_out/p4.err
  echo -n "$cfg rc=$? "; python -c "
import json; d=json.loads(open('gpurun_out/p4.json').read().strip().splitlines()[-1]); print(round(d['per_dest_GBps'],1), 'e2e', round(d['e2e']['value'],1), d['bit_exact'], d['config']['workload'][-60:])"
done 2>&1 | tee gpurun_out/pull4c.log
timeout 1200 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider --timeout 600 2>&1 | tail -2
