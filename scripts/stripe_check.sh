#!/bin/bash
# striped host-cache load: parity (mgpu_check) and e2e rate with / without striping
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 $R --nproc-per-node 4 --master-port 29971 scripts/mgpu_check.py > gpurun_out/stripe_mgpu.log 2>&1; echo "mgpu rc=$?"
grep '^{' gpurun_out/stripe_mgpu.log | cut -c1-200
X="--no-c3 --no-coop --no-live --no-realclock --no-cpu --steps 3 --warmup 3"
for n in 2 4; do
  timeout 300 $R --nproc-per-node $n --master-port 2997$n bench.py --gpus $n $X > gpurun_out/stripe_n$n.log 2>&1; echo "stripe n$n rc=$?"
  timeout 300 $R --nproc-per-node $n --master-port 2998$n bench.py --gpus $n $X --no-stripe > gpurun_out/nostripe_n$n.log 2>&1; echo "nostripe n$n rc=$?"
done
for f in stripe_n2 nostripe_n2 stripe_n4 nostripe_n4; do
  python -c "
import json,sys
l=[x for x in open('gpurun_out/$f.log') if x.startswith('{')]
d=json.loads(l[-1]); e=d['e2e']; print('$f', 'e2e', round(e['value'],1), 'stripe', e.get('host_stripe'), 'bit_exact', e.get('bit_exact'))
" || tail -20 gpurun_out/$f.log
done
grep "e2e steps" gpurun_out/stripe_n4.log gpurun_out/nostripe_n4.log | head
