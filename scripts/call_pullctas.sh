TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
X="--steps 5 --warmup 3 --no-c3 --no-coop --no-live --no-realclock --no-cpu"
p=29940
for c in 48 96 148 48 148; do
  p=$((p+1))
  timeout 600 $TR --master-port $p bench.py --gpus 2 $X --nctas $c > gpurun_out/pc.json 2> gpurun_out/pc.err
  echo -n "nctas $c (pull uses max(nctas,64)) rc=$? "; python -c "
import json; d=json.loads(open('gpurun_out/pc.json').read().strip().splitlines()[-1]); print(round(d['per_dest_GBps'],1), d['bit_exact'])"
done 2>&1 | tee gpurun_out/pullctas.log
