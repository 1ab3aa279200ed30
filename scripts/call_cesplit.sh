TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
X="--steps 5 --warmup 3 --no-c3 --no-coop --no-live --no-realclock --no-cpu"
p=29900
for cfg in "1 --gpus 4" "2 --gpus 4" "2 --gpus 4 --ce2-tiles 128" "1 --gpus 4" "2 --gpus 4"; do
  set -- $cfg; split=$1; shift
  p=$((p+1))
  BZ_CE_SPLIT=$split timeout 600 $TR --master-port $p bench.py $X "$@" > gpurun_out/cs.json 2> gpurun_out/cs.err
  echo -n "split=$split $@ rc=$? "; python -c "
import json; d=json.loads(open('gpurun_out/cs.json').read().strip().splitlines()[-1]); print(round(d['per_dest_GBps'],1), d['bit_exact'])"
done 2>&1 | tee gpurun_out/cesplit.log
