R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for v in "BZ_STRIPE=1"; do
  echo "=== $v"
  env $v BZ_WATCHDOG_S=90 timeout 120 $R --master-port $((29900 + RANDOM % 90)) scripts/stripe_probe.py 2>&1 | grep "^\[r" | grep -v "fill:" | tail -40
done
