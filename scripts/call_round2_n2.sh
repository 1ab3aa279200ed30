# 2-GPU box: GPU tests, NVLink probe (incl. copy-engine hop sweep), bench N=2 (default) and
# the live pair with the copy-engine push
nvidia-smi --query-gpu=index,name --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -rs -s -p no:cacheprovider > gpurun_out/pytest_gpu_n2.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_gpu_n2.log | tail -2
timeout 300 python scripts/nvlink_probe.py --ctas 24,48 --unrolls 8 > gpurun_out/nvl_probe2_n2.jsonl 2>&1; echo "probe rc=$?"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29711"
timeout 900 $TR bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench rc=$?"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29712"
timeout 900 $TR bench.py --gpus 2 --steps 3 --warmup 3 --no-c3 --no-coop --no-realclock --no-cpu --no-e2e --live-engine ce > gpurun_out/bench_n2_livece.json 2> gpurun_out/bench_n2_livece.err; echo "bench ce rc=$?"
