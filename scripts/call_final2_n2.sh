# 2-GPU box after the swapped decode GEMM: GPU suite (cross-GPU hand-offs, live pair, real clock) and the N=2 bench line
nvidia-smi --query-gpu=index,name --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > gpurun_out/pytest_gpu_n2s.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_gpu_n2s.log | tail -2
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29731"
timeout 900 $TR bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2s.json 2> gpurun_out/bench_n2s.err; echo "bench rc=$?"
