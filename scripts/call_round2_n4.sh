# 4-GPU box: GPU tests (multi-GPU cases at 4), NVLS probe with 4 members, bench N=4 (default,
# with interference + executed C3), 13B TP=2 (C4 shape: 1 -> 2 instances), and the
# host -> group -> group realisation (--no-stripe e2e: C5 shape at TP=2)
nvidia-smi --query-gpu=index,name --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -rs -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_n4.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_gpu_n4.log | tail -2
timeout 300 python scripts/nvlink_probe.py --ctas 48,96 --unrolls 8 > gpurun_out/nvl_probe_n4.jsonl 2>&1; echo "probe rc=$?"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1200 $TR --master-port 29721 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo "bench rc=$?"
timeout 900 $TR --master-port 29722 bench.py --gpus 4 --tp 2 --arch llama2-13b --steps 5 --warmup 3 --no-c3 --no-coop > gpurun_out/bench_n4_13b_tp2.json 2> gpurun_out/bench_n4_13b_tp2.err; echo "bench tp2 rc=$?"
timeout 900 $TR --master-port 29723 bench.py --gpus 4 --tp 2 --arch llama2-13b --steps 3 --warmup 3 --no-c3 --no-coop --no-cpu --no-stripe > gpurun_out/bench_n4_13b_tp2_nostripe.json 2> gpurun_out/bench_n4_13b_tp2_nostripe.err; echo "bench tp2 nostripe rc=$?"
