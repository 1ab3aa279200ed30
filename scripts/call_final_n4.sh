# 4 GPUs: the whole GPU suite, the default N=4 bench line (+ reference arm), 13B TP=2
nvidia-smi --query-gpu=index,name --format=csv,noheader
timeout 1800 python -m pytest tests -m gpu -q -rs -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_n4f.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_gpu_n4f.log | tail -3
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29760 bench.py --impl reference --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_n4f_ref.json 2> gpurun_out/bench_n4f_ref.err; echo "ref rc=$?"
timeout 1500 $TR --master-port 29761 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_n4f.json 2> gpurun_out/bench_n4f.err; echo "bench rc=$?"
timeout 900 $TR --master-port 29762 bench.py --gpus 4 --tp 2 --arch llama2-13b --steps 5 --warmup 3 --no-c3 --no-coop > gpurun_out/bench_n4f_13b.json 2> gpurun_out/bench_n4f_13b.err; echo "bench 13b rc=$?"
