# 8 ranks on a 4-GPU box (BZ_OVERSUBSCRIBE=4, gloo): functional check of the N=8 bench path
nvidia-smi --query-gpu=index,name,memory.used --format=csv,noheader
export BZ_OVERSUBSCRIBE=4
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29781 bench.py --impl reference --gpus 8 --steps 2 --warmup 1 > gpurun_out/bench_over8_ref.json 2> gpurun_out/bench_over8_ref.err; echo "ref rc=$?"
timeout 900 $TR --master-port 29782 bench.py --gpus 8 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_over8.json 2> gpurun_out/bench_over8.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_over8.json; echo; tail -20 gpurun_out/bench_over8.err
