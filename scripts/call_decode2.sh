timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_realclock_gpu.py tests/test_multigpu.py -q -rs -p no:cacheprovider --timeout 600 > gpurun_out/pytest_decode2.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error" gpurun_out/pytest_decode2.log | tail -5
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29731"
timeout 1200 $TR bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2b.json 2> gpurun_out/bench_n2b.err; echo "bench rc=$?"
tail -5 gpurun_out/bench_n2b.err
