#!/bin/bash
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/full_n1.log 2>&1; echo "n1 rc=$?"; tail -1 gpurun_out/full_n1.log | cut -c1-600
timeout 300 python bench.py --impl reference > gpurun_out/full_ref_n1.log 2>&1; echo "ref n1 rc=$?"; tail -1 gpurun_out/full_ref_n1.log | cut -c1-400
timeout 500 $R --master-port 29701 bench.py --gpus 4 > gpurun_out/full_n4.log 2>&1; echo "n4 rc=$?"; tail -1 gpurun_out/full_n4.log | cut -c1-600
timeout 300 $R --master-port 29702 bench.py --gpus 4 --impl reference > gpurun_out/full_ref_n4.log 2>&1; echo "ref n4 rc=$?"; tail -1 gpurun_out/full_ref_n4.log | cut -c1-400
timeout 400 $R --master-port 29703 bench.py --gpus 4 --arch llama2-13b --tp 2 --no-c3 > gpurun_out/full_n4_13b_tp2.log 2>&1; echo "13b tp2 rc=$?"; tail -1 gpurun_out/full_n4_13b_tp2.log | cut -c1-600
