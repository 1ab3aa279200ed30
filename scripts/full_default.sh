#!/bin/bash
# the driver's default invocations (N=1 and N=NG), timed end to end
NG=${NG:-4}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
s=$(date +%s); timeout 600 python bench.py > gpurun_out/def_n1.log 2>&1; echo "n1 rc=$? $(( $(date +%s)-s ))s"
s=$(date +%s); timeout 300 python bench.py --impl reference > gpurun_out/def_ref_n1.log 2>&1; echo "ref n1 rc=$? $(( $(date +%s)-s ))s"
s=$(date +%s); timeout 900 $R --master-port 29961 bench.py --gpus $NG > gpurun_out/def_n$NG.log 2>&1; echo "n$NG rc=$? $(( $(date +%s)-s ))s"
s=$(date +%s); timeout 300 $R --master-port 29962 bench.py --gpus $NG --impl reference > gpurun_out/def_ref_n$NG.log 2>&1; echo "ref n$NG rc=$? $(( $(date +%s)-s ))s"
timeout 600 python -m pytest tests -q -m gpu > gpurun_out/def_pytest.log 2>&1; echo "pytest gpu rc=$? $(tail -1 gpurun_out/def_pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/def_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/def_smoke.log)"
