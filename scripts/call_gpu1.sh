# one GPU: the whole GPU suite (the driver's GPUTEST), smoke, and the default N=1 bench line
timeout 1800 python -m pytest tests -m gpu -q -rs -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_n1.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_gpu_n1.log | tail -2
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_n1_ref.json 2> gpurun_out/bench_n1_ref.err; echo "ref rc=$?"
