# pytest -m gpu on the box (all visible GPUs), then ncu NVLink counters of one
# multicast launch with application replay (kernel replay cannot save multicast memory)
nvidia-smi --query-gpu=index,name --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q -rs -s -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
M=gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
if [ "$(nvidia-smi -L | wc -l)" -ge 2 ]; then
timeout 200 python scripts/nvlink_probe.py --once mc --gb 2 > gpurun_out/plain_mc.log 2>&1 && \
timeout 600 ncu --replay-mode application --metrics $M --clock-control none -k regex:k_multicast --csv --log-file gpurun_out/ncu_nvl_mc.csv python scripts/nvlink_probe.py --once mc --gb 2 > gpurun_out/ncu_mc.log 2>&1; echo "ncu mc rc=$?"
fi
