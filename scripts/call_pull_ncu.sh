timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum \
  --replay-mode application --clock-control none -k regex:k_push_tiles --csv --log-file gpurun_out/ncu_nvlink_pull_n2.csv \
  python scripts/nvlink_probe.py --once pull --gb 2 --nctas 64 > gpurun_out/ncu_pull.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_pull.log
grep -E "nvl|dram|duration" gpurun_out/ncu_nvlink_pull_n2.csv | head -12
