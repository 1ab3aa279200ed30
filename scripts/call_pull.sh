timeout 900 python scripts/nvlink_probe.py --ctas 48,64,96,148 2>&1 | grep -E '"case": "(ceiling|push|pull)"' | tee gpurun_out/pull_probe2.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['case'], d.get('engine',''), d.get('nctas', d.get('tiles_per_copy','')), round(d['GBps'],1), d.get('ok',''))"
