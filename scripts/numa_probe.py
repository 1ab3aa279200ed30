"""H2D copy-engine bandwidth from pinned host memory placed on the GPU's NUMA node
vs the other node (first-touch under a CPU affinity mask)."""
import json
import os

import torch


def cpulist(s):
    out = []
    for part in s.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


p = torch.cuda.get_device_properties(0)
bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
base = f"/sys/bus/pci/devices/{bdf}"
info = {"bdf": bdf}
try:
    info["numa_node"] = open(f"{base}/numa_node").read().strip()
    local = cpulist(open(f"{base}/local_cpulist").read())
except OSError as e:
    info["err"] = str(e)
    local = []
allc = sorted(os.sched_getaffinity(0))
remote = [c for c in allc if c not in set(local)]
info["local_cpus"] = len(local)
info["remote_cpus"] = len(remote)
nbytes = 4 << 30
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
for label, cpus in (("local", local), ("remote", remote), ("any", allc)):
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    h = torch.empty(nbytes, dtype=torch.uint8)
    h.fill_(1)  # first touch under this affinity
    torch.cuda.cudart().cudaHostRegister(h.data_ptr(), nbytes, 0)
    s = torch.cuda.Stream()
    best = 0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            dev.copy_(h, non_blocking=True)
            e1.record()
        e1.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    info[f"h2d_{label}_GBps"] = best
    torch.cuda.cudart().cudaHostUnregister(h.data_ptr())
    del h
os.sched_setaffinity(0, allc)
print(json.dumps(info))
