"""One-off hardware probe for the GPU box: device attributes that decide the
data-plane transport (P2P, VMM POSIX-FD / fabric handles, NVLS multicast)."""
import ctypes, os, subprocess, sys
import torch

cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
n = torch.cuda.device_count()
print("devices", n, torch.cuda.get_device_name(0), flush=True)
attrs = {"vmm": 102, "posix_fd": 103, "fabric": 128, "multicast": 132, "gdr": 116}
for d in range(n):
    dev = ctypes.c_int()
    cu.cuDeviceGet(ctypes.byref(dev), d)
    out = {}
    for k, a in attrs.items():
        v = ctypes.c_int(-1)
        r = cu.cuDeviceGetAttribute(ctypes.byref(v), a, dev)
        out[k] = (v.value, r)
    print("dev", d, out, flush=True)
for a in range(n):
    print("p2p", a, [torch.cuda.can_device_access_peer(a, b) if a != b else None for b in range(n)])
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
print(subprocess.run(["nvidia-smi", "-q", "-d", "CLOCK"], capture_output=True, text=True).stdout[:1500])
print("nproc", os.cpu_count())
print(open("/proc/sys/kernel/yama/ptrace_scope").read() if os.path.exists("/proc/sys/kernel/yama/ptrace_scope") else "no yama")
print(subprocess.run(["bash", "-c", "ls -la /dev/nvidia* | head -30; cat /proc/cpuinfo | grep 'model name' | head -1; free -g; lspci 2>/dev/null | grep -i nvidia | head"], capture_output=True, text=True).stdout)
