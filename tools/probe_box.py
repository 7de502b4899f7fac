"""Probe the GPU box: topology, P2P, multicast, host cores. Writes gpurun_out/probe.txt."""
import ctypes, os, subprocess
out = []
def p(*a):
    s = " ".join(str(x) for x in a); print(s); out.append(s)
p("nproc", os.cpu_count(), "sched_getaffinity", len(os.sched_getaffinity(0)))
for cmd in ["nvidia-smi", "nvidia-smi topo -m", "nvidia-smi -q -d CLOCK | head -40", "nvidia-smi nvlink -s | head -40", "lscpu | head -20", "free -g"]:
    try:
        p("$", cmd); p(subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout)
    except Exception as e:
        p("ERR", e)
import torch
n = torch.cuda.device_count(); p("device_count", n)
for i in range(n):
    pr = torch.cuda.get_device_properties(i)
    p(i, pr.name, pr.multi_processor_count, pr.total_memory // 2**20, "MiB")
for i in range(n):
    for j in range(n):
        if i != j:
            p("p2p", i, j, torch.cuda.can_device_access_peer(i, j))
cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
for i in range(n):
    dev = ctypes.c_int(); cu.cuDeviceGet(ctypes.byref(dev), i)
    for name, attr in [("MULTICAST", 132), ("FABRIC", 128), ("POSIX_FD", 103), ("VMM", 102), ("MEMOPS64", 122), ("WAIT_NOR", 123)]:
        v = ctypes.c_int(-1); r = cu.cuDeviceGetAttribute(ctypes.byref(v), attr, dev)
        p("dev", i, name, v.value, "rc", r)
os.makedirs("gpurun_out", exist_ok=True)
open("gpurun_out/probe.txt", "w").write("\n".join(out))
