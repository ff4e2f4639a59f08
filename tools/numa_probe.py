"""Print the GPU's NVML CPU affinity and the host topology (for e2e variance)."""
import os
import sys

import torch
import pynvml

pynvml.nvmlInit()
props = torch.cuda.get_device_properties(0)
uuid = "GPU-" + str(props.uuid)
h = pynvml.nvmlDeviceGetHandleByUUID(uuid)
n = (os.cpu_count() + 63) // 64
mask = pynvml.nvmlDeviceGetCpuAffinity(h, n)
cpus = [w * 64 + b for w, word in enumerate(mask) for b in range(64) if (word >> b) & 1]
print("cpu_count", os.cpu_count(), "gpu-local cpus", len(cpus), cpus[:8], "...", cpus[-4:])
print("current affinity", len(os.sched_getaffinity(0)))
try:
    print("numa nodes", sorted(os.listdir("/sys/devices/system/node")))
except Exception as e:
    print("numa", e)
