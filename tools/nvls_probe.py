"""Probe (development tool): does this box support NVLink SHARP multicast (NVLS), and
does NCCL use it?  Prints CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED per GPU (libcuda via
ctypes) and, under torchrun, runs one NCCL fp16 all-reduce with NCCL_DEBUG=INFO (grep
the log for NVLS)."""
import ctypes
import os

import torch
import torch.distributed as dist

cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
rank = int(os.environ.get("RANK", 0))
if rank == 0:
    for d in range(torch.cuda.device_count()):
        v = ctypes.c_int(-1)
        dev = ctypes.c_int(0)
        cu.cuDeviceGet(ctypes.byref(dev), d)
        cu.cuDeviceGetAttribute(ctypes.byref(v), CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
        print(f"gpu {d}: multicast_supported={v.value}", flush=True)
if "WORLD_SIZE" in os.environ:
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    x = torch.ones(1 << 24, dtype=torch.float16, device="cuda")
    for _ in range(3):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    dist.destroy_process_group()
