"""Probe: does this box give NVLink-SHARP multicast (NVLS) to a one-rank group?

Prints the driver's multicast attribute and what torch's symmetric memory
reports for a 512 KiB buffer (the histogram all-reduce's size)."""
import ctypes, os, sys
import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29561")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
cu = ctypes.CDLL("libcuda.so.1")
v = ctypes.c_int(-1)
# CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
rc = cu.cuDeviceGetAttribute(ctypes.byref(v), 132, 0)
print("cuDeviceGetAttribute(MULTICAST_SUPPORTED) rc", rc, "value", v.value, flush=True)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
import torch.distributed._symmetric_memory as symm_mem
try:
    t = symm_mem.empty(65536, dtype=torch.uint64, device=dev)
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    print("has_multicast_support", h.has_multicast_support(), "multicast_ptr", hex(h.multicast_ptr),
          "buffer_ptrs", [hex(p) for p in h.buffer_ptrs], "backend", symm_mem.get_backend(dev), flush=True)
except Exception as e:  # noqa: BLE001 -- a probe reports whatever fails
    print("symm_mem failed:", type(e).__name__, e, flush=True)
dist.destroy_process_group()
