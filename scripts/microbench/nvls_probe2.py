"""Probe cuMulticastCreate argument combinations on this box (NVLS availability)."""
import torch
from cuda.bindings import driver as cu
torch.cuda.init(); torch.zeros(1, device="cuda")
err, d = cu.cuDeviceGet(0)
for a in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
          "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED", "CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED"):
    print(a, cu.cuDeviceGetAttribute(getattr(cu.CUdevice_attribute, a), d))
T = cu.CUmemAllocationHandleType
for ht in (T.CU_MEM_HANDLE_TYPE_NONE, T.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, T.CU_MEM_HANDLE_TYPE_FABRIC):
    for nd in (1, 2, 8):
        p = cu.CUmulticastObjectProp()
        p.numDevices = nd
        p.handleTypes = ht
        p.size = 2 << 20
        r1 = cu.cuMulticastGetGranularity(p, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        r2 = cu.cuMulticastGetGranularity(p, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        res = []
        for size in (2 << 20, 512 << 20):
            p.size = size
            e, h = cu.cuMulticastCreate(p)
            res.append((size >> 20, str(e).split(".")[-1]))
            if e == cu.CUresult.CUDA_SUCCESS:
                ea = cu.cuMulticastAddDevice(h, d)
                res.append(("add", str(ea[0] if isinstance(ea, tuple) else ea).split(".")[-1]))
                cu.cuMemRelease(h)
        print(str(ht).split(".")[-1], nd, "gran min/rec", r1, r2, res, flush=True)
