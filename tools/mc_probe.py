"""Which cuMulticastCreate configurations does this GPU accept (1-GPU box)?"""
import torch
from cuda.bindings import driver as cu
torch.zeros(1, device="cuda")
err, dev = cu.cuCtxGetDevice()
for attr in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    a = getattr(cu.CUdevice_attribute, attr, None)
    print(attr, cu.cuDeviceGetAttribute(a, dev) if a is not None else "n/a")
H = cu.CUmemAllocationHandleType
for nd in (1, 2):
    for ht in (0, H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, getattr(H, "CU_MEM_HANDLE_TYPE_FABRIC", None)):
        if ht is None:
            continue
        mp = cu.CUmulticastObjectProp()
        mp.numDevices = nd
        mp.handleTypes = ht
        mp.flags = 0
        mp.size = 2 << 20
        r = cu.cuMulticastGetGranularity(mp, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        g = r[1] if r[0] == cu.CUresult.CUDA_SUCCESS else None
        if g:
            mp.size = max(g, 2 << 20)
        r2 = cu.cuMulticastCreate(mp)
        print("numDevices", nd, "handleTypes", ht, "gran", r[0], g, "create", r2[0])
