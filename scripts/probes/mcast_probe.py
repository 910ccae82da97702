"""Which multicast-object properties does this box's driver accept (1 device)?"""
import torch
from cuda.bindings import driver as cu

torch.cuda.init()
torch.zeros(1, device="cuda")
dev = cu.cuDeviceGet(0)[1]
for ht in (0, cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
           cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC):
    prop = cu.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.size = 1 << 21
    prop.handleTypes = int(ht)
    err, gran = cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    print("handleTypes", int(ht), "granularity", err, gran)
    if err == cu.CUresult.CUDA_SUCCESS:
        prop.size = max(prop.size, gran)
    err, h = cu.cuMulticastCreate(prop)
    print("  create", err)
    if err == cu.CUresult.CUDA_SUCCESS:
        print("  add device", cu.cuMulticastAddDevice(h, dev))
for nd in (2, 4, 8):
    prop = cu.CUmulticastObjectProp()
    prop.numDevices = nd
    prop.size = 1 << 21
    prop.handleTypes = int(cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR)
    err, h = cu.cuMulticastCreate(prop)
    print("numDevices", nd, "create", err)
    if err == cu.CUresult.CUDA_SUCCESS:
        print("  add device", cu.cuMulticastAddDevice(h, dev), "again", cu.cuMulticastAddDevice(h, dev))
