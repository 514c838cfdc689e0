"""Does this box support CUDA multicast objects (NVLS, multimem.*)?"""
import torch
from cuda.bindings import driver as drv

torch.cuda.init()
(err,) = drv.cuInit(0)
err, dev = drv.cuDeviceGet(0)
err, mc = drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
print("multicast supported:", err, mc)
err, n = drv.cuDeviceGetCount()
print("visible devices:", n)
if mc:
    prop = drv.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.size = 2 << 20
    prop.handleTypes = drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
    err, gran = drv.cuMulticastGetGranularity(prop, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    print("granularity:", err, gran)
    err, h = drv.cuMulticastCreate(prop)
    print("create (1 device):", err)
