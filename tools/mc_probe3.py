"""Probe: cuMulticastCreate at the recommended granularity, and the device's multicast-related attributes."""
import torch
from cuda.bindings import driver as drv

torch.zeros(1, device="cuda")
drv.cuInit(0)
err, dev = drv.cuDeviceGet(0)
for name in dir(drv.CUdevice_attribute):
    if any(k in name for k in ("MULTICAST", "FABRIC", "IPC", "VIRTUAL_MEMORY", "GPU_DIRECT")):
        print(name, drv.cuDeviceGetAttribute(getattr(drv.CUdevice_attribute, name), dev)[1])
for size in (2 << 20, 512 << 20, 1 << 30):
    prop = drv.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.size = size
    prop.handleTypes = int(drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR)
    prop.flags = 0
    e3, h = drv.cuMulticastCreate(prop)
    print("size", size, "create", e3, drv.cuGetErrorString(e3)[1] if e3 else "")
print("driver", drv.cuDriverGetVersion())
