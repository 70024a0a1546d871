"""Probe the multicast object API step by step on one device (driver results printed)."""
import torch
from cuda.bindings import driver as drv

torch.cuda.init()
torch.zeros(1, device="cuda")  # primary context current
print(drv.cuInit(0))
err, dev = drv.cuDeviceGet(0)
for ht in (drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE,
           drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
           drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC):
    for nd in (1, 2):
        prop = drv.CUmulticastObjectProp()
        prop.numDevices = nd
        prop.size = 32 << 20
        prop.handleTypes = int(ht)
        e1, gmin = drv.cuMulticastGetGranularity(prop, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        e2, grec = drv.cuMulticastGetGranularity(prop, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        prop.size = max(prop.size, gmin)
        e3, h = drv.cuMulticastCreate(prop)
        print(ht.name, "nd", nd, "gran", e1, gmin, e2, grec, "create", e3)
        if e3 == drv.CUresult.CUDA_SUCCESS:
            e4, = drv.cuMulticastAddDevice(h, dev)
            print("   add_device", e4)
            if nd == 1 and e4 == drv.CUresult.CUDA_SUCCESS:
                mp = drv.CUmemAllocationProp()
                mp.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
                mp.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
                mp.location.id = 0
                e5, mem = drv.cuMemCreate(prop.size, mp, 0)
                e6, = drv.cuMulticastBindMem(h, 0, mem, 0, prop.size, 0)
                print("   memcreate", e5, "bind", e6)
            if int(ht) == int(drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR):
                print("   export", drv.cuMemExportToShareableHandle(h, ht, 0)[0])
            drv.cuMemRelease(h)
