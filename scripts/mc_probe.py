"""Probe: can this box create / export / bind / map a multicast (NVLS) object
with one device and POSIX-fd handles?  (cuda-python driver API)"""
from cuda.bindings import driver as d


def ck(r, what):
    err = r[0] if isinstance(r, tuple) else r
    print(f"{what}: {err}")
    if err != d.CUresult.CUDA_SUCCESS:
        raise SystemExit(1)
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None


ck(d.cuInit(0), "cuInit")
dev = ck(d.cuDeviceGet(0), "cuDeviceGet")
ctx = ck(d.cuDevicePrimaryCtxRetain(dev), "retain")
ck(d.cuCtxSetCurrent(ctx), "setcurrent")
for ht_name in ("CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC"):
    print("==", ht_name)
    ht = getattr(d.CUmemAllocationHandleType, ht_name)
    prop = d.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.handleTypes = ht
    prop.size = 1 << 21
    gran = d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    print("granularity", gran)
    prop.size = max(gran[1], 1 << 21)
    r = d.cuMulticastCreate(prop)
    print("create", r[0])
    if r[0] != d.CUresult.CUDA_SUCCESS:
        continue
    mc = r[1]
    r = d.cuMemExportToShareableHandle(mc, ht, 0)
    print("export", r[0], type(r[1]) if len(r) > 1 else None)
    print("adddevice", d.cuMulticastAddDevice(mc, dev))
    aprop = d.CUmemAllocationProp()
    aprop.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    aprop.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    aprop.location.id = 0
    aprop.requestedHandleTypes = ht
    r = d.cuMemCreate(prop.size, aprop, 0)
    print("memcreate", r[0])
    mem = r[1]
    print("bind", d.cuMulticastBindMem(mc, 0, mem, 0, prop.size, 0))
    r = d.cuMemAddressReserve(prop.size, 0, 0, 0)
    print("reserve", r[0])
    va = r[1]
    print("map mc", d.cuMemMap(va, prop.size, 0, mc, 0))
    acc = d.CUmemAccessDesc()
    acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    acc.location.id = 0
    acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    print("setaccess", d.cuMemSetAccess(va, prop.size, [acc], 1))
    print("mc va", hex(int(va)))
