"""Probe: is an NVLS multicast object usable on this box (1 GPU)?  Prints attributes
and the result of creating / binding / mapping a 1-device multicast object."""
from cuda.bindings import driver as d


def chk(r, what):
    err = r[0] if isinstance(r, tuple) else r
    print(what, err)
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None


chk(d.cuInit(0), "init")
dev = chk(d.cuDeviceGet(0), "dev")
ctx = chk(d.cuDevicePrimaryCtxRetain(dev), "ctx")
chk(d.cuCtxSetCurrent(ctx), "setctx")
for a in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
          "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    print(a, d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, a), dev))
prop = d.CUmulticastObjectProp()
prop.numDevices = 1
prop.size = 2 << 20
prop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
gran = chk(d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED), "gran")
print("granularity", gran)
for nd, ht in ((1, 0), (2, 0), (1, d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC), (2, d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR)):
    p2 = d.CUmulticastObjectProp()
    p2.numDevices = nd
    p2.size = gran
    p2.handleTypes = ht
    p2.flags = 0
    print("variant", nd, ht, d.cuMulticastCreate(p2))
mc = chk(d.cuMulticastCreate(prop), "mc create")
chk(d.cuMulticastAddDevice(mc, dev), "add dev")
ap = d.CUmemAllocationProp()
ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
ap.location.id = 0
ap.requestedHandleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
h = chk(d.cuMemCreate(2 << 20, ap, 0), "memcreate")
chk(d.cuMulticastBindMem(mc, 0, h, 0, 2 << 20, 0), "bind")
va = chk(d.cuMemAddressReserve(2 << 20, 2 << 20, 0, 0), "reserve")
chk(d.cuMemMap(va, 2 << 20, 0, mc, 0), "map mc")
acc = d.CUmemAccessDesc()
acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
acc.location.id = 0
acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
chk(d.cuMemSetAccess(va, 2 << 20, [acc], 1), "access")
print("multicast VA", va)
