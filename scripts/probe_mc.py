"""Probe NVSwitch multicast object creation on this box (diagnostics only)."""
from cuda.bindings import driver as d

def chk(r):
    err = r[0] if isinstance(r, tuple) else r
    return err

print(d.cuInit(0))
err, dev = d.cuDeviceGet(0)
err, ctx = d.cuDevicePrimaryCtxRetain(dev)
print(d.cuCtxSetCurrent(ctx))
for attr in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED", "CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED"]:
    try:
        print(attr, d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, attr), dev))
    except Exception as e:
        print(attr, e)
for nd in (1, 2):
    for ht in (0, 1, 8):
        p = d.CUmulticastObjectProp()
        p.numDevices = nd
        p.handleTypes = ht
        p.size = 2 << 20
        err, g = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        err2, gmin = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        p.size = g if g else (2 << 20)
        r = d.cuMulticastCreate(p)
        print("numDevices", nd, "handleTypes", ht, "gran", err, g, gmin, "create", r[0])
        if r[0] == d.CUresult.CUDA_SUCCESS:
            print(" add", d.cuMulticastAddDevice(r[1], dev))
            d.cuMemRelease(r[1])
