"""Probe NVSwitch multicast object creation with larger sizes (diagnostics)."""
from cuda.bindings import driver as d
d.cuInit(0)
err, dev = d.cuDeviceGet(0)
err, ctx = d.cuDevicePrimaryCtxRetain(dev)
d.cuCtxSetCurrent(ctx)
for size_mb in (2, 64, 512, 1024, 4096):
    for nd in (1, 2, 8):
        for ht in (0, 1):
            p = d.CUmulticastObjectProp()
            p.numDevices = nd
            p.handleTypes = ht
            p.size = size_mb << 20
            p.flags = 0
            r = d.cuMulticastCreate(p)
            print("size_MB", size_mb, "numDevices", nd, "handleTypes", ht, "->", r[0])
            if r[0] == d.CUresult.CUDA_SUCCESS:
                print("   add:", d.cuMulticastAddDevice(r[1], dev))
                d.cuMemRelease(r[1])
print(d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
import subprocess
print(subprocess.run(["nvidia-smi", "-q", "-d", "FABRIC"], capture_output=True, text=True).stdout[-1500:])
