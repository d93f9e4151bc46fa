"""Probe (diagnostics): can this GPU create an NVLS multicast object, with which handle types?"""
import ctypes

cuda = ctypes.CDLL("libcuda.so.1")
cuda.cuInit(0)
dev = ctypes.c_int(0)
cuda.cuDeviceGet(ctypes.byref(dev), 0)
ctx = ctypes.c_void_p()
cuda.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev)
cuda.cuCtxSetCurrent(ctx)
for name, attr in [("MULTICAST_SUPPORTED", 132), ("HANDLE_TYPE_FABRIC_SUPPORTED", 128),
                   ("HANDLE_TYPE_POSIX_FD_SUPPORTED", 101)]:
    v = ctypes.c_int(-1)
    print(name, cuda.cuDeviceGetAttribute(ctypes.byref(v), attr, dev), v.value)


class Prop(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong),
                ("flags", ctypes.c_ulonglong)]


for ht, hname, nd in [(0x8, "FABRIC", 1), (0x1, "POSIX_FD", 1), (0x0, "NONE", 1), (0x8, "FABRIC", 2),
                      (0x1, "POSIX_FD", 2), (0x8, "FABRIC", 8)]:
    p = Prop(nd, 2 << 20, ht, 0)
    hname = f"{hname} x{nd}"
    g = ctypes.c_size_t(0)
    r1 = cuda.cuMulticastGetGranularity(ctypes.byref(g), ctypes.byref(p), 1)
    p.size = max(g.value, 2 << 20)
    h = ctypes.c_ulonglong(0)
    r2 = cuda.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
    r3 = -1
    if r2 == 0:
        buf = ctypes.create_string_buffer(64)
        r3 = cuda.cuMemExportToShareableHandle(buf, h, ht, 0) if ht else -2
        r4 = cuda.cuMulticastAddDevice(h, dev)
        print(hname, "granularity", r1, g.value, "create", r2, "export", r3, "add", r4)
    else:
        print(hname, "granularity", r1, g.value, "create", r2)
