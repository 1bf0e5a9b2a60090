"""Probe NVLink SHARP multicast on this box: device attributes, then
cuMulticastCreate over a sweep of (numDevices, handleTypes, size)."""
import ctypes as C
cu = C.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = C.c_int(); cu.cuDeviceGet(C.byref(dev), 0)
v = C.c_int()
for name, a in [("MULTICAST_SUPPORTED", 132), ("HANDLE_TYPE_FABRIC_SUPPORTED", 128),
                ("HANDLE_TYPE_POSIX_FD_SUPPORTED", 103)]:
    cu.cuDeviceGetAttribute(C.byref(v), a, dev); print(name, v.value, flush=True)
class Prop(C.Structure):
    _fields_ = [("numDevices", C.c_uint), ("size", C.c_size_t), ("handleTypes", C.c_ulonglong), ("flags", C.c_ulonglong)]
ctx = C.c_void_p(); cu.cuDevicePrimaryCtxRetain(C.byref(ctx), dev); cu.cuCtxSetCurrent(ctx)
es = C.c_char_p()
cu.cuMulticastCreate.argtypes = [C.POINTER(C.c_ulonglong), C.POINTER(Prop)]
for nd in (1, 2, 8):
    for ht in (0, 1, 8):
        for sz in (2 << 20, 512 << 20):
            p = Prop(nd, sz, ht, 0)
            h = C.c_ulonglong(); r = cu.cuMulticastCreate(C.byref(h), C.byref(p))
            cu.cuGetErrorString(r, C.byref(es))
            print(nd, ht, sz, r, es.value, flush=True)
            if r == 0:
                print("  addDevice", cu.cuMulticastAddDevice(h, dev))
