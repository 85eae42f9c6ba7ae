"""Developer probe: does this GPU support multicast objects (NVLS multimem) for a 1-device group?"""
import ctypes
import torch

torch.cuda.init()
torch.zeros(1, device="cuda")
cu = ctypes.CDLL("libcuda.so.1")
v = ctypes.c_int()
CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
rc = cu.cuDeviceGetAttribute(ctypes.byref(v), CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, 0)
print("multicast supported:", rc, v.value)


class Prop(ctypes.Structure):   # CUmulticastObjectProp
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong),
                ("flags", ctypes.c_ulonglong)]


gran = ctypes.c_size_t()
p = Prop(1, 2 << 20, 0, 0)
rc = cu.cuMulticastGetGranularity(ctypes.byref(gran), ctypes.byref(p), 0)
print("granularity:", rc, gran.value)
for nd in (1, 2):
    for ht in (0, 1, 8):
        h = ctypes.c_ulonglong()
        p = Prop(nd, max(gran.value, 2 << 20), ht, 0)
        rc = cu.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
        extra = ""
        if rc == 0:
            extra = f" addDevice(0) -> {cu.cuMulticastAddDevice(h, 0)}"
        print(f"cuMulticastCreate(numDevices={nd}, handleTypes={ht}): {rc}{extra}")
