"""Does this box support NVLink multicast objects (NVLS)?  cuDeviceGetAttribute(MULTICAST_SUPPORTED)."""
import ctypes
cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
v = ctypes.c_int(-1)
CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
rc = cu.cuDeviceGetAttribute(ctypes.byref(v), CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
print("multicast_supported", v.value, "rc", rc)
n = ctypes.c_int()
cu.cuDeviceGetCount(ctypes.byref(n))
print("devices", n.value)
