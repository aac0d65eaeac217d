import ctypes as C
cuda = C.CDLL("libcuda.so.1")
cuda.cuInit(0)
dev = C.c_int()
cuda.cuDeviceGet(C.byref(dev), 0)
v = C.c_int()
# CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
for name, attr in (("multicast", 132), ("handle_type_fabric", 128), ("virtual_mem_mgmt", 102)):
    r = cuda.cuDeviceGetAttribute(C.byref(v), attr, dev)
    print(name, r, v.value)
