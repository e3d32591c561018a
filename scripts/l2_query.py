"""Query the L2 persistence limits of GPU 0 (cudaDeviceGetAttribute)."""
import ctypes, torch
torch.cuda.init()
rt = ctypes.CDLL("libcudart.so")
v = ctypes.c_int()
for name, attr in [("MaxPersistingL2CacheSize", 108), ("MaxAccessPolicyWindowSize", 109), ("L2CacheSize", 38)]:
    rc = rt.cudaDeviceGetAttribute(ctypes.byref(v), attr, 0)
    print(name, rc, v.value)
