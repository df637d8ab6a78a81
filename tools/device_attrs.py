"""Print the L2 persistence limits of device 0 (diagnostics)."""
import torch, ctypes
cu = ctypes.CDLL("libcudart.so") if False else None
from cuda import cudart
for attr in ["cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize", "cudaDevAttrL2CacheSize"]:
    err, v = cudart.cudaDeviceGetAttribute(getattr(cudart.cudaDeviceAttr, attr), 0)
    print(attr, v)
