import torch, ctypes
p = torch.cuda.get_device_properties(0)
print({k: getattr(p, k) for k in dir(p) if not k.startswith('_') and isinstance(getattr(p, k), (int, float, str))})
cudart = ctypes.CDLL("libcudart.so.12") if False else None
from cuda.bindings import runtime as rt
for attr in ["cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrL2CacheSize", "cudaDevAttrMaxSharedMemoryPerBlockOptin", "cudaDevAttrMaxSharedMemoryPerMultiprocessor", "cudaDevAttrMaxAccessPolicyWindowSize"]:
    try:
        err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, attr), 0)
        print(attr, v)
    except Exception as e:
        print(attr, "err", e)
