import torch
from cuda.bindings import runtime as rt  # noqa
err, dev = rt.cudaGetDevice()
for a in ("cudaDevAttrL2CacheSize", "cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize"):
    print(a, rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), dev))
