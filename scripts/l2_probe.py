#!/usr/bin/env python
"""Print the device's persisting-L2 limits (cudaDevAttrMaxPersistingL2CacheSize, max access-policy
window) through torch's CUDA runtime -- context for SPUMA_OPT_L2_PERSIST A/Bs."""
import json

import torch

torch.cuda.init()
p = torch.cuda.get_device_properties(0)
out = {"name": p.name, "l2_cache_size": getattr(p, "L2_cache_size", None)}
try:
    from cuda.bindings import runtime as cr  # cuda-python
    for name in ("cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize"):
        err, v = cr.cudaDeviceGetAttribute(getattr(cr.cudaDeviceAttr, name), 0)
        out[name] = v
except Exception as e:  # noqa: BLE001
    out["error"] = str(e)[:200]
print(json.dumps(out))
