timeout 600 python scripts/repeat_train.py c4 3 2>&1 | tail -2
SVMB200_NO_L2PERSIST=1 timeout 600 python scripts/repeat_train.py c4 2 2>&1 | tail -1
python -c "
import torch; p=torch.cuda.get_device_properties(0); print(p)
from cuda.bindings import runtime as rt
print(rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0), rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0), rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrL2CacheSize, 0))" 2>&1 | tail -2
