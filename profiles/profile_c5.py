import ctypes as C, os, sys
sys.path.insert(0, '/root/repo')
import torch
from paper_1903_10977_b200 import MgHierarchy, _ffi, build_case, configs
case = build_case(configs.c5())
h = MgHierarchy(case)
lib = _ffi.gpu(); vp = C.c_void_p
db = torch.from_numpy(case.b).cuda(); dx = torch.empty_like(db)
lib.ig_set_option(_ffi.IG_OPT_USE_GRAPH, 0)
for _ in range(2): lib.ig_vcycle_device(h.handle, vp(db.data_ptr()), vp(dx.data_ptr()))
torch.cuda.synchronize()
print("done")
