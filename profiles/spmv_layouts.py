import ctypes as C, sys, os
sys.path.insert(0,'/root/repo')
import torch
from paper_1903_10977_b200 import MgHierarchy, _ffi, build_case, configs
lib=_ffi.gpu(); case=build_case(configs.c4()); vp=C.c_void_p
db=torch.from_numpy(case.b).cuda(); dx=torch.empty_like(db)
for opt5, opt6 in ((0,0),(100000,0),(100000,1)):
    lib.ig_set_option(5,opt5); lib.ig_set_option(6,opt6)
    h=MgHierarchy(case); L=h.levels(); st=torch.cuda.ExternalStream(lib.ig_hier_stream(h.handle))
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    res={}
    for lvl in (L-1, L-2):
        for mode in (0,1,2):
            f=lambda: lib.ig_level_spmv_device(h.handle, lvl, vp(db.data_ptr()), vp(dx.data_ptr()), mode)
            f(); torch.cuda.synchronize(); e0.record(st)
            for _ in range(20): f()
            e1.record(st); torch.cuda.synchronize(); res[(lvl,mode)]=e0.elapsed_time(e1)/20*1e3
    print(opt5,opt6,' '.join(f'L{l}m{m}:{t:.1f}' for (l,m),t in res.items()), flush=True)
    h.close(); torch.cuda.synchronize()
