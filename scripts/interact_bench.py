"""Time dlrm_interact_fwd / dlrm_interact_bwd alone at the c2 / c3 / c4
shapes (CUDA events, 20 reps after warm-up, features in one [B, nf, d]
buffer like the training engine's Z).  Prints algorithmic GB/s."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import _lib

SHAPES = {"c2": (27, 16, 2048), "c3": (9, 64, 2048), "c4": (27, 128, 32768), "c1": (9, 16, 128)}
P = _lib.ptr
for name, (nf, d, B) in SHAPES.items():
    Z = torch.randn((B, nf * d), device="cuda")
    width = d + nf * (nf - 1) // 2
    R = torch.empty((B, (width + 3) // 4 * 4), device="cuda")
    gR = torch.randn_like(R)
    gZ = torch.empty_like(Z)
    feats = _lib.make_features([(Z.data_ptr() + 4 * f * d, nf * d) for f in range(nf)])
    fp = C.c_void_p(C.addressof(feats))
    gfeat = (C.c_void_p * nf)(*[gZ.data_ptr() + 4 * f * d for f in range(nf)])
    gstr = (C.c_int64 * nf)(*([nf * d] * nf))
    s = _lib.stream_handle()
    fwd = lambda: _lib.call("dlrm_interact_fwd", fp, nf, d, B, P(R), R.stride(0), R.shape[1], s)
    bwd = lambda: _lib.call("dlrm_interact_bwd", fp, nf, d, B, P(gR), gR.stride(0),
                            C.cast(gfeat, C.c_void_p), C.cast(gstr, C.c_void_p), 1, s)
    out = {"cfg": name, "nf": nf, "d": d, "B": B}
    for k, fn, nbytes in (("fwd", fwd, 4 * B * (nf * d + width)),
                          ("bwd", bwd, 4 * B * (width + 2 * nf * d))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        out[k + "_us"] = round(us, 2)
        out[k + "_GBs"] = round(nbytes / us / 1e3, 1)
    print(json.dumps(out), flush=True)
