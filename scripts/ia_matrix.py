"""Tensor-core vs SIMT dot interaction across shapes (dlrm_gemm_mode 2 =
tensor cores forced, 1 = SIMT), features in one [B, nf, d] buffer, CUDA
events over 20 back-to-back calls: the data behind the default dispatch
rule in csrc/interact_tc.cu (tensor cores from IA_TC_MIN_TILES tiles/SM)."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import _lib

P = _lib.ptr


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for nf, d in ((9, 64), (27, 128), (27, 64), (9, 128), (27, 32), (13, 64)):
    for B in (1024, 2048, 4096, 8192, 16384, 32768):
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
        out = {"nf": nf, "d": d, "B": B}
        for mode, tag in ((2, "tc"), (1, "simt")):
            _lib.call("dlrm_gemm_mode", mode)
            out[f"fwd_{tag}"] = round(timed(fwd), 2)
            out[f"bwd_{tag}"] = round(timed(bwd), 2)
        _lib.call("dlrm_gemm_mode", 0)
        out["fwd_default"] = round(timed(fwd), 2)
        out["bwd_default"] = round(timed(bwd), 2)
        print(json.dumps(out), flush=True)
