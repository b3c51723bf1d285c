"""One interaction shape, forward and backward, a few reps (for ncu)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import _lib
nf, d, B = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (27, 128, 32768)))
P = _lib.ptr
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
for _ in range(3):
    _lib.call("dlrm_interact_fwd", fp, nf, d, B, P(R), R.stride(0), R.shape[1], s)
    _lib.call("dlrm_interact_bwd", fp, nf, d, B, P(gR), gR.stride(0), C.cast(gfeat, C.c_void_p),
              C.cast(gstr, C.c_void_p), 1, s)
torch.cuda.synchronize()
print("ok")
