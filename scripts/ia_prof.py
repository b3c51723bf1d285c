"""Per-role phase times of the tcgen05 interaction backward (DLRM_IA_PROF
builds: python scripts/build_variant.py prof -DDLRM_IA_PROF), in % of the
role's kernel time, summed over CTAs."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_00091_b200 import _lib
nf, d, B = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (27, 128, 32768)))
L = _lib.lib()
P = _lib.ptr
Z = torch.randn((B, nf * d), device="cuda")
width = d + nf * (nf - 1) // 2
gR = torch.randn((B, (width + 3) // 4 * 4), device="cuda")
gZ = torch.empty_like(Z)
feats = _lib.make_features([(Z.data_ptr() + 4 * f * d, nf * d) for f in range(nf)])
fp = C.c_void_p(C.addressof(feats))
gfeat = (C.c_void_p * nf)(*[gZ.data_ptr() + 4 * f * d for f in range(nf)])
gstr = (C.c_int64 * nf)(*([nf * d] * nf))
s = _lib.stream_handle()
buf = (C.c_ulonglong * 32)()
for rep in range(3):
    L.dlrm_ia_prof(buf)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("dlrm_interact_bwd", fp, nf, d, B, P(gR), gR.stride(0), C.cast(gfeat, C.c_void_p),
              C.cast(gstr, C.c_void_p), 1, s)
    e1.record()
    torch.cuda.synchronize()
L.dlrm_ia_prof(buf)
v = list(buf)
print("kernel us", e0.elapsed_time(e1) * 1e3)
names = {0: ["ld:empty", "ld:issue", "ld:land", "ld:bar", "ld:lo", "ld:aempty", "ld:Abuild"],
         1: ["mma:afull", "mma:dempty"], 2: ["epi:prefetch", "epi:dfull", "epi:gzbar", "epi:tmem+st"]}
for role, ns in names.items():
    tot = v[8 * role + 7] or 1
    for k, n in enumerate(ns):
        print(f"{n:14s} {100.0 * v[8 * role + k] / tot:6.1f}%")
