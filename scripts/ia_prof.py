"""Barrier-wait share per role of the tcgen05 interaction backward
(DLRM_IA_PROF builds: python scripts/build_variant.py prof -DDLRM_IA_PROF;
run with DLRM_B200_LIB=gpurun_var/prof/libdlrmb200.so): cycles each role's
first thread spent in each wait, in % of that role's kernel time."""
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
buf = (C.c_ulonglong * 24)()
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
print(f"nf={nf} d={d} B={B}: kernel {e0.elapsed_time(e1) * 1e3:.1f} us")
roles = {"loader": (16, {0: "zempty"}), "splitter": (17, {1: "zfull", 2: "opempty", 9: "gzempty"}),
         "builder": (18, {3: "opempty", 10: "gzempty"}),
         "mma": (19, {4: "afull", 5: "bfull", 6: "dempty"}),
         "epilogue": (20, {7: "dfull", 11: "gzfull"})}
for role, (tot, waits) in roles.items():
    t = v[tot] or 1
    ws = ", ".join(f"{n} {100.0 * v[k] / t:5.1f}%" for k, n in waits.items())
    print(f"  {role:9s} waits: {ws}   busy {100.0 - 100.0 * sum(v[k] for k in waits) / t:5.1f}%")
