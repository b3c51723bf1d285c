"""Per-role phase times of the tcgen05 interaction forward (DLRM_IA_PROF
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
R = torch.empty((B, (width + 3) // 4 * 4), device="cuda")
feats = _lib.make_features([(Z.data_ptr() + 4 * f * d, nf * d) for f in range(nf)])
fp = C.c_void_p(C.addressof(feats))
s = _lib.stream_handle()
buf = (C.c_ulonglong * 32)()
for rep in range(3):
    L.dlrm_ia_prof(buf)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("dlrm_interact_fwd", fp, nf, d, B, P(R), R.stride(0), R.shape[1], s)
    e1.record()
    torch.cuda.synchronize()
L.dlrm_ia_prof(buf)
v = list(buf)
names = ["ld:empty", "ld:issue", "ld:cpwait", "ld:bar", "ld:lo", "ld:z0", "mma:full", "mma:tempty",
         "-", "epi:tfull", "epi:tmem", "epi:bar1", "epi:out", "-", "-"]
tot = {"epi": v[15], "ld": v[16], "mma": v[17]}
print("kernel us", e0.elapsed_time(e1) * 1e3)
for k, n in enumerate(names):
    if n == "-":
        continue
    role = n.split(":")[0]
    print(f"{n:12s} {100.0 * v[k] / max(tot[role], 1):6.1f}%")
