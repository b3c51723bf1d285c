"""Per-role barrier-wait share of the tcgen05 interaction forward
(DLRM_IF_PROF builds: scripts/build_variant.sh ifprof interact_tc
-DDLRM_IF_PROF; run with DLRM_B200_LIB=gpurun_var/ifprof.so).  Cycles per
CTA: each role's first thread, waits and total."""
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
buf = (C.c_ulonglong * 16)()
for _ in range(3):
    _lib.call("dlrm_interact_fwd", fp, nf, d, B, P(R), R.stride(0), R.shape[1], s)
torch.cuda.synchronize()
L.dlrm_if_prof(buf)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_lib.call("dlrm_interact_fwd", fp, nf, d, B, P(R), R.stride(0), R.shape[1], s)
e1.record(); torch.cuda.synchronize()
L.dlrm_if_prof(buf)
n = buf[11] or 1
print(f"fwd {e0.elapsed_time(e1) * 1e3:.1f} us, {n} CTAs")
names = {0: "loader wait empty", 1: "loader total", 2: "splitter wait land", 3: "splitter wait aempty",
         4: "splitter total", 5: "mma wait land", 6: "mma wait afull", 7: "mma wait tempty",
         8: "mma total", 9: "epilogue wait tfull", 10: "epilogue total"}
for k, v in names.items():
    print(f"{v:24s} {buf[k] / n:10.0f} cyc/CTA")
