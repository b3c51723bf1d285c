"""Diagnostic: from the same post-step-1 state, run step 2 with tcgen05 and
with SIMT GEMMs and diff every buffer."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1906_00091_b200 import _lib, DlrmConfig, init_model
from paper_1906_00091_b200.trainer import StepEngine
from tests.conftest import load_golden
from tests._util import traj_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c1s"
fx = load_golden(f"traj_{name}.npz")
c, batches = traj_inputs(fx)
model = init_model(DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=c["seed"]))
caps = [max(len(hb.indices[t]) for hb in batches) for t in range(len(c["tables"]))]
eng = StepEngine(model, c["batch"], caps, lr=c["lr"])
_lib.call("dlrm_gemm_mode", 0)
hb = batches[0]
eng.load(hb.dense, hb.offsets, hb.indices, hb.labels); eng.run(); torch.cuda.synchronize()
p0, w0 = eng.params.clone(), eng.W_all.clone()
def bufs():
    d = {"Z": eng.Z, "R": eng.R, "logits": eng.logits, "glogit": eng.glogit, "gR": eng.gR, "gZ": eng.gZ}
    for i, t in enumerate(eng.bact): d[f"bact{i}"] = t
    for i, t in enumerate(eng.tact): d[f"tact{i}"] = t
    for i, t in enumerate(eng.gtop): d[f"gtop{i}"] = t
    for i, t in enumerate(eng.gbot): d[f"gbot{i}"] = t
    for li, l in enumerate(eng.layers): d[f"W{li}"] = l.storage; d[f"b{li}"] = l.bias
    return {k: v.double().cpu().numpy().copy() for k, v in d.items()}
out = {}
for mode in (1, 0, 1, 0):
    eng.params.copy_(p0); eng.W_all.copy_(w0)
    _lib.call("dlrm_gemm_mode", mode)
    hb = batches[1]
    eng.load(hb.dense, hb.offsets, hb.indices, hb.labels); eng.run(); torch.cuda.synchronize()
    r = bufs()
    if mode in out:
        print("mode", mode, "rerun identical:", all(np.array_equal(r[k], out[mode][k]) for k in r))
    out[mode] = r
for k in out[0]:
    a, b = out[0][k], out[1][k]
    d = np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)
    flag = "  <<<" if d > 1e-4 else ""
    print(f"{k:8s} {str(a.shape):14s} diff={d:.2e} max|simt|={np.abs(b).max():.3e}{flag}")

# standalone re-run of the suspicious GEMM on the captured step-2 inputs
_lib.call("dlrm_gemm_mode", 0)
eng.params.copy_(p0); eng.W_all.copy_(w0)
hb = batches[1]
eng.load(hb.dense, hb.offsets, hb.indices, hb.labels); eng.run(); torch.cuda.synchronize()
l = eng.layers[5]
gz, W, mask = eng.gtop[1].clone(), None, eng.tact[0].clone()
eng.params.copy_(p0)
W = l.storage.clone()
np.savez("gpurun_out/step2_inputs.npz", gz=gz.cpu().numpy(), W=W.cpu().numpy(), mask=mask.cpu().numpy())
for mode in (0, 1):
    _lib.call("dlrm_gemm_mode", mode)
    dx = torch.zeros((128, 512), device="cuda")
    _lib.call("dlrm_linear_bwd_data", _lib.ptr(gz), gz.stride(0), _lib.ptr(W), W.stride(0), _lib.ptr(mask),
              mask.stride(0), _lib.ptr(dx), dx.stride(0), 128, l.n_out, l.n_in, _lib.stream_handle())
    ref = (gz[:, :l.n_out].double() @ W[:, :l.n_in].double()) * (mask[:, :l.n_in] > 0).double()
    print("standalone mode", mode, "err", float((dx.double() - ref).abs().max() / ref.abs().max()))

# (a) re-run the layer-5 data gradient on the engine's own buffers
_lib.call("dlrm_gemm_mode", 0)
eng.params.copy_(p0); eng.W_all.copy_(w0)
eng.load(hb.dense, hb.offsets, hb.indices, hb.labels); eng.run(); torch.cuda.synchronize()
eng.params.copy_(p0)
g0_engine = eng.gtop[0].clone()
_lib.call("dlrm_linear_bwd_data", _lib.ptr(eng.gtop[1]), eng.gtop[1].stride(0), _lib.ptr(l.storage),
          l.ldw, _lib.ptr(eng.tact[0]), eng.tact[0].stride(0), _lib.ptr(eng.gtop[0]),
          eng.gtop[0].stride(0), 128, l.n_out, l.n_in, _lib.stream_handle())
torch.cuda.synchronize()
ref = (eng.gtop[1][:, :l.n_out].double() @ l.storage[:, :l.n_in].double()) * (eng.tact[0] > 0).double()
print("engine-buffer rerun err", float((eng.gtop[0].double() - ref).abs().max() / ref.abs().max()),
      "engine step value err", float((g0_engine.double() - ref).abs().max() / ref.abs().max()))
