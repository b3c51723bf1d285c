"""Weight-gradient time per (BN, split-K) plan at one shape (measurement:
each plan in a fresh process via DLRM_WGRAD_PLAN).  SHAPE=M,N,K."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "one":
    sys.path.insert(0, ROOT)
    import torch
    from paper_1906_00091_b200 import _lib
    M, N, K = (int(x) for x in os.environ["SHAPE"].split(","))
    g = torch.Generator(device="cuda").manual_seed(0)
    gZ = torch.randn((M, N), device="cuda", generator=g); X = torch.randn((M, K), device="cuda", generator=g)
    dW = torch.empty((N, K), device="cuda"); db = torch.empty(N, device="cuda")
    wsb = _lib.size("dlrm_linear_bwd_weight_workspace_size", M, N, K)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    s = _lib.stream_handle()
    fn = lambda: _lib.call("dlrm_linear_bwd_weight", _lib.ptr(gZ), N, _lib.ptr(X), K, M, N, K, _lib.ptr(dW), K, _lib.ptr(db), None, 0, None, 0.0, None, _lib.ptr(ws), wsb, s)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    ref = gZ.double().T @ X.double()
    err = float((dW.double() - ref).abs().max() / ref.abs().max())
    print(json.dumps({"us": round(e0.elapsed_time(e1) / 20 * 1e3, 2), "err": f"{err:.1e}"}))
    sys.exit(0)
shape = os.environ.get("SHAPE", "32768,256,512")
plans = [None] + [f"{bn},{sp}" for bn in (128, 64, 32) for sp in (4, 8, 12, 16)]
for p in plans:
    env = dict(os.environ, SHAPE=shape)
    if p: env["DLRM_WGRAD_PLAN"] = p
    r = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    print(shape, p or "default", line[-1] if line else r.stderr[-300:], flush=True)
