"""c5: embedding-bag microbenchmark sweep (BASELINE.json configs[4]).

pooling {1,8,32,128} x d {16,64,128,256} x rows {1e5,1e6,1e7,1e8} x
{uniform, Zipf(1.05)} on one B200: forward (dlrm_emb_fwd) and backward+SGD
(dlrm_emb_bwd_sgd: keys + radix sort + segmented fold + row update) timed
with CUDA events (L2 flushed before each rep), reported as ALGORITHMIC
GB/s (SURVEY §8(d) byte formulas) and as a fraction of the measured HBM
copy peak.  Writes one JSON line per point.

    python scripts/emb_sweep.py [--quick] > profiles/round1/c5_sweep.jsonl
"""
import argparse, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1906_00091_b200 import _lib
from paper_1906_00091_b200.rng import zipf_indices

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--rows", type=int, nargs="*")
ap.add_argument("--d", type=int, nargs="*")
ap.add_argument("--pool", type=int, nargs="*")
ap.add_argument("--fwd-only", action="store_true")
ap.add_argument("--nnz", type=int, default=1 << 20, help="lookups per point")
ap.add_argument("--cpu", action="store_true",
                help="instead: the reference algorithm (oracle/port.py, float64 numpy) on the "
                     "host, 10^6-row tables, a 32k-lookup sample per point (SURVEY §8(d))")
a = ap.parse_args()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6553.6
rows_list = [10**5, 10**6, 10**7] if a.quick else [10**5, 10**6, 10**7, 10**8]
d_list = [16, 64, 128, 256]
pool_list = [1, 8, 32, 128]
rows_list = a.rows or rows_list
d_list = a.d or d_list
pool_list = a.pool or pool_list
if a.cpu:
    import time
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import port
    rng = np.random.default_rng(0)
    m = 10 ** 6
    for d in d_list:
        W = rng.standard_normal((m, d))
        for pool in pool_list:
            for dist in ("uniform", "zipf"):
                nnz = 1 << 15
                B = max(1, nnz // pool)
                nnz = B * pool
                idx = (rng.integers(0, m, nnz) if dist == "uniform"
                       else zipf_indices(m, nnz, 1.05, seed=d + pool))
                offs = np.arange(0, nnz + 1, pool, dtype=np.int64)
                g = rng.standard_normal((B, d))
                t0 = time.perf_counter()
                port.lookup(W, offs, idx)
                t1 = time.perf_counter()
                rows, vals = port.lookup_backward(W, offs, idx, g)
                W[rows] -= 0.0 * vals
                t2 = time.perf_counter()
                u = int(np.unique(idx).size)
                bf = nnz * (4 * d + 8) + (B + 1) * 8 + B * 4 * d
                bb = B * 4 * d + nnz * 8 + (B + 1) * 8 + 2 * u * 4 * d
                print(json.dumps(dict(impl="cpu-port (oracle/port.py, float64 numpy)",
                                      threads=os.cpu_count(), rows=m, d=d, pooling=pool,
                                      dist=dist, bags=B, nnz=nnz,
                                      fwd_GBs=round(bf / (t1 - t0) / 1e9, 3),
                                      bwd_sgd_GBs=round(bb / (t2 - t1) / 1e9, 3))), flush=True)
    sys.exit(0)

dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s = _lib.stream_handle()
P = _lib.ptr

def timeit(fn, reps):
    fn(); torch.cuda.synchronize()
    tot = 0.0
    for r in range(reps):
        flush.fill_(r & 0xff)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


for rows in rows_list:
    for d in d_list:
        if rows * d * 4 > 120e9:
            continue
        W = torch.empty(rows * d, device=dev)
        W.uniform_(-0.1, 0.1)
        for pool in pool_list:
            B = max(2048, a.nnz // pool)
            for dist in ("uniform", "zipf"):
                nnz = B * pool
                if dist == "uniform":
                    idx = torch.randint(0, rows, (nnz,), device=dev)
                else:
                    idx = torch.as_tensor(zipf_indices(rows, nnz, 1.05, seed=d + pool), device=dev)
                offs = torch.arange(0, nnz + 1, pool, device=dev, dtype=torch.int64)
                out = torch.empty((B, d), device=dev)
                grad = torch.randn((B, d), device=dev) * 1e-3
                desc = _lib.table_array([_lib.TableDesc(offs.data_ptr(), idx.data_ptr(), None, 0, rows, 0, nnz, 0)])
                ep = torch.empty(1, dtype=torch.int64, device=dev); ef = torch.zeros(1, dtype=torch.int32, device=dev)
                wsb = _lib.size("dlrm_emb_bwd_workspace_size", nnz, rows, d)
                ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
                def fwd():
                    _lib.call("dlrm_emb_fwd", P(W), d, C.cast(desc, C.c_void_p), 1, B, P(out), d, P(ep), P(ef), s)
                def bwd():
                    _lib.call("dlrm_emb_bwd_sgd", P(W), d, C.cast(desc, C.c_void_p), 1, B, P(grad), d, 0.01,
                              P(ef), rows, P(ws), wsb, s)
                _lib.call("dlrm_err_reset", P(ep), 1, P(ef), s)
                tf = timeit(fwd, a.reps)
                tb = float('nan') if a.fwd_only else timeit(bwd, a.reps)
                u = int(torch.unique(idx).numel())
                bf = nnz * (4 * d + 8) + (B + 1) * 8 + B * 4 * d
                bb = B * 4 * d + nnz * 8 + (B + 1) * 8 + 2 * u * 4 * d
                rec = dict(rows=rows, d=d, pooling=pool, dist=dist, bags=B, nnz=nnz, unique=u,
                           fwd_us=round(tf * 1e3, 2), fwd_GBs=round(bf / tf / 1e6, 1),
                           fwd_frac=round(bf / tf / 1e6 / peak, 3),
                           bwd_sgd_us=round(tb * 1e3, 2), bwd_GBs=round(bb / tb / 1e6, 1),
                           bwd_frac=round(bb / tb / 1e6 / peak, 3))
                print(json.dumps(rec), flush=True)
        del W
        torch.cuda.empty_cache()
