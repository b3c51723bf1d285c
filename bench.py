"""Benchmark: DLRM training samples/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
                    [--impl ours|reference]

* workload (default ``c3``): the paper's Big Basin shape — 8 tables x 1M rows,
  d=64, 512 dense features, multi-hot pooling U[1,100], bottom 512-512-64,
  top 1024-1024-1024-1, 2048 samples per GPU (weak scaling).  It is the
  configuration BASELINE.json quotes at 1/2/4/8 GPUs and the only one with a
  published training-throughput number (paper: ~33.0k samples/s, V100,
  Caffe2).  ``--config c2`` runs the Criteo-Kaggle shape.
* ``value``: whole-job samples/s with the batch pool resident in HBM; each
  timed step = the D2D load of the step's batch into the engine's input
  buffers + one replay of the captured training-step graph.  L2 is flushed
  (256 MiB write) between timed steps, outside the timed events.
* ``e2e``: the same step through the public engine API from PINNED HOST
  buffers — H2D of dense rows, offsets, indices and labels, the step, and a
  D2H read of the step result (loss sum, correct count) — every step.
* ``roofline``: the dominant single kernel of the step (the embedding
  backward apply: segmented fold + row update), its per-launch time from a
  replay of the step graph with event-record nodes at the stage boundaries,
  algorithmic bytes per launch, the copy-bandwidth peak of
  MEASURED_PEAKS.json, and ``traffic`` = DRAM bytes per launch from the
  committed ncu capture (profiles/ncu_traffic_<config>.json).
  ``embedding_roofline`` adds the forward and the standalone full backward;
  ``mlp_roofline`` the tcgen05 MLP GEMMs against the bf16 and 3xTF32 peaks.
* ``cpu_baseline``: the reference algorithm (oracle/port.py, float64, the
  reference's own numpy/BLAS path) on this host's cores over a bounded
  sample of the same workload.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KAGGLE = [1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683,
          8351593, 3194, 27, 14992, 5461306, 10, 5652, 2173, 4, 7046547, 18,
          15, 286181, 105, 142572]
TERABYTE_40M = [39884406, 39043, 17289, 7420, 20263, 3, 7120, 1543, 63,
                38532951, 2953546, 403346, 10, 2208, 11938, 155, 4, 976, 14,
                39979771, 25641295, 39664984, 585935, 12972, 108, 36]

CONFIGS = {
    "c1": dict(name="c1: 8x1e4, d=16, bot 13-512-256-64-16, top 512-256-1, "
               "B=128, 1 idx", tables=[10 ** 4] * 8, d=16,
               bot=[13, 512, 256, 64, 16], top=[512, 256, 1], batch=128, k=1,
               fixed=True, published=None),
    "c2": dict(name="Criteo-Kaggle-shaped synthetic: 26 tables (Kaggle "
               "cardinalities), d=16, bot 13-512-256-64-16, top 512-256-1, "
               "B=2048, 1 idx", tables=KAGGLE, d=16,
               bot=[13, 512, 256, 64, 16], top=[512, 256, 1], batch=2048, k=1,
               fixed=True, published=None),
    "c3": dict(name="Big Basin: 8 tables x 1M rows, d=64, 512 dense, pooling "
               "U[1,100], bot 512-512-64, top 1024-1024-1024-1, B=2048/GPU",
               tables=[10 ** 6] * 8, d=64, bot=[512, 512, 64],
               top=[1024, 1024, 1024, 1], batch=2048, k=100, fixed=False,
               published=33000.0),
    "c4": dict(name="Criteo-Terabyte-shaped synthetic: 26 tables (40M cap), "
               "d=128, bot 13-512-256-128, top 1024-1024-512-256-1, B=32768 "
               "global", tables=TERABYTE_40M, d=128, bot=[13, 512, 256, 128],
               top=[1024, 1024, 512, 256, 1], batch=32768, k=1, fixed=True,
               published=None, global_batch=True),
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0,
            "bf16_tflops_sustained": 1400.0}, "fallback"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region

class ClockSampler:
    def __init__(self, gpu_index=0):
        self.samples = []
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 10:
                time.sleep(0.02)   # sampler is live before the timed region
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# the reference CPU arm / baseline (oracle port = the reference algorithm)

def cpu_port_rate(c, batch, steps, warmup, seed=0):
    """samples/s of the float64 reference algorithm on this host."""
    from oracle import port
    from paper_1906_00091_b200.rng import RandomBatchSource
    # all host threads, also under torchrun (which sets OMP_NUM_THREADS=1 per
    # rank; only rank 0 runs the reference arm)
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    limiter = None
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        limiter = threadpool_limits(limits=ncpu)
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        threads = ncpu
    # tables capped at 2^20 rows per table for host memory (per-sample compute
    # does not depend on the row count); the cap is reported in `sample`
    cap = 1 << 20
    tables = [min(m, cap) for m in c["tables"]]
    model = port.init_params(tables, c["d"], c["bot"], c["top"], seed)
    src = RandomBatchSource(tables, c["bot"][0], batch, c["k"], c["fixed"], seed=seed)
    hbs = [src.next_batch() for _ in range(steps + warmup)]
    for hb in hbs[:warmup]:
        port.train_step(model, hb.dense, hb.offsets, hb.indices, hb.labels, 0.1)
    t0 = time.perf_counter()
    for hb in hbs[warmup:]:
        port.train_step(model, hb.dense, hb.offsets, hb.indices, hb.labels, 0.1)
    dt = time.perf_counter() - t0
    if limiter is not None:
        limiter.restore_original_limits()
    sample = (f"oracle/port.py float64 train_step (reference algorithm), batch "
              f"{batch} ({'the full' if batch == c['batch'] else 'part of the'} "
              f"{c['batch']}-sample step), {steps} timed steps after {warmup} warm-up, "
              f"tables capped at {cap} rows")
    return batch * steps / dt, threads, sample, dt / steps


def run_reference(args, c, rank, world):
    if rank != 0:
        return
    # the per-GPU batch of our arm's workload (at N = 1: exactly its config)
    batch = max(16, min(c["batch"] // world if c.get("global_batch") else c["batch"],
                        int(args.cpu_batch) if args.cpu_batch else 1 << 30))
    rate, threads, sample, per = cpu_port_rate(c, batch, args.steps, args.warmup)
    line = {"impl": "reference", "metric": "train samples/s", "value": rate,
            "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (reference random source)",
            "config": {"workload": c["name"],
                       "global_batch": c["batch"] if c.get("global_batch") else c["batch"] * world,
                       "per_step_batch": batch},
            "cpu_baseline": {"value": rate, "unit": "samples/s", "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": rate, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm

# Random-row gather ceiling on B200 (scripts/gather_bw.cu: 831k uniformly
# random rows of a 2 GiB table, fresh indices and a flushed L2 per rep; GB/s
# by row bytes) — the access pattern of the pooled lookup.  See
# profiles/round1/gather_ceiling.txt.
GATHER_CEILING = {64: 1610.0, 128: 3201.0, 256: 4223.0, 512: 4981.0}
# Read-modify-write of ~787k distinct random 256-byte rows of an 8M-row table
# (scripts/gather_rmw.cu, both directions counted; profiles/round1/gather_rmw.txt)
# — the sparse apply's access pattern.
RMW_CEILING = {256: 5008.0}
# Dense kind::tf32 tcgen05 MMA peak of this part, chip-wide (128x256x8 MMAs,
# profiles/round1/mma_rate.txt); MEASURED_PEAKS.json has bf16 only.
MEASURED_TF32 = 1093.0


def ncu_traffic(config, kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed
    ncu --set full capture of this config (profiles/ncu_traffic_<cfg>.json),
    or None."""
    p = os.path.join(ROOT, "profiles", f"ncu_traffic_{config}.json")
    try:
        return json.load(open(p)).get(kernel)
    except Exception:
        return None


def time_embedding_kernels(eng, flush, reps=5):
    """dlrm_emb_fwd and the full sparse backward (prepare + apply, lr = 0 so
    the tables stay unchanged) launched alone on the engine's buffers, CUDA
    events on the launching stream, L2 flushed before each rep."""
    import torch
    from paper_1906_00091_b200 import _lib
    P, call = _lib.ptr, _lib.call
    s = torch.cuda.current_stream()
    h = _lib.stream_handle(s)
    d, B, nf = eng.d, eng.B, eng.nf

    def fwd():
        call("dlrm_emb_fwd", P(eng.W_all), d, eng._descs_p, eng.T, B, P(eng.Z), nf * d,
             P(eng.err_pos), P(eng.err_flag), h)

    def bwd():
        call("dlrm_emb_bwd_prepare", d, eng._descs_p, eng.T, B, eng.total_rows,
             P(eng.emb_ws), eng.emb_ws_bytes, h)
        call("dlrm_emb_bwd_apply_sgd", P(eng.W_all), d, eng._descs_p, eng.T, B, P(eng.gZ),
             nf * d, 0.0, P(eng.err_flag), eng.total_rows, P(eng.emb_ws), eng.emb_ws_bytes, h)

    out = {}
    for name, fn in (("fwd_ms", fwd), ("bwd_ms", bwd)):
        fn()
        torch.cuda.synchronize()
        tot = 0.0
        for r in range(reps):
            flush.fill_(r & 0xff)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        out[name] = tot / reps
    return out


def hybrid_roofline(c, tr, hb, flush):
    """Embedding roofline of one rank of the hybrid step: its owned tables'
    lookup over the global batch and the full sparse backward (prepare +
    apply, lr = 0), launched alone (CUDA events, L2 flushed); algorithmic
    bytes from the rank's own batch."""
    import torch
    from paper_1906_00091_b200 import _lib
    e = tr.engine
    To = len(e.own)
    if To == 0:
        return None
    P, call = _lib.ptr, _lib.call
    s = torch.cuda.current_stream()
    h = _lib.stream_handle(s)
    d, Bg = e.d, e.Bg
    descs = C.cast(e._descs, C.c_void_p)
    upd = _lib.Update(_lib.UPD_SGD, 0.0, 0.0, 0)

    def fwd():
        call("dlrm_emb_fwd", P(e.W_own), d, descs, To, Bg, P(e.send), To * d,
             P(e.err_pos), P(e.err_flag), h)

    def bwd():
        call("dlrm_emb_bwd_prepare", d, descs, To, Bg, e.total_rows, P(e.emb_ws),
             e.emb_ws_bytes, h)
        call("dlrm_emb_bwd_apply", P(e.W_own), d, descs, To, Bg, P(e.grecv), To * d,
             C.byref(upd), P(e.err_flag), e.total_rows, P(e.emb_ws), e.emb_ws_bytes, h)

    ms = {}
    for name, fn in (("fwd", fwd), ("bwd", bwd)):
        fn()
        torch.cuda.synchronize()
        tot = 0.0
        for rep in range(5):
            flush.fill_(rep & 0xff)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        ms[name] = tot / 5
    fwd_b = bwd_b = 0.0
    for o, i in zip(hb[2], hb[3]):
        nnz, u = int(i.size), int(np.unique(i).size)
        fwd_b += nnz * (4 * d + 8) + (Bg + 1) * 8 + Bg * 4 * d
        bwd_b += Bg * 4 * d + nnz * 8 + (Bg + 1) * 8 + 2 * u * 4 * d
    pk, pk_kind = peaks()
    gbs = fwd_b / (ms["fwd"] / 1e3) / 1e9
    return {"kernel": "embedding_fwd (owned tables, global batch)", "bound": "hbm",
            "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": gbs / pk["hbm_gbs"], "traffic": None, "ms_per_launch": ms["fwd"],
            "algorithmic_bytes_per_launch": fwd_b,
            "embedding_bwd_full_standalone": {
                "GB/s": bwd_b / (ms["bwd"] / 1e3) / 1e9, "ms": ms["bwd"], "bytes": bwd_b,
                "frac": bwd_b / (ms["bwd"] / 1e3) / 1e9 / pk["hbm_gbs"]},
            "peak_kind": pk_kind + " copy bandwidth (MEASURED_PEAKS.json)"}


def algorithmic(c, B, hbs, eng):
    """Per-step algorithmic bytes/flops of the stages."""
    d = c["d"]
    fwd = bwd = 0.0
    for hb in hbs[:1]:
        for o, i in zip(hb.offsets, hb.indices):
            nnz = int(i.size)
            u = int(np.unique(i).size)
            fwd += nnz * (4 * d + 8) + (B + 1) * 8 + B * 4 * d
            bwd += B * 4 * d + nnz * 8 + (B + 1) * 8 + 2 * u * 4 * d
    fl = 0.0
    for li, l in enumerate(eng.layers):
        n, k = l.n_out, l.n_in
        fl += 2 * B * k * n * (2 if li == 0 else 3)
    return fwd, bwd, fl


def run_ours(args, c, rank, world, dist):
    import torch
    from paper_1906_00091_b200 import DlrmConfig, init_model, _lib
    from paper_1906_00091_b200.rng import RandomBatchSource
    from paper_1906_00091_b200.trainer import StepEngine

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dev = torch.device("cuda")
    B = c["batch"] // world if c.get("global_batch") else c["batch"]
    cfg = DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=0)
    model = init_model(cfg, table_init="device")
    src = RandomBatchSource(c["tables"], c["bot"][0], B, c["k"], c["fixed"],
                            seed=1 + rank)
    P = args.pool
    hbs = [src.next_batch() for _ in range(P)]
    # index capacity per table = the largest batch of the stream (the captured
    # graph is valid for every batch of the pool; the sort runs over it)
    caps = [max(int(hb.indices[t].size) for hb in hbs) for t in range(cfg.num_tables)]
    eng = StepEngine(model, B, caps, lr=0.1, input_sets=2)

    # The data pipeline packs every batch once into the engine's input-block
    # layout in pinned host memory (hpool); the device-resident pool (dpool)
    # holds the same blocks in HBM.  A step's inputs then move with ONE copy.
    hpool = [eng.pack_host_batch(hb.dense, hb.offsets, hb.indices, hb.labels)
             for hb in hbs]
    dpool = [hp.to(dev) for hp in hpool]
    h2d_bytes = int(eng.block_bytes)
    stream = torch.cuda.current_stream()

    # warm-up: one eager step per input set, then capture one graph per set
    for k in range(2):
        eng.use_set(k)
        eng.stage(dpool[k % P], k)
        eng.run()
    torch.cuda.synchronize()
    use_graph = not args.no_graph
    if use_graph:
        for k in range(2):
            eng.use_set(k)
            eng.capture()
    eng.use_set(0)
    launches = eng.launches_per_step
    for w in range(args.warmup):
        eng.stage(dpool[w % P], 0)
        eng.run()
    torch.cuda.synchronize()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    K = args.steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(torch.cuda.current_device()).__enter__()
    for s in range(K):
        flush.fill_(s & 0xff)
        starts[s].record(stream)
        eng.stage(dpool[s % P], 0)       # D2D copy of the resident batch
        eng.run()
        ends[s].record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends))
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * B * K / (ms / 1e3)
    eng.check_errors()
    if args.quick:  # A/B experiments: the device-timed number only
        if rank == 0:
            print(json.dumps({"metric": "train samples/s", "value": value, "ms_per_step": ms / K,
                              "config": {"workload": c["name"]}, "quick": True}), flush=True)
        return

    # e2e: pinned host batch -> H2D on a copy stream into the input set the
    # previous step is NOT using, step graph on the compute stream, D2H of
    # the step result (loss sum, #correct) every step.
    copy_s = torch.cuda.Stream()
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    for k in range(2):
        free[k].record(stream)
    res_host = torch.zeros((K, 2), dtype=torch.float32).pin_memory()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    e0.record(stream)
    copy_s.wait_event(e0)
    for s in range(K):
        k = s & 1
        copy_s.wait_event(free[k])
        eng.stage(hpool[s % P], k, copy_s)
        ready[k].record(copy_s)
        stream.wait_event(ready[k])
        eng.use_set(k)
        eng.run()
        res_host[s].copy_(eng.stats, non_blocking=True)
        free[k].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    eng.use_set(0)
    if dist is not None:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    clk.__exit__()
    e2e = world * B * K / (e2e_ms / 1e3)
    loss_last = float(res_host[K - 1, 0]) / B

    # per-stage breakdown (a replay of the same step graph with event-record
    # nodes at the stage boundaries, L2 flushed) and the rooflines
    stages = eng.profile_stages(reps=5, flush=flush)
    fwd_b, bwd_b, flops = algorithmic(c, B, hbs, eng)
    emb_alone = time_embedding_kernels(eng, flush)
    pk, pk_kind = peaks()
    hbm = pk["hbm_gbs"]
    emb_fwd_ms = stages.get("embedding_fwd", float("nan"))
    emb_apply_ms = stages.get("embedding_bwd_sgd", float("nan"))
    # embedding backward = index prepare (keys + radix sort; overlapped with
    # the dense step on a side stream) + apply (segmented fold + row update,
    # on the critical path); bytes: SURVEY §8(d) per lookup / per unique row
    cands = {
        "embedding_fwd": (fwd_b / (emb_fwd_ms / 1e3) / 1e9, emb_fwd_ms, fwd_b),
        "embedding_bwd_apply": (bwd_b / (emb_apply_ms / 1e3) / 1e9, emb_apply_ms, bwd_b),
        "embedding_bwd_full_standalone": (bwd_b / (emb_alone["bwd_ms"] / 1e3) / 1e9,
                                          emb_alone["bwd_ms"], bwd_b),
        "embedding_fwd_standalone": (fwd_b / (emb_alone["fwd_ms"] / 1e3) / 1e9,
                                     emb_alone["fwd_ms"], fwd_b),
    }
    # the dominant single kernel of the step is the embedding backward apply
    # (one fold + SGD launch; every GEMM launch is shorter, see profiles/)
    dom = max(("embedding_fwd", "embedding_bwd_apply"), key=lambda k: cands[k][1])
    gbs, kms, kb = cands[dom]
    traffic = None
    for kn in (("emb_fold_kernel",) if dom == "embedding_bwd_apply"
               else ("emb_fwd_stream_kernel", "emb_fwd_kernel")):
        traffic = traffic if traffic is not None else ncu_traffic(args.config, kn)
    roofline = {"kernel": dom, "bound": "hbm", "achieved": gbs, "peak": hbm,
                "unit": "GB/s", "frac": gbs / hbm, "traffic": traffic,
                "peak_kind": pk_kind + " copy bandwidth (MEASURED_PEAKS.json)",
                "algorithmic_bytes_per_launch": kb, "ms_per_launch": kms,
                "random_row_gather_ceiling_gbs": GATHER_CEILING.get(4 * c["d"])}
    if dom == "embedding_bwd_apply" and 4 * c["d"] in RMW_CEILING:
        # the apply reads AND writes its rows: its own measured ceiling
        roofline["random_row_rmw_ceiling_gbs"] = RMW_CEILING[4 * c["d"]]
    tf = flops / (stages["mlp_total"] / 1e3) / 1e12
    mlp_roof = {"bound": "tensor", "achieved": tf, "unit": "TFLOP/s",
                "peak": pk["bf16_tflops"], "frac": tf / pk["bf16_tflops"],
                "peak_tf32_measured": MEASURED_TF32,
                "peak_fp32_accurate": MEASURED_TF32 / 3.0,
                "frac_of_fp32_accurate_peak": tf / (MEASURED_TF32 / 3.0),
                "note": "fp32-accurate 3xTF32 = 3 kind::tf32 MMAs per product; peak_tf32 "
                        "measured by scripts/mma_rate.cu (128x256x8, chip-wide); "
                        "algorithmic flops 2*B*n_in*n_out per GEMM (fwd, dgrad, wgrad) over "
                        "the whole MLP stage incl. the loss head",
                "ms": stages["mlp_total"], "gflop_per_step": flops / 1e9}
    emb_roof = {k: {"GB/s": v[0], "ms": v[1], "bytes": v[2], "frac": v[0] / hbm}
                for k, v in cands.items()}

    # e2e through the drop-in API: the reference's host arrays (numpy, as
    # RandomBatchSource / dlrmkit produce them) -> Prefetcher (worker threads
    # pack each batch into a reused pinned block, one H2D copy on a copy
    # stream) -> train_step(model, dense, batches, labels, Sgd) -> the
    # StepResult's loss as a Python float (D2H + host sync) every step.
    e2e_api = e2e_train_step(model, cfg, hbs, B, K, args.warmup, dist, dev)

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            batch = max(16, min(c["batch"], int(args.cpu_batch) if args.cpu_batch else 1 << 30))
            rate, threads, sample, _ = cpu_port_rate(c, batch, 2, 1)
            cpu = {"value": rate, "unit": "samples/s", "cores": threads,
                   "kind": "port", "sample": sample}
        line = {
            "metric": "train samples/s", "value": value, "unit": "samples/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": (value / c["published"]) if c["published"] else None,
            "dtype": "f32", "data": "synthetic (reference random source; "
            "device-seeded tables)",
            "config": {"workload": c["name"], "global_batch": B * world,
                       "per_gpu_batch": B, "parallelism": f"hybrid{world}",
                       "l2": "flushed (256 MiB write) between timed steps",
                       "graph": use_graph},
            "e2e": {"value": world * B * K / (e2e_api["ms"] / 1e3), "unit": "samples/s",
                    "h2d_bytes_per_step": e2e_api["h2d_bytes"], "d2h_bytes_per_step": 12,
                    "ms_per_step": e2e_api["ms"] / K,
                    "path": "train_step(model, dense, batches, labels, Sgd, sync=False) on "
                            "Prefetcher batches packed from the reference's numpy arrays; "
                            "every step's loss read back (D2H + host wait), one step "
                            "behind", "loss_last": e2e_api["loss_last"],
                    "input_wait_ms_per_step": e2e_api["input_wait_ms"]},
            "e2e_engine": {"value": e2e, "unit": "samples/s", "h2d_bytes_per_step": h2d_bytes,
                           "d2h_bytes_per_step": 8, "ms_per_step": e2e_ms / K,
                           "path": "StepEngine: pre-packed pinned blocks, H2D of step s+1 "
                                   "overlapping step s, loss sum + #correct read back"},
            "gpu_launches": int(launches) * K if launches else None,
            "roofline": roofline, "embedding_roofline": emb_roof, "mlp_roofline": mlp_roof,
            "stages_ms": {k: v for k, v in stages.items() if k != "captured"},
            "stages_graph_events": stages.get("captured"), "mlp_gflop_per_step": flops / 1e9,
            "loss_last": loss_last, "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)


def e2e_train_step(model, cfg, hbs, B, K, warmup, dist, dev):
    """K steps of the public API (see run_ours); device-timed with CUDA events
    on the compute stream, max over ranks."""
    import torch
    from paper_1906_00091_b200 import Prefetcher, Sgd, train_step
    T = cfg.num_tables
    caps = [max(int(hb.indices[t].size) for hb in hbs) for t in range(T)]

    def source():
        s = 0
        while True:
            yield hbs[s % len(hbs)]
            s += 1
    # two packing workers x 4 native threads each (16-core GPU hosts: one
    # c3 batch packs in 0.32 ms on 4 threads, scripts/pack_bench.py; two
    # batches in flight keep the input ahead of the 0.4 ms step)
    pf = Prefetcher(source(), B, T, cfg.dense_dim, capacities=caps, depth=4,
                    threads=int(os.environ.get("DLRM_PF_THREADS", min(4, max(1, (os.cpu_count() or 2) // 4)))),
                    workers=int(os.environ.get("DLRM_PF_WORKERS", 2)))
    it = iter(pf)
    opt = Sgd(0.1)
    for _ in range(warmup + 2):   # eager step, graph capture, warm-up
        d, b, l = next(it)
        train_step(model, d, b, l, opt)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    loss = None
    waited = 0.0
    prev = None
    for _ in range(K):
        t0 = time.perf_counter()
        d, b, l = next(it)
        waited += time.perf_counter() - t0
        # issue this step, then read the PREVIOUS step's loss back (D2H +
        # host wait): every step's result is read, one step behind, so the
        # host stages step s+1 while step s runs (train_step(sync=False))
        r = train_step(model, d, b, l, opt, sync=False)
        if prev is not None:
            loss = prev.loss
        prev = r
    loss = prev.loss
    e1.record(stream)
    torch.cuda.synchronize()
    pf.close()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"ms": ms, "h2d_bytes": int(pf.layout.nbytes), "loss_last": loss,
            "input_wait_ms": waited * 1e3 / K}


def rank_batches(c, plan, rank, P, seed):
    """P synthetic batches for one rank: its dense/label shard and, for every
    table it owns, bags over the GLOBAL batch (the owner looks them up)."""
    rng = np.random.default_rng(seed + 1000 * rank)
    lo, hi = plan.shard(rank)
    Bg = plan.batch_size
    own = plan.owned(rank)
    out = []
    for _ in range(P):
        dense = rng.random((hi - lo, c["bot"][0]), dtype=np.float64)
        labels = (rng.random(hi - lo) < 0.5).astype(np.float64)
        offs, idxs = [], []
        for t in own:
            k = c["k"]
            lens = np.full(Bg, k, np.int64) if c["fixed"] else rng.integers(1, k + 1, Bg)
            o = np.zeros(Bg + 1, np.int64)
            np.cumsum(lens, out=o[1:])
            offs.append(o)
            idxs.append(rng.integers(0, c["tables"][t], int(o[-1])))
        out.append((dense, labels, offs, idxs))
    return out


def run_hybrid(args, c, rank, world, dist):
    """N > 1: one process per GPU, tables model-parallel (reference plan),
    MLPs data-parallel, NCCL all-to-all + overlapped allreduce."""
    import torch
    from paper_1906_00091_b200 import DlrmConfig, init_model, make_plan, _lib
    from paper_1906_00091_b200.distributed import HybridTrainer

    dev = torch.device("cuda")
    B = c["batch"] // world if c.get("global_batch") else c["batch"]
    Bg = B * world
    cfg = DlrmConfig(c["tables"], c["d"], c["bot"], c["top"], seed=0)
    model = init_model(cfg, table_init="device")
    pool = (c["k"] if c["fixed"] else (c["k"] + 1) / 2.0)
    plan = make_plan(cfg, Bg, world, policy=args.plan, pooling=[pool] * cfg.num_tables,
                     capacity_bytes=150e9)
    own = plan.owned(rank)
    P = args.pool
    hbs = rank_batches(c, plan, rank, P, seed=1)
    # index capacity per owned table = the largest batch of the pool (the
    # captured graph serves every batch; the sort runs over the capacity)
    caps = [max(int(b[3][j].size) for b in hbs) for j in range(len(own))]
    tr = HybridTrainer(model, plan, rank, caps, lr=0.1)

    # the data pipeline packs each batch once into the rank's input-block
    # layout (pinned host); the device pool holds the same blocks in HBM
    hpool = [tr.pack(*b) for b in hbs]
    dpool = [hp.to(dev) for hp in hpool]
    h2d = int(tr.engine.block_bytes)
    n0 = _lib.launch_count()
    tr.stage(dpool[0])
    tr.step()
    launches = _lib.launch_count() - n0
    captured = tr.capture()       # NCCL collectives inside the step graph
    for w in range(args.warmup):
        tr.stage(dpool[w % P])
        tr.step(sync=False)
    torch.cuda.synchronize()
    tr.check_errors()
    stream = torch.cuda.current_stream()
    K = args.steps
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(torch.cuda.current_device()).__enter__()
    for s in range(K):
        flush.fill_(s & 0xff)
        starts[s].record(stream)
        tr.stage(dpool[s % P])
        tr.step(sync=False)     # no host sync inside the step
        ends[s].record(stream)
    torch.cuda.synchronize()
    tr.check_errors()
    dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends))
    t = torch.tensor([ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = Bg * K / (ms / 1e3)
    # e2e from pinned host buffers: the H2D copy of batch s+1 (copy stream,
    # into the landing buffer step s is not reading) overlaps step s; each
    # step starts with a device copy landing -> input block, and ends with a
    # D2H read of its result
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    copy_s = torch.cuda.Stream()
    land = [torch.empty(h2d, dtype=torch.uint8, device=dev) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    for k in range(2):
        free[k].record(stream)
    dist.barrier()
    torch.cuda.synchronize()
    res_host = torch.zeros((K, 3), dtype=torch.float32).pin_memory()
    e0.record(stream)
    copy_s.wait_event(e0)
    for s in range(K):
        k = s & 1
        copy_s.wait_event(free[k])
        with torch.cuda.stream(copy_s):
            land[k].copy_(hpool[s % P], non_blocking=True)   # one H2D copy per batch
        ready[k].record(copy_s)
        stream.wait_event(ready[k])
        tr.stage(land[k])
        free[k].record(stream)
        tr.step(sync=False)
        res_host[s].copy_(tr.engine.stats, non_blocking=True)   # D2H of the step result
    e1.record(stream)
    torch.cuda.synchronize()
    r = tr.result()
    clk.__exit__()
    roofline = hybrid_roofline(c, tr, hbs[0], flush)
    t = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e = Bg * K / (float(t.item()) / 1e3)
    if rank == 0:
        line = {
            "metric": "train samples/s", "value": value, "unit": "samples/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": (value / c["published"]) if c["published"] else None,
            "dtype": "f32", "data": "synthetic (seeded numpy; device-seeded tables)",
            "config": {"workload": c["name"], "global_batch": Bg, "per_gpu_batch": B,
                       "parallelism": f"hybrid: tables model-parallel {plan.table_assignment} "
                                      f"({args.plan} plan), MLP data-parallel x{world}",
                       "l2": "flushed (256 MiB write) between timed steps",
                       "graph": captured},
            "e2e": {"value": e2e, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 12},
            "gpu_launches": launches * K, "loss_last": r.loss,
            "clocks": clk.summary(), "roofline": roofline, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pool", type=int, default=4)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--hybrid", action="store_true",
                    help="run the multi-process hybrid path even at N=1 (under torchrun)")
    ap.add_argument("--plan", default="size", choices=["size", "traffic"],
                    help="table placement for N > 1: the reference's size-balanced plan or "
                         "the traffic-balanced one")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true",
                    help="experiments: print only the device-timed step rate (no e2e, "
                         "stage profile, rooflines or CPU baseline)")
    ap.add_argument("--cpu-batch", type=int, default=0,
                    help="batch of the CPU reference / baseline sample (0: the workload's)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    c = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    dist = None
    if args.impl == "reference":
        run_reference(args, c, rank, world)
        return
    if world > 1 or args.hybrid:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    if world > 1 or args.hybrid:
        run_hybrid(args, c, rank, world, dist)
    else:
        run_ours(args, c, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
