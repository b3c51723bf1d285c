"""Shared test helpers (no reference import: runs on the GPU box too)."""

import hashlib
import json

import numpy as np

from paper_1906_00091_b200.rng import RandomBatchSource


def digest(arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def batch_arrays(hb):
    return [hb.dense, *hb.offsets, *hb.indices, hb.labels]


def port_arrays(m):
    out = []
    for w, b, _ in m["bottom"] + m["top"]:
        out += [w, b]
    return out + list(m["tables"])


def traj_inputs(fx):
    """Config dict and the host batches of a trajectory fixture."""
    c = json.loads(str(fx["config"]))
    src = RandomBatchSource(c["tables"], c["bot"][0], c["batch"], c["k"],
                            c["fixed"], seed=c["seed"], key=0)
    return c, [src.next_batch() for _ in range(c["steps"])]


def rel_err(got, ref, floor=1e-3):
    """max |got - ref| / (|ref| + floor * max|ref|)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    scale = np.abs(ref) + floor * max(np.abs(ref).max(), 1e-30)
    return float((np.abs(got - ref) / scale).max())


def maxnorm_err(got, ref):
    """max |got - ref| / max |ref| (normwise, per tensor)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


KSEG = 256  # csrc/emb.cu kSeg: runs up to this many slots fold strictly


def assert_fold_match(got, exp, absum, counts, rtol=1e-5, ulps=0):
    """Sparse-gradient rows (or the rows they updated): bit-identical to the
    strict ascending fold where the row's run is <= KSEG slots; where it is
    longer (a hot row reduced as a fixed tree of KSEG-slot strict folds),
    |got - exp| <= rtol * sum|contribution| elementwise.
    ``counts[i]`` is the run length of row i; ``absum[i]`` the fold of the
    absolute contributions; ``ulps`` widens the bound by that many ulps of
    ``exp`` (for weights after the SGD rounding)."""
    got = np.asarray(got, np.float32)
    exp = np.asarray(exp, np.float32)
    counts = np.asarray(counts)
    assert got.shape == exp.shape
    short = counts <= KSEG
    assert np.array_equal(got[short].view(np.uint32), exp[short].view(np.uint32))
    if (~short).any():
        d = np.abs(got[~short].astype(np.float64) - exp[~short])
        tol = (rtol * np.asarray(absum, np.float64)[~short]
               + ulps * np.spacing(np.abs(exp[~short])) + 1e-30)
        assert (d <= tol).all(), float((d / tol).max())
    return int((~short).sum())
