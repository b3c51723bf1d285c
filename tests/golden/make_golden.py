"""Generate the golden fixtures by running the REFERENCE (dlrmkit) itself.

Run in the build container, where the reference is mounted read-only:

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

For every trajectory config it
  1. builds the model with ``dlrmkit.init_model`` and checks that our host
     initialiser (``oracle.port.init_params``) reproduces it bit for bit;
  2. draws batches with ``dlrmkit``'s CLI random source and checks that our
     ``RandomBatchSource`` reproduces them bit for bit (digest stored);
  3. rounds the initial parameters and dense features to float32 (the GPU's
     starting point) and runs ``dlrmkit.parallel.train_step`` in float64;
  4. runs ``oracle.port.train_step`` on the same inputs and asserts it is
     bit-identical to dlrmkit (the oracle pin);
  5. stores per-step loss / accuracy / probabilities and the final
     parameters.

It also stores embedding-bag fixtures (weighted bags, empty bags, duplicate
rows) computed by ``dlrmkit.lookup_batch`` / ``lookup_backward``, a
checkpoint written by ``dlrmkit.cli.save_checkpoint`` (``ckpt_toy.dlrmkit``)
and the reference's ``_evaluate`` over validation batches (``eval_*.npz``).
The GPU box never runs this script; it only reads the ``.npz`` files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import dlrmkit  # noqa: E402  (the reference, from /root/reference/pkg/src)
from dlrmkit import cli as ref_cli  # noqa: E402
from dlrmkit.parallel import train_step as ref_train_step  # noqa: E402

from oracle import port  # noqa: E402
from paper_1906_00091_b200.rng import RandomBatchSource  # noqa: E402

KAGGLE = [1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683,
          8351593, 3194, 27, 14992, 5461306, 10, 5652, 2173, 4, 7046547, 18,
          15, 286181, 105, 142572]

TRAJ = {
    "toy": dict(tables=[7, 5, 9], d=3, bot=[4, 3], top=[10, 4, 1], seed=44,
                batch=9, k=3, fixed=False, steps=20, lr=0.1),
    "c1s": dict(tables=[600] * 8, d=16, bot=[13, 512, 256, 64, 16],
                top=[512, 256, 1], seed=0, batch=128, k=1, fixed=True,
                steps=4, lr=0.1),
    "c2s": dict(tables=[min(m, 300) for m in KAGGLE], d=16,
                bot=[13, 512, 256, 64, 16], top=[512, 256, 1], seed=2,
                batch=64, k=1, fixed=True, steps=2, lr=0.1),
    "c3s": dict(tables=[800] * 4, d=64, bot=[32, 64, 64], top=[64, 32, 1],
                seed=1, batch=96, k=12, fixed=False, steps=3, lr=0.1),
    # Adagrad: the reference's make_optimizer("adagrad").
    # eps well above fp32 rounding noise: with eps ~ 0 the first Adagrad step
    # is lr*sign(g), so a gradient that is 1e-12 in float64 and 1e-9 of the
    # other sign in float32 moves a weight by 2*lr — no fp32 implementation
    # can match float64 elementwise there.
    "c1a": dict(tables=[600] * 8, d=16, bot=[13, 512, 256, 64, 16],
                top=[512, 256, 1], seed=0, batch=128, k=1, fixed=True,
                steps=4, lr=0.01, opt="adagrad", eps=1e-2),
    "c3a": dict(tables=[800] * 4, d=64, bot=[32, 64, 64], top=[64, 32, 1],
                seed=1, batch=96, k=12, fixed=False, steps=3, lr=0.01,
                opt="adagrad", eps=1e-4),
}


def digest(arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def batch_arrays(hb):
    return [hb.dense, *hb.offsets, *hb.indices, hb.labels]


def ref_model_to_port(model):
    lay = lambda mlp: [(l.weight, l.bias, l.activation) for l in mlp.layers]
    return {"bottom": lay(model.bottom), "top": lay(model.top),
            "tables": [t.weights for t in model.tables]}


def port_arrays(m):
    out = []
    for w, b, _ in m["bottom"] + m["top"]:
        out += [w, b]
    return out + list(m["tables"])


def make_traj(name, c):
    cfg = dlrmkit.DlrmConfig(embedding_sizes=c["tables"], sparse_dim=c["d"],
                             bottom_mlp_dims=c["bot"], top_mlp_dims=c["top"],
                             seed=c["seed"])
    ref_model = dlrmkit.init_model(cfg)
    mine = port.init_params(c["tables"], c["d"], c["bot"], c["top"],
                            c["seed"])
    assert digest(port_arrays(mine)) == digest(
        port_arrays(ref_model_to_port(ref_model))), "init mismatch"

    # reference CLI random source vs ours
    opts = ref_cli.RunOptions(mini_batch_size=c["batch"],
                              num_indices_per_lookup=c["k"],
                              num_indices_per_lookup_fixed=c["fixed"])
    src = ref_cli._RandomSource(cfg, opts, key=0)
    ours = RandomBatchSource(c["tables"], c["bot"][0], c["batch"], c["k"],
                             c["fixed"], seed=c["seed"], key=0)
    batches = []
    for _ in range(c["steps"]):
        dense, sparse, labels = src.next_batch()
        hb = ours.next_batch()
        ref_arrays = [dense, *[s.offsets for s in sparse],
                      *[s.indices for s in sparse], labels]
        assert digest(ref_arrays) == digest(batch_arrays(hb)), "batch mismatch"
        batches.append(hb)
    input_digest = digest([a for hb in batches for a in batch_arrays(hb)])

    # GPU start point: float32-rounded params and dense rows, held in f64
    start = port.round_params_f32(mine)
    for (w, b, _), l in zip(start["bottom"] + start["top"],
                            ref_model.bottom.layers + ref_model.top.layers):
        l.weight[...] = w
        l.bias[...] = b
    for w, t in zip(start["tables"], ref_model.tables):
        t.weights[...] = w

    opt = dlrmkit.make_optimizer(c.get("opt", "sgd"), c["lr"], c.get("eps", 1e-10))
    losses, accs, probs = [], [], []
    for hb in batches:
        dense32 = hb.dense.astype(np.float32).astype(np.float64)
        sparse = [dlrmkit.SparseBatch(o, i) for o, i in
                  zip(hb.offsets, hb.indices)]
        r = ref_train_step(ref_model, dense32, sparse, hb.labels, opt)
        losses.append(r.loss)
        accs.append(r.accuracy)
        probs.append(r.probs)

    # the oracle pin: our float64 port must reproduce dlrmkit bit for bit
    pm = start
    ada = port.adagrad_state(pm) if c.get("opt") == "adagrad" else None
    for s, hb in enumerate(batches):
        dense32 = hb.dense.astype(np.float32).astype(np.float64)
        loss, acc, prob = port.train_step(pm, dense32, hb.offsets,
                                          hb.indices, hb.labels, c["lr"],
                                          adagrad=ada, eps=c.get("eps", 1e-10))
        assert loss == losses[s] and acc == accs[s], (name, s, loss, losses[s])
        assert np.array_equal(prob, probs[s])
    final_ref = port_arrays(ref_model_to_port(ref_model))
    final_port = port_arrays(pm)
    for a, b in zip(final_ref, final_port):
        assert np.array_equal(a, b), name

    small = sum(a.size for a in final_ref) < 20000
    store = {
        "config": np.array(json.dumps(c)),
        "input_digest": np.array(input_digest),
        "init_digest": np.array(digest(port_arrays(mine))),
        "losses": np.array(losses), "accs": np.array(accs),
        "probs": np.stack(probs),
    }
    for i, a in enumerate(final_ref):
        store[f"final_{i}"] = a if small else a.astype(np.float32)
    path = os.path.join(HERE, f"traj_{name}.npz")
    np.savez_compressed(path, **store)
    print(f"{name}: losses {losses[0]:.6f}..{losses[-1]:.6f} -> {path}")


def make_bags():
    """Embedding-bag fixtures through dlrmkit.lookup_batch/lookup_backward."""
    rng = np.random.default_rng(7)
    store = {}
    cases = [(50, 4, 9, 6, True), (300, 16, 40, 12, False),
             (1000, 64, 33, 30, True), (20, 3, 7, 5, True),
             (600, 128, 64, 3, False), (64, 256, 16, 9, True)]
    for n, (m, d, nb, maxlen, weighted) in enumerate(cases):
        W = rng.standard_normal((m, d)).astype(np.float32).astype(np.float64)
        lens = rng.integers(0, maxlen + 1, nb)
        lens[rng.integers(0, nb)] = 0            # at least one empty bag
        idx = rng.integers(0, m, int(lens.sum()))
        if idx.size > 2:
            idx[1] = idx[0]                       # a duplicate row
        w = (rng.standard_normal(idx.size).astype(np.float32)
             .astype(np.float64) if weighted else None)
        sb = dlrmkit.SparseBatch(dlrmkit.offsets_from_lengths(lens), idx, w)
        table = dlrmkit.EmbeddingTable(W.copy(), table_id=n)
        out = dlrmkit.lookup_batch(table, sb)
        g = rng.standard_normal((nb, d)).astype(np.float32).astype(np.float64)
        sg = dlrmkit.lookup_backward(table, sb, g)
        o2 = port.lookup(W, sb.offsets, sb.indices, w, n)
        r2, v2 = port.lookup_backward(W, sb.offsets, sb.indices, g, w, n)
        assert np.array_equal(out, o2) and np.array_equal(sg.rows, r2)
        assert np.array_equal(sg.values, v2)
        p = f"case{n}_"
        store.update({p + "W": W, p + "offsets": sb.offsets,
                      p + "indices": sb.indices, p + "grad": g,
                      p + "out": out, p + "rows": sg.rows,
                      p + "values": sg.values})
        if w is not None:
            store[p + "weights"] = w
    store["num_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "bags.npz"), **store)
    print("bags: ok")


def ref_start_model(c):
    """dlrmkit model of a trajectory config at the GPU start point (every
    parameter rounded to float32, held in float64)."""
    cfg = dlrmkit.DlrmConfig(embedding_sizes=c["tables"], sparse_dim=c["d"],
                             bottom_mlp_dims=c["bot"], top_mlp_dims=c["top"],
                             seed=c["seed"])
    m = dlrmkit.init_model(cfg)
    for l in m.bottom.layers + m.top.layers:
        l.weight[...] = l.weight.astype(np.float32)
        l.bias[...] = l.bias.astype(np.float32)
    for t in m.tables:
        t.weights[...] = t.weights.astype(np.float32)
    return cfg, m


def make_ckpt():
    """A reference-written checkpoint of the toy config's start point."""
    _, m = ref_start_model(TRAJ["toy"])
    path = os.path.join(HERE, "ckpt_toy.dlrmkit")
    ref_cli.save_checkpoint(path, m)
    back = ref_cli.load_checkpoint(path)
    for a, b in zip(port_arrays(ref_model_to_port(m)), port_arrays(ref_model_to_port(back))):
        assert np.array_equal(a, b)
    print("ckpt: ok ->", path)


def make_eval(name, nbatches=3):
    """dlrmkit's _evaluate (cli.py:542-552) over validation batches of the
    CLI random source (key 1, as run_training draws them), dense rounded to
    float32, from the float32 start point."""
    c = TRAJ[name]
    cfg, m = ref_start_model(c)
    ours = RandomBatchSource(c["tables"], c["bot"][0], c["batch"], c["k"], c["fixed"],
                             seed=c["seed"], key=1)
    opts = ref_cli.RunOptions(mini_batch_size=c["batch"], num_indices_per_lookup=c["k"],
                              num_indices_per_lookup_fixed=c["fixed"])
    src = ref_cli._RandomSource(cfg, opts, key=1)
    batches, hbs = [], []
    for _ in range(nbatches):
        dense, sparse, labels = src.next_batch()
        hb = ours.next_batch()
        assert digest([dense, *[s.offsets for s in sparse], *[s.indices for s in sparse],
                       labels]) == digest(batch_arrays(hb)), "batch mismatch"
        batches.append((dense.astype(np.float32).astype(np.float64), sparse, labels))
        hbs.append(hb)
    vloss, vacc = ref_cli._evaluate(m, batches)
    np.savez_compressed(os.path.join(HERE, f"eval_{name}.npz"), config=np.array(json.dumps(c)),
                        nbatches=np.array(nbatches), loss=np.array(vloss), acc=np.array(vacc),
                        input_digest=np.array(digest([a for hb in hbs for a in batch_arrays(hb)])))
    print(f"eval {name}: loss {vloss:.6f} acc {vacc:.4f}")


def make_criteo():
    """A Criteo-format TSV (empty fields, negative / large dense values,
    unicode tokens, a trailing carriage return, blank lines) and dlrmkit's
    read_criteo / parse_criteo results for it, plus malformed lines with the
    reference's error messages."""
    from dlrmkit import datagen
    import tempfile
    rng = np.random.default_rng(11)
    vocab = [int(v) for v in rng.integers(1, 10**7, 26)]
    vocab[3], vocab[7] = 1, 3
    words = ["", "68fd1e64", "80e26c9b", "fb936136", "7b4723c4", "25c83c98", "7e0ccccf",
             "de7995b8", "1f89b562", "a73ee510", "\u00e9t\u00e9", "\u6f22\u5b57", "x" * 140]
    lines = []
    for r in range(300):
        lab = "" if r % 37 == 5 else str(int(rng.integers(0, 2)))
        dense = []
        for i in range(13):
            u = rng.random()
            dense.append("" if u < 0.15 else str(int(rng.integers(-3, 0))) if u < 0.25
                         else str(int(rng.integers(0, 10**6))))
        cats = [words[int(rng.integers(0, len(words)))] if rng.random() < 0.5
                else format(int(rng.integers(0, 2**32)), "08x") for _ in range(26)]
        lines.append("\t".join([lab] + dense + cats))
        if r % 50 == 7:
            lines.append("")          # blank line (skipped, counted)
    lines[10] = lines[10] + "\r"     # stays in the last token
    text = "\n".join(lines) + "\n"
    with tempfile.NamedTemporaryFile("w", suffix=".tsv", delete=False, encoding="utf-8") as f:
        f.write(text)
        path = f.name
    samples = list(datagen.read_criteo(path, vocab))
    os.unlink(path)
    store = {"text": np.frombuffer(text.encode("utf-8"), np.uint8),
             "vocab": np.array(vocab, np.int64),
             "labels": np.array([s.label for s in samples], np.int64),
             "dense": np.stack([s.dense for s in samples]),
             "cat": np.stack([s.categorical for s in samples])}
    good = lines[0].split("\t")
    bad = [("\t".join(good[:-1]), 7),
           ("\t".join(["2"] + good[1:]), 3),
           ("\t".join(["x"] + good[1:]), 1),
           ("\t".join(good[:4] + ["1.5.2"] + good[5:]), 9),
           ("\t".join(good + ["extra"]), 12)]
    msgs = []
    for ln, lineno in bad:
        try:
            datagen.parse_criteo(ln, vocab, lineno)
            raise AssertionError("expected an error")
        except datagen.CriteoFormatError as e:
            msgs.append(str(e))
    store["bad_lines"] = np.array([b[0] for b in bad])
    store["bad_linenos"] = np.array([b[1] for b in bad])
    store["bad_msgs"] = np.array(msgs)
    np.savez_compressed(os.path.join(HERE, "criteo.npz"), **store)
    print(f"criteo: {len(samples)} records, errors {msgs}")


if __name__ == "__main__":
    only = sys.argv[1:]
    if "criteo" in only:
        make_criteo()
    if not only or "ckpt" in only:
        make_ckpt()
    if not only or "eval" in only:
        make_eval("c3s")
        make_eval("c1s")
    if not only:
        make_criteo()
        make_bags()
    for name, c in TRAJ.items():
        if not only or name in only:
            make_traj(name, c)
