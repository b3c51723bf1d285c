"""DLRMKIT1 v1 checkpoint format (ref cli.py:475-518) on the host: the
reference-written golden file parses, the digest and the error cases match
the reference's checks, and files written here load with the reference's own
loader when it is importable (this build container)."""

import json
import os
import sys

import numpy as np
import pytest

from paper_1906_00091_b200.checkpoint import (CHECKPOINT_MAGIC, CheckpointError,
                                              config_digest, read_arrays, write_arrays)

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "ckpt_toy.dlrmkit")
TOY = dict(embedding_sizes=[7, 5, 9], sparse_dim=3, bottom_mlp_dims=[4, 3],
           top_mlp_dims=[10, 4, 1], interaction="dot", seed=44)


def test_reference_checkpoint_parses():
    cfg, arrays = read_arrays(GOLD)
    assert cfg == TOY
    assert sorted(arrays) == sorted(["bottom_w_0", "bottom_b_0", "top_w_0", "top_b_0",
                                     "top_w_1", "top_b_1", "top_w_2", "top_b_2",
                                     "table_0", "table_1", "table_2"])
    assert arrays["bottom_w_0"].shape == (3, 4)
    assert arrays["top_w_0"].shape == (10, 3 + 6)   # d + P with nf = 4
    for t, m in enumerate(TOY["embedding_sizes"]):
        assert arrays[f"table_{t}"].shape == (m, 3)
    with open(GOLD, "rb") as f:
        assert f.readline().decode().split() == [CHECKPOINT_MAGIC, "v1", config_digest(TOY)]


def test_write_read_roundtrip(tmp_path):
    cfg, arrays = read_arrays(GOLD)
    arrays["adagrad_table_0"] = np.ones((7, 3), np.float32)
    p = str(tmp_path / "rt.dlrmkit")
    write_arrays(p, cfg, arrays)
    cfg2, arrays2 = read_arrays(p)
    assert cfg2 == cfg and sorted(arrays2) == sorted(arrays)
    for k in arrays:
        assert arrays2[k].dtype == arrays[k].dtype and np.array_equal(arrays2[k], arrays[k])


def test_header_errors(tmp_path):
    raw = open(GOLD, "rb").read()
    head, body = raw.split(b"\n", 1)
    for bad, msg in ((b"NOTDLRM v1 " + head.split()[2], "not a"),
                     (b"DLRMKIT1 v2 " + head.split()[2], "unsupported checkpoint version"),
                     (b"DLRMKIT1 v1 " + b"0" * 64, "digest mismatch"),
                     (b"DLRMKIT1 v1", "not a")):
        p = tmp_path / "bad.dlrmkit"
        p.write_bytes(bad + b"\n" + body)
        with pytest.raises(CheckpointError, match=msg):
            read_arrays(str(p))


def _reference():
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        return None
    if src not in sys.path:
        sys.path.insert(0, src)
    try:
        from dlrmkit import cli
        return cli
    except Exception:
        return None


def test_reference_loader_reads_our_file(tmp_path):
    cli = _reference()
    if cli is None:
        pytest.skip("reference not importable here")
    cfg, arrays = read_arrays(GOLD)
    arrays = {k: v.astype(np.float32) for k, v in arrays.items()}   # our training dtype
    arrays["opt_kind"] = np.frombuffer(b"adagrad", np.uint8)        # extras are ignored
    arrays["adagrad_table_1"] = np.zeros((5, 3), np.float32)
    p = str(tmp_path / "ours.dlrmkit")
    write_arrays(p, cfg, arrays)
    m = cli.load_checkpoint(p)
    assert json.loads(json.dumps(m.config.__dict__)) == TOY
    for l, layer in enumerate(m.bottom.layers):
        assert np.array_equal(layer.weight, arrays[f"bottom_w_{l}"])
    for l, layer in enumerate(m.top.layers):
        assert np.array_equal(layer.weight, arrays[f"top_w_{l}"])
        assert np.array_equal(layer.bias, arrays[f"top_b_{l}"])
    for t, table in enumerate(m.tables):
        assert np.array_equal(table.weights, arrays[f"table_{t}"])
