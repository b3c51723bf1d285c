"""Criteo ingestion vs dlrmkit.datagen: the native
parser's labels / categorical indices are bit-identical to the reference's
read_criteo on a fixture with empty fields, negative and large dense values,
unicode and >128-byte tokens, a trailing carriage return and blank lines;
dense values equal the reference's float64 rounded to fp32; malformed lines
raise the reference's messages.  Host code only (no GPU)."""

import gzip
import hashlib
import os

import numpy as np
import pytest

from paper_1906_00091_b200.criteo import (CriteoBatchReader, CriteoFormatError, hash_token,
                                          parse_criteo, parse_criteo_block, read_criteo)

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def fx():
    return dict(np.load(os.path.join(HERE, "golden", "criteo.npz")))


def check(fx, labels, dense, cat):
    assert np.array_equal(labels.astype(np.int64), fx["labels"])
    assert np.array_equal(dense, fx["dense"].astype(np.float32))
    assert np.array_equal(cat, fx["cat"])


def test_block_parse_matches_reference(fx):
    text = fx["text"].tobytes()
    labels, dense, cat, used = parse_criteo_block(text, fx["vocab"])
    assert used == len(text)
    check(fx, labels, dense, cat.T)


def test_multithreaded_parse_is_identical(fx):
    text = fx["text"].tobytes() * 20     # > 4096 records: the threaded path
    a = parse_criteo_block(text, fx["vocab"], nthreads=1)
    b = parse_criteo_block(text, fx["vocab"], nthreads=7)
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)
    n = fx["labels"].size
    assert a[0].size == 20 * n
    check(fx, a[0][-n:], a[1][-n:], a[2][:, -n:].T)


@pytest.mark.parametrize("gz", [False, True])
def test_read_criteo_and_batches(fx, tmp_path, gz):
    p = tmp_path / ("d.tsv.gz" if gz else "d.tsv")
    data = fx["text"].tobytes()
    if gz:
        with gzip.open(p, "wb") as f:
            f.write(data)
    else:
        p.write_bytes(data)
    # small chunks: records straddle chunk boundaries
    samples = list(read_criteo(str(p), fx["vocab"], chunk_bytes=4096))
    check(fx, np.array([s.label for s in samples]), np.stack([s.dense for s in samples]),
          np.stack([s.categorical for s in samples]))
    B = 64
    batches = list(CriteoBatchReader(str(p), fx["vocab"], B, drop_last=False, chunk_bytes=5000))
    n = fx["labels"].size
    assert [b.labels.shape[0] for b in batches] == [B] * (n // B) + [n % B]
    dense = np.concatenate([b.dense for b in batches])
    labels = np.concatenate([b.labels for b in batches])
    cat = np.stack([np.concatenate([b.indices[i] for b in batches]) for i in range(26)], 1)
    check(fx, labels, dense, cat)
    for b in batches:
        assert all(np.array_equal(o, np.arange(b.labels.shape[0] + 1)) for o in b.offsets)
    assert len(list(CriteoBatchReader(str(p), fx["vocab"], B))) == n // B


def test_errors_match_reference(fx):
    for line, lineno, msg in zip(fx["bad_lines"], fx["bad_linenos"], fx["bad_msgs"]):
        with pytest.raises(CriteoFormatError) as e:
            parse_criteo(str(line), fx["vocab"], int(lineno))
        assert str(e.value) == str(msg)
    with pytest.raises(ValueError, match="need 26 vocabulary sizes, got 3"):
        parse_criteo(fx["text"].tobytes().split(b"\n")[0].decode(), [1, 2, 3])


def test_first_bad_line_wins_across_threads(fx):
    good = fx["text"].tobytes() * 20
    lines = good.split(b"\n")
    lines[6000] = b"1\t2"          # late bad line (other thread)
    lines[2500] = b"x" + lines[2500]
    with pytest.raises(CriteoFormatError, match=r"^line 2501: "):
        parse_criteo_block(b"\n".join(lines), fx["vocab"], nthreads=8)


def test_single_record_api(fx):
    first = fx["text"].tobytes().split(b"\n")[0].decode()
    s = parse_criteo(first + "\n", fx["vocab"])
    assert s.label == fx["labels"][0]
    assert np.array_equal(s.dense, fx["dense"][0].astype(np.float32))
    assert np.array_equal(s.categorical, fx["cat"][0])
    empty = parse_criteo("\t" * 39, fx["vocab"])
    assert empty.label == 0 and not empty.dense.any() and not empty.categorical.any()


def test_hash_token():
    for tok in ["", "a", "68fd1e64", "été", "z" * 300]:
        ref = int.from_bytes(hashlib.blake2b(tok.encode(), digest_size=8).digest(), "little")
        assert hash_token(tok) == ref
