"""Pins for the oracle's naive fixed-width index encoding (no GPU).

PAPER.md:387: "stores the non-zeros as two 1D arrays, idx and val ... int32 or int64
(depending on tensor size)"; the "naive int32/64 index encoding" the paper
measures LEB128 against (414 MB vs 202 MB).  DESIGN.md reading R18 fixes the bytes: the
SPEC.md:148 record with the index stream = the absolute indices, little-endian, 4 bytes
iff N - 1 <= 2^31 - 1, else 8.

Against: a hand-derived golden record (tests/golden/record_w_bf16_fixed.txt), the width
boundary at N = 2^31 worked by hand, the closed-form size 27 + name + nnz (iw + w), brute
force vs numpy, the LEB128 record of the same change set (independent decode), and the
round-trip / rejection invariants.
"""

import numpy as np
import pytest

from conftest import golden_lines, hexbytes
from oracle import DeltaError, brute, codec, payload


def _kv(name):
    d = {}
    for ln in golden_lines(name):
        k, _, v = ln.partition(" ")
        d[k] = v
    return d


def test_golden_fixed_record():
    g = _kv("record_w_bf16_fixed.txt")
    old = [int(t, 16) for t in g["old"].split()]
    new = [int(t, 16) for t in g["new"].split()]
    want = hexbytes(g["record"])
    assert len(want) == 34 == 27 + 1 + 4 + 2
    body, table = brute.extract([(g["name"], [old], [new])], width=2, index_codec="fixed")
    assert body == want
    nb, ntab = codec.extract([(g["name"], [np.array(old, np.uint16)], [np.array(new, np.uint16)])],
                             index_codec="fixed")
    assert nb == want
    assert table == ntab == [(0, 3, 1, 27, 4, 31, 34)]
    assert brute.apply([("w", old)], body, 2, index_codec="fixed") == [new]


def test_width_boundary_by_hand():
    # N = 2^31: largest index 2^31 - 1 is INT32_MAX -> 4 bytes; N = 2^31 + 1 -> 8 bytes
    assert brute.fixed_index_width(2**31) == 4 == codec.fixed_index_width(2**31)
    assert brute.fixed_index_width(2**31 + 1) == 8 == codec.fixed_index_width(2**31 + 1)
    assert brute.encode_indices_fixed([0, 2**31 - 1], 2**31) == bytes.fromhex("00000000ffffff7f")
    assert brute.encode_indices_fixed([5, 2**31], 2**31 + 1) == bytes.fromhex(
        "0500000000000000" "0000008000000000")
    s = codec.encode_fixed(np.array([5, 2**31], np.uint64), 2**31 + 1).tobytes()
    assert s == bytes.fromhex("0500000000000000" "0000008000000000")
    assert codec.decode_fixed(np.frombuffer(s, np.uint8), 2**31 + 1).tolist() == [5, 2**31]
    # agrees with the payload model's naive width (PAPER.md:387 reading)
    for n in (1, 3, 2**31, 2**31 + 1, 2**40):
        assert brute.fixed_index_width(n) == payload.naive_index_width(n)


@pytest.mark.parametrize("seed", range(12))
def test_fixed_brute_vs_numpy_and_size(seed):
    rng = np.random.default_rng(1000 + seed)
    width = 2 if seed % 2 == 0 else 4
    dt = np.uint16 if width == 2 else np.uint32
    tensors_np, tensors_py = [], []
    for k in range(3):
        nsp = 1 + (seed + k) % 3
        olds = [rng.integers(0, 2**(8 * width), rng.integers(0, 40), dtype=np.uint64).astype(dt)
                for _ in range(nsp)]
        news = []
        for o in olds:
            n = o.copy()
            m = rng.random(o.size) < 0.3
            n[m] ^= dt(1 + seed)
            news.append(n)
        name = f"t{k}.ü"
        tensors_np.append((name, olds, news))
        tensors_py.append((name, [o.tolist() for o in olds], [n.tolist() for n in news]))
    bb, bt = brute.extract(tensors_py, width, index_codec="fixed")
    nb, nt = codec.extract(tensors_np, index_codec="fixed")
    assert bb == nb and bt == [tuple(r) for r in nt]
    lb, lt = codec.extract(tensors_np)  # LEB128 record of the same change sets
    lrecs = codec.parse(lb, width)
    frecs = codec.parse(nb, width, index_codec="fixed")
    for (name, n, li, lv, _), (fname, fn, fi, fv, _), row in zip(lrecs, frecs, bt):
        assert (name, n) == (fname, fn)
        assert np.array_equal(li, fi) and np.array_equal(lv, fv)
        nl = len(name.encode())
        assert row[6] == 27 + nl + fi.size * (brute.fixed_index_width(n) + width)
        assert row[4] == payload.naive_bytes(fi.size, n, width) - fi.size * width
    # round trip
    for (name, olds, news), got in zip(tensors_np, codec.apply(
            [(nm, codec.fuse(o)) for nm, o, _ in tensors_np], nb, width, index_codec="fixed")):
        assert np.array_equal(got, codec.fuse(news))


def _one(old, new, width=2):
    return codec.extract([("x", [np.array(old, np.uint16)], [np.array(new, np.uint16)])],
                         index_codec="fixed")[0]


@pytest.mark.parametrize("kind", ["truncated", "nonincreasing", "range", "count"])
def test_fixed_rejects_and_leaves_targets(kind):
    old = np.arange(10, dtype=np.uint16)
    new = old.copy()
    new[[2, 7]] += 1
    body = bytearray(_one(old, new))
    p = 2 + 1 + 24  # index stream: 02 00 00 00 07 00 00 00
    if kind == "truncated":  # idx_len = 7 (not a multiple of 4), nnz 2; shift values
        body = body[:p + 7] + body[p + 8:]
        body[2 + 1 + 16] = 7
    elif kind == "nonincreasing":
        body[p + 4] = 2  # second index = first
    elif kind == "range":
        body[p + 4] = 10  # index 10 >= N = 10
    else:  # nnz says 3, the stream holds 2 indices; one more value byte pair
        body[2 + 1 + 8] = 3
        body = body[:-1] + b"\x00\x00" + body[-1:]
    w = old.copy()
    for fn in (lambda: codec.apply([("x", w)], bytes(body), 2, inplace=True, index_codec="fixed"),
               lambda: brute.apply([("x", w.tolist())], bytes(body), 2, index_codec="fixed")):
        with pytest.raises(DeltaError) as e:
            fn()
        assert e.value.kind == kind
    assert np.array_equal(w, old)
