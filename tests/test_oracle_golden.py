"""Pins for the oracle's record layout, extract, apply and rho (no GPU).

Against: the hand-derived golden record of SPEC.md:102's example
(tests/golden/record_w_bf16.txt), SPEC.md:104's fused q/k/v example, the apply
examples of SPEC.md:112-114 and the Eq. 1 examples of SPEC.md:122-124.
"""

import numpy as np
import pytest

from conftest import golden_lines, hexbytes
from oracle import DeltaError, brute, codec


def _kv(name):
    d = {}
    for ln in golden_lines(name):
        k, _, v = ln.partition(" ")
        d[k] = v
    return d


def test_golden_record_bf16():
    g = _kv("record_w_bf16.txt")
    old = [int(t, 16) for t in g["old"].split()]
    new = [int(t, 16) for t in g["new"].split()]
    want = hexbytes(g["record"])
    assert len(want) == 31 == 27 + 1 + 1 + 2
    body, table = brute.extract([(g["name"], [old], [new])], width=2)
    assert body == want
    nb, ntab = codec.extract([(g["name"], [np.array(old, np.uint16)], [np.array(new, np.uint16)])])
    assert nb == want
    # offset table O7: record_off, N, nnz, idx_off = 0+2+1+24, idx_len, val_off, bytes
    assert table == ntab == [(0, 3, 1, 27, 1, 28, 31)]
    # apply gives new back
    assert brute.apply([("w", old)], body, 2) == [new]
    assert codec.apply([("w", np.array(old, np.uint16))], body, 2)[0].tolist() == new


def test_golden_fused_qkv():
    g = _kv("fused_qkv.txt")
    sp = {k: np.array([int(t, 16) for t in g[k].split()], np.uint16)
          for k in ("q_old", "q_new", "k_old", "k_new", "v_old", "v_new")}
    olds = [sp["q_old"], sp["k_old"], sp["v_old"]]
    news = [sp["q_new"], sp["k_new"], sp["v_new"]]
    want_idx = [int(t) for t in g["indices"].split()]
    assert codec.changed_indices(codec.fuse(olds), codec.fuse(news)).tolist() == want_idx
    body, table = codec.extract([(g["name"], olds, news)])
    stream = body[table[0][3]:table[0][3] + table[0][4]]
    assert stream == hexbytes(g["stream"])
    bbody, _ = brute.extract([(g["name"], [o.tolist() for o in olds], [n.tolist() for n in news])], 2)
    assert bbody == body
    # SPEC.md:128 fusion correctness: fused extract+apply == per-source apply then concatenation
    fused_new = codec.apply([("qkv", codec.fuse(olds))], body, 2)[0]
    assert np.array_equal(fused_new, codec.fuse(news))


def test_spec_apply_examples():
    # params=[1,2,3], delta {idx:[1], val:[5]} -> [1,5,3]
    body, _ = brute.extract([("p", [[1, 2, 3]], [[1, 5, 3]])], 2)
    assert brute.apply([("p", [1, 2, 3])], body, 2) == [[1, 5, 3]]
    # empty delta -> unchanged
    body0, tab0 = brute.extract([("p", [[1, 2, 3]], [[1, 2, 3]])], 2)
    assert tab0[0][2] == 0 and tab0[0][4] == 0
    assert brute.apply([("p", [7, 8, 9])], body0, 2) == [[7, 8, 9]]


def test_identity_gives_empty_records():
    # old == new -> zero nnz in every tensor, every tensor still has a record
    rng = np.random.default_rng(0)
    ts = [(f"t{i}", [rng.integers(0, 2**16, n, dtype=np.uint16)]) for i, n in enumerate([1, 5, 1000])]
    body, table = codec.extract([(nm, a, [x.copy() for x in a]) for nm, a in ts])
    assert [r[2] for r in table] == [0, 0, 0]
    assert [r[6] for r in table] == [27 + 2, 27 + 2, 27 + 2]
    assert len(body) == sum(r[6] for r in table)


def test_rho_examples():
    # sizes 4 and 6 with 1 and 2 changed -> 3/10
    a = ([0, 0, 0, 0], [0, 1, 0, 0])
    b = ([0] * 6, [1, 0, 0, 0, 0, 1])
    assert brute.rho([a, b]) == pytest.approx(0.3)
    assert codec.rho([(np.array(x, np.uint16), np.array(y, np.uint16)) for x, y in (a, b)]) == pytest.approx(0.3)
    # identical -> 0
    assert brute.rho([([1, 2], [1, 2])]) == 0.0


def test_bitwise_semantics_signed_zero_and_nan():
    # DESIGN.md reading R2: -0.0 vs +0.0 is a change; identical NaN bits are not;
    # different NaN payloads are.
    old = np.array([0x0000, 0x7FC0, 0x7FC0, 0x3F80], np.uint16)
    new = np.array([0x8000, 0x7FC0, 0x7FC1, 0x3F80], np.uint16)
    assert codec.changed_indices(old, new).tolist() == [0, 2]
    assert brute.changed_indices(old.tolist(), new.tolist()) == [0, 2]


def test_shape_mismatch():
    with pytest.raises(DeltaError) as e:
        codec.extract([("x", [np.zeros(3, np.uint16)], [np.zeros(4, np.uint16)])])
    assert e.value.kind == "shape"
    with pytest.raises(DeltaError) as e:
        brute.extract([("x", [[0, 0]], [[0, 0], [1]])], 2)
    assert e.value.kind == "shape"


def test_record_from_sparse_equals_record_on_dense():
    """brute.record_from_sparse (the expected value of the >2^32-lane GPU test) is the same
    O3-O6 record as brute.record when the change set comes from dense lists."""
    rng = np.random.default_rng(7)
    for trial in range(40):
        n = int(rng.integers(0, 400))
        width = 2 if trial % 2 else 4
        old = rng.integers(0, 1 << (8 * width), n, dtype=np.uint64).tolist()
        new = list(old)
        for j in rng.choice(n, size=int(rng.integers(0, n + 1)) if n else 0, replace=False).tolist():
            new[j] = (new[j] + int(rng.integers(1, 1 << (8 * width)))) % (1 << (8 * width))
        idx = [j for j in range(n) if old[j] != new[j]]
        name = f"t{trial}.weight" + ("é" if trial % 3 == 0 else "")
        assert brute.record_from_sparse(name, n, idx, [new[j] for j in idx], width) == \
            brute.record(name, old, new, width)


def test_record_from_sparse_golden_2p32():
    """Hand-derived record of a tensor with 2^32 + 1000 lanes (tests/golden/record_sparse_2p32.txt):
    u64 element count above 2^32, a 5-byte LEB128 gap (reading R13)."""
    g = _kv("record_sparse_2p32.txt")
    want = hexbytes(g["record"])
    n = int(g["numel"])
    assert n == 2 ** 32 + 1000 and len(want) == 40
    got = brute.record_from_sparse(g["name"], n, [int(t) for t in g["idx"].split()],
                                   [int(t, 16) for t in g["vals"].split()], int(g["width"]))
    assert got == want
