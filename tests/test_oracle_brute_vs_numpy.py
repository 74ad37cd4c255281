"""oracle.codec (numpy) against oracle.brute (pure-Python definition) on random
tiny inputs, and both against hand-built malformed bodies (no GPU)."""

import struct

import numpy as np
import pytest

from oracle import DeltaError, brute, codec


def _rand_case(rng, width):
    dt = np.uint16 if width == 2 else np.uint32
    hi = 2**16 if width == 2 else 2**32
    tensors = []
    for t in range(rng.integers(1, 5)):
        nspans = int(rng.integers(1, 4))
        olds, news = [], []
        for _ in range(nspans):
            n = int(rng.integers(0, 300)) if rng.random() < 0.9 else int(rng.integers(300, 40000))
            o = rng.integers(0, hi, n, dtype=np.uint64).astype(dt)
            p = rng.choice([0.0, 0.001, 0.01, 0.3, 1.0])
            m = rng.random(n) < p
            nw = o.copy()
            nw[m] = (o[m].astype(np.uint64) ^ rng.integers(1, hi, int(m.sum()), dtype=np.uint64)).astype(dt)
            olds.append(o)
            news.append(nw)
        name = "".join(chr(int(c)) for c in rng.integers(97, 123, int(rng.integers(1, 40))))
        if rng.random() < 0.2:
            name += "é中"  # non-ASCII: name_len counts UTF-8 bytes
        tensors.append((name + str(t), olds, news))
    return tensors


@pytest.mark.parametrize("width", [2, 4])
def test_extract_apply_match(width):
    rng = np.random.default_rng(42 + width)
    for _ in range(60):
        ts = _rand_case(rng, width)
        body, table = codec.extract(ts)
        bbody, btable = brute.extract([(n, [o.tolist() for o in os_], [x.tolist() for x in ns])
                                       for n, os_, ns in ts], width)
        assert body == bbody
        assert table == btable
        targets = [(n, codec.fuse(os_)) for n, os_, _ in ts]
        got = codec.apply(targets, body, width)
        bgot = brute.apply([(n, w.tolist()) for n, w in targets], body, width)
        for g, bg, (_, _, ns) in zip(got, bgot, ts):
            assert g.tolist() == bg == codec.fuse(ns).tolist()


def _rec(name, n, nnz, stream, vals, mode=0, width=2):
    nb = name.encode()
    return (struct.pack("<H", len(nb)) + nb + struct.pack("<QQQ", n, nnz, len(stream))
            + bytes(stream) + bytes(vals) + bytes([mode]))


# (kind, body, targets)   each body carries exactly one fault
_BAD = [
    ("truncated", _rec("a", 10, 1, b"\x85", b"\x01\x00"), [("a", 10)]),
    ("overlong", _rec("a", 10, 1, b"\x85\x00", b"\x01\x00"), [("a", 10)]),
    ("overflow", _rec("a", 10, 1, b"\xff" * 9 + b"\x02", b"\x01\x00"), [("a", 10)]),
    ("overflow", _rec("a", 10, 1, b"\xff" * 10 + b"\x01", b"\x01\x00"), [("a", 10)]),
    ("nonincreasing", _rec("a", 10, 2, b"\x05\x00", b"\x01\x00\x02\x00"), [("a", 10)]),
    ("range", _rec("a", 10, 2, b"\x05\x05", b"\x01\x00\x02\x00"), [("a", 10)]),
    ("range", _rec("a", 10, 1, b"\x0a", b"\x01\x00"), [("a", 10)]),
    ("count", _rec("a", 10, 1, b"\x01\x01", b"\x01\x00"), [("a", 10)]),
    ("count", _rec("a", 10, 3, b"\x01\x01", b"\x01\x00\x02\x00\x03\x00"), [("a", 10)]),
    ("name", _rec("a", 10, 1, b"\x01", b"\x01\x00"), [("b", 10)]),
    ("numel", _rec("a", 10, 1, b"\x01", b"\x01\x00"), [("a", 11)]),
    ("mode", _rec("a", 10, 1, b"\x01", b"\x01\x00", mode=2), [("a", 10)]),
    ("layout", _rec("a", 10, 1, b"\x01", b"\x01\x00")[:-1], [("a", 10)]),
    ("layout", _rec("a", 10, 1, b"\x01", b"\x01\x00") + b"\x00", [("a", 10)]),
    ("layout", _rec("a", 10, 1, b"\x01", b"\x01\x00"), [("a", 10), ("b", 3)]),
    ("layout", _rec("a", 10, 1, b"\x01", b"\x01\x00")[:5], [("a", 10)]),
]


@pytest.mark.parametrize("kind,body,tgt", _BAD)
def test_malformed_rejected_and_untouched(kind, body, tgt):
    with pytest.raises(DeltaError) as e1:
        brute.apply([(n, [0] * k) for n, k in tgt], body, 2)
    arrs = [(n, np.arange(k, dtype=np.uint16)) for n, k in tgt]
    before = [a.copy() for _, a in arrs]
    with pytest.raises(DeltaError) as e2:
        codec.apply(arrs, body, 2, inplace=True)
    assert e1.value.kind == e2.value.kind == kind
    for (_, a), b in zip(arrs, before):
        assert np.array_equal(a, b)  # all-or-nothing


def test_valid_control_for_malformed_set():
    body = _rec("a", 10, 2, b"\x05\x04", b"\x01\x00\x02\x00")
    out = codec.apply([("a", np.zeros(10, np.uint16))], body, 2)[0]
    assert out.tolist() == [0, 0, 0, 0, 0, 1, 0, 0, 0, 2]
    assert brute.apply([("a", [0] * 10)], body, 2)[0] == out.tolist()


@pytest.mark.parametrize("width", [2, 4])
def test_additive_mode_brute_vs_numpy(width):
    """Additive mode: values = new - old in the lane's float type; apply
    adds.  numpy (float32 arrays) against the per-element definition (Python floats rounded
    to fp32, then RNE to bf16), on random bit patterns incl. NaN / Inf / subnormals."""
    rng = np.random.default_rng(7 + width)
    for _ in range(30):
        ts = _rand_case(rng, width)
        body, table = codec.extract(ts, mode=codec.MODE_ADDITIVE)
        bbody, btable = brute.extract([(n, [o.tolist() for o in os_], [x.tolist() for x in ns])
                                       for n, os_, ns in ts], width, mode=brute.MODE_ADDITIVE)
        assert body == bbody and table == btable
        targets = [(n, codec.fuse(os_)) for n, os_, _ in ts]
        got = codec.apply(targets, body, width)
        bgot = brute.apply([(n, w.tolist()) for n, w in targets], body, width)
        for g, bg in zip(got, bgot):
            assert g.tolist() == bg


def test_additive_hand_examples():
    # bf16: 1.0 = 0x3F80, 1.0078125 = 0x3F81 -> difference 2^-7 = 0x3C00; 1.0 + 2^-7 = 0x3F81
    assert brute.lane_op(0x3F81, 0x3F80, 2, -1) == 0x3C00
    assert brute.lane_op(0x3F80, 0x3C00, 2, +1) == 0x3F81
    # tie: 256 (0x4380) + 1.0 = 257 lies halfway between 256 and 258 -> even mantissa: 256
    assert brute.lane_op(0x4380, 0x3F80, 2, +1) == 0x4380
    # ... and 258 (0x4381) + 1.0 = 259 -> halfway between 258 and 260 -> 260 (0x4382)
    assert brute.lane_op(0x4381, 0x3F80, 2, +1) == 0x4382
    # fp32: 1.0 + 2^-24 is a tie between 1.0 and 1 + 2^-23 -> 1.0 (even)
    assert brute.lane_op(0x3F800000, 0x33800000, 4, +1) == 0x3F800000
    # numpy agrees on the same lanes
    assert codec.lane_add(np.array([0x4380, 0x4381], np.uint16), np.array([0x3F80, 0x3F80], np.uint16)).tolist() \
        == [0x4380, 0x4382]
    # additive with exactly representable differences reconstructs new exactly
    old = np.array([0x3F80, 0x4000, 0x4040], np.uint16)   # 1, 2, 3
    new = np.array([0x3F80, 0x40A0, 0x4040], np.uint16)   # 1, 5, 3
    body, _ = codec.extract([("w", [old], [new])], mode=codec.MODE_ADDITIVE)
    assert body[-1] == 1 and body[-3:-1] == bytes([0x40, 0x40])  # value 3.0 = 5 - 2
    assert codec.apply([("w", old)], body, 2)[0].tolist() == new.tolist()
