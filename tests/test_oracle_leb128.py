"""Pins for oracle.leb128 / oracle.codec varints (no GPU).

Pinned against: the paper's worked example, SPEC's vectors
(SPEC.md:71-94), hand-derived boundary values, hand-built rejection strings
(SPEC.md:80), and protobuf's independent unsigned-varint implementation
(protobuf varints are ULEB128) over an exhaustive range plus random u64.
"""

import random

import numpy as np
import pytest
from google.protobuf.internal import decoder as pb_dec
from google.protobuf.internal import encoder as pb_enc

from conftest import golden_lines, hexbytes
from oracle import DeltaError, brute, codec, leb128


def _pairs(name):
    out = []
    for ln in golden_lines(name):
        v, *bs = ln.split()
        out.append((int(v), bytes(int(b, 16) for b in bs)))
    return out


@pytest.mark.parametrize("fixture", ["paper_varint.txt", "spec_varint.txt", "leb128_boundaries.txt"])
def test_golden_encode_decode(fixture):
    for v, b in _pairs(fixture):
        assert leb128.encode(v) == b, (v, b.hex())
        assert leb128.decode(b) == (v, len(b))
        assert leb128.length(v) == len(b)
        # numpy vectorised encoder / decoder agree on the same vectors
        assert codec.encode_gaps(np.array([v], dtype=np.uint64)).tobytes() == b
        assert codec.decode_gaps(np.frombuffer(b, dtype=np.uint8)).tolist() == [v]


def test_paper_example_bit_by_bit():
    # C6 = 1100 0110 carries payload 70 with the continuation bit.
    b = leb128.encode(198)
    assert b[0] == 0b11000110 and b[0] & 0x7F == 70 and b[0] & 0x80
    assert b[1] == 0x01 and 70 + (1 << 7) == 198


def test_reject_vectors():
    for ln in golden_lines("varint_reject.txt"):
        kind, *bs = ln.split()
        b = bytes(int(x, 16) for x in bs)
        with pytest.raises(DeltaError) as e:
            leb128.decode(b)
        assert e.value.kind == kind, (ln, e.value)
        with pytest.raises(DeltaError) as e2:
            codec.decode_gaps(np.frombuffer(b, dtype=np.uint8))
        assert e2.value.kind == kind, (ln, e2.value)


def test_spec_encode_indices():
    for ln in golden_lines("spec_indices.txt"):
        lhs, rhs = ln.split("|")
        idx = [int(t) for t in lhs.split(",") if t.strip()]
        want = hexbytes(rhs)
        assert brute.encode_indices(idx) == want
        assert codec.encode_gaps(codec.gaps(np.array(idx, dtype=np.uint64))).tobytes() == want
        assert brute.decode_indices(want) == idx


def test_encode_indices_rejects_nonincreasing():
    with pytest.raises(DeltaError) as e:
        brute.encode_indices([3, 3])
    assert e.value.kind == "nonincreasing"


def test_exhaustive_vs_protobuf_0_to_2p20():
    # SPEC.md:533 (acceptance 2): exhaustive round trip for 0..2^20.
    for v in range(0, 1 << 20):
        b = leb128.encode(v)
        assert b == pb_enc._VarintBytes(v)
    g = np.arange(0, 1 << 20, dtype=np.uint64)
    enc = codec.encode_gaps(g)
    assert enc.tobytes() == b"".join(pb_enc._VarintBytes(int(v)) for v in range(0, 1 << 20))
    assert np.array_equal(codec.decode_gaps(enc), g)


def test_random_u64_vs_protobuf():
    rng = random.Random(1234)
    vals = [rng.getrandbits(rng.choice([7, 8, 14, 15, 21, 28, 32, 35, 49, 56, 63, 64]))
            for _ in range(100_000)]
    vals += [(1 << 64) - 1, (1 << 63), (1 << 63) - 1]
    for v in vals:
        b = leb128.encode(v)
        assert b == pb_enc._VarintBytes(v)
        dv, pos = pb_dec._DecodeVarint(b, 0)
        assert dv == v and pos == len(b)
        assert leb128.decode(b) == (v, len(b))
    g = np.array(vals, dtype=np.uint64)
    enc = codec.encode_gaps(g)
    assert enc.tobytes() == b"".join(pb_enc._VarintBytes(v) for v in vals)
    assert np.array_equal(codec.decode_gaps(enc), g)


def test_length_formula_closed_form():
    # len(g) = 1 + #{t in 7,14,..,63 : g >= 2^t} at and around every boundary
    for t in range(7, 64, 7):
        for v in ((1 << t) - 1, 1 << t):
            want = 1 + sum(1 for s in range(7, 64, 7) if v >= (1 << s))
            assert leb128.length(v) == want == len(leb128.encode(v))
            assert codec.varint_lengths(np.array([v], dtype=np.uint64))[0] == want
