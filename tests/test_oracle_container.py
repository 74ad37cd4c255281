"""Pins for oracle.container: the SPDC header layout of SPEC.md:145-149 (no GPU)."""

import struct

import pytest

from conftest import golden_lines, hexbytes
from oracle import DeltaError, container


def _golden_body():
    for ln in golden_lines("record_w_bf16.txt"):
        if ln.startswith("record "):
            return hexbytes(ln[len("record "):])


def test_header_layout_by_hand():
    body = _golden_body()
    blob = container.pack(body, version=5, base_version=4, width=2, n_tensors=1)
    assert container.HEADER_BYTES == 67 == 4 + 2 + 8 + 8 + 1 + 4 + 8 + 32
    assert blob[:4] == b"SPDC"
    assert blob[4:6] == b"\x01\x00"                       # format_version 1 (R9)
    assert blob[6:14] == (5).to_bytes(8, "little")
    assert blob[14:22] == (4).to_bytes(8, "little")
    assert blob[22] == 0                                   # 16-bit element code
    assert blob[23:27] == (1).to_bytes(4, "little")
    assert blob[27:35] == len(body).to_bytes(8, "little")
    assert blob[67:] == body
    assert container.unpack(blob) == (5, 4, 2, 1, body)


def test_reject():
    body = _golden_body()
    blob = bytearray(container.pack(body, 1, 0, 2, 1))
    bad = bytearray(blob)
    bad[-1] ^= 1                                           # body hash mismatch
    with pytest.raises(DeltaError):
        container.unpack(bytes(bad))
    bad = bytearray(blob)
    bad[4] = 2                                             # unknown format_version
    with pytest.raises(DeltaError):
        container.unpack(bytes(bad))
    with pytest.raises(DeltaError):
        container.pack(body, 3, 1, 2, 1)                   # version != base + 1


def test_fixed_codec_container_version():
    # reading R18: format_version 2 marks fixed-width index streams; a LEB128 reader rejects it
    body = b"\x01\x00w" + bytes(24) + b"\x00"
    blob = container.pack(body, 2, 1, 2, 1, index_codec="fixed")
    assert blob[4:6] == b"\x02\x00"
    assert container.unpack(blob, index_codec="fixed") == (2, 1, 2, 1, body)
    with pytest.raises(DeltaError):
        container.unpack(blob)


def _kat():
    out = []
    for ln in golden_lines("blake3_kat.txt"):
        n, h = ln.split()
        out.append((int(n), bytes.fromhex(h)))
    return out


def test_digest_blake3_known_answers():
    """container.digest against the official BLAKE3 vectors (tests/golden/blake3_kat.txt): the
    empty input, 1 byte, chunk boundaries 1023/1024/1025 and multi-chunk trees."""
    kat = _kat()
    assert [n for n, _ in kat][:5] == [0, 1, 1023, 1024, 1025]
    for n, h in kat:
        assert container.digest(bytes(i % 251 for i in range(n))) == h, n


def test_header_digest_field_is_the_body_hash():
    """The 32 header bytes 35..67 are the BLAKE3 of exactly the body, pinned
    through a KAT body: a 1025-byte body of i mod 251 carries the 1025-byte vector."""
    n, h = _kat()[4]
    body = bytes(i % 251 for i in range(n))
    blob = container.pack(body, version=2, base_version=1, width=2, n_tensors=0)
    assert blob[35:67] == h
