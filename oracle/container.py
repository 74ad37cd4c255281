"""SPDC delta-checkpoint container (test infrastructure only).

SPEC.md:145-149 (codec › External Interfaces): header = magic "SPDC" |
format_version u16 | version u64 | base_version u64 | element-type code u8
(0 = 16-bit, 1 = 32-bit) | tensor count u32 | body length u64 | body hash
(32 bytes); "the hash covers exactly the body bytes"; readers reject unknown
format_version.  PAPER.md:368-370: D_v is "versioned, immutable ... complete
with a unique identifier and integrity hash".

Readings (R9, R10, R18): format_version = 1 for LEB128 index streams,
2 for the naive fixed-width index encoding; the digest is
BLAKE3-256 of exactly the body bytes.  A reader names the codec it reads and
rejects the other format_version.
"""

import struct

import blake3

from .errors import DeltaError

MAGIC = b"SPDC"
FORMAT_VERSION = {"leb128": 1, "fixed": 2}
HEADER_BYTES = 4 + 2 + 8 + 8 + 1 + 4 + 8 + 32  # = 67
ELEM_CODE = {2: 0, 4: 1}


def digest(body: bytes) -> bytes:
    return blake3.blake3(bytes(body)).digest(32)


def pack(body: bytes, version: int, base_version: int, width: int, n_tensors: int,
         index_codec: str = "leb128") -> bytes:
    if version != base_version + 1:
        raise DeltaError("layout", "version must equal base_version + 1 (SPEC.md:46)")
    hdr = (MAGIC + struct.pack("<HQQBIQ", FORMAT_VERSION[index_codec], version, base_version,
                               ELEM_CODE[width], n_tensors, len(body)) + digest(body))
    assert len(hdr) == HEADER_BYTES
    return hdr + bytes(body)


def unpack(blob: bytes, index_codec: str = "leb128"):
    """-> (version, base_version, width, n_tensors, body); verifies the hash."""
    if len(blob) < HEADER_BYTES or blob[:4] != MAGIC:
        raise DeltaError("layout", "not an SPDC container")
    fv, ver, base, code, nt, blen = struct.unpack_from("<HQQBIQ", blob, 4)
    if fv != FORMAT_VERSION[index_codec]:
        raise DeltaError("layout", f"unknown format_version {fv}")
    h = blob[35:67]
    body = blob[HEADER_BYTES:]
    if len(body) != blen:
        raise DeltaError("layout", "body length mismatch")
    if digest(body) != h:
        raise DeltaError("layout", "body hash mismatch")
    width = {0: 2, 1: 4}[code]
    return ver, base, width, nt, body
