"""SPDC delta-checkpoint container, host side.

Header (67 bytes, little-endian): "SPDC" | format_version u16 (= 1) | version u64 |
base_version u64 | element-type code u8 (0 = 16-bit, 1 = 32-bit) | tensor count u32 |
body length u64 | BLAKE3-256 of exactly the body bytes (readings R9, R10).
The body is what ``delta_extract`` writes.  Hashing runs on the host in this version (a
GPU tree hash is the next step).
"""

import struct

import blake3

_MAGIC = b"SPDC"
_FMT = "<4sHQQBIQ32s"
HEADER_BYTES = struct.calcsize(_FMT)


def pack_container(body: bytes, version: int, base_version: int, width: int, n_tensors: int) -> bytes:
    if version != base_version + 1:
        raise ValueError("version must be base_version + 1")
    body = bytes(body)
    code = {2: 0, 4: 1}[width]
    return struct.pack(_FMT, _MAGIC, 1, version, base_version, code, n_tensors, len(body),
                       blake3.blake3(body).digest()) + body


def unpack_container(blob: bytes):
    """-> (version, base_version, width, n_tensors, body); raises ValueError if the
    magic, format version, length or hash does not match."""
    if len(blob) < HEADER_BYTES:
        raise ValueError("short container")
    magic, fv, ver, base, code, nt, blen, h = struct.unpack_from(_FMT, blob, 0)
    if magic != _MAGIC or fv != 1 or code not in (0, 1):
        raise ValueError("not an SPDC v1 container")
    body = bytes(blob[HEADER_BYTES:])
    if len(body) != blen or blake3.blake3(body).digest() != h:
        raise ValueError("body length or hash mismatch")
    return ver, base, 2 if code == 0 else 4, nt, body
