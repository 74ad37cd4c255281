"""Unsigned LEB128 of a single integer, pure Python (test infrastructure only).

PAPER.md:389-391 (§5.1 "Sparse encoding"): "encodes the delta sequence using
unsigned LEB128, a variable-length integer representation in which the most
significant bit of each byte indicates continuation. Differences smaller than
128 therefore occupy a single byte ... the value 198 is encoded as two bytes
(C6 01) ... 70 + (1 << 7) = 198".

SPEC.md:65-84 (codec › varint_encode / varint_decode): little-endian base-128
groups, high bit = continuation, minimal length; decode rejects a truncated
stream, an overlong (non-minimal) encoding and a value exceeding 64 bits.
"""

from .errors import DeltaError

U64_MAX = (1 << 64) - 1


def encode(value: int) -> bytes:
    """7-bit groups, least significant first; every byte but the
    last has its high bit set.  Minimal by construction (stops as soon as the
    remaining value fits in 7 bits)."""
    if value < 0 or value > U64_MAX:
        raise ValueError("LEB128 value must fit in 64 unsigned bits (SPEC.md:67)")
    out = bytearray()
    while value >= 0x80:
        out.append((value & 0x7F) | 0x80)
        value >>= 7
    out.append(value)
    return bytes(out)


def decode(buf: bytes, pos: int = 0) -> tuple[int, int]:
    """returns (value, new position).

    Errors:
      * ``truncated`` — the buffer ends while the continuation bit is set;
      * ``overflow``  — more than 64 bits of payload (an 11th byte, or a 10th
        byte carrying more than bit 63);
      * ``overlong``  — a multi-byte encoding whose last byte is 0x00 (its
        value would fit in fewer bytes, so the encoding is not minimal).
    """
    value = 0
    shift = 0
    start = pos
    while True:
        if pos >= len(buf):
            raise DeltaError("truncated", f"varint starting at byte {start}")
        b = buf[pos]
        pos += 1
        nbytes = pos - start
        if nbytes > 10:
            raise DeltaError("overflow", f"varint at byte {start} longer than 10 bytes")
        payload = b & 0x7F
        if nbytes == 10 and payload > 1:
            raise DeltaError("overflow", f"varint at byte {start} exceeds 64 bits")
        value |= payload << shift
        shift += 7
        if b & 0x80 == 0:
            if nbytes > 1 and b == 0:
                raise DeltaError("overlong", f"varint at byte {start} is not minimal")
            return value, pos


def length(value: int) -> int:
    """Number of bytes ``encode(value)`` produces: 1 + #{t in 7,14,...,63 : value >= 2^t}."""
    n = 1
    while value >= 0x80:
        value >>= 7
        n += 1
    return n
