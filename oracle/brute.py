"""The sparse-delta codec written per element and per byte in pure Python.

TEST INFRASTRUCTURE ONLY (see oracle/__init__).  For tiny inputs: this is the
definition, read off the paper and the SPEC byte layout, with no vectorisation.
``oracle.codec`` (numpy) is checked against it.

Definitions followed, in order (SURVEY.md §8(c) O1-O10 restates them):
  O1  A logical tensor is the concatenation of its spans in fusion order
      ("stacking split HuggingFace blocks in a fixed order";
      SPEC.md:52-57 FusionMap offsets = prefix sums).  Lanes are unsigned
      integers of width w in {2, 4} bytes ("opaque fixed-width
      byte lanes").
  O2  changed lanes: j with old[j] != new[j] as integers (SPEC.md:136,
      DESIGN.md reading R2), ascending ("stores the non-zeros as
      two 1D arrays, idx and val").
  O3  gaps: first index as-is, then differences.
  O4  LEB128 of every gap, concatenated (oracle.leb128).
  O5  values: the NEW lanes at idx (replace mode, reading R1).
  O6  record = u16 name_len | name | u64 N | u64 nnz | u64 idx_len |
      idx_stream | values | u8 mode(=0), little-endian.
  O7  offset table row per record (north_star "per-tensor offset tables").
  O9  apply: validate every record fully, then W[idx_i] = val_i
      ("validate fully before mutating").
  O10 rho = sum nnz / sum N (Eq. 1).
  F   the naive fixed-width index encoding the paper compares against
      ("a naive int32/64 index encoding"; "two 1D arrays, idx and
      val ... int32 or int64 (depending on tensor size)"): the
      index stream is the nnz absolute indices, each as a little-endian
      unsigned integer of 4 bytes if N - 1 <= 2^31 - 1, else 8 (DESIGN.md
      reading R18); every other byte of the record is as in O6.
  M   merge of two consecutive deltas D_a (v-1 -> v) and D_b (v -> v+1) into one
      (v-1 -> v+1) for a laggard's catch-up ("laggards catch up
      asynchronously"; SPEC.md:476 leaves merging open; reading R19):
      per tensor the union of the two index sets, each value taken from D_b
      where D_b has the index, else from D_a — so applying the merge equals
      applying D_a then D_b.  Replace mode only.
"""

import math
import struct

from . import leb128
from .errors import DeltaError

MODE_REPLACE, MODE_ADDITIVE = 0, 1


def _f32(bits: int) -> float:
    return struct.unpack("<f", struct.pack("<I", bits & 0xFFFFFFFF))[0]


def _f32_bits(x: float) -> int:
    """Round a Python float (f64) to fp32, round-to-nearest-even (struct 'f'); for the
    sum / difference of two fp32 values this equals the fp32 operation (53 >= 2*24 + 2)."""
    if math.isnan(x):
        return 0x7FC00000
    try:
        return struct.unpack("<I", struct.pack("<f", x))[0]
    except OverflowError:  # beyond fp32 range after rounding: +-Inf
        return 0x7F800000 if x > 0 else 0xFF800000


def _bf16_rne(bits32: int) -> int:
    """fp32 bits -> bf16 bits, round to nearest even; NaN -> 0x7FC0 (R17)."""
    if (bits32 & 0x7FFFFFFF) > 0x7F800000:
        return 0x7FC0
    return ((bits32 + 0x7FFF + ((bits32 >> 16) & 1)) >> 16) & 0xFFFF


def lane_op(a: int, b: int, width: int, sign: int) -> int:
    """a + sign * b in the lane's float type: bf16 (width 2) via fp32, or fp32."""
    if width == 2:
        fa, fb = _f32(a << 16), _f32(b << 16)
        return _bf16_rne(_f32_bits(fa + sign * fb))
    return _f32_bits(_f32(a) + sign * _f32(b))

HEADER_FIXED = 2 + 8 + 8 + 8 + 1  # u16 name_len, u64 N, u64 nnz, u64 idx_len, u8 mode


def _u(n: int, nbytes: int) -> bytes:
    """Little-endian unsigned integer of ``nbytes`` bytes, written byte by byte."""
    return bytes((n >> (8 * i)) & 0xFF for i in range(nbytes))


def _read_u(buf: bytes, pos: int, nbytes: int) -> tuple[int, int]:
    if pos + nbytes > len(buf):
        raise DeltaError("layout", f"header field at byte {pos} runs past the body")
    v = 0
    for i in range(nbytes):
        v |= buf[pos + i] << (8 * i)
    return v, pos + nbytes


def fuse(spans: list[list[int]]) -> list[int]:
    """O1: the fused tensor's flat lanes are the spans concatenated in order."""
    out: list[int] = []
    for s in spans:
        out.extend(s)
    return out


def changed_indices(old: list[int], new: list[int]) -> list[int]:
    """O2: ascending j where the lanes differ bitwise."""
    if len(old) != len(new):
        raise DeltaError("shape", "old and new have different element counts")
    return [j for j in range(len(old)) if old[j] != new[j]]


def encode_indices(idx: list[int]) -> bytes:
    """O3+O4: LEB128(idx[0]) then LEB128(idx[i]-idx[i-1])."""
    out = bytearray()
    prev = None
    for x in idx:
        if prev is not None and x <= prev:
            raise DeltaError("nonincreasing", "encode_indices needs strictly increasing input")
        out += leb128.encode(x if prev is None else x - prev)
        prev = x
    return bytes(out)


def decode_indices(stream: bytes) -> list[int]:
    """Inverse of encode_indices with the strict checks of SPEC.md:80 and
    the strictly-increasing invariant: every gap after the
    first must be >= 1."""
    idx: list[int] = []
    pos = 0
    while pos < len(stream):
        g, pos = leb128.decode(stream, pos)
        if idx and g == 0:
            raise DeltaError("nonincreasing", f"zero gap after index {idx[-1]}")
        idx.append(g if not idx else idx[-1] + g)
    return idx


def fixed_index_width(n: int) -> int:
    """F ("int32 or int64 (depending on tensor size)"): 4 bytes iff the
    largest index n - 1 fits a signed 32-bit integer."""
    return 4 if n - 1 <= 2**31 - 1 else 8


def encode_indices_fixed(idx: list[int], n: int) -> bytes:
    """F: each absolute index as a little-endian integer of fixed_index_width(n) bytes."""
    iw = fixed_index_width(n)
    return b"".join(_u(x, iw) for x in idx)


def decode_indices_fixed(stream: bytes, n: int) -> list[int]:
    """Inverse of encode_indices_fixed: the stream must hold a whole number of
    indices, strictly increasing."""
    iw = fixed_index_width(n)
    if len(stream) % iw:
        raise DeltaError("truncated", f"fixed-width index stream of {len(stream)} bytes, width {iw}")
    idx: list[int] = []
    for pos in range(0, len(stream), iw):
        x, _ = _read_u(stream, pos, iw)
        if idx and x <= idx[-1]:
            raise DeltaError("nonincreasing", f"index {x} after {idx[-1]}")
        idx.append(x)
    return idx


def record(name: str, old: list[int], new: list[int], width: int, mode: int = MODE_REPLACE,
           index_codec: str = "leb128") -> bytes:
    """O2..O6 for one fused tensor.  Additive mode: values are new - old.
    index_codec "fixed": the index stream of F instead of O3+O4."""
    nb = name.encode("utf-8")
    if len(nb) > 0xFFFF:
        raise DeltaError("layout", "name longer than the u16 length field (SPEC.md:148)")
    idx = changed_indices(old, new)
    stream = encode_indices(idx) if index_codec == "leb128" else encode_indices_fixed(idx, len(old))
    if mode == MODE_REPLACE:
        vals = b"".join(_u(new[j], width) for j in idx)
    else:
        vals = b"".join(_u(lane_op(new[j], old[j], width, -1), width) for j in idx)
    return (_u(len(nb), 2) + nb + _u(len(old), 8) + _u(len(idx), 8)
            + _u(len(stream), 8) + stream + vals + _u(mode, 1))


def record_from_sparse(name: str, n: int, idx: list[int], vals: list[int], width: int) -> bytes:
    """O3..O6 when the change set is given directly (a tensor too large to hold as a
    Python list, e.g. one with more than 2^32 lanes): idx ascending, vals the new lanes."""
    nb = name.encode("utf-8")
    stream = encode_indices(idx)
    return (_u(len(nb), 2) + nb + _u(n, 8) + _u(len(idx), 8) + _u(len(stream), 8) + stream
            + b"".join(_u(v, width) for v in vals) + _u(0, 1))


def extract(tensors: list[tuple[str, list[list[int]], list[list[int]]]], width: int,
            mode: int = MODE_REPLACE, index_codec: str = "leb128"):
    """Body and offset table for (name, old_spans, new_spans) in list order.

    Table rows: (record_off, N, nnz, idx_off, idx_len, val_off, record_bytes),
    with idx_off = record_off + 2 + name_len + 24 and val_off = idx_off +
    idx_len (O7, from the O6 layout)."""
    body = bytearray()
    table = []
    for name, old_spans, new_spans in tensors:
        if len(old_spans) != len(new_spans) or any(
                len(a) != len(b) for a, b in zip(old_spans, new_spans)):
            raise DeltaError("shape", f"tensor {name!r}: span structure differs")
        old, new = fuse(old_spans), fuse(new_spans)
        rec = record(name, old, new, width, mode, index_codec)
        nl = len(name.encode("utf-8"))
        nnz = sum(1 for j in range(len(old)) if old[j] != new[j])
        idx_off = len(body) + 2 + nl + 24
        idx_len, _ = _read_u(rec, 2 + nl + 16, 8)
        table.append((len(body), len(old), nnz, idx_off, idx_len, idx_off + idx_len, len(rec)))
        body += rec
    return bytes(body), table


def parse(body: bytes, width: int, index_codec: str = "leb128"):
    """Split a body into records [(name, N, idx list, value list, mode)],
    decoding and validating everything."""
    recs = []
    pos = 0
    while pos < len(body):
        nl, pos = _read_u(body, pos, 2)
        if pos + nl > len(body):
            raise DeltaError("layout", "name runs past the body")
        name = body[pos:pos + nl].decode("utf-8", errors="strict")
        pos += nl
        n, pos = _read_u(body, pos, 8)
        nnz, pos = _read_u(body, pos, 8)
        ilen, pos = _read_u(body, pos, 8)
        if pos + ilen > len(body):
            raise DeltaError("layout", f"index stream of {name!r} runs past the body")
        stream = body[pos:pos + ilen]
        idx = decode_indices(stream) if index_codec == "leb128" else decode_indices_fixed(stream, n)
        pos += ilen
        if len(idx) != nnz:
            raise DeltaError("count", f"{name!r}: {len(idx)} indices decoded, nnz says {nnz}")
        if idx and idx[-1] >= n:
            raise DeltaError("range", f"{name!r}: index {idx[-1]} >= element_count {n}")
        vals = []
        for _ in range(nnz):
            v, pos = _read_u(body, pos, width)
            vals.append(v)
        mode, pos = _read_u(body, pos, 1)
        if mode not in (MODE_REPLACE, MODE_ADDITIVE):
            raise DeltaError("mode", f"{name!r}: mode byte {mode} (replace=0, additive=1)")
        recs.append((name, n, idx, vals, mode))
    return recs


def apply(targets: list[tuple[str, list[int]]], body: bytes, width: int,
          index_codec: str = "leb128") -> list[list[int]]:
    """O9: returns new lane lists; raises DeltaError (inputs untouched) if any
    record is malformed or does not match its target (name, element count,
    record count)."""
    recs = parse(body, width, index_codec)
    if len(recs) != len(targets):
        raise DeltaError("layout", f"{len(recs)} records for {len(targets)} targets")
    for (name, n, _, _, _), (tname, lanes) in zip(recs, targets):
        if name != tname:
            raise DeltaError("name", f"record {name!r} vs target {tname!r}")
        if n != len(lanes):
            raise DeltaError("numel", f"{name!r}: record N={n}, target has {len(lanes)}")
    out = []
    for (_, _, idx, vals, mode), (_, lanes) in zip(recs, targets):
        w = list(lanes)
        for j, v in zip(idx, vals):
            w[j] = v if mode == MODE_REPLACE else lane_op(w[j], v, width, +1)
        out.append(w)
    return out


def merge(body_a: bytes, body_b: bytes, width: int, index_codec: str = "leb128") -> bytes:
    """M: the delta equivalent to applying body_a then body_b (replace mode)."""
    ra, rb = parse(body_a, width, index_codec), parse(body_b, width, index_codec)
    if len(ra) != len(rb):
        raise DeltaError("layout", f"{len(ra)} records vs {len(rb)}")
    out = b""
    for (na, n_a, ia, va, ma), (nb, n_b, ib, vb, mb) in zip(ra, rb):
        if na != nb:
            raise DeltaError("name", f"record {na!r} vs {nb!r}")
        if n_a != n_b:
            raise DeltaError("numel", f"{na!r}: N={n_a} vs {n_b}")
        if ma != MODE_REPLACE or mb != MODE_REPLACE:
            raise DeltaError("mode", f"{na!r}: merge needs replace-mode records")
        d = {}
        for j, v in zip(ia, va):
            d[j] = v
        for j, v in zip(ib, vb):  # the later delta wins
            d[j] = v
        idx = sorted(d)
        if index_codec == "leb128":
            out += record_from_sparse(na, n_a, idx, [d[j] for j in idx], width)
        else:
            nbytes = na.encode("utf-8")
            stream = encode_indices_fixed(idx, n_a)
            out += (_u(len(nbytes), 2) + nbytes + _u(n_a, 8) + _u(len(idx), 8) + _u(len(stream), 8) + stream
                    + b"".join(_u(d[j], width) for j in idx) + _u(0, 1))
    return out


def rho(pairs: list[tuple[list[int], list[int]]]) -> float:
    """O10, Eq. 1 with bitwise inequality as 'nonzero'."""
    total = sum(len(o) for o, _ in pairs)
    nz = sum(1 for o, n in pairs for a, b in zip(o, n) if a != b)
    return nz / total if total else 0.0
