"""The sparse-delta codec in plain vectorised numpy (test infrastructure only).

Same definitions as ``oracle.brute`` (
SPEC.md:86-149), written with numpy primitives so that M1..M5 tensors (up to
7.8e8 lanes) finish in seconds.  The library primitives used as steps are
``flatnonzero`` (the change set), ``diff`` (gaps), ``cumsum`` (byte offsets /
absolute indices) and fancy indexing (gather of values, scatter on apply).
Nothing is blocked, fused or reordered beyond the definition.  Checked
against ``oracle.brute`` on random tiny inputs (tests/test_oracle_brute_vs_numpy.py).

Lanes are unsigned integer arrays: ``uint16`` for 16-bit element types
(bf16/fp16), ``uint32`` for 32-bit (fp32) — SPEC.md:33, reading R2.
"""

import struct

import numpy as np

from .errors import DeltaError

HEADER_FIXED = 27  # u16 name_len + u64 N + u64 nnz + u64 idx_len + u8 mode
_LANE = {2: np.dtype("<u2"), 4: np.dtype("<u4")}


def lanes(a: np.ndarray) -> np.ndarray:
    """View any 2- or 4-byte array as flat unsigned lanes (bitwise identity)."""
    a = np.ascontiguousarray(a).reshape(-1)
    return a.view(_LANE[a.dtype.itemsize])


def fuse(spans) -> np.ndarray:
    """O1: concatenate spans in fusion order."""
    if len(spans) == 1:
        return lanes(spans[0])
    return np.concatenate([lanes(s) for s in spans])


def changed_indices(old: np.ndarray, new: np.ndarray) -> np.ndarray:
    """O2: ascending flat positions where the lanes differ as integers."""
    if old.shape != new.shape or old.dtype != new.dtype:
        raise DeltaError("shape", "old and new differ in element count or width")
    return np.flatnonzero(old != new).astype(np.uint64)


def gaps(idx: np.ndarray) -> np.ndarray:
    """O3: first index as-is, then differences."""
    return np.diff(idx, prepend=np.uint64(0)).astype(np.uint64)


def varint_lengths(g: np.ndarray) -> np.ndarray:
    """len(g) = 1 + [g >= 2^7] + [g >= 2^14] + ... + [g >= 2^63]."""
    n = np.ones(g.shape, dtype=np.int64)
    for t in range(7, 64, 7):
        n += (g >= np.uint64(1 << t))
    return n


def encode_gaps(g: np.ndarray) -> np.ndarray:
    """O4: LEB128 of every gap, concatenated.
    Byte j of a varint carries bits 7j..7j+6; all but its last byte have the
    high (continuation) bit set."""
    g = g.astype(np.uint64)
    n = varint_lengths(g)
    off = np.cumsum(n) - n
    out = np.empty(int(n.sum()), dtype=np.uint8)
    for j in range(10):
        m = n > j
        payload = ((g[m] >> np.uint64(7 * j)) & np.uint64(0x7F)).astype(np.uint8)
        cont = (n[m] > j + 1).astype(np.uint8) << np.uint8(7)
        out[off[m] + j] = payload | cont
    return out


def decode_gaps(stream: np.ndarray) -> np.ndarray:
    """Inverse of encode_gaps with SPEC.md:80's checks: truncated (stream ends
    on a continuation byte), overflow (> 10 bytes, or a 10th byte > 0x01),
    overlong (a multi-byte varint whose last byte is 0x00)."""
    stream = np.asarray(stream, dtype=np.uint8)
    if stream.size == 0:
        return np.zeros(0, dtype=np.uint64)
    term = np.flatnonzero((stream & 0x80) == 0)
    if term.size == 0 or term[-1] != stream.size - 1:
        raise DeltaError("truncated", "index stream ends inside a varint")
    starts = np.concatenate(([0], term[:-1] + 1))
    n = term - starts + 1
    if (n > 10).any():
        raise DeltaError("overflow", "varint longer than 10 bytes")
    if ((n == 10) & (stream[term] > 1)).any():
        raise DeltaError("overflow", "varint exceeds 64 bits")
    if ((n > 1) & (stream[term] == 0)).any():
        raise DeltaError("overlong", "non-minimal varint")
    g = np.zeros(term.size, dtype=np.uint64)
    for j in range(10):
        m = n > j
        g[m] |= (stream[starts[m] + j] & np.uint8(0x7F)).astype(np.uint64) << np.uint64(7 * j)
    return g


# ---- naive fixed-width index encoding (reading R18): the
# index stream is the absolute indices as little-endian u32 if N - 1 <= 2^31 - 1, else u64.
def fixed_index_width(n: int) -> int:
    return 4 if n - 1 <= 2**31 - 1 else 8


def encode_fixed(idx: np.ndarray, n: int) -> np.ndarray:
    dt = np.dtype("<u4") if fixed_index_width(n) == 4 else np.dtype("<u8")
    return idx.astype(dt).view(np.uint8)


def decode_fixed(stream: np.ndarray, n: int) -> np.ndarray:
    """Inverse of encode_fixed; strictly increasing is checked by the caller (parse)."""
    iw = fixed_index_width(n)
    stream = np.ascontiguousarray(stream, dtype=np.uint8)
    if stream.size % iw:
        raise DeltaError("truncated", f"fixed-width index stream of {stream.size} bytes, width {iw}")
    return stream.view("<u4" if iw == 4 else "<u8").astype(np.uint64)


# ---- additive mode ("the arithmetic difference when mode=additive";
# scatter-ADD on apply).  Lanes are read as bf16 (16-bit) or fp32 (32-bit);
# the difference and the sum are taken in fp32 and rounded to the lane type with
# round-to-nearest-even; a NaN result becomes the canonical quiet NaN (R17).
MODE_REPLACE, MODE_ADDITIVE = 0, 1


def bf16_to_f32(lanes16: np.ndarray) -> np.ndarray:
    """bf16 bit patterns -> float32 (exact: the bf16 bits are the top half)."""
    return (lanes16.astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns, round to nearest, ties to even; NaN -> 0x7FC0."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)
    return np.where(np.isnan(x), np.uint16(0x7FC0), r)


def lane_sub(new: np.ndarray, old: np.ndarray) -> np.ndarray:
    """Additive value: new - old in the lane's float type (fp32 arithmetic)."""
    with np.errstate(all="ignore"):  # Inf - Inf, overflow: IEEE results are intended
        if new.dtype.itemsize == 2:
            return f32_to_bf16_rne(bf16_to_f32(new) - bf16_to_f32(old))
        return _canon_f32(new.view(np.float32) - old.view(np.float32))


def _canon_f32(d: np.ndarray) -> np.ndarray:
    bits = d.astype(np.float32).view(np.uint32)
    return np.where(np.isnan(d), np.uint32(0x7FC00000), bits)


def lane_add(w: np.ndarray, val: np.ndarray) -> np.ndarray:
    """Additive apply: w + val in the lane's float type (fp32 arithmetic)."""
    with np.errstate(all="ignore"):
        if w.dtype.itemsize == 2:
            return f32_to_bf16_rne(bf16_to_f32(w) + bf16_to_f32(val))
        return _canon_f32(w.view(np.float32) + val.view(np.float32))


def record(name: str, old: np.ndarray, new: np.ndarray, mode: int = MODE_REPLACE,
           index_codec: str = "leb128") -> bytes:
    """O2..O6 for one fused tensor (SPEC.md:148 layout, little-endian).  mode 0: values are
    the new lanes (replace, reading R1); mode 1: the arithmetic differences (additive).
    index_codec "fixed": absolute fixed-width indices (reading R18) instead of O3+O4."""
    nb = name.encode("utf-8")
    if len(nb) > 0xFFFF:
        raise DeltaError("layout", "name longer than the u16 length field")
    idx = changed_indices(old, new)
    stream = encode_gaps(gaps(idx)) if index_codec == "leb128" else encode_fixed(idx, old.size)
    ii = idx.astype(np.int64)
    vals = new[ii] if mode == MODE_REPLACE else lane_sub(new[ii], old[ii])
    vals = vals.astype(new.dtype.newbyteorder("<"), copy=False)
    return b"".join((struct.pack("<H", len(nb)), nb,
                     struct.pack("<QQQ", old.size, idx.size, stream.size),
                     stream.tobytes(), vals.tobytes(), bytes([mode])))


def table_row(record_off: int, rec: bytes) -> tuple:
    """O7: (record_off, N, nnz, idx_off, idx_len, val_off, record_bytes) read
    back from the record's own header."""
    nl = struct.unpack_from("<H", rec, 0)[0]
    n, nnz, ilen = struct.unpack_from("<QQQ", rec, 2 + nl)
    idx_off = record_off + 2 + nl + 24
    return (record_off, n, nnz, idx_off, ilen, idx_off + ilen, len(rec))


def extract(tensors, mode: int = MODE_REPLACE, index_codec: str = "leb128"):
    """tensors: [(name, old_spans, new_spans)] -> (body bytes, table rows).
    Records appear in list order (reading R15), one per tensor even
    when nothing changed (R12)."""
    parts, table, off = [], [], 0
    for name, old_spans, new_spans in tensors:
        if len(old_spans) != len(new_spans):
            raise DeltaError("shape", f"{name!r}: span count differs")
        rec = record(name, fuse(old_spans), fuse(new_spans), mode, index_codec)
        table.append(table_row(off, rec))
        parts.append(rec)
        off += len(rec)
    return b"".join(parts), table


def parse(body, width: int, index_codec: str = "leb128"):
    """Walk and fully validate a body: [(name, N, idx uint64, vals)]."""
    body = memoryview(bytes(body))
    recs, pos = [], 0
    dt = _LANE[width]
    while pos < len(body):
        if pos + 2 > len(body):
            raise DeltaError("layout", "record header runs past the body")
        nl = struct.unpack_from("<H", body, pos)[0]
        if pos + 2 + nl + 24 > len(body):
            raise DeltaError("layout", "record header runs past the body")
        name = bytes(body[pos + 2:pos + 2 + nl]).decode("utf-8")
        n, nnz, ilen = struct.unpack_from("<QQQ", body, pos + 2 + nl)
        p = pos + 2 + nl + 24
        if ilen > len(body) - p or nnz > (len(body) - p - ilen) // width:
            raise DeltaError("layout", f"{name!r}: record runs past the body")
        end = p + ilen + nnz * width + 1
        if end > len(body):
            raise DeltaError("layout", f"{name!r}: record runs past the body")
        stream = np.frombuffer(body[p:p + ilen], dtype=np.uint8)
        if index_codec == "leb128":
            g = decode_gaps(stream)
            if g.size != nnz:
                raise DeltaError("count", f"{name!r}: {g.size} indices decoded, nnz says {nnz}")
            if g.size > 1 and (g[1:] == 0).any():
                raise DeltaError("nonincreasing", f"{name!r}: zero gap")
            idx = np.cumsum(g, dtype=np.uint64)
        else:
            idx = decode_fixed(stream, n)
            if idx.size != nnz:
                raise DeltaError("count", f"{name!r}: {idx.size} indices decoded, nnz says {nnz}")
            if idx.size > 1 and (idx[1:] <= idx[:-1]).any():
                raise DeltaError("nonincreasing", f"{name!r}: indices not strictly increasing")
        if idx.size and ((idx[1:] <= idx[:-1]).any() or idx[-1] >= np.uint64(n)):
            # a wrap of the 64-bit running sum also lands here: such an index
            # is >= 2^64 > N, i.e. out of range.
            raise DeltaError("range", f"{name!r}: index >= element_count {n}")
        vals = np.frombuffer(body[p + ilen:p + ilen + nnz * width], dtype=dt)
        mode = body[end - 1]
        if mode not in (MODE_REPLACE, MODE_ADDITIVE):
            raise DeltaError("mode", f"{name!r}: mode byte {mode}")
        recs.append((name, n, idx, vals, mode))
        pos = end
    return recs


def apply(targets, body, width: int, inplace: bool = False, index_codec: str = "leb128"):
    """O9: targets [(name, lanes)]; validate everything, then
    W[idx] = vals.  Returns the updated lane arrays (copies unless inplace).
    On any DeltaError no target has been modified."""
    recs = parse(body, width, index_codec)
    if len(recs) != len(targets):
        raise DeltaError("layout", f"{len(recs)} records for {len(targets)} targets")
    for (name, n, _, _, _), (tname, w) in zip(recs, targets):
        if name != tname:
            raise DeltaError("name", f"record {name!r} vs target {tname!r}")
        if n != lanes(w).size:
            raise DeltaError("numel", f"{name!r}: N={n} vs target {lanes(w).size}")
    out = []
    for (_, _, idx, vals, mode), (_, w) in zip(recs, targets):
        dst = lanes(w) if inplace else lanes(w).copy()
        ii = idx.astype(np.int64)
        dst[ii] = vals if mode == MODE_REPLACE else lane_add(dst[ii], vals)
        out.append(dst)
    return out


def merge(body_a, body_b, width: int, index_codec: str = "leb128") -> bytes:
    """Merge of two consecutive replace-mode deltas (reading R19; brute.merge):
    per tensor idx = union (numpy union1d), values of body_b where it has the index, else
    body_a's.  apply(merge(a, b)) == apply(b) after apply(a)."""
    ra, rb = parse(body_a, width, index_codec), parse(body_b, width, index_codec)
    if len(ra) != len(rb):
        raise DeltaError("layout", f"{len(ra)} records vs {len(rb)}")
    parts = []
    for (na, n_a, ia, va, ma), (nb, n_b, ib, vb, mb) in zip(ra, rb):
        if na != nb:
            raise DeltaError("name", f"record {na!r} vs {nb!r}")
        if n_a != n_b:
            raise DeltaError("numel", f"{na!r}: N={n_a} vs {n_b}")
        if ma != MODE_REPLACE or mb != MODE_REPLACE:
            raise DeltaError("mode", f"{na!r}: merge needs replace-mode records")
        idx = np.union1d(ia, ib).astype(np.uint64)
        vals = np.empty(idx.size, dtype=_LANE[width])
        vals[np.searchsorted(idx, ia)] = va
        vals[np.searchsorted(idx, ib)] = vb  # the later delta wins
        stream = encode_gaps(gaps(idx)) if index_codec == "leb128" else encode_fixed(idx, n_a)
        nbytes = na.encode("utf-8")
        parts.append(b"".join((struct.pack("<H", len(nbytes)), nbytes,
                               struct.pack("<QQQ", n_a, idx.size, stream.size),
                               stream.tobytes(), vals.astype(_LANE[width], copy=False).tobytes(), b"\x00")))
    return b"".join(parts)


def rho(pairs) -> float:
    """O10, Eq. 1: sum_k ||dW_k||_0 / sum_k |W_k|, with
    bitwise inequality as nonzero (reading R2)."""
    total = sum(lanes(o).size for o, _ in pairs)
    nz = sum(int(np.count_nonzero(lanes(o) != lanes(n))) for o, n in pairs)
    return nz / total if total else 0.0
