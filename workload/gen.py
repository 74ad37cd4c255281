"""Counter-based generator of (old, new) lane pairs, device-agnostic.

Every lane's bits are a pure function of (seed, tensor index k, lane index j),
computed with integer-only torch ops (a 32-bit "lowbias32" mix evaluated in
int64 without overflow) plus one correctly rounded float multiply and cast, so
CPU and CUDA produce identical tensors and a tensor's data do not depend on
which rank generates it (SURVEY.md §8(d) "per-tensor seeds").

Recipe:
  * old, "matrix" tensors: bf16/fp32 of sigma * IH4 / 147.8, IH4 = sum of the
    four bytes of a 32-bit hash minus 510 (Irwin-Hall(4): mean 0, sd 147.8),
    sigma = 0.02 — an integer stand-in for N(0, 0.02) init;
  * old, "norm" tensors: 1 + the same;
  * changed lanes: new = old XOR r, r uniform in [1, 15] (low mantissa bits),
    a small-ulp step that guarantees bitwise inequality;
  * change positions: ``uniform`` Bernoulli(rho) per lane; ``exact`` exactly
    k = round(rho N) positions without replacement (configs[0]); ``rowblock``
    round(rho R) whole rows of a 2-D tensor (1-D tensors fall back to uniform);
  * ``values="bits"``: old lanes are uniformly random bit patterns (NaN, +-0,
    Inf, subnormals all occur) and changed lanes get another random pattern —
    the edge-case set of SPEC.md:465.
No compare, compaction, encoding or scatter happens here.
"""

import torch

M32 = 0xFFFFFFFF
CHUNK = 1 << 25


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for int64 x in [0, 2^32), without int64 overflow."""
    lo, hi = c & 0xFFFF, c >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & M32


def hash32(x: torch.Tensor) -> torch.Tensor:
    """lowbias32 (x in [0, 2^32)) on int64 tensors."""
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    return x ^ (x >> 16)


def hash32_py(x: int) -> int:
    x &= M32
    x ^= x >> 16
    x = (x * 0x7FEB352D) & M32
    x ^= x >> 15
    x = (x * 0x846CA68B) & M32
    return x ^ (x >> 16)


def tensor_key(seed: int, k: int, stream: int) -> int:
    return hash32_py(hash32_py(hash32_py(seed) ^ (k * 0x9E3779B1 & M32)) ^ (stream * 0x85EBCA77 & M32))


def _lane_hash(j: torch.Tensor, key: int) -> torch.Tensor:
    return hash32(hash32((j & M32) ^ key) ^ ((j >> 32) + 0x632BE5AB))


def _old_bits(h: torch.Tensor, kind: str, width: int, values: str) -> torch.Tensor:
    """int64 lane bit patterns of ``old`` from a 32-bit hash."""
    if values == "bits":
        return h & (0xFFFF if width == 2 else M32)
    ih4 = (h & 0xFF) + ((h >> 8) & 0xFF) + ((h >> 16) & 0xFF) + ((h >> 24) & 0xFF) - 510
    v = ih4.to(torch.float32) * (0.02 / 147.8)
    if kind == "norm":
        v = v + 1.0
    if width == 2:
        return v.to(torch.bfloat16).view(torch.int16).to(torch.int64) & 0xFFFF
    return v.view(torch.int32).to(torch.int64) & M32


def _to_lanes(bits: torch.Tensor, width: int) -> torch.Tensor:
    if width == 2:
        b = torch.where(bits >= 0x8000, bits - 0x10000, bits)
        return b.to(torch.int16)
    b = torch.where(bits >= 0x80000000, bits - 0x100000000, bits)
    return b.to(torch.int32)


def change_positions_exact(n: int, k: int, seed: int, key: int) -> torch.Tensor:
    """k distinct positions in [0, n), uniform (CPU generator, any device after)."""
    g = torch.Generator().manual_seed((seed * 1000003 + key) & ((1 << 63) - 1))
    return torch.randperm(n, generator=g)[:k]


def rowblock_rows(rows: int, rho: float, seed: int, key: int) -> torch.Tensor:
    k = int(round(rho * rows))
    g = torch.Generator().manual_seed((seed * 1000003 + key) & ((1 << 63) - 1))
    return torch.randperm(rows, generator=g)[:k]


def generate_pair(spec, k: int, seed: int, *, rho: float, pattern: str = "uniform",
                  dtype=torch.bfloat16, device="cpu", values: str = "weights",
                  old_out: torch.Tensor = None, new_out: torch.Tensor = None):
    """Fill (or allocate) flat ``old``/``new`` tensors of ``spec.numel`` lanes of
    ``dtype`` (bf16/fp16 -> 16-bit lanes, fp32 -> 32-bit lanes).  Returns
    (old, new) as 1-D tensors of ``dtype``."""
    n = spec.numel
    width = torch.empty(0, dtype=dtype).element_size()
    lane_t = torch.int16 if width == 2 else torch.int32
    if old_out is None:
        old_out = torch.empty(n, dtype=dtype, device=device)
    if new_out is None:
        new_out = torch.empty(n, dtype=dtype, device=device)
    ov, nv = old_out.view(lane_t), new_out.view(lane_t)
    dev = old_out.device
    k_old, k_mask, k_r = (tensor_key(seed, k, s) for s in (1, 2, 3))
    thr = int(round(rho * 2**32))

    if pattern == "exact":
        pos = change_positions_exact(n, int(round(rho * n)), seed, k_mask)
        mask_all = torch.zeros(n, dtype=torch.bool)
        mask_all[pos] = True
        mask_all = mask_all.to(dev)
    elif pattern == "rowblock" and len(spec.shape) == 2:
        rows = rowblock_rows(spec.shape[0], rho, seed, k_mask)
        rowmask = torch.zeros(spec.shape[0], dtype=torch.bool)
        rowmask[rows] = True
        rowmask = rowmask.to(dev)
        cols = spec.shape[1]
    elif pattern not in ("uniform", "rowblock"):
        raise ValueError(f"unknown pattern {pattern!r}")

    for s in range(0, n, CHUNK):
        e = min(n, s + CHUNK)
        j = torch.arange(s, e, dtype=torch.int64, device=dev)
        old_bits = _old_bits(_lane_hash(j, k_old), spec.kind, width, values)
        if pattern == "exact":
            m = mask_all[s:e]
        elif pattern == "rowblock" and len(spec.shape) == 2:
            m = rowmask[j // cols]
        else:
            m = _lane_hash(j, k_mask) < thr
        hr = _lane_hash(j, k_r)
        if values == "bits":
            full = 0xFFFF if width == 2 else M32
            r = 1 + hr % full          # any other pattern
        else:
            r = 1 + hr % 15            # low 4 mantissa bits
        new_bits = torch.where(m, old_bits ^ r, old_bits)
        ov[s:e] = _to_lanes(old_bits, width)
        nv[s:e] = _to_lanes(new_bits, width)
    return old_out, new_out
