"""Closed-form payload model (test infrastructure only).

SPEC.md:499-503 (harness › payload_model): expected bytes = nnz x (width +
E[varint bytes per gap]) + per-tensor headers.  For uniformly random change
positions (each lane changes independently with probability rho, the
Bernoulli workload of DESIGN.md §5) the gaps between consecutive changed lanes
are geometric, P(g >= m) = (1 - rho)^(m - 1), so

    E[len] = 1 + sum_{t = 7, 14, ..., 63} P(g >= 2^t)
           = 1 + sum_t (1 - rho)^(2^t - 1)

(len(g) = 1 + #{t : g >= 2^t}).  This is a derivation from
the LEB128 definition and the geometric law, independent of the codec code, so
it pins the oracle's varint lengths statistically (tests/test_oracle_payload.py).
"""

import math

HEADER_FIXED = 27  # u16 + 3 x u64 + u8


def expected_varint_len(rho: float) -> float:
    """E[LEB128 bytes per gap] for Bernoulli(rho) positions."""
    if rho <= 0.0:
        return float("nan")
    q = 1.0 - rho
    return 1.0 + sum(q ** ((1 << t) - 1) for t in range(7, 64, 7))


def expected_record_bytes(n: int, rho: float, width: int, name_len: int) -> float:
    """Header + E[nnz] x (width + E[len]); E[nnz] = rho n."""
    return HEADER_FIXED + name_len + rho * n * (width + expected_varint_len(rho))


def naive_index_width(n: int) -> int:
    """PAPER.md:387 'int32 or int64 (depending on tensor size)': int32 iff the
    largest index n - 1 fits a signed 32-bit integer (reading R6)."""
    return 4 if n - 1 <= 2**31 - 1 else 8


def naive_bytes(nnz: int, n: int, width: int) -> int:
    """Fixed-width (index, value) encoding of PAPER.md:387."""
    return nnz * (naive_index_width(n) + width)


def payload_ratio(full_bytes: int, body_bytes: int) -> float:
    return full_bytes / body_bytes if body_bytes else math.inf
