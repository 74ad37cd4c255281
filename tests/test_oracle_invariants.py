"""Invariants and closed forms that pin the oracle (no GPU).

SPEC.md:126-132 (losslessness, determinism, strictly increasing indices,
index compression bound), SPEC.md:532-535 (acceptance 1, 3, 4), the closed
form payload model (oracle.payload) and the O7 size
formula record_bytes = 27 + name_len + idx_len + w * nnz.
"""

import numpy as np
import pytest
import torch

from oracle import codec, payload
from workload import TensorSpec, generate_pair


def _np_lanes(t):
    return t.view(torch.int16 if t.element_size() == 2 else torch.int32).numpy().view(
        np.uint16 if t.element_size() == 2 else np.uint32)


def test_roundtrip_randomized_acceptance1():
    # randomized (W, W') pairs, N in 1e3..1e6, rho in {0.001,0.01,0.03},
    # mixed clustered/uniform positions, zero tolerance.
    rng = np.random.default_rng(7)
    for case in range(120):
        n = int(10 ** rng.uniform(3, 6))
        rho = float(rng.choice([0.001, 0.01, 0.03]))
        pattern = "rowblock" if case % 3 == 0 else "uniform"
        cols = int(rng.choice([64, 128, 1000]))
        rows = max(1, n // cols)
        spec = TensorSpec(f"t{case}", (rows, cols), "matrix")
        values = "bits" if case % 4 == 0 else "weights"
        dtype = torch.float32 if case % 5 == 0 else torch.bfloat16
        old, new = generate_pair(spec, case, 11, rho=rho, pattern=pattern, values=values, dtype=dtype)
        o, w = _np_lanes(old), _np_lanes(new)
        body, table = codec.extract([(spec.name, [o], [w])])
        width = o.dtype.itemsize
        got = codec.apply([(spec.name, o)], body, width)[0]
        assert np.array_equal(got, w)
        # idempotent re-apply (replace mode, R14)
        assert np.array_equal(codec.apply([(spec.name, got)], body, width)[0], w)
        # deterministic re-serialization
        assert codec.extract([(spec.name, [o], [w])])[0] == body
        # sum nnz == number of differing lanes; O7 size formula
        nnz = int(np.count_nonzero(o != w))
        r = table[0]
        assert r[2] == nnz
        assert r[6] == 27 + len(spec.name) + r[4] + width * nnz == len(body)


@pytest.mark.parametrize("rho", [0.001, 0.01, 0.1])
def test_index_bytes_match_closed_form(rho):
    # SPEC.md:534 (acceptance 3): at rho = 1% uniform, mean index bytes/entry < 2 and
    # within +-5% of the payload model; we hold it to +-1% at N = 2e7.
    n = 20_000_000
    spec = TensorSpec("x", (n,), "matrix")
    old, new = generate_pair(spec, 0, 3, rho=rho, pattern="uniform")
    o, w = _np_lanes(old), _np_lanes(new)
    idx = codec.changed_indices(o, w)
    g = codec.gaps(idx)
    mean_len = codec.encode_gaps(g).size / g.size
    assert mean_len == pytest.approx(payload.expected_varint_len(rho), rel=0.01)
    if rho == 0.01:
        assert mean_len < 2.0
        assert payload.expected_varint_len(0.01) == pytest.approx(1.2790, abs=1e-4)


def test_payload_ratio_and_naive_ratio():
    # SPEC.md:535 (acceptance 4): delta payload / full payload <= 2.5 rho at rho = 1%,
    # and within 10% of the analytic model; naive int32 / varint in [1.4, 2.1].
    n = 16_777_216
    spec = TensorSpec("model.layers.0.self_attn.o_proj.weight", (4096, 4096), "matrix")
    old, new = generate_pair(spec, 0, 0, rho=0.01, pattern="exact")
    o, w = _np_lanes(old), _np_lanes(new)
    body, table = codec.extract([(spec.name, [o], [w])])
    full = 2 * n
    assert len(body) / full <= 2.5 * 0.01
    model = payload.expected_record_bytes(n, 0.01, 2, len(spec.name))
    assert len(body) == pytest.approx(model, rel=0.10)
    nnz = table[0][2]
    assert nnz == round(0.01 * n) == 167_772
    naive = payload.naive_bytes(nnz, n, 2)
    assert 1.4 <= naive / (len(body) - 27 - len(spec.name)) <= 2.1


def test_strictly_increasing_decoded():
    rng = np.random.default_rng(5)
    o = rng.integers(0, 2**16, 100000, dtype=np.uint16)
    w = o.copy()
    w[rng.random(o.size) < 0.05] ^= 1
    body, _ = codec.extract([("x", [o], [w])])
    (_, _, idx, _, _), = codec.parse(body, 2)
    assert np.all(idx[1:] > idx[:-1])
    assert np.array_equal(idx, np.flatnonzero(o != w).astype(np.uint64))
