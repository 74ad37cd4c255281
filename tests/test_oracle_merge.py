"""Pins for the oracle's delta merge (no GPU).  DESIGN.md reading R19: merging D_a
(v-1 -> v) with D_b (v -> v+1) gives, per tensor, the union of the index sets with
D_b's value wherever D_b has the index (PAPER.md:355 laggard catch-up; SPEC.md:476
leaves merging open).

Against: hand-derived merged records (tests/golden/merge_w_bf16.txt), the composition
identity apply(merge(a, b), X) == apply(b, apply(a, X)) for ARBITRARY bases X (not only
the version the deltas were extracted from), the index-set identity idx(merge) =
idx(a) U idx(b), brute force vs numpy, both index codecs, and the rejection kinds.
"""

import numpy as np
import pytest

from conftest import golden_lines, hexbytes
from oracle import DeltaError, brute, codec


def _kv():
    d = {}
    for ln in golden_lines("merge_w_bf16.txt"):
        k, _, v = ln.partition(" ")
        d[k] = v
    return d


def _lanes(s):
    return [int(t, 16) for t in s.split()]


@pytest.mark.parametrize("pre,key", [("w", "merged"), ("v", "merged2")])
def test_merge_golden(pre, key):
    g = _kv()
    x0, x1, x2 = (_lanes(g[f"{pre}{i}"]) for i in range(3))
    a, _ = brute.extract([("w", [x0], [x1])], 2)
    b, _ = brute.extract([("w", [x1], [x2])], 2)
    want = hexbytes(g[key])
    assert brute.merge(a, b, 2) == want
    assert codec.merge(a, b, 2) == want
    assert brute.apply([("w", x0)], want, 2) == [x2]


def _random_versions(rng, width, sizes, rho):
    dt = np.uint16 if width == 2 else np.uint32
    vs = []
    base = [rng.integers(0, 2**(8 * width), n, dtype=np.uint64).astype(dt) for n in sizes]
    vs.append(base)
    for _ in range(2):
        nxt = []
        for t in vs[-1]:
            u = t.copy()
            m = rng.random(t.size) < rho
            u[m] = rng.integers(0, 2**(8 * width), int(m.sum()), dtype=np.uint64).astype(dt)
            nxt.append(u)
        vs.append(nxt)
    return vs


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("index_codec", ["leb128", "fixed"])
def test_merge_composition(seed, index_codec):
    rng = np.random.default_rng(500 + seed)
    width = 2 if seed % 2 == 0 else 4
    sizes = [int(rng.integers(0, 300)) for _ in range(3)] + [0, 1]
    names = [f"t{k}" for k in range(len(sizes))]
    v0, v1, v2 = _random_versions(rng, width, sizes, rho=[0.02, 0.3, 0.7][seed % 3])
    a, _ = codec.extract([(n, [x], [y]) for n, x, y in zip(names, v0, v1)], index_codec=index_codec)
    b, _ = codec.extract([(n, [x], [y]) for n, x, y in zip(names, v1, v2)], index_codec=index_codec)
    m = codec.merge(a, b, width, index_codec)
    assert m == brute.merge(a, b, width, index_codec)
    # apply(m, v0) == v2, and the composition identity on an arbitrary base X
    got = codec.apply(list(zip(names, v0)), m, width, index_codec=index_codec)
    assert all(np.array_equal(g, w) for g, w in zip(got, v2))
    xs = _random_versions(rng, width, sizes, 0.0)[0]
    lhs = codec.apply(list(zip(names, xs)), m, width, index_codec=index_codec)
    mid = codec.apply(list(zip(names, xs)), a, width, index_codec=index_codec)
    rhs = codec.apply(list(zip(names, mid)), b, width, index_codec=index_codec)
    assert all(np.array_equal(p, q) for p, q in zip(lhs, rhs))
    # index sets: union of the two
    for (_, _, im, _, _), (_, _, ia, _, _), (_, _, ib, _, _) in zip(
            codec.parse(m, width, index_codec), codec.parse(a, width, index_codec), codec.parse(b, width, index_codec)):
        assert set(im.tolist()) == set(ia.tolist()) | set(ib.tolist())


def test_merge_rejects():
    a, _ = codec.extract([("x", [np.arange(5, dtype=np.uint16)], [np.arange(5, dtype=np.uint16) + 1])])
    b, _ = codec.extract([("y", [np.arange(5, dtype=np.uint16)], [np.arange(5, dtype=np.uint16) + 1])])
    c, _ = codec.extract([("x", [np.arange(6, dtype=np.uint16)], [np.arange(6, dtype=np.uint16) + 1])])
    add, _ = codec.extract([("x", [np.arange(5, dtype=np.uint16)], [np.arange(5, dtype=np.uint16) + 1])],
                           mode=codec.MODE_ADDITIVE)
    for mod, x, y, kind in ((codec, a, b, "name"), (codec, a, c, "numel"), (codec, a, a + a, "layout"),
                            (codec, a, add, "mode"), (brute, a, b, "name"), (brute, a, add, "mode")):
        with pytest.raises(DeltaError) as e:
            mod.merge(x, y, 2)
        assert e.value.kind == kind
