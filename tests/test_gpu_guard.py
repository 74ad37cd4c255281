"""Guard-band tests (stand-in for compute-sanitizer's memcheck, which is closed on this GPU
pool): every buffer a kernel writes is a view into a larger buffer whose surrounding bytes
hold a canary pattern; after extract / apply / merge / assemble / container header the
canaries must be intact and the results equal to the oracle's.  Also a seeded fuzz of
corrupted bodies: the GPU accepts exactly the bodies the oracle accepts (with the oracle's
result), and rejected bodies leave every target (and its guard bands) bitwise untouched
(SPEC.md:109 all-or-nothing).  A mutation can create several faults at once, so only the
accept / reject verdict is compared (reading R16: the kinds agree on single-fault bodies,
tests/test_gpu_parity.py::test_corruption_suite)."""

import numpy as np
import pytest
import torch

import oracle
from gpu_helpers import assert_body_equal, oracle_extract, to_np
from workload import TensorSpec, generate_pair

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)
G = 4096  # guard bytes on each side
CANARY = 0xA7


@pytest.fixture(scope="module")
def sd():
    import __graft_entry__ as entry
    entry.build()
    import paper_2602_11456_b200 as m
    torch.cuda.set_device(DEV)
    return m


def _guarded(nbytes, shift=0):
    """(whole buffer, the n-byte view at offset G + shift) with canary bytes around it."""
    whole = torch.full((2 * G + nbytes + 16,), CANARY, dtype=torch.uint8, device=DEV)
    return whole, whole[G + shift:G + shift + nbytes]


def _intact(whole, lo, hi):
    w = whole.cpu().numpy()
    return bool((w[:lo] == CANARY).all() and (w[hi:] == CANARY).all())


def _tensors(sizes, rho, seed):
    out = []
    for k, n in enumerate(sizes):
        spec = TensorSpec(f"g{k}.weight", (n,), "matrix")
        o, w = generate_pair(spec, k, seed, rho=rho, device=DEV)
        out.append((spec.name, o, w))
    return out


@pytest.mark.parametrize("shift", [0, 1, 3, 7])
@pytest.mark.parametrize("rho", [0.001, 0.01, 0.3])
def test_extract_writes_only_the_body(sd, shift, rho):
    tensors = _tensors([16_384 * 3 + 5, 1, 0, 100_003, 16_384], rho, seed=int(rho * 1000) + shift)
    want, table = oracle_extract(tensors)
    ctx = sd.DeltaContext(DEV)
    whole, out = _guarded(len(want), shift)
    body, _ = ctx.delta_extract(tensors, out=out)
    torch.cuda.synchronize()
    assert body.numel() == len(want)
    assert_body_equal(body, want)
    assert _intact(whole, G + shift, G + shift + len(want))
    # the async path with an exact-capacity buffer, size on the device
    whole2, out2 = _guarded(len(want), shift)
    size = torch.zeros(1, dtype=torch.int64, device=DEV)
    ctx.delta_extract_async(tensors, out2, size)
    assert ctx.extract_wait() == len(want)
    assert_body_equal(out2, want)
    assert _intact(whole2, G + shift, G + shift + len(want))
    ctx.close()


@pytest.mark.parametrize("rho", [0.001, 0.01, 0.3, 1.0])
def test_apply_writes_only_the_targets(sd, rho):
    tensors = _tensors([16_384 * 2 + 3, 7, 0, 250_001], rho, seed=int(rho * 100) + 3)
    body_b, _ = oracle_extract(tensors)
    body = torch.frombuffer(bytearray(body_b), dtype=torch.uint8).to(DEV)
    ctx = sd.DeltaContext(DEV)
    wholes, targets = [], []
    for name, o, _ in tensors:
        whole, view = _guarded(o.numel() * 2, 0)
        view.copy_(o.view(torch.uint8).reshape(-1))
        wholes.append(whole)
        targets.append((name, view.view(torch.bfloat16)))
    ctx.delta_apply(targets, body)
    torch.cuda.synchronize()
    for (name, t), (_, _, w), whole in zip(targets, tensors, wholes):
        assert torch.equal(t.view(torch.int16), w.view(torch.int16))
        assert _intact(whole, G, G + 2 * w.numel())
    ctx.close()


def test_merge_and_container_write_only_their_outputs(sd):
    rng = np.random.default_rng(9)
    v0 = rng.integers(0, 65536, 300_007, dtype=np.uint64).astype(np.uint16)
    v1 = v0.copy()
    v1[rng.random(v0.size) < 0.02] ^= 3
    v2 = v1.copy()
    v2[rng.random(v0.size) < 0.02] ^= 5
    a, _ = oracle.codec.extract([("m", [v0], [v1])])
    b, _ = oracle.codec.extract([("m", [v1], [v2])])
    want = oracle.codec.merge(a, b, 2)
    ctx = sd.DeltaContext(DEV)
    ta = torch.frombuffer(bytearray(a), dtype=torch.uint8).to(DEV)
    tb = torch.frombuffer(bytearray(b), dtype=torch.uint8).to(DEV)
    whole, out = _guarded(len(a) + len(b), 1)
    merged = ctx.delta_merge(ta, tb, 1, width=2, out=out)
    torch.cuda.synchronize()
    assert_body_equal(merged, want)
    assert _intact(whole, G + 1, G + 1 + len(want))
    # the SPDC header writes exactly 67 bytes
    hwhole, hview = _guarded(sd.container.HEADER_BYTES, 3)
    ctx.container_header(merged, 2, 1, 2, 1, hview)
    torch.cuda.synchronize()
    assert hview.cpu().numpy().tobytes() == oracle.container.pack(want, 2, 1, 2, 1)[:sd.container.HEADER_BYTES]
    assert _intact(hwhole, G + 3, G + 3 + sd.container.HEADER_BYTES)
    ctx.close()


def _mutate(body, rng):
    b = bytearray(body)
    kind = rng.integers(0, 4)
    if kind == 0:  # flip a byte
        i = int(rng.integers(0, len(b)))
        b[i] ^= int(rng.integers(1, 256))
    elif kind == 1:  # truncate
        b = b[:int(rng.integers(0, len(b)))]
    elif kind == 2:  # insert a byte
        i = int(rng.integers(0, len(b) + 1))
        b[i:i] = bytes([int(rng.integers(0, 256))])
    else:  # set a continuation bit somewhere
        i = int(rng.integers(0, len(b)))
        b[i] |= 0x80
    return bytes(b)


def test_fuzzed_bodies_all_or_nothing(sd):
    """120 seeded single mutations of a valid 3-record body: the GPU accepts exactly when the
    oracle does (and then produces the oracle's lanes); on rejection the targets and their
    guard bands are untouched."""
    rng = np.random.default_rng(2024)
    olds = [rng.integers(0, 65536, n, dtype=np.uint64).astype(np.uint16) for n in (5000, 300, 40_000)]
    news = [o.copy() for o in olds]
    for nw in news:
        idx = rng.choice(nw.size, size=max(1, nw.size // 20), replace=False)
        nw[idx] ^= 1
    names = ["f.a", "f.b", "f.c"]
    body, _ = oracle.codec.extract([(n, [o], [w]) for n, o, w in zip(names, olds, news)])
    ctx = sd.DeltaContext(DEV)
    accepted = rejected = 0
    for trial in range(120):
        bad = _mutate(body, rng)
        try:
            ref = oracle.codec.apply([(n, o.copy()) for n, o in zip(names, olds)], bad, 2)
            ref_kind = None
        except oracle.DeltaError as e:
            ref, ref_kind = None, e.kind
        wholes, targets = [], []
        for n, o in zip(names, olds):
            whole, view = _guarded(o.size * 2, 0)
            view.copy_(torch.from_numpy(o.view(np.int16).copy()).to(DEV).view(torch.uint8))
            wholes.append(whole)
            targets.append((n, view.view(torch.bfloat16)))
        tbody = torch.frombuffer(bytearray(bad) or bytearray(1), dtype=torch.uint8).to(DEV)[:len(bad)]
        try:
            ctx.delta_apply(targets, tbody)
            kind = None
        except sd.DeltaError as e:
            kind = e.kind or "other"
        torch.cuda.synchronize()
        for (n, t), o, whole in zip(targets, olds, wholes):
            assert _intact(whole, G, G + 2 * o.size), trial
        if ref_kind is None:
            assert kind is None, (trial, kind)
            for (_, t), r in zip(targets, ref):
                assert np.array_equal(to_np(t), r), trial
            accepted += 1
        else:
            assert kind is not None, (trial, ref_kind)
            for (_, t), o in zip(targets, olds):
                assert np.array_equal(to_np(t), o), trial
            rejected += 1
    assert rejected > 60
    ctx.close()


def _dense_lanes(n, rho, pattern, width, rng):
    """old / new lane arrays with a `pattern` change set: "uniform" (each lane with
    probability rho), "runs" (runs of 1-64 changed lanes, rho of the lanes), "late" (the
    first 3000 lanes unchanged, then uniform)."""
    dt = np.uint16 if width == 2 else np.uint32
    old = rng.integers(0, 1 << (8 * width), n, dtype=np.uint64).astype(dt)
    if pattern == "runs":
        m = np.zeros(n, bool)
        p = 0
        while p < n:
            run = int(rng.integers(1, 65))
            if rng.random() < rho:
                m[p:p + run] = True
            p += run
    else:
        m = rng.random(n) < rho
        if pattern == "late":
            m[:3000] = False
    flip = rng.integers(1, 1 << (8 * width), n, dtype=np.uint64).astype(dt)
    new = np.where(m, old ^ flip, old).astype(dt)
    if width == 2:  # keep additive arithmetic away from NaN patterns (bf16 0x7F80+ exponents)
        old &= 0xBFFF
        new &= 0xBFFF
    else:
        old &= 0xBFFFFFFF
        new &= 0xBFFFFFFF
    return old, new


@pytest.mark.parametrize("width", [2, 4])
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("shift", [0, 1, 3, 7])
def test_dense_scatter_unaligned_targets(sd, width, mode, shift):
    """A4's dense-chunk path (whole 16-byte vectors rewritten inside a chunk's window, the
    window's edge vectors lane by lane): targets at every lane alignment, densities from
    the path's threshold (>= 256 entries, gap sum < 4 per entry) to every lane, runs and a
    late first change; replace and additive records; lanes equal the oracle's apply and
    the bytes around every target stay untouched."""
    rng = np.random.default_rng(100 * width + 10 * mode + shift)
    cases = [(50_000, 0.26, "uniform"), (200_003, 0.5, "uniform"), (70_001, 0.95, "uniform"),
             (33_333, 1.0, "uniform"), (120_000, 0.5, "runs"), (60_000, 0.6, "late"), (9, 1.0, "uniform"),
             (300, 1.0, "uniform")]
    tensors, np_pairs = [], []
    for k, (n, rho, pat) in enumerate(cases):
        o, w = _dense_lanes(n, rho, pat, width, rng)
        np_pairs.append((f"d{k}.weight", o, w))
    body_b, _ = oracle.codec.extract([(nm, [o], [w]) for nm, o, w in np_pairs], mode=mode)
    want = oracle.codec.apply([(nm, o) for nm, o, _ in np_pairs], body_b, width)
    body = torch.frombuffer(bytearray(body_b), dtype=torch.uint8).to(DEV)
    tdt = torch.bfloat16 if width == 2 else torch.float32
    ctx = sd.DeltaContext(DEV)
    wholes, targets = [], []
    for nm, o, _ in np_pairs:
        nb = o.size * width
        whole, view = _guarded(nb, shift * width)
        view.copy_(torch.from_numpy(o.view(np.uint8).copy()).to(DEV))
        wholes.append(whole)
        targets.append((nm, view.view(tdt)))
    ctx.delta_apply(targets, body)
    torch.cuda.synchronize()
    for (nm, t), exp, whole in zip(targets, want, wholes):
        got = t.view(torch.int16 if width == 2 else torch.int32).cpu().numpy().view(exp.dtype)
        assert np.array_equal(got, exp), f"{nm}: {np.flatnonzero(got != exp)[:10]}"
        assert _intact(whole, G + shift * width, G + shift * width + exp.size * width)
    ctx.close()
