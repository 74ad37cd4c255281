"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element, on the same seeded inputs.  Bit-exact for every byte of the packed body, every
offset-table row and every lane of the reconstructed weights (integer views).

Cases: configs[0] (M1), ragged / multi-tile / multi-span / unaligned tensors, full-range
bit patterns (NaN, +-0, Inf, subnormals), gap boundaries of the LEB128 encoding, the
degenerate cases (nothing / everything / first / last lane changed, empty tensors),
workspace regrowth, the two-phase size+extract path, the corruption suite (error kind
equal to the oracle's, targets untouched) and, at full size, Qwen3-8B (configs[2], in
the launch configuration bench.py times) in tests/test_gpu_fullsize.py, every record.
"""

import numpy as np
import pytest
import torch

import oracle
from gpu_helpers import (as_list, assert_body_equal, assert_lanes_equal, fused, lane_view,
                         oracle_extract, to_np)
from workload import TensorSpec, generate_pair, m1_specs, qwen3

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def sd():
    import __graft_entry__ as entry
    entry.build()
    import paper_2602_11456_b200 as m
    torch.cuda.set_device(DEV)
    return m


def _roundtrip(sd, tensors, ctx=None, check_oracle=True):
    """Extract on the GPU, compare with the oracle, apply (with and without the table
    hint) to copies of old, compare with new."""
    ctx = ctx or sd.context()
    body, table = ctx.delta_extract(tensors)
    torch.cuda.synchronize()
    if check_oracle:
        ref_body, ref_table = oracle_extract(tensors)
        assert_body_equal(body, ref_body)
        assert [tuple(r) for r in table] == [tuple(r) for r in ref_table]
    for hint in ("host", "none", "device", "chain"):
        targets = [(n, fused(o).clone()) for n, o, _ in tensors]
        if hint == "chain":  # extract -> apply with size and table on the device, one wait
            out = torch.full((body.numel() + 64,), 0xA5, dtype=torch.uint8, device=DEV)
            size = torch.zeros(1, dtype=torch.int64, device=DEV)
            assert ctx.round_trip(tensors, targets, out, size) == body.numel()
            assert int(size.item()) == body.numel()
            assert torch.equal(out[:body.numel()], body)
        elif hint == "device":  # the table left on the device by a second extract
            dbody, dtab = ctx.delta_extract(tensors, table="device")
            assert torch.equal(dbody, body)
            ctx.delta_apply(targets, dbody, table=dtab)
        else:
            ctx.delta_apply(targets, body, table=table if hint == "host" else None)
        torch.cuda.synchronize()
        for (_, w), (_, _, nw) in zip(targets, tensors):
            assert_lanes_equal(w, fused(nw))
    return body, table


def test_m1_config0(sd):
    spec = m1_specs()[0]
    old, new = generate_pair(spec, 0, 0, rho=0.01, pattern="exact", device=DEV)
    body, table = _roundtrip(sd, [(spec.name, old, new)])
    assert table[0][2] == 167_772
    # idempotent re-apply on new (replace mode, R14)
    w = new.clone()
    sd.delta_apply([(spec.name, w)], body, table=table)
    assert_lanes_equal(w, new)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("rho", [0.0, 0.001, 0.01, 0.3, 1.0])
def test_ragged_bit_patterns(sd, dtype, rho):
    sizes = [1, 7, 8, 9, 1000, 8191, 8192, 16384, 16385, 16384 * 3 + 5, 100_003, 0, 2]
    tensors = []
    for k, n in enumerate(sizes):
        spec = TensorSpec(f"t.{k}.weight", (n,), "matrix")
        o, w = generate_pair(spec, k, 17, rho=rho, dtype=dtype, device=DEV, values="bits")
        tensors.append((spec.name, o, w))
    _roundtrip(sd, tensors)


def test_fused_unaligned_spans(sd):
    # spans are slices of one buffer at odd lane offsets (not 16-byte aligned), including
    # an empty span: exercises the lane-by-lane path and span-local tiling.
    n = 300_001
    spec = TensorSpec("buf", (n,), "matrix")
    o, w = generate_pair(spec, 0, 5, rho=0.02, device=DEV, values="bits")
    cuts = [1, 50_001, 50_001, 50_002, 130_001, 299_999]
    so = [o[a:b] for a, b in zip(cuts[:-1], cuts[1:])]
    sw = [w[a:b] for a, b in zip(cuts[:-1], cuts[1:])]
    tensors = [("model.layers.0.self_attn.qkv_proj.weight", so, sw),
               ("aligned.tail", o[299_999:].clone(), w[299_999:].clone())]
    _roundtrip(sd, tensors)


def _with_changes(n, positions, dtype=torch.bfloat16):
    old = torch.zeros(n, dtype=dtype, device=DEV)
    new = old.clone()
    if positions:
        p = torch.tensor(positions, dtype=torch.int64, device=DEV)
        lane_view(new)[p] = 0x3F80 if dtype == torch.bfloat16 else 0x3F800000
    return old, new


def test_gap_boundaries(sd):
    gaps = [0, 127, 128, 16383, 16384, 2**21 - 1, 2**21, 1, 1, 300]
    pos = list(np.cumsum(gaps))
    n = pos[-1] + 5
    old, new = _with_changes(n, pos)
    body, table = _roundtrip(sd, [("gaps", old, new)])
    # index stream by hand: first index 0 -> 00; 127 -> 7F; 128 -> 80 01; ...
    ref = oracle.brute.encode_indices([int(x) for x in pos])
    s = body[table[0][3]:table[0][3] + table[0][4]].cpu().numpy().tobytes()
    assert s == ref


def test_degenerate_change_sets(sd):
    n = 16384 * 2 + 3
    cases = {"none": [], "first": [0], "last": [n - 1], "first_last": [0, n - 1],
             "all": list(range(n))}
    tensors = []
    for name, p in cases.items():
        o, w = _with_changes(n, p)
        tensors.append((name, o, w))
    body, table = _roundtrip(sd, tensors)
    assert [r[2] for r in table] == [0, 1, 1, 2, n]


def test_many_small_tensors(sd):
    rng = np.random.default_rng(3)
    tensors = []
    for k in range(400):
        n = int(rng.integers(0, 5000))
        spec = TensorSpec(f"layer.{k}", (n,), "norm")
        o, w = generate_pair(spec, k, 2, rho=float(rng.choice([0, 0.01, 0.5])), device=DEV)
        tensors.append((spec.name + "é" * (k % 3), o, w))
    _roundtrip(sd, tensors)


def test_workspace_regrowth_high_density(sd):
    ctx = sd.DeltaContext(DEV)  # fresh: initial entry workspace is max(1M, N/32)
    spec = TensorSpec("dense", (4096, 2048), "matrix")
    o, w = generate_pair(spec, 0, 9, rho=0.5, device=DEV)
    _roundtrip(sd, [(spec.name, o, w)], ctx=ctx)
    o2, w2 = generate_pair(spec, 1, 9, rho=0.99, device=DEV)  # grows again
    _roundtrip(sd, [(spec.name, o2, w2)], ctx=ctx)
    ctx.close()


def test_size_then_extract_and_capacity(sd):
    spec = TensorSpec("x", (100_000,), "matrix")
    o, w = generate_pair(spec, 0, 1, rho=0.05, device=DEV)
    tl = sd.TensorList([(spec.name, o, w)])
    ctx = sd.context()
    size = ctx.delta_size(tl)
    out = torch.empty(size, dtype=torch.uint8, device=DEV)
    body, table = ctx.delta_extract(tl, out=out)  # consumes the cached compaction
    ref_body, ref_table = oracle_extract([(spec.name, o, w)])
    assert size == len(ref_body)
    assert_body_equal(body, ref_body)
    small = torch.empty(size - 1, dtype=torch.uint8, device=DEV)
    with pytest.raises(sd.DeltaError) as e:
        ctx.delta_extract(tl, out=small)
    assert e.value.status == -3  # DELTA_ECAPACITY


def test_compute_rho_and_size_table(sd):
    """SPEC.md:116-119 compute_rho (Eq. 1): per-tensor nnz and rho from the GPU compaction
    equal the oracle's; the cached compaction still serves the following extract."""
    specs = [TensorSpec("a", (4096, 33), "matrix"), TensorSpec("b", (70_001,), "matrix"),
             TensorSpec("c", (257,), "norm")]
    tensors = []
    for i, (spec, r) in enumerate(zip(specs, (0.01, 0.3, 0.0))):
        o, w = generate_pair(spec, 0, i, rho=r, device=DEV)
        tensors.append((spec.name, o, w))
    pairs = [(to_np(o), to_np(w)) for _, o, w in tensors]
    ctx = sd.context()
    tl = sd.TensorList(tensors)
    rho, nnz = ctx.compute_rho(tl)
    ref_body, ref_table = oracle_extract(tensors)
    assert nnz == [r[2] for r in ref_table]
    assert nnz[2] == 0
    assert rho == oracle.codec.rho(pairs)
    assert [tuple(r) for r in ctx.size_table(len(tensors))] == [tuple(r) for r in ref_table]
    body, _ = ctx.delta_extract(tl)  # consumes the cached compaction
    assert_body_equal(body, ref_body)
    with pytest.raises(sd.DeltaError):
        ctx.size_table(len(tensors))  # nothing cached any more
    ctx.delta_size(tl)
    with pytest.raises(sd.DeltaError):
        ctx.size_table(len(tensors) + 1)  # n mismatch


def test_compute_rho_spec_example(sd):
    """SPEC.md:121 worked example: tensors of 4 and 6 lanes with 1 and 2 changed -> 0.3."""
    a_old = torch.tensor([1.0, 2.0, 3.0, 4.0], dtype=torch.bfloat16, device=DEV)
    a_new = a_old.clone()
    a_new[2] = 5.0
    b_old = torch.arange(6, dtype=torch.float32, device=DEV).to(torch.bfloat16)
    b_new = b_old.clone()
    b_new[0] = -0.0  # +0.0 -> -0.0 is a change (bitwise, reading R2)
    b_new[5] = 7.0
    rho, nnz = sd.compute_rho([("a", a_old, a_new), ("b", b_old, b_new)])
    assert nnz == [1, 2]
    assert rho == 3 / 10


def test_fp32_m1_shape(sd):
    spec = m1_specs()[0]
    o, w = generate_pair(spec, 0, 4, rho=0.01, dtype=torch.float32, device=DEV)
    _roundtrip(sd, [(spec.name, o, w)])


# ------------------------------------------------------------------ corruption suite
def _small_valid():
    spec_a = TensorSpec("a", (5000,), "matrix")
    spec_b = TensorSpec("b", (300,), "norm")
    oa, wa = generate_pair(spec_a, 0, 3, rho=0.05)
    ob, wb = generate_pair(spec_b, 1, 3, rho=0.05)
    return [("a", oa, wa), ("b", ob, wb)]


def _mutations(body: bytes, table):
    """(label, mutated body, targets numel overrides) — each with exactly one fault."""
    b = bytearray(body)
    ra, rb = table[0], table[1]
    out = []
    m = bytearray(b)
    m[ra[3] + ra[4] - 1] |= 0x80                         # last stream byte keeps going
    out.append(("truncated", m, None))
    # zero gap: find a 1-byte varint after the first entry and make it 0
    s = ra[3]
    m = bytearray(b)
    pos = s + 1
    while m[pos - 1] & 0x80 or m[pos] & 0x80:
        pos += 1
    m[pos] = 0x00
    out.append(("nonincreasing", m, None))
    m = bytearray(b)
    m[ra[6] - 1] = 2                                     # mode byte (0 replace, 1 additive)
    out.append(("mode", m, None))
    m = bytearray(b)
    m[2] ^= 0x01                                         # name byte of record a ('a' -> '`')
    out.append(("name", m, None))
    out.append(("numel", bytearray(b), {"a": 5001}))
    out.append(("layout", bytearray(b[:-1]), None))
    out.append(("layout", bytearray(b + b"\x00"), None))
    # count: nnz field of record b says one more (values region shifts: also make room)
    m = bytearray(b)
    nl = 1
    nnz_off = rb[0] + 2 + nl + 8
    nnz = int.from_bytes(m[nnz_off:nnz_off + 8], "little")
    m[nnz_off:nnz_off + 8] = (nnz + 1).to_bytes(8, "little")
    m[rb[0] + rb[6] - 1:rb[0] + rb[6] - 1] = b"\x00\x00"  # two more value bytes before mode
    out.append(("count", m, None))
    return out


def _hand_record(name, n, nnz, stream, vals, mode=0):
    import struct
    nb = name.encode()
    return (struct.pack("<H", len(nb)) + nb + struct.pack("<QQQ", n, nnz, len(stream))
            + bytes(stream) + bytes(vals) + bytes([mode]))


_HAND = [
    ("overlong", _hand_record("a", 10, 1, b"\x85\x00", b"\x01\x00")),
    ("overflow", _hand_record("a", 10, 1, b"\xff" * 9 + b"\x02", b"\x01\x00")),
    ("overflow", _hand_record("a", 10, 1, b"\xff" * 10 + b"\x01", b"\x01\x00")),
    ("range", _hand_record("a", 10, 2, b"\x05\x05", b"\x01\x00\x02\x00")),
    ("range", _hand_record("a", 10, 1, b"\x0a", b"\x01\x00")),
    ("truncated", _hand_record("a", 10, 1, b"\x85", b"\x01\x00")),
    ("count", _hand_record("a", 10, 1, b"\x01\x01", b"\x01\x00")),
]


def _expect_reject(sd, body: bytes, targets_np, kind_expected):
    """targets_np: [(name, np lanes)]; the oracle and the GPU must both reject with the
    same kind, and the GPU targets must be bitwise untouched."""
    with pytest.raises(oracle.DeltaError) as eo:
        oracle.codec.apply(targets_np, body, 2)
    assert eo.value.kind == kind_expected
    dev_body = torch.tensor(list(body), dtype=torch.uint8, device=DEV)
    targets = [(n, torch.from_numpy(a.view(np.int16).copy()).to(DEV).view(torch.bfloat16))
               for n, a in targets_np]
    before = [t.clone() for _, t in targets]
    for hint in (None, "valid-looking"):
        table = None
        if hint:  # a hint computed from the body's own (corrupt) headers
            table = _naive_table(body, len(targets))
            if table is None:
                continue
        with pytest.raises(sd.DeltaError) as eg:
            sd.delta_apply(targets, dev_body, table=table)
        assert eg.value.kind == kind_expected, (eg.value, kind_expected)
        for (_, t), b in zip(targets, before):
            assert_lanes_equal(t, b)


def _naive_table(body: bytes, n):
    import struct
    rows, pos = [], 0
    try:
        for _ in range(n):
            nl = struct.unpack_from("<H", body, pos)[0]
            N, nnz, il = struct.unpack_from("<QQQ", body, pos + 2 + nl)
            io = pos + 2 + nl + 24
            rb = 27 + nl + il + 2 * nnz
            rows.append((pos, N, nnz, io, il, io + il, rb))
            pos += rb
    except struct.error:
        return None
    return rows


def test_corruption_suite(sd):
    ts = _small_valid()
    body, table = oracle_extract(ts)
    for kind, mbody, override in _mutations(body, table):
        targets = [(n, to_np(o).copy()) for n, o, _ in ts]
        if override:
            targets = [(n, np.zeros(override.get(n, a.size), np.uint16)) for n, a in targets]
        _expect_reject(sd, bytes(mbody), targets, kind)


@pytest.mark.parametrize("kind,body", _HAND)
def test_corruption_hand(sd, kind, body):
    _expect_reject(sd, body, [("a", np.arange(10, dtype=np.uint16))], kind)


def test_corruption_deep_in_a_multichunk_stream(sd):
    # a fault in a later 4 KiB chunk of a long stream (M1-sized record)
    spec = m1_specs()[0]
    o, w = generate_pair(spec, 0, 0, rho=0.01, pattern="exact")
    body, table = oracle.codec.extract([(spec.name, [to_np(o)], [to_np(w)])])
    r = table[0]
    assert r[4] > 5 * 4096
    m = bytearray(body)
    p = r[3] + 3 * 4096 + 100
    while m[p - 1] & 0x80 or m[p] & 0x80:  # a 1-byte varint that is not the first
        p += 1
    m[p] = 0
    _expect_reject(sd, bytes(m), [(spec.name, to_np(o).copy())], "nonincreasing")


def test_u64_index_path(sd):
    """A tensor with more than 2^32 lanes (reading R13): 64-bit indices and 5-byte gaps."""
    n = 2**32 + 1000
    pos = [0, 2**31, 2**32 - 1, 2**32, 2**32 + 999]
    old, new = _with_changes(n, pos)
    ctx = sd.DeltaContext(DEV)
    body, table = ctx.delta_extract([("huge", old, new)])
    want = oracle.brute.record_from_sparse("huge", n, pos, [0x3F80] * len(pos), 2)
    assert body.cpu().numpy().tobytes() == want
    w = old.clone()
    del old
    ctx.delta_apply([("huge", w)], body, table=table)
    assert_lanes_equal(w, new)
    ctx.close()


# ------------------------------------------------------------------ pipelined round trip
def test_pipelined_roundtrip_matches_oracle(sd):
    from paper_2602_11456_b200.pipeline import RoundTrip
    rng = np.random.default_rng(11)
    tensors = []
    for k in range(23):
        n = int(rng.integers(0, 200_000))
        spec = TensorSpec(f"model.layers.{k}.w", (n,), "matrix")
        o, w = generate_pair(spec, k, 5, rho=float(rng.choice([0.0, 0.01, 0.2])), device=DEV)
        tensors.append((spec.name, o, w))
    targets = [(n, o.clone()) for n, o, _ in tensors]
    for groups, ctas in ((1, None), (4, 2), (7, None)):
        for _, t in targets:
            t.zero_()
        rt = RoundTrip(tensors, targets, groups=groups, device=DEV, apply_ctas_per_sm=ctas)
        for (n, t), (_, o, _) in zip(targets, tensors):
            t.copy_(o)
        body = rt.step()
        torch.cuda.synchronize()
        ref_body, ref_table = oracle_extract(tensors)
        assert_body_equal(body, ref_body)
        assert rt.table() == [tuple(r) for r in ref_table]
        for (_, t), (_, _, w) in zip(targets, tensors):
            assert_lanes_equal(t, w)
        rt.close()


def test_async_apply_error_is_reported_at_wait(sd):
    ts = _small_valid()
    body, table = oracle_extract(ts)
    bad = bytearray(body)
    bad[table[0][6] - 1] = 2  # mode byte of record a (0 replace, 1 additive)
    targets = [(n, torch.from_numpy(to_np(o).view(np.int16).copy()).to(DEV).view(torch.bfloat16))
               for n, o, _ in ts]
    before = [t.clone() for _, t in targets]
    ctx = sd.DeltaContext(DEV)
    ctx.delta_apply(targets, torch.tensor(list(bad), dtype=torch.uint8, device=DEV), wait=False)
    with pytest.raises(sd.DeltaError) as e:
        ctx.apply_wait()
    assert e.value.kind == "mode"
    for (_, t), b in zip(targets, before):
        assert_lanes_equal(t, b)
    # the sticky error is cleared by the wait: a valid body now applies
    ctx.delta_apply(targets, torch.tensor(list(body), dtype=torch.uint8, device=DEV), wait=False)
    ctx.apply_wait()
    for (_, t), (_, _, w) in zip(targets, ts):
        assert_lanes_equal(t, w.to(DEV))
    ctx.close()


# ------------------------------------------------------------------ K1 launch variants
@pytest.mark.parametrize("kernel", [1])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_scan_kernel_variants_parity(sd, dtype, kernel):
    """The compare+compaction kernel (DELTA_OPT_SCAN_KERNEL = 1, the only form) on ragged /
    unaligned / multi-tile / dense inputs, byte-exact against the oracle; the retired forms
    2-5 are rejected."""
    from paper_2602_11456_b200 import _abi
    ctx = sd.DeltaContext(DEV)
    for bad in (2, 3, 4, 5, 6):
        with pytest.raises(sd.DeltaError):
            ctx.set_option(_abi.DELTA_OPT_SCAN_KERNEL, bad)
    ctx.set_option(_abi.DELTA_OPT_SCAN_KERNEL, kernel)
    rng = np.random.default_rng(21)
    tensors = []
    for k, n in enumerate([1, 9, 16384, 16385, 16384 * 7 + 3, 250_001, 0, 3_000_000]):
        spec = TensorSpec(f"t{k}", (n,), "matrix")
        o, w = generate_pair(spec, k, 3, rho=float(rng.choice([0.0, 0.01, 0.5, 1.0])), dtype=dtype,
                             device=DEV, values="bits")
        tensors.append((spec.name, o, w))
    # an unaligned multi-span tensor
    spec = TensorSpec("u", (100_003,), "matrix")
    o, w = generate_pair(spec, 99, 3, rho=0.05, dtype=dtype, device=DEV)
    tensors.append(("unaligned", [o[1:40_000], o[40_000:]], [w[1:40_000], w[40_000:]]))
    _roundtrip(sd, tensors, ctx=ctx)
    ctx.close()


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("scatter_ctas", [1, 8])
def test_scatter_launch_options_parity(sd, order, scatter_ctas):
    """Scatter store order (thread-major / entry-major) and grid size change only speed."""
    from paper_2602_11456_b200 import _abi
    ctx = sd.DeltaContext(DEV)
    ctx.set_option(_abi.DELTA_OPT_SCATTER_ORDER, order)
    ctx.set_option(_abi.DELTA_OPT_SCATTER_CTAS_PER_SM, scatter_ctas)
    ctx.set_option(_abi.DELTA_OPT_PREFETCH_TILES, 1000)
    tensors = []
    for k, (n, rho) in enumerate([(16_777_216, 0.01), (100_003, 0.9), (5, 1.0), (0, 0.0), (70_000, 0.0005)]):
        spec = TensorSpec(f"s{k}", (n,), "matrix")
        o, w = generate_pair(spec, k, 8, rho=rho, device=DEV, values="bits")
        tensors.append((spec.name, o, w))
    _roundtrip(sd, tensors, ctx=ctx)
    ctx.close()


def test_mixed_varint_lengths(sd):
    """Index streams mixing 1-, 2-, 3- and 4-byte gaps at every alignment (exercises the
    bit-parallel decode fast path and its byte-loop fallback at window boundaries)."""
    rng = np.random.default_rng(77)
    n = 1 << 26
    gaps, pos, cur = [], [], 0
    while True:
        kind = rng.choice([1, 1, 1, 2, 2, 3, 4], p=[0.3, 0.2, 0.1, 0.15, 0.1, 0.1, 0.05])
        g = {1: int(rng.integers(1, 128)), 2: int(rng.integers(128, 16384)),
             3: int(rng.integers(16384, 2**21)), 4: int(rng.integers(2**21, 2**22))}[kind]
        if cur + g >= n:
            break
        cur += g
        pos.append(cur)
    pos = [0] + pos  # first index 0 (a 0x00 first varint)
    old, new = _with_changes(n, pos)
    body, table = _roundtrip(sd, [("mixed", old, new)])
    assert table[0][2] == len(pos)


# ------------------------------------------------------------------ GPU digest (NEXT f1)
def test_gpu_digest_and_container(sd):
    """delta_digest (BLAKE3-256 on the GPU) equals the oracle container's digest (the
    `blake3` package) for sizes around every chunk / tree boundary, and the product's SPDC
    container is byte-identical to the oracle's."""
    import oracle
    rng = np.random.default_rng(5)
    ctx = sd.DeltaContext(DEV)
    for n in [0, 1, 63, 64, 65, 1023, 1024, 1025, 2047, 2048, 2049, 3072, 4097, 65536, 100_000,
              1 << 20, (1 << 20) + 7, 5_000_001]:
        data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        buf = torch.tensor(list(data) if n < 5000 else np.frombuffer(data, np.uint8).copy(),
                           dtype=torch.uint8, device=DEV)
        assert ctx.digest(buf) == oracle.container.digest(data), n
        # unaligned start
        if n > 3:
            assert ctx.digest(buf[3:]) == oracle.container.digest(data[3:]), n
    spec = m1_specs()[0]
    o, w = generate_pair(spec, 0, 0, rho=0.01, pattern="exact", device=DEV)
    body, table = ctx.delta_extract([(spec.name, o, w)])
    blob = sd.pack_container(body, 9, 8, 2, 1, ctx=ctx)
    ref = oracle.container.pack(body.cpu().numpy().tobytes(), 9, 8, 2, 1)
    assert blob == ref
    # the container built on the device: the extract writes straight into it, the header
    # (digest included) is written by the library's kernel — no host copy of the body
    cont = torch.empty(sd.container.HEADER_BYTES + body.numel(), dtype=torch.uint8, device=DEV)
    b2, _ = ctx.delta_extract([(spec.name, o, w)], out=cont[sd.container.HEADER_BYTES:], table=False)
    dev_blob = sd.pack_container_device(b2, 9, 8, 2, 1, ctx=ctx, out=cont)
    assert dev_blob.data_ptr() == cont.data_ptr()
    assert dev_blob.cpu().numpy().tobytes() == ref
    # fixed-width codec: format_version 2 in the header
    ref_f = oracle.container.pack(body.cpu().numpy().tobytes(), 9, 8, 2, 1, index_codec="fixed")
    dev_f = sd.pack_container_device(body, 9, 8, 2, 1, ctx=ctx, index_codec="fixed")
    assert dev_f.cpu().numpy().tobytes() == ref_f
    with pytest.raises(sd.DeltaError):
        ctx.container_header(body, 9, 7, 2, 1, cont)  # version != base_version + 1
    ctx.close()


# ------------------------------------------------------------------ additive mode (NEXT f3)
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_additive_mode_parity(sd, dtype):
    """DELTA_OPT_MODE = 2: values are new - old (fp32 arithmetic, RNE to bf16) and apply
    adds them — body bytes and the applied lanes byte-exact against the
    oracle's additive codec, on sparse, dense (whole-vector window rewrite) and full-range bit patterns."""
    import oracle
    from paper_2602_11456_b200 import _abi
    ctx = sd.DeltaContext(DEV)
    ctx.set_option(_abi.DELTA_OPT_MODE, 2)
    tensors = []
    for k, (n, rho, vals) in enumerate([(16_777_216, 0.01, "weights"), (300_001, 0.6, "weights"),
                                        (100_003, 0.3, "bits"), (9, 1.0, "bits"), (0, 0.0, "weights")]):
        spec = TensorSpec(f"a{k}", (n,), "matrix")
        o, w = generate_pair(spec, k, 12, rho=rho, dtype=dtype, device=DEV, values=vals)
        tensors.append((spec.name, o, w))
    body, table = ctx.delta_extract(tensors)
    ref_body, ref_table = oracle.codec.extract([(n, [to_np(o)], [to_np(w)]) for n, o, w in tensors],
                                               mode=oracle.codec.MODE_ADDITIVE)
    assert_body_equal(body, ref_body)
    assert [tuple(r) for r in table] == [tuple(r) for r in ref_table]
    width = 2 if dtype == torch.bfloat16 else 4
    ref_out = oracle.codec.apply([(n, to_np(o)) for n, o, _ in tensors], ref_body, width)
    for hint in (True, False):
        targets = [(n, o.clone()) for n, o, _ in tensors]
        ctx.delta_apply(targets, body, table=table if hint else None)
        torch.cuda.synchronize()
        for (_, t), r in zip(targets, ref_out):
            assert np.array_equal(to_np(t), r)
    ctx.close()


def test_chained_round_trip_overflow_and_capacity(sd):
    """delta_extract_async -> delta_apply_async_chain: a first call at a higher density
    overflows the tile slots (EAGAIN, workspace grown, the chained apply refuses and
    mutates nothing); a too-small output closes the emit gate (ECAPACITY, size = -1,
    targets untouched); round_trip retries the overflow and matches the oracle."""
    ctx = sd.DeltaContext(DEV)
    spec = TensorSpec("d", (2048, 1024), "matrix")
    o, w = generate_pair(spec, 0, 21, rho=0.4, device=DEV)  # > the initial 1/16 slots
    tensors = [(spec.name, o, w)]
    ref_body, _ = oracle_extract(tensors)
    out = torch.zeros(len(ref_body) + 16, dtype=torch.uint8, device=DEV)
    size = torch.zeros(1, dtype=torch.int64, device=DEV)
    tgt = [(spec.name, o.clone())]
    table = ctx.delta_extract_async(tensors, out, size)
    ctx.delta_apply(tgt, out, table=table, size=size, wait=False)
    with pytest.raises(sd.DeltaError) as e:
        ctx.extract_wait()
    assert e.value.status == -8  # DELTA_EAGAIN
    with pytest.raises(sd.DeltaError) as e:
        ctx.apply_wait()
    assert e.value.kind == "layout"
    assert int(size.item()) == -1
    assert_lanes_equal(tgt[0][1], o)  # untouched
    # the grown workspace now fits: the same calls succeed
    n = ctx.round_trip(tensors, tgt, out, size)
    assert n == len(ref_body)
    assert_body_equal(out[:n], ref_body)
    assert_lanes_equal(tgt[0][1], w)
    # capacity: one byte short
    small = torch.zeros(len(ref_body) - 1, dtype=torch.uint8, device=DEV)
    tgt2 = [(spec.name, o.clone())]
    table = ctx.delta_extract_async(tensors, small, size)
    ctx.delta_apply(tgt2, small, table=table, size=size, wait=False)
    with pytest.raises(sd.DeltaError) as e:
        ctx.extract_wait()
    assert e.value.status == -3
    with pytest.raises(sd.DeltaError):
        ctx.apply_wait()
    assert int(size.item()) == -1
    assert_lanes_equal(tgt2[0][1], o)
    assert int(small.count_nonzero().item()) == 0  # nothing written
    # a fresh context: round_trip absorbs the first-call overflow by itself
    ctx2 = sd.DeltaContext(DEV)
    tgt3 = [(spec.name, o.clone())]
    assert ctx2.round_trip(tensors, tgt3, out, size) == len(ref_body)
    assert_lanes_equal(tgt3[0][1], w)
    ctx.close()
    ctx2.close()


# ------------------------------------------------------------------ fixed-width index codec (NEXT f4)
def _fixed_ctx(sd):
    from paper_2602_11456_b200 import _abi
    ctx = sd.DeltaContext(DEV)
    ctx.set_option(_abi.DELTA_OPT_INDEX_CODEC, 2)
    return ctx


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_fixed_codec_parity(sd, dtype):
    """DELTA_OPT_INDEX_CODEC = 2, the naive int32/64 encoding (R18):
    body bytes and table rows equal the oracle's fixed-width codec; apply (host, device and
    no table hint) reconstructs new bit for bit.  Multi-chunk, dense, ragged, fused and
    empty tensors, full-range bit patterns."""
    ctx = _fixed_ctx(sd)
    tensors = []
    for k, (n, rho, vals) in enumerate([(16_777_216, 0.01, "weights"), (300_001, 0.6, "weights"),
                                        (100_003, 0.3, "bits"), (9, 1.0, "bits"), (0, 0.0, "weights"),
                                        (16385, 0.001, "weights")]):
        spec = TensorSpec(f"f{k}.w", (n,), "matrix")
        o, w = generate_pair(spec, k, 21, rho=rho, dtype=dtype, device=DEV, values=vals)
        tensors.append((spec.name, o, w))
    o, w = tensors[1][1], tensors[1][2]  # a fused, unaligned 3-span tensor
    tensors.append(("f.qkv", [o[:1001], o[1001:50001], o[50001:]], [w[:1001], w[1001:50001], w[50001:]]))
    body, table = ctx.delta_extract(tensors)
    ref_body, ref_table = oracle.codec.extract(
        [(n, [to_np(s) for s in as_list(a)], [to_np(s) for s in as_list(b)]) for n, a, b in tensors],
        index_codec="fixed")
    assert_body_equal(body, ref_body)
    assert [tuple(r) for r in table] == [tuple(r) for r in ref_table]
    for hint in ("host", "none", "device"):
        targets = [(n, fused(a).clone()) for n, a, _ in tensors]
        if hint == "device":
            dbody, dtab = ctx.delta_extract(tensors, table="device")
            ctx.delta_apply(targets, dbody, table=dtab)
        else:
            ctx.delta_apply(targets, body, table=table if hint == "host" else None)
        torch.cuda.synchronize()
        for (_, t), (_, _, b) in zip(targets, tensors):
            assert_lanes_equal(t, fused(b))
    ctx.close()


def test_fixed_codec_u64_indices(sd):
    """N = 2^31 + 1000 lanes: N - 1 > INT32_MAX -> 8-byte indices (R18)."""
    n = 2**31 + 1000
    pos = [0, 5, 2**31 - 1, 2**31, 2**31 + 999]
    old, new = _with_changes(n, pos)
    ctx = _fixed_ctx(sd)
    body, table = ctx.delta_extract([("big", old, new)])
    import struct
    vals = b"".join(struct.pack("<H", int(x)) for x in to_np(new[torch.tensor(pos, device=DEV)]))
    stream = oracle.brute.encode_indices_fixed(pos, n)
    assert len(stream) == 8 * len(pos)
    want = _hand_record("big", n, len(pos), stream, vals)
    assert body.cpu().numpy().tobytes() == want
    w = old
    del old
    ctx.delta_apply([("big", w)], body, table=table)
    assert_lanes_equal(w, new)
    ctx.close()


_HAND_FIXED = [
    ("truncated", _hand_record("a", 10, 1, b"\x01\x00\x00", b"\x01\x00")),
    ("count", _hand_record("a", 10, 1, b"\x01\x00\x00\x00\x02\x00\x00\x00", b"\x01\x00")),
    ("nonincreasing", _hand_record("a", 10, 2, b"\x03\x00\x00\x00\x03\x00\x00\x00", b"\x01\x00\x02\x00")),
    ("nonincreasing", _hand_record("a", 10, 2, b"\x04\x00\x00\x00\x03\x00\x00\x00", b"\x01\x00\x02\x00")),
    ("range", _hand_record("a", 10, 2, b"\x03\x00\x00\x00\x0a\x00\x00\x00", b"\x01\x00\x02\x00")),
]


@pytest.mark.parametrize("kind,body", _HAND_FIXED)
def test_fixed_codec_rejects(sd, kind, body):
    """Single-fault fixed-width bodies: the GPU's error kind equals the oracle's and the
    targets stay bitwise untouched (all-or-nothing)."""
    a = np.arange(10, dtype=np.uint16)
    with pytest.raises(oracle.DeltaError) as eo:
        oracle.codec.apply([("a", a.copy())], body, 2, index_codec="fixed")
    assert eo.value.kind == kind
    ctx = _fixed_ctx(sd)
    t = torch.from_numpy(a.view(np.int16).copy()).to(DEV).view(torch.bfloat16)
    before = t.clone()
    with pytest.raises(sd.DeltaError) as eg:
        ctx.delta_apply([("a", t)], torch.tensor(list(body), dtype=torch.uint8, device=DEV))
    assert eg.value.kind == kind
    assert_lanes_equal(t, before)
    ctx.close()


def test_fixed_codec_fault_in_a_later_chunk(sd):
    """A non-increasing index deep in a multi-chunk fixed-width stream (chunk boundary
    carries the previous entry)."""
    spec = m1_specs()[0]
    o, w = generate_pair(spec, 0, 0, rho=0.01, pattern="exact")
    body, table = oracle.codec.extract([(spec.name, [to_np(o)], [to_np(w)])], index_codec="fixed")
    r = table[0]
    m = bytearray(body)
    e = 3 * 1024  # the first entry of the fourth 4 KiB chunk repeats the previous index
    m[r[3] + 4 * e:r[3] + 4 * e + 4] = m[r[3] + 4 * (e - 1):r[3] + 4 * e]
    ctx = _fixed_ctx(sd)
    t = o.to(DEV)
    before = t.clone()
    with pytest.raises(sd.DeltaError) as eg:
        ctx.delta_apply([(spec.name, t)], torch.tensor(list(m), dtype=torch.uint8, device=DEV))
    assert eg.value.kind == "nonincreasing"
    assert_lanes_equal(t, before)
    ctx.close()


# ------------------------------------------------------------------ extract-and-advance (NEXT f3)
def test_extract_and_advance(sd):
    """DELTA_OPT_ADVANCE = 2: the body equals the oracle's, and afterwards every old span
    equals its new span bitwise (fused, unaligned and ragged spans included).  The first
    call runs at a density that overflows the default slots, so the retry path (slots
    regrown with the fitted tiles' compaction kept, only overflowed tiles redone) is
    exercised; a second extract of the same pair sees no change."""
    from paper_2602_11456_b200 import _abi
    ctx = sd.DeltaContext(DEV)
    ctx.set_option(_abi.DELTA_OPT_ADVANCE, 2)
    tensors, keep_old = [], []
    for k, (n, rho) in enumerate([(16_777_216, 0.01), (2_000_003, 0.3), (100_003, 0.001), (7, 1.0), (0, 0.0)]):
        spec = TensorSpec(f"adv{k}", (n,), "matrix")
        o, w = generate_pair(spec, k, 31, rho=rho, device=DEV)
        tensors.append((spec.name, o, w))
    o, w = generate_pair(TensorSpec("adv.qkv", (60_001,), "matrix"), 9, 31, rho=0.05, device=DEV)
    tensors.append(("adv.qkv", [o[:1001].clone(), o[1001:50001].clone(), o[50001:].clone()],
                    [w[:1001], w[1001:50001], w[50001:]]))
    ref_body, ref_table = oracle_extract(tensors)
    keep_old = [[s.clone() for s in as_list(a)] for _, a, _ in tensors]
    body, table = ctx.delta_extract(tensors)
    torch.cuda.synchronize()
    assert_body_equal(body, ref_body)
    assert [tuple(r) for r in table] == [tuple(r) for r in ref_table]
    for (_, a, b) in tensors:
        for sa, sb in zip(as_list(a), as_list(b)):
            assert_lanes_equal(sa, sb)
    # the body still applies onto the pre-advance copy
    targets = [(n, fused(ko).clone()) for (n, _, _), ko in zip(tensors, keep_old)]
    ctx.delta_apply(targets, body, table=table)
    torch.cuda.synchronize()
    for (_, t), (_, _, b) in zip(targets, tensors):
        assert_lanes_equal(t, fused(b))
    body2, table2 = ctx.delta_extract(tensors)
    assert all(r[2] == 0 for r in table2)
    with pytest.raises(sd.DeltaError):  # asynchronous extract refuses advance
        ctx.delta_extract_async(tensors, torch.empty(1 << 20, dtype=torch.uint8, device=DEV),
                                torch.zeros(1, dtype=torch.int64, device=DEV))
    ctx.close()


# ------------------------------------------------------------------ delta merge (NEXT f4)
def _three_versions(n, seed, rho1, rho2, overlap, dt=np.uint16):
    """v0 -> v1 (rho1 uniform), v1 -> v2 (rho2 uniform, plus a share `overlap` of v1's
    changed lanes changed again); lanes as numpy uint16 (bf16) or uint32 (fp32)."""
    rng = np.random.default_rng(seed)
    v0 = rng.integers(0, 2**(8 * np.dtype(dt).itemsize), n, dtype=np.uint64).astype(dt)
    m1 = rng.random(n) < rho1
    v1 = v0.copy()
    v1[m1] ^= rng.integers(1, 16, int(m1.sum()), dtype=np.uint64).astype(dt)
    m2 = rng.random(n) < rho2
    again = np.flatnonzero(m1)
    m2[again[rng.random(again.size) < overlap]] = True
    v2 = v1.copy()
    v2[m2] ^= rng.integers(1, 16, int(m2.sum()), dtype=np.uint64).astype(dt)
    return v0, v1, v2


def _dev(a):
    if a.dtype == np.uint32:
        return torch.from_numpy(a.view(np.int32).copy()).to(DEV).view(torch.float32)
    return torch.from_numpy(a.view(np.int16).copy()).to(DEV).view(torch.bfloat16)


@pytest.mark.parametrize("dt", [np.uint16, np.uint32])
def test_merge_parity(sd, dt):
    """delta_merge on the GPU == oracle.codec.merge byte for byte, and applying the merge
    to v0 gives v2 (M1-sized multi-chunk record, dense, overlapping, empty, 1-lane;
    16- and 32-bit lanes)."""
    cases = [(16_777_216, 0.01, 0.01, 0.3), (300_001, 0.4, 0.2, 0.5), (5000, 0.0, 0.05, 0.0),
             (5000, 0.05, 0.0, 0.0), (0, 0.0, 0.0, 0.0), (1, 1.0, 1.0, 1.0), (100_003, 0.001, 0.001, 1.0)]
    if dt == np.uint32:
        cases[0] = (4_000_037, 0.01, 0.01, 0.3)
    width = np.dtype(dt).itemsize
    names = [f"m{k}.weight" for k in range(len(cases))]
    vs = [_three_versions(n, 70 + k, r1, r2, ov, dt) for k, (n, r1, r2, ov) in enumerate(cases)]
    ctx = sd.DeltaContext(DEV)
    # the two input bodies come from the oracle (not from the GPU's extract)
    a_ref, _ = oracle.codec.extract([(nm, [v[0]], [v[1]]) for nm, v in zip(names, vs)])
    b_ref, _ = oracle.codec.extract([(nm, [v[1]], [v[2]]) for nm, v in zip(names, vs)])
    a = torch.frombuffer(bytearray(a_ref), dtype=torch.uint8).to(DEV)
    b = torch.frombuffer(bytearray(b_ref), dtype=torch.uint8).to(DEV)
    merged = ctx.delta_merge(a, b, len(names), width=width)
    torch.cuda.synchronize()
    want = oracle.codec.merge(a_ref, b_ref, width)
    assert_body_equal(merged, want)
    targets = [(nm, _dev(v[0])) for nm, v in zip(names, vs)]
    ctx.delta_apply(targets, merged)
    torch.cuda.synchronize()
    for (_, t), v in zip(targets, vs):
        assert np.array_equal(to_np(t), v[2])
    ctx.close()


def test_merge_rejects(sd):
    """Faults in either body: the GPU's error kind equals the oracle's (and nothing is
    written to out)."""
    x = np.arange(50, dtype=np.uint16)
    y = x.copy()
    y[[3, 30]] += 1

    def body(name, o, n, mode=0):
        bb, _ = oracle.codec.extract([(name, [o], [n])], mode=mode)
        return bb
    good = body("p", x, y)
    cases = [("name", good, body("q", x, y)), ("numel", good, body("p", np.arange(51, dtype=np.uint16),
                                                                     np.arange(51, dtype=np.uint16) + 1)),
             ("mode", good, body("p", x, y, mode=oracle.codec.MODE_ADDITIVE)),
             ("layout", good, good + good)]
    trunc = bytearray(good)
    trunc[2 + 1 + 24 + 1] |= 0x80  # second varint keeps going into the values
    cases.append(("truncated", good, bytes(trunc)))
    ctx = sd.DeltaContext(DEV)
    for kind, ba, bb in cases:
        with pytest.raises(oracle.DeltaError) as eo:
            oracle.codec.merge(ba, bb, 2)
        if kind is not None:
            assert eo.value.kind == kind
        out = torch.full((256,), 0x5A, dtype=torch.uint8, device=DEV)
        with pytest.raises(sd.DeltaError) as eg:
            ctx.delta_merge(torch.tensor(list(ba), dtype=torch.uint8, device=DEV),
                            torch.tensor(list(bb), dtype=torch.uint8, device=DEV), 1, out=out)
        assert eg.value.kind == eo.value.kind, (eg.value, eo.value.kind)
        assert bool((out == 0x5A).all())
    ctx.close()


# ------------------------------------------------------------------ option combinations
def test_fixed_codec_with_additive_and_advance(sd):
    """The index codec, the record mode and extract-and-advance are independent: additive
    records with fixed-width indices match the oracle (and apply adds), and advance with
    fixed-width indices leaves old == new with the body unchanged."""
    from paper_2602_11456_b200 import _abi
    tensors = []
    for k, (n, rho) in enumerate([(1_000_003, 0.02), (70_001, 0.4), (0, 0.0)]):
        spec = TensorSpec(f"c{k}", (n,), "matrix")
        o, w = generate_pair(spec, k, 41, rho=rho, device=DEV, values="bits")
        tensors.append((spec.name, o, w))
    ctx = sd.DeltaContext(DEV)
    ctx.set_option(_abi.DELTA_OPT_INDEX_CODEC, 2)
    ctx.set_option(_abi.DELTA_OPT_MODE, 2)
    body, table = ctx.delta_extract(tensors)
    npt = [(n, [to_np(o)], [to_np(w)]) for n, o, w in tensors]
    ref, ref_table = oracle.codec.extract(npt, mode=oracle.codec.MODE_ADDITIVE, index_codec="fixed")
    assert_body_equal(body, ref)
    assert [tuple(r) for r in table] == [tuple(r) for r in ref_table]
    want = oracle.codec.apply([(n, to_np(o)) for n, o, _ in tensors], ref, 2, index_codec="fixed")
    targets = [(n, o.clone()) for n, o, _ in tensors]
    ctx.delta_apply(targets, body, table=table)
    torch.cuda.synchronize()
    for (_, t), r in zip(targets, want):
        assert np.array_equal(to_np(t), r)
    ctx.close()
    ctx = sd.DeltaContext(DEV)
    ctx.set_option(_abi.DELTA_OPT_INDEX_CODEC, 2)
    ctx.set_option(_abi.DELTA_OPT_ADVANCE, 2)
    ref, _ = oracle.codec.extract(npt, index_codec="fixed")
    body, _ = ctx.delta_extract(tensors)
    torch.cuda.synchronize()
    assert_body_equal(body, ref)
    for _, o, w in tensors:
        assert_lanes_equal(o, w)
    ctx.close()


def test_merge_degenerate(sd):
    """delta_merge of bodies with no change at all, of an empty tensor list, and of a body
    with itself (idempotent replace: the merge equals the body)."""
    x = np.arange(300, dtype=np.uint16)
    same, _ = oracle.codec.extract([("s", [x], [x]), ("t", [x[:7]], [x[:7]])])
    y = x.copy()
    y[[0, 5, 299]] ^= 3
    one, _ = oracle.codec.extract([("s", [x], [y]), ("t", [x[:7]], [x[:7]])])
    ctx = sd.DeltaContext(DEV)
    dev = lambda b: torch.tensor(list(b), dtype=torch.uint8, device=DEV)
    for a, b in ((same, same), (same, one), (one, same), (one, one)):
        got = ctx.delta_merge(dev(a), dev(b), 2)
        torch.cuda.synchronize()
        assert_body_equal(got, oracle.codec.merge(a, b, 2))
    assert_body_equal(ctx.delta_merge(dev(one), dev(one), 2), one)
    empty = torch.empty(0, dtype=torch.uint8, device=DEV)
    assert ctx.delta_merge(empty, empty, 0).numel() == 0
    ctx.close()


def test_pipelined_round_trips_and_accumulated_timing(sd):
    """round_trip(wait=False) back to back (the host never waits between steps) ends in the
    same state as waited steps, and profiling mode 2 accumulates every step's kernel times
    (delta_timing_totals) without host synchronisation."""
    spec = m1_specs()[0]
    o, w = generate_pair(spec, 0, 5, rho=0.01, device=DEV)
    ref_body, _ = oracle_extract([(spec.name, o, w)])
    ctx = sd.DeltaContext(DEV)
    tl = sd.TensorList([(spec.name, o, w)])
    target = o.clone()
    tg = sd.TargetList([(spec.name, target)])
    out = torch.empty(len(ref_body) * 2 + 4096, dtype=torch.uint8, device=DEV)
    size = torch.zeros(1, dtype=torch.int64, device=DEV)
    assert ctx.round_trip(tl, tg, out, size) == len(ref_body)  # first call sizes the workspace
    ctx.set_profiling(2)
    for _ in range(5):
        assert ctx.round_trip(tl, tg, out, size, wait=False) is None
    assert ctx.extract_wait() == len(ref_body)
    ctx.apply_wait()
    tot, calls = ctx.timing_totals()
    assert calls == 5 and tot["scan_ms"] > 0 and tot["scatter_ms"] > 0
    assert_body_equal(out[:len(ref_body)], ref_body)
    assert_lanes_equal(target, w)
    ctx.close()
