"""GPU tests of boundary calls beyond extract/apply, against the oracle:

* delta_digest against the official BLAKE3 known-answer vectors (tests/golden/blake3_kat.txt;
  reading R10);
* the multi-GPU assembly kernels on ONE GPU into a local destination (S3):
  delta_assemble (contiguous shards), delta_record_sizes + delta_assemble_records (any
  partition), each body byte-equal to the oracle's whole-list body; the capacity gate and a
  closed extract gate (~0 size) write nothing;
* extract-and-advance across DELTA_ECAPACITY (the retry emits the same body);
* compute_rho refused on an advancing context; the sticky outcome of several async
  extracts (an earlier call's overflow is reported at the wait).
"""

import numpy as np
import pytest
import torch

import oracle
from conftest import golden_lines
from gpu_helpers import assert_body_equal, assert_lanes_equal, oracle_extract
from workload import TensorSpec, generate_pair

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def sd():
    import __graft_entry__ as entry
    entry.build()
    import paper_2602_11456_b200 as m
    torch.cuda.set_device(DEV)
    return m


def _tensors(n_list, seed=3, rho=0.01):
    out = []
    for k, n in enumerate(n_list):
        spec = TensorSpec(f"layer.{k}.weight", (n,), "matrix")
        o, w = generate_pair(spec, k, seed, rho=rho, device=DEV)
        out.append((spec.name, o, w))
    return out


def test_digest_known_answers(sd):
    ctx = sd.DeltaContext(DEV)
    for ln in golden_lines("blake3_kat.txt"):
        n, h = ln.split()
        data = torch.tensor([i % 251 for i in range(int(n))], dtype=torch.uint8, device=DEV)
        assert ctx.digest(data) == bytes.fromhex(h), n
    ctx.close()


def test_assemble_contiguous_local(sd):
    """Three simulated ranks with contiguous shards: ranks 1, 2 copy their bodies into rank
    0's buffer at the offsets delta_assemble computes from the sizes on the device."""
    tensors = _tensors([300_001, 70_000, 1_000_003, 5, 0, 250_000, 33])
    want, _ = oracle_extract(tensors)
    shards = [tensors[0:2], tensors[2:5], tensors[5:]]
    ctx = sd.DeltaContext(DEV)
    bodies = [ctx.delta_extract(sh, table=False)[0].clone() for sh in shards]
    sizes = torch.tensor([b.numel() for b in bodies], dtype=torch.int64, device=DEV)
    dst = torch.full((len(want) + 100,), 0xEE, dtype=torch.uint8, device=DEV)
    dst[:bodies[0].numel()].copy_(bodies[0])
    for r in (1, 2):
        ctx.assemble(bodies[r], dst, sizes, r)
    ctx.assemble_wait()
    assert_body_equal(dst[:len(want)], want)
    assert bool((dst[len(want):] == 0xEE).all())
    # capacity gate: a destination one byte short takes nothing from rank 2
    small = torch.full((len(want) - 1,), 0x11, dtype=torch.uint8, device=DEV)
    ctx.assemble(bodies[2], small, sizes, 2)
    with pytest.raises(sd.DeltaError) as e:
        ctx.assemble_wait()
    assert e.value.status == sd._abi.DELTA_ECAPACITY
    assert bool((small == 0x11).all())
    # a closed extract gate (~0 size) on an earlier rank: nothing is written
    bad = sizes.clone()
    bad[0] = -1
    ctx.assemble(bodies[1], small, bad, 1)
    with pytest.raises(sd.DeltaError):
        ctx.assemble_wait()
    assert bool((small == 0x11).all())
    ctx.close()


def test_assemble_records_any_partition(sd):
    """An interleaved (LPT-like) partition over two simulated ranks: each rank's record
    sizes scattered into global order (delta_record_sizes), summed, then every local record
    copied to its global offset (delta_assemble_records)."""
    tensors = _tensors([200_000, 1_000_003, 17, 0, 640_000, 999])
    want, want_table = oracle_extract(tensors)
    parts = [[0, 2, 3], [1, 4, 5]]
    ctx = [sd.DeltaContext(DEV) for _ in parts]
    n = len(tensors)
    bodies, sizes = [], []
    for c, p in zip(ctx, parts):
        body, dt = c.delta_extract([tensors[k] for k in p], table="device")
        gidx = torch.tensor(p, dtype=torch.int32, device=DEV)
        s = torch.full((n,), 77, dtype=torch.int64, device=DEV)
        c.record_sizes(dt.ptr, len(p), gidx, s)
        bodies.append((body.clone(), gidx))
        sizes.append(s)
    torch.cuda.synchronize()
    for s, p in zip(sizes, parts):  # own entries = record sizes, every other entry 0
        got = s.tolist()
        for k in range(n):
            assert got[k] == (want_table[k][6] if k in p else 0)
    total = sizes[0] + sizes[1]
    dst = torch.full((len(want),), 0xEE, dtype=torch.uint8, device=DEV)
    for c, (body, gidx) in zip(ctx, bodies):
        c.assemble_records(body, gidx, total, dst)
        c.assemble_wait()
    assert_body_equal(dst, want)
    # capacity gate: nothing written
    small = torch.full((len(want) - 1,), 0x11, dtype=torch.uint8, device=DEV)
    ctx[1].assemble_records(bodies[1][0], bodies[1][1], total, small)
    with pytest.raises(sd.DeltaError):
        ctx[1].assemble_wait()
    assert bool((small == 0x11).all())
    for c in ctx:
        c.close()


def test_advance_survives_ecapacity(sd):
    """DELTA_OPT_ADVANCE: a delta_extract that fails with ECAPACITY keeps its compaction (old
    already equals new), so the retry with a large enough buffer emits the oracle's body."""
    from paper_2602_11456_b200 import _abi
    tensors = _tensors([1_000_003, 4096, 77_777], seed=11, rho=0.02)
    want, want_table = oracle_extract(tensors)
    keep = [o.clone() for _, o, _ in tensors]
    ctx = sd.DeltaContext(DEV)
    ctx.set_option(_abi.DELTA_OPT_ADVANCE, 2)
    with pytest.raises(sd.DeltaError) as e:
        ctx.delta_extract(tensors, out=torch.empty(16, dtype=torch.uint8, device=DEV))
    assert e.value.status == _abi.DELTA_ECAPACITY
    for (_, o, w) in tensors:  # advanced already
        assert_lanes_equal(o, w)
    body, table = ctx.delta_extract(tensors, out=torch.empty(len(want) + 8, dtype=torch.uint8, device=DEV))
    assert_body_equal(body, want)
    assert [tuple(r) for r in table] == [tuple(r) for r in want_table]
    targets = [(n, k) for (n, _, _), k in zip(tensors, keep)]
    ctx.delta_apply(targets, body, table=table)
    torch.cuda.synchronize()
    for (_, t), (_, _, w) in zip(targets, tensors):
        assert_lanes_equal(t, w)
    with pytest.raises(sd.DeltaError) as e:  # compute_rho would overwrite old: refused
        ctx.compute_rho(tensors)
    assert e.value.status == _abi.DELTA_EINVAL
    ctx.close()


def test_compute_rho_in_library(sd):
    """delta_compute_rho: rho and the per-tensor counts equal the oracle's Eq. 1."""
    tensors = _tensors([100_000, 5000, 0, 31], seed=5, rho=0.03)
    ctx = sd.DeltaContext(DEV)
    rho, nnz = ctx.compute_rho(tensors)
    pairs = [(o.view(torch.int16).cpu().numpy().view(np.uint16), w.view(torch.int16).cpu().numpy().view(np.uint16))
             for _, o, w in tensors]
    assert rho == oracle.codec.rho(pairs)
    assert nnz == [int((a != b).sum()) for a, b in pairs]
    ctx.close()


def test_async_extract_sticky_overflow(sd):
    """Two async extracts before one wait: the first overflows the tile slots (a new, higher
    density), the second fits.  The wait reports EAGAIN (not just the last call's state)."""
    from paper_2602_11456_b200 import _abi
    dense = _tensors([2_000_000], seed=21, rho=0.5)
    sparse = _tensors([2_000_000], seed=22, rho=0.001)
    ctx = sd.DeltaContext(DEV)
    out = torch.empty(8 << 20, dtype=torch.uint8, device=DEV)
    size = torch.zeros(1, dtype=torch.int64, device=DEV)
    ctx.delta_extract_async(dense, out, size)
    ctx.delta_extract_async(sparse, out, size)
    with pytest.raises(sd.DeltaError) as e:
        ctx.extract_wait()
    assert e.value.status == _abi.DELTA_EAGAIN
    # after the wait the sticky state is cleared and the slots are grown: both succeed
    ctx.delta_extract_async(dense, out, size)
    n = ctx.extract_wait()
    want, _ = oracle_extract(dense)
    assert n == len(want)
    assert_body_equal(out[:n], want)
    ctx.delta_extract_async(sparse, out[:16], size)  # too small: ECAPACITY, nothing written
    with pytest.raises(sd.DeltaError) as e:
        ctx.extract_wait()
    assert e.value.status == _abi.DELTA_ECAPACITY
    ctx.close()


@pytest.mark.parametrize("prefix", [0, 1, 2, 3, 5, 4096 + 7])
def test_fused_emit_peer_destination(sd, prefix):
    """delta_extract_scan_async + delta_extract_emit_async with a peer destination (here a
    local buffer standing in for the root's IPC mapping): the body lands in out AND at
    sum(sizes[:rank]) of the peer buffer, for every alignment of that offset; the bytes
    around it are untouched; a ~0 size of another rank or a short peer buffer skips the peer
    copy (local body still written) and is reported by extract_wait."""
    from paper_2602_11456_b200 import _abi
    tensors = _tensors([300_001, 17, 0, 65_536 * 3 + 5], seed=prefix + 40, rho=0.02)
    want, _ = oracle_extract(tensors)
    ctx = sd.DeltaContext(DEV)
    out = torch.empty(len(want) + 64, dtype=torch.uint8, device=DEV)
    size = torch.zeros(1, dtype=torch.int64, device=DEV)
    peer = torch.full((prefix + len(want) + 99,), 0x5A, dtype=torch.uint8, device=DEV)
    ctx.delta_extract_scan_async(tensors, size)
    torch.cuda.synchronize()
    assert int(size.item()) == len(want)
    sizes = torch.tensor([prefix, len(want), 12345], dtype=torch.int64, device=DEV)
    ctx.delta_extract_emit_async(out, size, peer=peer, sizes=sizes, rank=1)
    assert ctx.extract_wait() == len(want)
    assert_body_equal(out[:len(want)], want)
    assert_body_equal(peer[prefix:prefix + len(want)], want)
    assert bool((peer[:prefix] == 0x5A).all()) and bool((peer[prefix + len(want):] == 0x5A).all())
    # another rank's extract did not complete (~0 size): no peer copy, EAGAIN at the wait
    peer.fill_(0x5A)
    bad = sizes.clone()
    bad[2] = -1
    ctx.delta_extract_scan_async(tensors, size)
    ctx.delta_extract_emit_async(out, size, peer=peer, sizes=bad, rank=1)
    with pytest.raises(sd.DeltaError) as e:
        ctx.extract_wait()
    assert e.value.status == _abi.DELTA_EAGAIN
    assert bool((peer == 0x5A).all())
    assert_body_equal(out[:len(want)], want)
    # the peer buffer one byte short: no peer copy, ECAPACITY
    short = peer[:prefix + len(want) - 1]
    ctx.delta_extract_scan_async(tensors, size)
    ctx.delta_extract_emit_async(out, size, peer=short, sizes=sizes, rank=1)
    with pytest.raises(sd.DeltaError) as e:
        ctx.extract_wait()
    assert e.value.status == _abi.DELTA_ECAPACITY
    assert bool((peer == 0x5A).all())
    ctx.close()
