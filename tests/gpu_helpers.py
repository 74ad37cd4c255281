"""Helpers for the -m gpu parity tests: move lanes to numpy, run the oracle on the same
inputs, compare element by element (bytes of the body, rows of the table, lanes of the
reconstructed weights — always on integer views, never float ==)."""

import numpy as np
import torch

import oracle


def lane_view(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.int16 if t.element_size() == 2 else torch.int32)


def to_np(t: torch.Tensor) -> np.ndarray:
    a = lane_view(t).detach().cpu().numpy()
    return a.view(np.uint16 if t.element_size() == 2 else np.uint32)


def as_list(x):
    return [x] if isinstance(x, torch.Tensor) else list(x)


def oracle_extract(tensors):
    """tensors: [(name, old or [spans], new or [spans])] on any device."""
    return oracle.codec.extract([(n, [to_np(s) for s in as_list(o)], [to_np(s) for s in as_list(w)])
                                 for n, o, w in tensors])


def fused(x):
    xs = as_list(x)
    return xs[0] if len(xs) == 1 else torch.cat([s.reshape(-1) for s in xs])


def assert_body_equal(got: torch.Tensor, want: bytes):
    g = got.cpu().numpy()
    w = np.frombuffer(want, dtype=np.uint8)
    assert g.size == w.size, f"body size {g.size} != oracle {w.size}"
    if not np.array_equal(g, w):
        bad = np.flatnonzero(g != w)
        raise AssertionError(f"{bad.size} body bytes differ; first at {bad[0]}: "
                             f"got {g[bad[0]:bad[0] + 8].tolist()} want {w[bad[0]:bad[0] + 8].tolist()}")


def assert_lanes_equal(a: torch.Tensor, b: torch.Tensor):
    assert a.numel() == b.numel()
    assert torch.equal(lane_view(a.reshape(-1)), lane_view(b.reshape(-1)))


# ---------------------------------------------------------------- full-size oracle parity
# The workers are forked after the host copies are made: they inherit the arrays (no
# pickling of GB-sized inputs) and never touch CUDA.
_FULL = None


def _full_task(k):
    names, olds, news, body, table, mode = _FULL
    r = table[k]
    want = oracle.codec.record(names[k], olds[k], news[k], mode=mode)
    got = body[r[0]:r[0] + r[6]].tobytes()
    if got == want and oracle.codec.table_row(r[0], want) == tuple(r):
        return k, None
    n = min(len(got), len(want))
    bad = next((i for i in range(n) if got[i] != want[i]), n)
    return k, f"record {k} ({names[k]}): {len(got)} vs {len(want)} bytes, first difference at {bad}"


def oracle_check_all(tensors, body: torch.Tensor, table, group_bytes: int = 12 << 30, mode: int = 0):
    """Every record of ``body`` (uint8 CUDA tensor) and every offset-table row against
    oracle.codec.record / table_row of the same tensor, in tensor groups of at most
    ``group_bytes`` of host copies, over all host cores.  Returns the number of records
    checked; raises AssertionError listing the first mismatches."""
    import multiprocessing as mp
    import os
    import warnings
    global _FULL
    rows = [tuple(r) for r in table]
    assert len(rows) == len(tensors)
    off = 0
    for r in rows:
        assert r[0] == off, f"table rows do not tile the body at {off}"
        off += r[6]
    assert off == body.numel(), f"table covers {off} bytes, body has {body.numel()}"
    body_np = body.cpu().numpy()
    procs = max(1, len(os.sched_getaffinity(0)))
    errors, checked, k0 = [], 0, 0
    while k0 < len(tensors):
        k1, acc = k0, 0
        while k1 < len(tensors) and (k1 == k0 or acc + 2 * fused(tensors[k1][1]).numel() * 4 <= group_bytes):
            acc += 2 * fused(tensors[k1][1]).numel() * 4
            k1 += 1
        names = {k: tensors[k][0] for k in range(k0, k1)}
        olds = {k: to_np(fused(tensors[k][1])) for k in range(k0, k1)}
        news = {k: to_np(fused(tensors[k][2])) for k in range(k0, k1)}
        _FULL = (names, olds, news, body_np, rows, mode)
        with warnings.catch_warnings():  # the forked workers run numpy only (no CUDA, no threads)
            warnings.simplefilter("ignore", DeprecationWarning)
            with mp.get_context("fork").Pool(min(procs, k1 - k0)) as pool:
                for k, err in pool.imap_unordered(_full_task, range(k0, k1)):
                    checked += 1
                    if err:
                        errors.append(err)
        _FULL = None
        del olds, news
        k0 = k1
    assert not errors, f"{len(errors)} records differ from the oracle: {errors[:5]}"
    return checked
