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
