"""Pipelined extract + apply of one weight set on one GPU (the in-box analog of the paper's
"pipelines extraction with cut-through forwarding").

The tensor list is split into G contiguous groups (balanced by lanes, the same partition
as the multi-GPU sharding, dist.shard_plan).  Because records are self-contained and
appear in list order (R4, R15), the bodies of consecutive groups written back to
back ARE the body of the whole list.  Group g is extracted on the extract stream; as soon
as its records are written, its apply is enqueued on the apply stream (delta_apply_async),
so the scatter of group g — bound by DRAM row activations, not bandwidth — overlaps the
streaming compare of group g+1.  One delta_apply_wait at the end reports the first error.

Everything still runs in the library's kernels; this module only orders calls on streams.
"""

import torch

from . import _abi
from .binding import DeltaContext, TargetList, TensorList, rebase
from .dist import shard_plan


class RoundTrip:
    """extract(old, new) -> body; apply(body) onto ``targets``, as G pipelined groups.

    tensors: [(name, old, new)] (old/new CUDA tensors or span lists); targets:
    [(name, w)] in the same order; groups: G >= 1 (G = 1 is the plain sequential path).
    """

    def __init__(self, tensors, targets, groups=8, device=None, apply_ctas_per_sm=None,
                 apply_priority=-1, scan_kernel=None):
        assert len(tensors) == len(targets)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        numels = [sum(x.numel() for x in ([o] if isinstance(o, torch.Tensor) else o))
                  for _, o, _ in tensors]
        ranges = [r for r in shard_plan(numels, max(1, min(groups, len(tensors)))) if r[1] > r[0]]
        self.groups = [(TensorList(tensors[a:b]), TargetList(targets[a:b])) for a, b in ranges]
        # one extract context per group: each caches its own plan (tile table) and slots
        self.cxs = [DeltaContext(self.device) for _ in self.groups]
        self.cx = self.cxs[0]
        if scan_kernel:
            for cx in self.cxs:
                cx.set_option(_abi.DELTA_OPT_SCAN_KERNEL, scan_kernel)
        self.ca = DeltaContext(self.device)
        if apply_ctas_per_sm:
            self.ca.set_option(_abi.DELTA_OPT_APPLY_CTAS_PER_SM, apply_ctas_per_sm)
        self.sx = torch.cuda.Stream(self.device)
        self.sa = torch.cuda.Stream(self.device, priority=apply_priority)
        sizes = [cx.delta_size(tl, stream=self.sx) for cx, (tl, _) in zip(self.cxs, self.groups)]
        total = sum(sizes)
        self.out = torch.empty(total + total // 8 + 4096, dtype=torch.uint8, device=self.device)
        self.tables = None
        self.body_bytes = 0

    def set_profiling(self, on: bool):
        for cx in self.cxs:
            cx.set_profiling(on)
        self.ca.set_profiling(on)

    def step(self, timing=None):
        """One extract + apply of the whole set.  Returns the body (uint8 view of ``out``)."""
        cur = torch.cuda.current_stream(self.device)
        self.sx.wait_stream(cur)
        self.sa.wait_stream(cur)
        off, tables = 0, []
        for cx, (tl, tg) in zip(self.cxs, self.groups):
            size = cx.delta_size(tl, stream=self.sx)
            if timing is not None:
                t = cx.last_timing()
                for k in ("scan_ms", "lens_ms", "finalize_ms"):
                    timing[k] = timing.get(k, 0.0) + t[k]
            if off + size > self.out.numel():
                raise RuntimeError("body buffer too small (weights changed density?)")
            body, table = cx.delta_extract(tl, out=self.out[off:], stream=self.sx, table=True)
            if timing is not None:
                t = cx.last_timing()
                for k in ("emit_ms", "headers_ms"):
                    timing[k] = timing.get(k, 0.0) + t[k]
            ev = torch.cuda.Event()
            ev.record(self.sx)
            self.sa.wait_event(ev)
            self.ca.delta_apply(tg, body, table=table, stream=self.sa, wait=False)
            tables.append((off, table))
            off += size
        self.ca.apply_wait(stream=self.sa)
        cur.wait_stream(self.sx)
        cur.wait_stream(self.sa)
        self.tables, self.body_bytes = tables, off
        return self.out[:off]

    def table(self):
        """Offset table of the whole body (rows shifted to global offsets)."""
        rows = []
        for off, tab in self.tables or []:
            rows += list(rebase(tab, off))
        return rows

    def close(self):
        for cx in self.cxs:
            cx.close()
        self.ca.close()
