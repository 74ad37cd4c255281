"""Scatter-store probe (calibration, not product): how the 1 % uniform apply pattern uses HBM.

Decomposes the scatter's DRAM work into its parts on the same sorted positions (81.9 M
uniform 1 % lanes of a Qwen3-8B-sized 16.4 GB buffer):
  plain        one thread per entry, grid-stride (the shape of A4's stores)
  window/G/U   the whole grid sweeps the entries together (warp w of W takes entries
               [(kW + w) 32, +32)), so the stores in flight span about W x 32 entries:
               tests whether DRAM row locality (a narrow address window) lifts the rate
  gather       2-byte loads of the same lanes (the L2 fills alone)
  sector_read  whole 32-byte loads of every touched sector
  sector_write whole 32-byte stores of every touched sector (the write-backs alone, no fill)
One JSON line per measurement.  Run under ncu with -k regex:"k_scatter|k_gather|k_sector" for
the DRAM counters (dram__cycles_active vs dram__bytes)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from membench import build, timeit  # noqa: E402


def main():
    L = build()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    reps = int(os.environ.get("PROBE_REPS", "5"))
    n = 8_190_735_360
    w = torch.empty(n, dtype=torch.int16, device="cuda")
    w.random_(-32768, 32767)
    g = torch.Generator(device="cuda").manual_seed(0)
    chunks = []
    for s0 in range(0, n, 1 << 28):
        e = min(n, s0 + (1 << 28))
        r = torch.rand(e - s0, device="cuda", generator=g)
        chunks.append(torch.nonzero(r < 0.01).flatten() + s0)
        del r
    pos = torch.cat(chunks).to(torch.int64)
    del chunks
    val = torch.randint(0, 65535, (pos.numel(),), dtype=torch.int32, device="cuda").to(torch.int16)
    sec = torch.unique_consecutive(pos >> 4)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    P, V, S, O, Wp = (ctypes.c_void_p(t.data_ptr()) for t in (pos, val, sec, out, w))
    ne, ns = ctypes.c_size_t(pos.numel()), ctypes.c_size_t(sec.numel())
    base = {"entries": pos.numel(), "sectors": sec.numel(), "buffer_bytes": 2 * n}

    def emit(name, ms, **kw):
        print(json.dumps({"bench": name, "ms": round(ms, 4), **kw, **base}), flush=True)

    ref = None
    only = os.environ.get("PROBE_ONLY", "")
    cases = [("plain", 0, sm * 32, 256), ("plain", 0, sm * 8, 256)]
    for wpb, ctas in ((2, 1), (8, 1), (8, 2), (8, 4), (8, 8), (8, 32)):
        cases.append((f"window_u4", 7, sm * ctas, 32 * wpb))
    cases.append(("window_u1", 8, sm * 8, 256))
    for name, variant, grid, block in cases:
        if only and name not in only:
            continue
        run = lambda: L.mb_scatter(variant, Wp, P, V, ne, grid, block, st)  # noqa: E731
        ms = timeit(run, reps)
        if ref is None:
            ref = w.clone()
            ok = True
        else:
            ok = bool(torch.equal(w, ref))
        window = grid * (block // 32) * 32 if variant in (7, 8) else grid * block
        emit(f"scatter_{name}", ms, grid=grid, block=block, window_entries=window,
             window_mb=round(window * 200 / 1e6, 1), same_result=ok, Gstores_per_s=round(pos.numel() / ms / 1e6, 2))
    if not only or "gather" in only:
        for grid in (sm * 8, sm * 32):
            ms = timeit(lambda: L.mb_gather(Wp, P, ne, O, grid, 256, st), reps)
            emit("gather_u16", ms, grid=grid, block=256, sector_GBps=round(sec.numel() * 32 / ms / 1e6, 1))
    if not only or "sector" in only:
        for wr in (0, 1):
            for grid in (sm * 8, sm * 32):
                ms = timeit(lambda: L.mb_sector(wr, Wp, S, ns, O, grid, 256, st), reps)
                emit("sector_write" if wr else "sector_read", ms, grid=grid, block=256,
                     GBps=round(sec.numel() * 32 / ms / 1e6, 1))


if __name__ == "__main__":
    sys.exit(main())
