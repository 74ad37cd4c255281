"""Calibration microbenchmarks on the GPU box (not part of the product): read roofline and
scatter-store variants at 1 % uniform density into a Qwen3-8B-sized (16.4 GB) buffer.
Prints one JSON line per measurement; results summarised in profiles/."""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmembench.so")


def build():
    src = os.path.join(HERE, "membench.cu")
    if not os.path.exists(SO) or os.path.getmtime(src) > os.path.getmtime(SO):
        subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
                        "-shared", "-o", SO, src], check=True)
    return ctypes.CDLL(SO)


def timeit(fn, reps=5):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    L = build()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    n = 8_190_735_360  # Qwen3-8B lanes
    buf = torch.empty(2 * n, dtype=torch.uint8, device="cuda")
    buf.random_(0, 255)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    for grid_mul, block in (() if os.environ.get("MB_SCATTER") else ((4, 512), (8, 256), (16, 256), (32, 256))):
        ms = timeit(lambda: L.mb_read(ctypes.c_void_p(buf.data_ptr()), ctypes.c_size_t(buf.numel()),
                                      ctypes.c_void_p(out.data_ptr()), sm * grid_mul, block, st))
        print(json.dumps({"bench": "read", "grid": sm * grid_mul, "block": block, "ms": ms,
                          "GBps": buf.numel() / ms / 1e6}), flush=True)
    # sorted uniform 1 % positions
    g = torch.Generator(device="cuda").manual_seed(0)
    m = torch.rand(n, device="cuda", generator=g) < 0.01 if False else None
    pos_chunks = []
    step = 1 << 28
    for s0 in range(0, n, step):
        e = min(n, s0 + step)
        r = torch.rand(e - s0, device="cuda", generator=g)
        pos_chunks.append(torch.nonzero(r < 0.01).flatten() + s0)
        del r
    pos = torch.cat(pos_chunks).to(torch.int64)
    del pos_chunks
    val = torch.randint(0, 65535, (pos.numel(),), dtype=torch.int32, device="cuda").to(torch.int16)
    w = buf.view(torch.int16)
    only = os.environ.get("MB_SCATTER")
    variants = ((0, "plain"), (1, "prefetch_L2"), (2, "sector_merge"), (3, "batch_sector_rmw"),
                (4, "batch_sector_rmw_noL1"), (5, "plain_evict_first"), (6, "plain_evict_last"))
    init = w.clone()
    ref = None
    for variant, name in variants:
        if only and str(variant) not in only.split(","):
            continue
        shapes = ((8, 256), (32, 256)) if variant < 3 or variant > 4 else ((16, 128), (64, 128))
        for grid_mul, block in shapes:
            def run():
                return L.mb_scatter(variant, ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(pos.data_ptr()),
                                    ctypes.c_void_p(val.data_ptr()), ctypes.c_size_t(pos.numel()),
                                    sm * grid_mul, block, st)
            w.copy_(init)
            run()
            torch.cuda.synchronize()
            if ref is None:
                ref = w.clone()
                ok = True
            else:
                ok = bool(torch.equal(w, ref))
            ms = timeit(run)
            print(json.dumps({"bench": f"scatter_{name}", "entries": pos.numel(), "grid": sm * grid_mul,
                              "block": block, "ms": ms, "matches_plain": ok,
                              "Gstores_per_s": pos.numel() / ms / 1e6}), flush=True)

if __name__ == "__main__":
    sys.exit(main())
