"""Apply of one M3 body with a host table hint, a device table hint and no hint (A1 walks
the records itself): per-kernel times from the library's events (profiling mode 1) and the
whole call (torch events).  Diagnostics for the hint-less A1 walk."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import __graft_entry__ as entry
    entry.build()
    import paper_2602_11456_b200 as sd
    from workload import generate_pair, qwen3
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    specs = qwen3("8B")
    olds, news = [], []
    for k, s in enumerate(specs):
        o, w = generate_pair(s, k, 0, rho=0.01, device=dev)
        olds.append(o)
        news.append(w)
    ctx = sd.DeltaContext(dev)
    tl = sd.TensorList([(s.name, o, w) for s, o, w in zip(specs, olds, news)])
    body, table = ctx.delta_extract(tl)
    body = body.clone()
    _, dtab = ctx.delta_extract(tl, table="device")
    tg = sd.TargetList([(s.name, o) for s, o in zip(specs, olds)])
    ctx.set_profiling(True)
    for hint in ("host", "device", "none", "host", "none"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.delta_apply(tg, body, table={"host": table, "device": dtab, "none": None}[hint])
        e1.record()
        torch.cuda.synchronize()
        t = ctx.last_timing()
        print(json.dumps({"hint": hint, "call_ms": round(e0.elapsed_time(e1), 3),
                          **{k: round(t[k], 4) for k in ("locate_ms", "decode_ms", "apply_scan_ms", "scatter_ms")}}),
              flush=True)


if __name__ == "__main__":
    main()
