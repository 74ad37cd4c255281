"""delta_merge (NEXT f4, reading R19) on the bench workload: two consecutive deltas of a
Qwen3-8B-shaped bf16 set at 1 % uniform (v0 -> v1 -> v2; v2 = v1 XOR the change pattern of a
second seeded pair), merged on the GPU.  Reports the merge time (CUDA events around the call,
host syncs included), the merged size, and a laggard's catch-up: applying the merge once vs
applying both deltas in turn.  One JSON line."""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="8B")
    ap.add_argument("--rho", type=float, default=0.01)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import __graft_entry__ as entry
    entry.build()
    import paper_2602_11456_b200 as sd
    from workload import generate_pair, qwen3
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    specs = qwen3(args.model)
    v0, v1, v2 = [], [], []
    for k, s in enumerate(specs):
        o, w = generate_pair(s, k, 0, rho=args.rho, device=dev)
        o2, w2 = generate_pair(s, k, 1, rho=args.rho, device=dev)
        x = (o2.view(torch.int16) ^ w2.view(torch.int16))
        del o2, w2
        v0.append(o)
        v1.append(w)
        v2.append((w.view(torch.int16) ^ x).view(torch.bfloat16))
        del x
    ctx = sd.DeltaContext(dev)
    tl01 = sd.TensorList([(s.name, a, b) for s, a, b in zip(specs, v0, v1)])
    tl12 = sd.TensorList([(s.name, a, b) for s, a, b in zip(specs, v1, v2)])
    a, ta = ctx.delta_extract(tl01)
    a = a.clone()
    b, tb = ctx.delta_extract(tl12)
    b = b.clone()
    out = torch.empty(a.numel() + b.numel(), dtype=torch.uint8, device=dev)
    n = len(specs)

    def ev(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    m = ctx.delta_merge(a, b, n, out=out)
    ts = [ev(lambda: ctx.delta_merge(a, b, n, out=out)) for _ in range(args.reps)]
    merged = m.numel()
    # laggard catch-up on a copy of v0: merged apply vs the two applies in turn
    tgt = [t.clone() for t in v0]
    tg = sd.TargetList([(s.name, t) for s, t in zip(specs, tgt)])
    ctx.delta_apply(tg, m)  # untimed: grows the apply workspace to the merged body's size
    t_two = [ev(lambda: (ctx.delta_apply(tg, a, table=ta), ctx.delta_apply(tg, b, table=tb))) for _ in range(args.reps)]
    t_one = [ev(lambda: ctx.delta_apply(tg, m)) for _ in range(args.reps)]
    for t, x in zip(tgt, v0):  # the catch-up check below starts again from v0
        t.copy_(x)
    ctx.delta_apply(tg, m)
    torch.cuda.synchronize()
    ok = all(torch.equal(t.view(torch.int16), w.view(torch.int16)) for t, w in zip(tgt, v2))
    print(json.dumps({"bench": "delta_merge", "model": args.model, "rho": args.rho,
                      "body_a": a.numel(), "body_b": b.numel(), "merged": merged,
                      "merge_ms": round(statistics.median(ts), 3),
                      "merge_input_GBps": round((a.numel() + b.numel()) / statistics.median(ts) / 1e6, 1),
                      "apply_a_then_b_ms": round(statistics.median(t_two), 3),
                      "apply_merged_ms": round(statistics.median(t_one), 3), "catch_up_equals_v2": ok,
                      "timing": "CUDA events, median of reps after one untimed call each"}),
          flush=True)


if __name__ == "__main__":
    main()
