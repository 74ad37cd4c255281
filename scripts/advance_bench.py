"""Extract-and-advance cost (NEXT f3) on the bench workload (default M3: Qwen3-8B bf16, 1 %
uniform): K1 time with DELTA_OPT_ADVANCE off vs on, beside the two ways a trainer would
otherwise advance its shadow copy W_t -> W_{t+1}: a full device copy of new into old, or
applying the body to the shadow (the actor-side apply).  CUDA events (the library's K1
events; torch events on the current stream for copy_ / apply).  One JSON line per variant."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="8B")
    ap.add_argument("--rho", type=float, default=0.01)
    ap.add_argument("--pattern", default="uniform")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import __graft_entry__ as entry
    entry.build()
    import paper_2602_11456_b200 as sd
    from paper_2602_11456_b200 import _abi
    from workload import generate_pair, qwen3
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    specs = qwen3(args.model)
    olds, news, pristine = [], [], []
    for k, s in enumerate(specs):
        o, w = generate_pair(s, k, 0, rho=args.rho, pattern=args.pattern, device=dev)
        olds.append(o)
        news.append(w)
        pristine.append(o.clone())
    tensors = [(s.name, o, w) for s, o, w in zip(specs, olds, news)]
    lanes = sum(s.numel for s in specs)

    def restore():
        for o, p in zip(olds, pristine):
            o.copy_(p)
        torch.cuda.synchronize()

    def ev_time(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    out = {}
    for adv in (1, 2):
        ctx = sd.DeltaContext(dev)
        ctx.set_option(_abi.DELTA_OPT_ADVANCE, adv)
        ctx.set_profiling(True)
        ts = []
        for r in range(args.reps + 2):
            restore()
            ctx.delta_size(sd.TensorList(tensors))
            if r >= 2:
                ts.append(ctx.last_timing()["scan_ms"])
            if adv == 2:
                assert all(torch.equal(o.view(torch.int16), w.view(torch.int16)) for o, w in zip(olds, news))
        out[adv] = sum(ts) / len(ts)
        print(json.dumps({"variant": "k1_advance" if adv == 2 else "k1_plain", "k1_ms": round(out[adv], 4),
                          "scanned_GBps": round(2 * lanes * 2 / out[adv] / 1e6, 1)}), flush=True)
        ctx.close()
    restore()
    ts = [ev_time(lambda: [o.copy_(w) for o, w in zip(olds, news)]) for _ in range(args.reps)]
    print(json.dumps({"variant": "shadow_copy_new_to_old", "ms": round(sum(ts) / len(ts), 4)}), flush=True)
    restore()
    ctx = sd.DeltaContext(dev)
    body, table = ctx.delta_extract(sd.TensorList(tensors))
    tg = sd.TargetList([(s.name, o) for s, o in zip(specs, olds)])
    ts = [ev_time(lambda: ctx.delta_apply(tg, body, table=table)) for _ in range(args.reps)]
    print(json.dumps({"variant": "shadow_apply_body", "ms": round(sum(ts) / len(ts), 4)}), flush=True)
    print(json.dumps({"summary": "advance adds %.3f ms to K1" % (out[2] - out[1])}), flush=True)


if __name__ == "__main__":
    main()
