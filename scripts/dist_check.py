"""Multi-GPU check (run under torchrun on >= 2 GPUs): every rank extracts its contiguous
shard of a small Qwen-shaped tensor set, sizes are all-gathered over NCCL, the bodies are
assembled on rank 0 and compared byte-for-byte with (a) the single-GPU body of the whole
list and (b) the CPU oracle; every rank then applies its own records and checks the
round trip.  Exit code 0 iff all checks pass on all ranks."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    import paper_2602_11456_b200 as sd
    from paper_2602_11456_b200 import dist as sdist
    from workload import TensorSpec, generate_pair
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    specs = [TensorSpec(f"model.layers.{i}.w{j}", (shape, 512), "matrix")
             for i, shape in enumerate([64, 3000, 17, 1024, 4096, 5, 2048, 999, 300, 4000])
             for j in range(2)]
    ranges = sdist.shard_plan([s.numel for s in specs], world)
    a, b = ranges[rank]
    pairs = {k: generate_pair(specs[k], k, 7, rho=0.02, device=dev) for k in range(len(specs))}
    mine = [(specs[k].name, pairs[k][0], pairs[k][1]) for k in range(a, b)]
    ctx = sd.DeltaContext(dev)
    if mine:
        body, table = ctx.delta_extract(mine)
    else:
        body, table = torch.empty(0, dtype=torch.uint8, device=dev), []
    sizes, off, tot = sdist.gather_sizes(body.numel(), dev)
    root_out = torch.empty(max(tot, 1), dtype=torch.uint8, device=dev) if rank == 0 else None
    got = sdist.assemble(body, sizes, root_out)
    ok = True
    if rank == 0:
        full_body, full_table = ctx.delta_extract([(s.name, pairs[k][0], pairs[k][1]) for k, s in enumerate(specs)])
        ok &= torch.equal(got.cpu(), full_body.cpu())
        from gpu_helpers import oracle_extract
        ref_body, ref_table = oracle_extract([(s.name, pairs[k][0], pairs[k][1]) for k, s in enumerate(specs)])
        ok &= got.cpu().numpy().tobytes() == ref_body
        print(f"[rank0] assembled {tot} bytes from sizes {sizes}: match single-GPU and oracle = {ok}", flush=True)
    # the same assembly through the delta_assemble kernel over NVLink (CUDA IPC mapping)
    asm = sdist.NvlinkAssembler(ctx, tot + 4096, dev)
    if rank == 0 and mine:
        b0, _ = ctx.delta_extract(mine, out=asm.buf)
        body = b0
    got2 = asm.assemble(body, body.numel())
    torch.cuda.synchronize()
    ctx.assemble_wait()
    if rank == 0:
        ok2 = torch.equal(got2[:tot].cpu(), full_body.cpu())
        print(f"[rank0] NVLink delta_assemble: match = {ok2}", flush=True)
        ok &= ok2
    # flag-based assembly (no collective): three steps over two buffers
    fasm = sdist.FlagAssembler(ctx, tot + 4096, dev, nbuf=2)
    for step in range(3):
        slot = step % 2
        if rank == 0 and mine:
            bf, _ = ctx.delta_extract(mine, out=fasm.bufs[slot])
        elif mine:
            bf, _ = ctx.delta_extract(mine)
        else:
            bf = torch.empty(0, dtype=torch.uint8, device=dev)
        sz = torch.tensor([bf.numel()], dtype=torch.int64, device=dev)
        got4 = fasm.assemble(bf, sz, slot=slot)
        torch.cuda.synchronize()
        rc4 = 0
        try:
            ctx.assemble_wait()
        except Exception:
            rc4 = 1
        if rank == 0:
            ok4 = rc4 == 0 and torch.equal(got4[:tot].cpu(), full_body.cpu())
            print(f"[rank0] flag assembly step {step} slot {slot}: match = {ok4}", flush=True)
            ok &= ok4
        ok &= rc4 == 0
    fasm.close()
    # LPT partition + record-granular assembly (delta_record_sizes / delta_assemble_records)
    lpt = sdist.shard_lpt([s.numel for s in specs], world)[rank]
    mine_l = [(specs[k].name, pairs[k][0], pairs[k][1]) for k in lpt]
    rasm = sdist.RecordAssembler(ctx, tot + 4096, dev, lpt, len(specs))
    for slot in (0, 1):
        if mine_l:
            bl, _ = ctx.delta_extract(mine_l, table="device")
        else:
            bl = torch.empty(0, dtype=torch.uint8, device=dev)
            rasm.sizes[slot].zero_()
        if mine_l:
            rasm.record_sizes(ctx.table_dev_ptr(), slot=slot)
        got3 = rasm.assemble(bl, slot=slot)
        torch.cuda.synchronize()
        ctx.assemble_wait()
        if rank == 0:
            ok3 = torch.equal(got3[:tot].cpu(), full_body.cpu())
            print(f"[rank0] LPT {[len(p) for p in sdist.shard_lpt([s.numel for s in specs], world)]} "
                  f"record assembly slot {slot}: match = {ok3}", flush=True)
            ok &= ok3
    rasm.close()
    # LPT + record assembly through the root's board (no collective)
    rfa = sdist.RecordAssembler(ctx, tot + 4096, dev, lpt, len(specs), mode="flags")
    for step in range(3):
        slot = step % 2
        if mine_l:
            bl, _ = ctx.delta_extract(mine_l, table="device")
            rfa.record_sizes(ctx.table_dev_ptr(), slot=slot)
        else:
            bl = torch.empty(0, dtype=torch.uint8, device=dev)
            rfa.sizes[slot].zero_()
        got5 = rfa.assemble(bl, slot=slot)
        torch.cuda.synchronize()
        rc5 = 0
        try:
            ctx.assemble_wait()
        except Exception:
            rc5 = 1
        if rank == 0:
            ok5 = rc5 == 0 and torch.equal(got5[:tot].cpu(), full_body.cpu())
            print(f"[rank0] LPT record flags assembly step {step} slot {slot}: match = {ok5}", flush=True)
            ok &= ok5
        ok &= rc5 == 0
    rfa.close()
    if mine:
        targets = [(n, o.clone()) for n, o, _ in mine]
        ctx.delta_apply(targets, body, table=table)
        for (_, t), (_, _, w) in zip(targets, mine):
            ok &= torch.equal(t.view(torch.int16), w.view(torch.int16))
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    ctx.close()
    dist.destroy_process_group()
    return int(flag.item() != 0)


if __name__ == "__main__":
    sys.exit(main())
