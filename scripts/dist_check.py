"""Multi-GPU check (run under torchrun on >= 2 GPUs): every rank extracts its contiguous
shard of a small Qwen-shaped tensor set, sizes are all-gathered over NCCL, the bodies are
assembled on rank 0 — NCCL P2P, the delta_assemble copy kernel over NVLink, and the fused
emit (K4/K5 storing each rank's records at their global offsets in rank 0's buffer) — and
compared byte-for-byte with (a) the single-GPU body of the whole list and (b) the CPU oracle;
every rank then applies its own records and checks the round trip.  Exit code 0 iff all
checks pass on all ranks."""
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
    del got2
    asm.close()  # consumers drop their IPC mappings before the root may free its buffer
    # the fused emit + assembly: scan, size all-gather, emit into the local body AND straight
    # into rank 0's buffer at the global offset (three steps over two root buffers)
    fu = sdist.FusedAssembler(ctx, tot + 4096, dev, nbuf=2)
    comm = torch.cuda.Stream(dev)
    local = torch.empty(max(body.numel(), 1) + 4096, dtype=torch.uint8, device=dev)
    size = torch.zeros(1, dtype=torch.int64, device=dev)
    for step in range(3):
        slot = step % 2
        if rank == 0:
            fu.bufs[slot].fill_(0xEE)
            torch.cuda.synchronize()
        dist.barrier()
        buf, dtab = fu.extract(mine, local, size, slot=slot)
        comm.wait_stream(torch.cuda.current_stream())
        fu.token(comm)
        torch.cuda.current_stream().wait_stream(comm)
        torch.cuda.synchronize()
        rc6 = 0
        try:
            n6 = ctx.extract_wait()
        except Exception as e:  # noqa: BLE001
            print(f"[rank{rank}] fused extract_wait: {e}", flush=True)
            rc6, n6 = 1, -1
        ok &= rc6 == 0 and n6 == body.numel() and torch.equal(buf[:n6], body[:n6])
        if rank == 0:
            ok6 = rc6 == 0 and torch.equal(fu.bufs[slot][:tot].cpu(), full_body.cpu())
            print(f"[rank0] fused emit + NVLink assembly step {step} slot {slot}: match = {ok6}", flush=True)
            ok &= ok6
    fu.close()
    # a destination too small for the last rank: the peer copy is skipped and reported
    fu2 = sdist.FusedAssembler(ctx, max(tot - 1, 1), dev, nbuf=1)
    if rank == 0:
        fu2.bufs[0].fill_(0x11)
        torch.cuda.synchronize()
    dist.barrier()
    fu2.extract(mine, local, size, slot=0)
    fu2.token(torch.cuda.current_stream())
    torch.cuda.synchronize()
    failed = False
    try:
        ctx.extract_wait()
    except Exception:  # noqa: BLE001
        failed = True
    if rank == world - 1:
        ok &= failed or not mine  # the last rank's records end past tot - 1
        print(f"[rank{rank}] fused assembly into a short buffer reported: {failed}", flush=True)
    fu2.close()
    # any partition (LPT): record sizes all-reduced, record-by-record NVLink copies (rank 0 too)
    lpt = sdist.shard_lpt([s.numel for s in specs], world)[rank]
    lmine = [(specs[k].name, pairs[k][0], pairs[k][1]) for k in lpt]
    cx2 = sd.DeltaContext(dev)
    rsm = sdist.RecordAssembler(cx2, tot + 4096, dev, lpt, len(specs), nbuf=1)
    if lmine:
        lbody, _ = cx2.delta_extract(lmine, table="device")
    else:
        lbody = torch.empty(0, dtype=torch.uint8, device=dev)
    if rank == 0:
        rsm.bufs[0].fill_(0xEE)
        torch.cuda.synchronize()
    dist.barrier()
    rsm.record_sizes(0)
    got3 = rsm.assemble(lbody, 0)
    torch.cuda.synchronize()
    cx2.assemble_wait()
    if rank == 0:
        ok3 = torch.equal(got3[:tot].cpu(), full_body.cpu())
        print(f"[rank0] LPT partition {[len(p) for p in sdist.shard_lpt([s.numel for s in specs], world)]} "
              f"records per rank, delta_assemble_records over NVLink: match = {ok3}", flush=True)
        ok &= ok3
    del got3
    rsm.close()
    cx2.close()
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
