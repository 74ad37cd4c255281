"""Tensor-granular sharding of the delta path across the GPUs of one box.

S1  ``shard_plan``: a deterministic partition of the tensor list into G contiguous ranges
    (identical on every rank) that minimises the largest shard in bytes.  Contiguous
    ranges keep each rank's records one contiguous byte range of the global body, because
    records are self-contained (the gap chain restarts per tensor, reading R4) and appear
    in list order (R15): the global body is the concatenation of the rank bodies.
S2  ``gather_sizes``: all-gather of every rank's body size (one int64 per rank) over the
    process group (NCCL on GPUs) -> each rank's byte offset in the global body.
S3  ``assemble``: the rank bodies are sent to the root into their final offsets
    (point-to-point over NVLink, one batched group).  This is the only data movement
    between GPUs; apply needs none (each rank applies its own records).
"""

import torch
import torch.distributed as dist


def shard_plan(numels, world: int):
    """Split range(len(numels)) into ``world`` contiguous [begin, end) ranges minimising
    the largest sum (binary search on the bound + greedy fill).  Deterministic."""
    n = len(numels)
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * (world - 1 if world > 1 else 0)
    lo, hi = max(numels), sum(numels)

    def fits(bound):
        parts, acc = 1, 0
        for x in numels:
            if acc + x > bound:
                parts += 1
                acc = x
            else:
                acc += x
        return parts <= world

    while lo < hi:
        mid = (lo + hi) // 2
        if fits(mid):
            hi = mid
        else:
            lo = mid + 1
    bound = lo
    ranges, begin, acc = [], 0, 0
    for i, x in enumerate(numels):
        # close the current range if adding x would exceed the bound, as long as enough
        # tensors remain for the ranks still to fill
        if acc + x > bound and i > begin:
            ranges.append((begin, i))
            begin, acc = i, 0
        acc += x
    ranges.append((begin, n))
    while len(ranges) < world:
        ranges.append((n, n))
    return ranges


def gather_sizes(local_bytes: int, device, group=None):
    """S2: all-gather of one int64 per rank; returns (sizes list, my offset, total)."""
    world = dist.get_world_size(group)
    t = torch.tensor([local_bytes], dtype=torch.int64, device=device)
    out = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, t, group=group)
    sizes = out.tolist()
    rank = dist.get_rank(group)
    return sizes, sum(sizes[:rank]), sum(sizes)


def assemble(local_body: torch.Tensor, sizes, root_out: torch.Tensor = None, root: int = 0,
             group=None):
    """S3: concatenate every rank's body into ``root_out`` on the root (uint8 tensor of at
    least sum(sizes) bytes, required on the root).  Other ranks send.  Returns the
    assembled view on the root, None elsewhere."""
    rank = dist.get_rank(group)
    total = sum(sizes)
    if rank == root:
        offs = [sum(sizes[:r]) for r in range(len(sizes))]
        root_out[offs[root]:offs[root] + sizes[root]].copy_(local_body[:sizes[root]])
        ops = [dist.P2POp(dist.irecv, root_out[offs[r]:offs[r] + sizes[r]], r, group)
               for r in range(len(sizes)) if r != root and sizes[r] > 0]
    else:
        ops = [dist.P2POp(dist.isend, local_body[:sizes[rank]], root, group)] if sizes[rank] > 0 else []
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return root_out[:total] if rank == root else None


def shift_table(rows, offset: int):
    """Offset-table rows of a rank's body, shifted to the global body's byte offsets."""
    return [(r[0] + offset, r[1], r[2], r[3] + offset, r[4], r[5] + offset, r[6]) for r in rows]
