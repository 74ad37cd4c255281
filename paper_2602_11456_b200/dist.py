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
from torch.multiprocessing.reductions import reduce_tensor
from .binding import rebase


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


def shard_lpt(numels, world: int):
    """S1, LPT (max/ideal 1.0078 at G = 8 for Qwen3-8B vs 1.0406 for
    contiguous ranges): tensors in decreasing size (ties: lower index first) each go to the
    rank with the smallest load so far (ties: lower rank).  Deterministic; returns one
    ascending list of global tensor indices per rank."""
    loads = [0] * max(world, 1)
    parts = [[] for _ in range(max(world, 1))]
    for k in sorted(range(len(numels)), key=lambda i: (-numels[i], i)):
        r = min(range(len(loads)), key=lambda q: (loads[q], q))
        parts[r].append(k)
        loads[r] += numels[k]
    return [sorted(p) for p in parts]


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
    return list(rebase(rows, offset))


def _ipc_teardown(device, group):
    """Release order for CUDA IPC mappings: every consumer drops its mappings (and lets the
    garbage collector free the rebuilt tensors), then the producer reclaims what the
    consumers released (torch.cuda.ipc_collect) before anything is freed or the process
    exits — so no rank exits while a peer still maps its memory."""
    import gc
    gc.collect()
    torch.cuda.synchronize(device)
    dist.barrier(group=group)
    torch.cuda.ipc_collect()
    dist.barrier(group=group)


def _map_root_buffers(bufs, rank: int, world: int, root: int, device, group):
    """CUDA IPC: the root's buffers mapped into every other rank.  The root shares each buffer
    once PER CONSUMER (every reduce_tensor call carries its own sent-data reference counter,
    which exactly one consumer's rebuild releases), so after the consumers drop their mappings
    the root's torch.cuda.ipc_collect() reclaims every share and no counter is left pending
    at exit.  Returns the mapped tensors on non-root ranks, [] on the root."""
    shared = ({r: [reduce_tensor(b) for b in bufs] for r in range(world) if r != root}
              if rank == root else None)
    handles = [None] * world
    dist.all_gather_object(handles, shared, group=group)
    peers = []
    if rank != root:
        for fn, args in handles[root][rank]:
            args = list(args)
            args[6] = torch.device(device).index  # rebuild on this process's device (peer mapping)
            peers.append(fn(*args))
    return peers


class NvlinkAssembler:
    """S3 as one kernel over NVLink peer memory (delta_assemble): the root owns the
    assembled-body buffer ``buf``; every other rank maps it into its own address space with
    CUDA IPC once, and per step writes its body straight into it at the offset the kernel
    computes on the device from the all-gathered sizes (no host round trip, no receive
    posted on the root).  A one-element all-reduce on the same stream after the copies
    orders them before anything the root does next.  Rank 0's own body is extracted
    directly into ``buf`` (offset 0)."""

    def __init__(self, ctx, capacity: int, device, group=None, root: int = 0, nbuf: int = 1):
        assert root == 0, "the assembled body starts with rank 0's records"
        self.ctx, self.group, self.root = ctx, group, root
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.device = torch.device(device)
        # nbuf assembled-body buffers on the root (2: step t's assembly overlaps step t+1)
        self.bufs = ([torch.empty(capacity, dtype=torch.uint8, device=self.device) for _ in range(nbuf)]
                     if self.rank == root else [None] * nbuf)
        self.buf = self.bufs[0]
        self.peers = _map_root_buffers(self.bufs, self.rank, self.world, root, self.device, group)
        self.peer = self.peers[0] if self.peers else None
        self.sizes = torch.zeros(self.world, dtype=torch.int64, device=self.device)
        self.size1 = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.token = torch.zeros(1, dtype=torch.float32, device=self.device)

    def assemble(self, body: torch.Tensor, size, stream=None, slot: int = 0):
        """Enqueue: sizes all-gather, this rank's NVLink copy into the root's buffer
        ``slot``, completion all-reduce.  ``size``: the body size as an int, or a one-element
        int64 CUDA tensor (delta_extract_async's device-resident size: no host value needed).
        Returns the assembled buffer on the root, None elsewhere."""
        stream = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.stream(stream):
            if isinstance(size, torch.Tensor):
                self.size1.copy_(size)
            else:
                self.size1.fill_(size)
            dist.all_gather_into_tensor(self.sizes, self.size1, group=self.group)
            if self.rank != self.root:
                self.ctx.assemble(body, self.peers[slot], self.sizes, self.rank, stream=stream)
            dist.all_reduce(self.token, group=self.group)
        return self.bufs[slot] if self.rank == self.root else None

    def close(self):
        """Release the IPC mapping (non-root ranks) before the root frees or exits."""
        torch.cuda.synchronize(self.device)
        self.peer = None
        self.peers = []
        _ipc_teardown(self.device, self.group)


class RecordAssembler:
    """S3 for ANY tensor partition (e.g. ``shard_lpt``): the root owns ``nbuf`` assembled-body
    buffers, mapped into every other rank with CUDA IPC once.  Per step: ``record_sizes`` (on
    the extract's stream, right after it: reads this rank's device offset table) writes this
    rank's record sizes into a global-order vector (zeros elsewhere); ``assemble`` (on a comm
    stream) sums the vectors over the ranks (one NCCL all-reduce of T int64), then one
    delta_assemble_records kernel copies every local record to its global offset in the
    root's buffer (over NVLink; the root copies its own records locally), and a one-element
    all-reduce orders the copies before the root's readers."""

    def __init__(self, ctx, capacity: int, device, gidx, n_global: int, group=None, root: int = 0,
                 nbuf: int = 2):
        self.ctx, self.group, self.root = ctx, group, root
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.device = torch.device(device)
        self.bufs = ([torch.empty(capacity, dtype=torch.uint8, device=self.device) for _ in range(nbuf)]
                     if self.rank == root else [None] * nbuf)
        self.peers = _map_root_buffers(self.bufs, self.rank, self.world, root, self.device, group)
        self.gidx = torch.tensor(list(gidx), dtype=torch.int32, device=self.device)
        self.sizes = [torch.zeros(n_global, dtype=torch.int64, device=self.device) for _ in range(nbuf)]
        self.token = torch.zeros(1, dtype=torch.float32, device=self.device)

    def record_sizes(self, slot: int = 0, stream=None):
        """Enqueue on ``stream`` (the extract's, after it): this rank's record sizes."""
        if self.gidx.numel():
            self.ctx.record_sizes(self.ctx.table_dev_ptr(), self.gidx.numel(), self.gidx, self.sizes[slot],
                                  stream=stream)
        else:
            with torch.cuda.stream(stream or torch.cuda.current_stream(self.device)):
                self.sizes[slot].zero_()

    def assemble(self, body: torch.Tensor, slot: int = 0, stream=None):
        """Enqueue on ``stream``: size all-reduce, the record copies, completion all-reduce.
        Returns the assembled buffer on the root, None elsewhere."""
        stream = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.stream(stream):
            dist.all_reduce(self.sizes[slot], group=self.group)
            if self.gidx.numel():
                dst = self.bufs[slot] if self.rank == self.root else self.peers[slot]
                self.ctx.assemble_records(body, self.gidx, self.sizes[slot], dst, stream=stream)
            dist.all_reduce(self.token, group=self.group)
        return self.bufs[slot] if self.rank == self.root else None

    def close(self):
        torch.cuda.synchronize(self.device)
        self.peers = []
        _ipc_teardown(self.device, self.group)


class FusedAssembler:
    """S2 + S3 fused into the emit (NEXT f2; PAPER.md:405-409 cut-through): the root owns
    ``nbuf`` assembled-body buffers, mapped into every other rank with CUDA IPC once.  Per step
    each rank runs the scan phase (its body size lands on the device), one NCCL all-gather of
    the sizes on the same stream, then the emit phase: K4/K5 store this rank's records into its
    local body (for its own apply) AND straight into the root's buffer at their global offset
    (delta_extract_emit_async with a peer destination) — no separate copy kernel.  Rank 0 emits
    directly into the root buffer (its records head the body).  ``token()`` enqueues the
    completion all-reduce on a comm stream: the root's readers wait for it."""

    def __init__(self, ctx, capacity: int, device, group=None, root: int = 0, nbuf: int = 2):
        assert root == 0, "the assembled body starts with rank 0's records"
        self.ctx, self.group, self.root = ctx, group, root
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.device = torch.device(device)
        self.bufs = ([torch.empty(capacity, dtype=torch.uint8, device=self.device) for _ in range(nbuf)]
                     if self.rank == root else [None] * nbuf)
        self.peers = _map_root_buffers(self.bufs, self.rank, self.world, root, self.device, group)
        self.sizes = [torch.zeros(self.world, dtype=torch.int64, device=self.device) for _ in range(nbuf)]
        self.token_t = torch.zeros(1, dtype=torch.float32, device=self.device)

    def extract(self, tensors, out, size, slot: int = 0, stream=None):
        """Scan, size all-gather, fused emit, all on ``stream`` (default: current).  ``out``:
        this rank's local body buffer (ignored on the root, whose body is the root buffer);
        ``size``: one-element int64 CUDA tensor.  Returns (body buffer, DeviceTable)."""
        stream = stream or torch.cuda.current_stream(self.device)
        self.ctx.delta_extract_scan_async(tensors, size, stream=stream)
        with torch.cuda.stream(stream):
            dist.all_gather_into_tensor(self.sizes[slot], size, group=self.group)
        if self.rank == self.root:
            dst = self.bufs[slot]
            table = self.ctx.delta_extract_emit_async(dst, size, stream=stream)
        else:
            dst = out
            table = self.ctx.delta_extract_emit_async(out, size, peer=self.peers[slot], sizes=self.sizes[slot],
                                                      rank=self.rank, stream=stream)
        return dst, table

    def token(self, stream):
        """The completion token: one all-reduce on ``stream`` after the emit (the caller makes
        ``stream`` wait for the emit first).  The root's body is complete once it returns."""
        with torch.cuda.stream(stream):
            dist.all_reduce(self.token_t, group=self.group)

    def close(self):
        torch.cuda.synchronize(self.device)
        self.peers = []
        _ipc_teardown(self.device, self.group)
