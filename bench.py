#!/usr/bin/env python
"""Benchmark of the sparse-delta hot path (SparrowRL, arXiv 2602.11456 §5.1) on B200.

One step = one pass of the whole path over one synthetic weight set:
    delta_size (K1 compare+compaction, K2 LEB128 lengths, K3 offset table, size readback)
  + delta_extract (K4 LEB128 bytes + values, K5 headers; consumes the cached scan)
  + [N>1: NCCL size all-gather + assembly of the packed body on rank 0]
  + delta_apply (A1 locate, A2 decode+validate, A3 scans, A4 gated scatter-store)
Metric (BASELINE.json): GB/s of weights scanned (old + new bytes compared, all ranks) per
second of step time; the payload ratio W / body is reported beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config M3] [--impl reference]

Multi-GPU: launched by torchrun (one rank per GPU, NCCL); tensors are sharded by
contiguous balanced ranges (paper_2602_11456_b200.dist), the step time is the max over
ranks of the CUDA-event time of the K timed steps.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (model or None, rho, pattern, description)
    "M1": ("M1", 0.01, "exact", "single 16M-element bf16 tensor, 1% changed (configs[0])"),
    "M2": ("4B", 0.01, "uniform", "Qwen3-4B-shaped bf16 set, 1% uniform (configs[1])"),
    "M3": ("8B", 0.01, "uniform", "Qwen3-8B-shaped bf16 set, 1% uniform (configs[2])"),
    "M4": ("14B", 0.01, "uniform", "Qwen3-14B-shaped bf16 set, 1% uniform (configs[3])"),
    "M5": ("8B", None, None, "Qwen3-8B sweep (configs[4]); pick --rho/--pattern"),
}
METRIC = "delta extract+apply GB/s of weights scanned vs HBM peak; payload ratio, Qwen3-8B"
PAPER_CPU = "paper: ~5 s CPU extraction for Qwen3-8B (PAPER.md:405), 79x payload (PAPER.md:51), other hardware"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="M3", choices=sorted(CONFIGS))
    p.add_argument("--rho", type=float, default=None)
    p.add_argument("--pattern", default=None, choices=[None, "uniform", "rowblock", "exact"])
    p.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--host-sync", default="end", choices=["end", "step"],
                   help="chained path: 'end' = the host enqueues the timed steps without waiting "
                        "(one wait after the last; kernel times accumulated on the device), "
                        "'step' = the host waits for every step")
    p.add_argument("--index-codec", default="leb128", choices=["leb128", "fixed"],
                   help="fixed: the paper's naive int32/64 index encoding (PAPER.md:387, 609; R18)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=4)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    p.add_argument("--no-clocks", action="store_true")
    p.add_argument("--assembly", default="nvlink", choices=["nvlink", "fused", "nccl", "none"],
                   help="N>1: 'nvlink' = a delta_assemble copy kernel over NVLink on a comm stream, "
                        "overlapping the apply (default: measured fastest); 'fused' = the emit kernel "
                        "stores each rank's records at their global offsets in rank 0's buffer over "
                        "NVLink (sizes by one NCCL all-gather; the transfer then sits inside the emit); "
                        "'nccl' = NCCL P2P (baseline); 'none' = diagnostics only, no S2/S3")
    p.add_argument("--assemble-ctas", type=int, default=0, help="CTAs of the NVLink assembly kernel (0 = default)")
    p.add_argument("--partition", default="auto", choices=["auto", "contiguous", "lpt"],
                   help="N>1 S1: 'contiguous' = balanced tensor ranges (each rank's records are one byte "
                        "range of the body); 'lpt' = longest-processing-time tensor sets (better balance; "
                        "the NVLink assembly then copies record by record to global offsets); 'auto' "
                        "(default) = lpt from 4 GPUs with the nvlink (or no) assembly, else contiguous "
                        "(measured: lpt 1.3 %% faster at N=4, 1 %% slower at N=2 where ranges balance exactly)")
    p.add_argument("--comm-priority", type=int, default=0,
                   help="CUDA stream priority of the assembly stream (negative = higher)")
    p.add_argument("--sync-step", action="store_true",
                   help="host-sized step (size readback between extract and apply) instead of the "
                        "chained device-sized one")
    p.add_argument("--pipeline", type=int, default=1,
                   help="G > 1: extract and apply in G pipelined groups on two streams")
    p.add_argument("--apply-ctas", type=int, default=0, help="apply kernels' CTAs per SM (0 = default)")
    p.add_argument("--scatter-ctas", type=int, default=0, help="scatter kernel CTAs per SM (0 = default)")
    p.add_argument("--emit-ctas", type=int, default=0, help="extract emit kernel CTAs per SM (0 = default)")
    p.add_argument("--prefetch-tiles", type=int, default=0, help="K1 L2 prefetch distance in tiles + 1 (0 = default)")
    p.add_argument("--scatter-order", type=int, default=0, help="1 thread-major, 2 entry-major (0 = default)")
    p.add_argument("--scan-kernel", type=int, default=0,
                   help="compare kernel form: 1 (the only one; 0 = library default)")
    p.add_argument("--tensors", type=int, default=0,
                   help="profiling only: keep the first N tensors of the config")
    return p.parse_args()


def workload(args):
    from workload import m1_specs, qwen3
    model, rho, pattern, desc = CONFIGS[args.config]
    rho = args.rho if args.rho is not None else (rho if rho is not None else 0.01)
    pattern = args.pattern or pattern or "uniform"
    specs = m1_specs() if model == "M1" else qwen3(model)
    if getattr(args, "tensors", 0):
        specs = specs[:args.tensors]
        desc += f" [first {args.tensors} tensors only: profiling run]"
    return specs, rho, pattern, desc


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index, enabled=True):
        self.index, self.enabled, self.proc, self.lines = index, enabled, None, []

    def start(self):
        if not self.enabled:
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append((time.time(), ln.strip()))

    def mark(self):
        """Call right before and right after the timed region."""
        return time.time()

    def stop(self, t0=None, t1=None):
        if not self.proc:
            return None
        time.sleep(0.3)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        window = [(ts, ln) for ts, ln in self.lines
                  if t0 is None or (t0 - 0.15 <= ts <= t1 + 0.25)]
        if not window:  # timed region shorter than the sampling period: nearest samples
            window = sorted(self.lines, key=lambda x: abs(x[0] - (t0 or 0)))[:3]
        for _, ln in window:
            f = [x.strip() for x in ln.split(",")][1:]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ oracle timing (CPU)
class OracleSample:
    """A bounded sample of the workload for timing the oracle (oracle.codec, plain numpy,
    as it stands) on the host: whole tensors in list order (the embedding moved last so a
    short sample is layer tensors), generated once with the shared seeded generator (on
    cuda:0 when there is one, then copied to host) until the estimated oracle time reaches
    ``budget_s``."""

    def __init__(self, specs, rho, pattern, seed, dtype, budget_s, index_codec="leb128"):
        self.index_codec = index_codec
        import numpy as np
        import torch

        import oracle
        from workload import generate_pair
        self.oracle = oracle
        gdev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
        order = list(range(len(specs)))
        if len(order) > 3:
            order = order[1:] + order[:1]
        self.items, est, self.lanes, self.scanned = [], 0.0, 0, 0
        for k in order:
            s = specs[k]
            o, w = generate_pair(s, k, seed, rho=rho, pattern=pattern, dtype=dtype, device=gdev)
            lt = torch.int16 if o.element_size() == 2 else torch.int32
            nt = np.uint16 if o.element_size() == 2 else np.uint32
            on, wn = o.view(lt).cpu().numpy().view(nt), w.view(lt).cpu().numpy().view(nt)
            self.items.append((s.name, on, wn))
            self.lanes += s.numel
            self.scanned += 2 * s.numel * on.dtype.itemsize
            if not est:  # calibrate on the first tensor
                t0 = time.perf_counter()
                self._one(self.items[0])
                per_byte = (time.perf_counter() - t0) / self.scanned
            est = per_byte * self.scanned
            if est >= budget_s:
                break
        self.sample = (f"{len(self.items)} whole tensors ({self.lanes} lanes, "
                       f"{self.scanned / 1e9:.3f} GB of old+new) of the same workload; "
                       f"oracle.codec extract+apply (plain numpy, one thread per process); inputs from the shared "
                       f"seeded generator on {gdev}")

    def _one(self, item):
        name, on, wn = item
        body, _ = self.oracle.codec.extract([(name, [on], [wn])], index_codec=self.index_codec)
        got = self.oracle.codec.apply([(name, on)], body, on.dtype.itemsize, index_codec=self.index_codec)[0]
        return got

    def run(self, procs: int = 1):
        """One timed pass: returns (GB/s of weights scanned, seconds).  procs > 1: the
        sample's tensors spread over that many forked worker processes (one tensor per
        task, the oracle unchanged); seconds = wall time of the pool's pass."""
        import numpy as np
        if procs > 1:
            import multiprocessing as mp
            global _ORACLE_SAMPLE
            _ORACLE_SAMPLE = self
            with mp.get_context("fork").Pool(procs) as pool:
                pool.map(_oracle_noop, range(procs))  # workers up before the clock starts
                t0 = time.perf_counter()
                ok = pool.map(_oracle_task, range(len(self.items)), chunksize=1)
                spent = time.perf_counter() - t0
            if not all(ok):
                raise SystemExit("oracle round trip mismatch")
            return self.scanned / spent / 1e9, spent
        spent = 0.0
        for item in self.items:
            t0 = time.perf_counter()
            got = self._one(item)
            spent += time.perf_counter() - t0
            if not np.array_equal(got, item[2]):
                raise SystemExit("oracle round trip mismatch")
        return self.scanned / spent / 1e9, spent


_ORACLE_SAMPLE = None  # set before the fork: the workers inherit the sample's arrays


def _oracle_noop(_):
    return 0


def _oracle_task(i):
    import numpy as np
    item = _ORACLE_SAMPLE.items[i]
    return bool(np.array_equal(_ORACLE_SAMPLE._one(item), item[2]))


def ops_view(k, lanes, width, nnz, idx_bytes, body, peak, value, scanned_total, total_lanes, nnz_total,
             idx_total):
    """Extract / apply split of this rank's kernel time with their algorithmic bytes
    (extract: 2 w N read + body written; apply: body read + nnz w stored) and the round trip
    against the measured copy peak."""
    ex = sum(k.get(x, 0.0) for x in ("scan_ms", "lens_ms", "finalize_ms", "emit_ms", "headers_ms"))
    ap = sum(k.get(x, 0.0) for x in ("locate_ms", "decode_ms", "apply_scan_ms", "scatter_ms"))
    ex_b = 2 * lanes * width + body
    ap_b = body + nnz * width
    rt_per_lane = (2 * width * total_lanes + 2 * idx_total + 3 * width * nnz_total) / total_lanes
    return {"extract": {"ms": round(ex, 4), "algorithmic_bytes": ex_b,
                        "GBps": round(ex_b / ex / 1e6, 1) if ex else None},
            "apply": {"ms": round(ap, 4), "algorithmic_bytes": ap_b,
                      "GBps": round(ap_b / ap / 1e6, 1) if ap else None},
            "round_trip": {"algorithmic_bytes_per_lane": round(rt_per_lane, 4),
                           "algorithmic_GBps": round(value * rt_per_lane / (2 * width), 1),
                           "frac_of_measured_peak": round(value * rt_per_lane / (2 * width) / peak, 4),
                           "scanned_frac_of_measured_peak": round(value / peak, 4),
                           # north_star quotes "~8 TB/s" as the HBM peak (B200 nominal); the measured
                           # copy bandwidth above is what the box delivers
                           "frac_of_nominal_8TBps": round(value * rt_per_lane / (2 * width) / 8000.0, 4)}}


def host_info() -> dict:
    """CPU model, logical CPUs, affinity and RAM of the host the oracle ran on."""
    info = {"cpu_count": os.cpu_count(), "affinity": host_cores()}
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                info["cpu_model"] = ln.split(":", 1)[1].strip()
                break
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                info["ram_gb"] = round(int(ln.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    return info


def brute_m1(smp) -> dict:
    """oracle.brute (pure Python, per element / per byte) extract + apply of the M1 tensor,
    one thread; GB/s of old+new scanned."""
    import oracle
    name, on, wn = smp.items[0]
    old, new = on.tolist(), wn.tolist()
    t0 = time.perf_counter()
    body, _ = oracle.brute.extract([(name, [old], [new])], on.dtype.itemsize)
    got = oracle.brute.apply([(name, old)], body, on.dtype.itemsize)[0]
    secs = time.perf_counter() - t0
    if got != new:
        raise SystemExit("brute-force oracle round trip mismatch")
    return {"value": round(2 * len(old) * on.dtype.itemsize / secs / 1e9, 5), "unit": "GB/s", "cores": 1,
            "seconds": round(secs, 2), "kind": "oracle.brute (pure Python)"}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args):
    """--impl reference: the oracle as it stands, on the host cores, per step a bounded
    sample of this workload; rank 0 only (other ranks exit 0)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import torch
    specs, rho, pattern, desc = workload(args)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    budget = max(0.5, min(args.cpu_seconds, 90.0 / max(1, args.steps + args.warmup)))
    smp = OracleSample(specs, rho, pattern, args.seed, dtype, budget, args.index_codec)
    cores = host_cores()
    for _ in range(args.warmup):
        smp.run(cores)
    vals, secs = [], 0.0
    for _ in range(args.steps):
        v, s = smp.run(cores)
        vals.append(v)
        secs += s
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * secs / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u16" if args.dtype == "bf16" else "u32",
        "data": "synthetic", "config": {"workload": desc, "config": args.config, "rho": rho,
                                        "pattern": pattern},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": smp.sample + f"; {cores} worker processes (one tensor per task)",
                         "host": host_info()},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def resolve_partition(partition: str, world: int, assembly: str) -> str:
    """S1 choice: 'auto' = LPT tensor sets from 4 GPUs when the assembly can place records at
    scattered offsets (nvlink: delta_assemble_records; none), else contiguous ranges."""
    if partition == "auto":
        return "lpt" if world >= 4 and assembly in ("nvlink", "none") else "contiguous"
    if partition == "lpt" and world > 1 and assembly not in ("nvlink", "none"):
        raise SystemExit("bench: --partition lpt supports --assembly nvlink or none")
    return partition


def launch_ranks(args):
    """--gpus N with no WORLD_SIZE in the environment: re-exec this command under
    torch.distributed.run, one rank per GPU (rendezvous on 127.0.0.1).  Under a launcher,
    WORLD_SIZE must equal --gpus.  Returns an exit code, or None to run in this process."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if args.gpus <= 1:
            return None
        import random
        import socket
        # a free port BELOW the kernel's ephemeral range (32768+), so no socket the ranks or
        # NCCL open in the meantime can be handed the same number
        rng = random.Random(os.getpid() ^ int(time.time() * 1e6))
        for _ in range(100):
            port = rng.randrange(20000, 32000)
            with socket.socket() as sk:
                try:
                    sk.bind(("127.0.0.1", port))
                    break
                except OSError:
                    continue
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        print(f"bench: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
        return subprocess.call(cmd)
    if int(world) != args.gpus:
        print(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr, flush=True)
        return 2
    return None


def main():
    args = parse()
    rc = launch_ranks(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import __graft_entry__ as entry
    entry.build()
    import paper_2602_11456_b200 as sd
    from paper_2602_11456_b200 import dist as sdist
    from workload import generate_pair

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm_info = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        # the communicator as NCCL sees it (one all-reduce over it), logged per rank
        probe = torch.ones(1, dtype=torch.int64, device=dev)
        dist.all_reduce(probe)
        comm_info = {"backend": dist.get_backend(), "nranks": dist.get_world_size(),
                     "ranks_seen_by_allreduce": int(probe.item()),
                     "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version())}
        print(f"bench: rank {rank}/{world} on cuda:{local} {comm_info}", file=sys.stderr, flush=True)
        if comm_info["ranks_seen_by_allreduce"] != world:
            raise SystemExit(f"bench: NCCL all-reduce saw {comm_info['ranks_seen_by_allreduce']} ranks, expected {world}")

    specs, rho, pattern, desc = workload(args)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    width = 2 if args.dtype == "bf16" else 4
    args.partition = resolve_partition(args.partition, world, args.assembly)
    if args.partition == "lpt":  # LPT tensor sets, ascending global order within the rank
        mine = sdist.shard_lpt([s.numel for s in specs], world)[rank]
    else:  # contiguous ranges: each rank's records are one byte range of the global body
        b, e = sdist.shard_plan([s.numel for s in specs], world)[rank]
        mine = list(range(b, e))

    # ---- inputs resident in HBM before timing (per-tensor seeds: rank-independent data)
    olds, news, targets = [], [], []
    for k in mine:
        o, w = generate_pair(specs[k], k, args.seed, rho=rho, pattern=pattern, dtype=dtype, device=dev)
        olds.append(o)
        news.append(w)
        targets.append(o.clone())
    torch.cuda.synchronize()
    local_lanes = sum(specs[k].numel for k in mine)
    total_lanes = sum(s.numel for s in specs)
    scanned_total = 2 * total_lanes * width            # old + new bytes, all ranks
    tensors = [(specs[k].name, o, w) for k, o, w in zip(mine, olds, news)]
    tgts = [(specs[k].name, t) for k, t in zip(mine, targets)]
    root_out = None
    stream = torch.cuda.current_stream()

    comm = torch.cuda.Stream(dev, priority=args.comm_priority) if world > 1 else None
    nvasm = None
    fuasm = None
    rasm = None

    slot = {"t": 0, "cur": 0}

    def assemble(size, body):
        """S2+S3 on a side stream: the transfer of the body to rank 0 overlaps this rank's
        apply (which needs no collective) and, with two body buffers, the next step."""
        nonlocal root_out
        if args.assembly == "none":
            return
        if rasm is not None:  # record sizes from this rank's device table, before the next extract
            rasm.record_sizes(slot["cur"], stream=torch.cuda.current_stream())
        comm.wait_stream(torch.cuda.current_stream())
        if rasm is not None:  # record-granular NVLink copies (any partition)
            rasm.assemble(body, slot["cur"], stream=comm)
            return
        if fuasm is not None:  # the body is already there (fused emit): completion token only
            fuasm.token(comm)
            return
        if nvasm is not None:  # delta_assemble kernel over NVLink peer memory
            nvasm.assemble(body, size, stream=comm, slot=slot["cur"])
            return
        with torch.cuda.stream(comm):
            sizes, off, tot = sdist.gather_sizes(size, dev)
            if rank == 0 and (root_out is None or root_out.numel() < tot):
                root_out = torch.empty(tot + tot // 8, dtype=torch.uint8, device=dev)
            sdist.assemble(body, sizes, root_out)

    if args.pipeline > 1:
        from paper_2602_11456_b200.pipeline import RoundTrip
        rt = RoundTrip(tensors, tgts, groups=args.pipeline, device=dev,
                       apply_ctas_per_sm=args.apply_ctas or None, scan_kernel=args.scan_kernel or None)
        rt.set_profiling(True)
        ctx = rt.cx

        def step(acc=None):
            body = rt.step(acc)
            if world > 1:
                assemble(body.numel(), body)
                torch.cuda.current_stream().wait_stream(comm)
            return body, rt.table()
    else:
        tl = sd.TensorList(tensors)
        tg = sd.TargetList(tgts)
        ctx = sd.DeltaContext(dev)
        if args.apply_ctas:
            ctx.set_option(1, args.apply_ctas)
        if args.emit_ctas:
            ctx.set_option(2, args.emit_ctas)
        if args.scan_kernel:
            ctx.set_option(3, args.scan_kernel)
        if args.scatter_ctas:
            ctx.set_option(4, args.scatter_ctas)
        if args.prefetch_tiles:
            ctx.set_option(5, args.prefetch_tiles)
        if args.scatter_order:
            ctx.set_option(6, args.scatter_order)
        if args.index_codec == "fixed":
            ctx.set_option(8, 2)
        if args.assemble_ctas:
            ctx.set_option(10, args.assemble_ctas)
        ctx.set_profiling(True)
        size0 = ctx.delta_size(tl)
        out = torch.empty(size0 + size0 // 8 + 4096, dtype=torch.uint8, device=dev)
        if world > 1 and args.assembly in ("nvlink", "fused"):
            tot0 = torch.tensor([size0], dtype=torch.int64, device=dev)
            dist.all_reduce(tot0)
            total0 = int(tot0.item())
            if args.assembly == "fused":
                fuasm = sdist.FusedAssembler(ctx, total0 + total0 // 8 + 4096, dev, nbuf=2)
                if rank == 0:
                    out = fuasm.bufs[0]  # rank 0's records are the head of the assembled body
            elif args.partition == "lpt":  # records go to scattered global offsets: rank 0 copies too
                rasm = sdist.RecordAssembler(ctx, total0 + total0 // 8 + 4096, dev, mine, len(specs), nbuf=2)
            else:
                nvasm = sdist.NvlinkAssembler(ctx, total0 + total0 // 8 + 4096, dev, nbuf=2)
                if rank == 0:
                    out = nvasm.buf  # rank 0's records are the head of the assembled body

        size_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        # two (body, size) slots when the NVLink assembly runs on the comm stream: step t+1
        # extracts into the other slot while step t's body is still being copied to rank 0
        nslots = 2 if (nvasm is not None or fuasm is not None or rasm is not None) else 1
        root_bufs = nvasm.bufs if nvasm is not None else (fuasm.bufs if fuasm is not None else None)
        outs = [out] + ([root_bufs[1] if (rank == 0 and root_bufs is not None) else torch.empty_like(out)]
                        if nslots == 2 else [])
        size_devs = [size_dev] + ([torch.zeros(1, dtype=torch.int64, device=dev)] if nslots == 2 else [])
        slot_free = [None] * nslots  # comm-stream event: the slot's last assembly is done

        def record(acc):
            t = ctx.last_timing()
            if acc is not None:
                for kname in ("scan_ms", "lens_ms", "finalize_ms", "emit_ms", "headers_ms",
                              "locate_ms", "decode_ms", "apply_scan_ms", "scatter_ms"):
                    acc[kname] = acc.get(kname, 0.0) + t[kname]

        if args.sync_step or (world > 1 and nvasm is None and fuasm is None and rasm is None
                               and args.assembly != "none"):
            def step(acc=None):
                # host-sized path: delta_extract reads the size back (sync), the apply takes
                # the device table; 2 host syncs per step
                body, table = ctx.delta_extract(tl, out=out, table="device")
                if world > 1:
                    assemble(body.numel(), body)
                ctx.delta_apply(tg, body, table=table)
                if world > 1:
                    torch.cuda.current_stream().wait_stream(comm)
                record(acc)
                return body, table
        else:
            def before_apply(buf, size):
                if world > 1:
                    assemble(size, buf)

            def step(acc=None, wait=True):
                # one stream of kernels: extract (size + table stay on the device) -> [assembly
                # on the comm stream] -> chained apply; the host waits once, at the end (or,
                # wait=False, not at all: errors surface at the next extract_wait/apply_wait)
                s = slot["t"] % nslots
                slot["t"] += 1
                slot["cur"] = s
                if slot_free[s] is not None:  # the slot's previous body has reached rank 0
                    torch.cuda.current_stream().wait_event(slot_free[s])
                fx = None
                if fuasm is not None:  # fused emit + assembly: scan, size all-gather, emit to both
                    def fx(tl_, o_, sz_, st_, s=s):
                        return fuasm.extract(tl_, o_, sz_, slot=s, stream=st_)[1]
                n = ctx.round_trip(tl, tg, outs[s], size_devs[s], before_apply=before_apply, wait=wait, extract=fx)
                if world > 1:
                    if nslots == 1:
                        torch.cuda.current_stream().wait_stream(comm)
                    else:
                        ev = torch.cuda.Event()
                        ev.record(comm)
                        slot_free[s] = ev
                    if wait:
                        torch.cuda.current_stream().wait_stream(comm)
                if wait:
                    record(acc)
                return (outs[s][:n] if n is not None else None), None

    chained = args.pipeline <= 1 and not (args.sync_step or (world > 1 and nvasm is None and fuasm is None
                                                             and rasm is None
                                                             and args.assembly != "none"))
    pipelined = chained and args.host_sync == "end"
    for _ in range(max(args.warmup, 0)):
        body, table = step()
    if pipelined:  # K1's time accumulated on the device over the timed region (events around
        ctx.set_profiling(3)  # K1 only: events between every kernel cost ~30 us per step)
        step()  # one more waited warm-up step with the accumulating event ring
        ctx.timing_totals()
    clocks = Clocks(local, enabled=not args.no_clocks)
    acc = {}
    clocks.start()
    time.sleep(1.0)  # sampler up and running before the timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    ev0.record(stream)
    for _ in range(args.steps):
        if pipelined:
            step(wait=False)
        else:
            body, table = step(acc)
    if comm is not None:  # the last step's assembly is part of the timed work
        stream.wait_stream(comm)
    ev1.record(stream)
    torch.cuda.synchronize()
    if pipelined:
        nb = ctx.extract_wait()   # raises if any step's extract overflowed (never after warm-up)
        ctx.apply_wait()          # raises if any step's apply gate was closed
        body, table = outs[(slot["t"] - 1) % nslots][:nb], None
        tot, calls = ctx.timing_totals()
        if calls != args.steps:
            raise SystemExit(f"bench: {calls} extract scans timed for {args.steps} steps")
        acc = {k: v for k, v in tot.items()}
    w1 = time.time()
    if world > 1:
        dist.barrier()
    clk = clocks.stop(w0, w1)
    # correctness guard on the timed configuration: apply(extract(old,new)) == new
    ok = all(torch.equal(t.view(torch.int16 if width == 2 else torch.int32),
                         w.view(torch.int16 if width == 2 else torch.int32))
             for t, w in zip(targets, news))
    if not ok:
        raise SystemExit("bench: round trip mismatch")
    ms = ev0.elapsed_time(ev1)
    breakdown_steps = None
    if pipelined:  # the other kernels' times: the same loop again, events around every kernel
        ctx.set_profiling(2)
        step()
        ctx.timing_totals()
        breakdown_steps = max(3, args.steps // 2)
        if world > 1:
            dist.barrier()
        for _ in range(breakdown_steps):
            step(wait=False)
        if comm is not None:
            stream.wait_stream(comm)
        torch.cuda.synchronize()
        ctx.extract_wait()
        ctx.apply_wait()
        tb, cb = ctx.timing_totals()
        acc = {**{k: v * args.steps / max(cb, 1) for k, v in tb.items()}, "scan_ms": acc.get("scan_ms", 0.0)}
    rank_view = None
    if world > 1:  # max over ranks; every rank's time and K1 / scatter time for the record
        k1_local = acc.get("scan_ms", 0.0) / args.steps
        sc_local = acc.get("scatter_ms", 0.0) / args.steps
        t = torch.tensor([ms, k1_local, sc_local], dtype=torch.float64, device=dev)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        rank_view = {"ms_per_step": [round(float(x[0]) / args.steps, 4) for x in allt],
                     "k1_ms": [round(float(x[1]), 4) for x in allt],
                     "scatter_ms": [round(float(x[2]), 4) for x in allt]}
        ms = max(float(x[0]) for x in allt)
    ms_step = ms / args.steps
    value = scanned_total * args.steps / (ms / 1e3) / 1e9

    # ---- payload (global) and kernel-level roofline of the dominant kernel (K1)
    if table is None or isinstance(table, sd.DeviceTable):  # host rows for the statistics (untimed)
        body, table = ctx.delta_extract(tl, out=out, table=True)
    body_local = body.numel()
    nnz_local = sum(r[2] for r in table)
    idx_local = sum(r[4] for r in table)
    # the paper's "naive" fixed-width encoding of the same change set (int32
    # or int64 index "depending on tensor size" + the value; reading R6), for the
    # naive-vs-varint payload ablation (414 MB -> 202 MB)
    naive_local = sum((27 + len(specs[k].name.encode())) + r[2] * ((4 if r[1] - 1 <= 2**31 - 1 else 8) + width)
                      for k, r in zip(mine, table))
    if world > 1:
        t = torch.tensor([body_local, nnz_local, idx_local, naive_local], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        body_total, nnz_total, idx_total, naive_total = (int(x) for x in t.tolist())
    else:
        body_total, nnz_total, idx_total, naive_total = body_local, nnz_local, idx_local, naive_local
    k1_ms = acc.get("scan_ms", 0.0) / args.steps
    k1_bytes = 2 * local_lanes * width  # K1's algorithmic bytes = the 2wN it compares
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    # DRAM traffic of one K1 launch from the committed ncu capture of this exact workload
    # (profiles/ncu_traffic.json; null for other configurations)
    k1_traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        c = tr["config"]
        if (c["config"] == args.config and abs(c["rho"] - rho) < 1e-12 and c["pattern"] == pattern
                and c["dtype"] == args.dtype and c["n_gpus"] == world):
            k = tr["kernels"]["k_scan_tiles"]
            k1_traffic = k["dram_read_bytes"] + k["dram_write_bytes"]
    except (OSError, ValueError, KeyError):
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = k1_bytes / (k1_ms / 1e3) / 1e9 if k1_ms > 0 else None
    kernel_ms = {k: round(v / args.steps, 4) for k, v in acc.items()}

    result = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u16" if width == 2 else "u32", "data": "synthetic",
        "config": {"workload": desc, "config": args.config, "tensors": len(specs),
                   "lanes": total_lanes, "weights_bytes": total_lanes * width,
                   "scanned_bytes_per_step": scanned_total, "rho": rho, "pattern": pattern,
                   "seed": args.seed, "index_codec": args.index_codec,
                   "shard": ("one GPU: every tensor" if world == 1 else
                             "LPT tensor sets (dist.shard_lpt)" if args.partition == "lpt" else
                             "contiguous balanced tensor ranges (dist.shard_plan)"),
                   "l2": f"inputs ({scanned_total / 1e9:.1f} GB per step) larger than L2 (126 MB); no flush"},
        "payload": {"body_bytes": body_total, "ratio": round(total_lanes * width / body_total, 3),
                    "nnz": nnz_total, "rho_measured": nnz_total / total_lanes,
                    "index_bytes_per_entry": round(idx_total / max(nnz_total, 1), 4),
                    "naive_fixed_width_bytes": naive_total,
                    "varint_saving_vs_naive": round(naive_total / body_total, 3),
                    "paper_context": PAPER_CPU},
        "kernel_ms_per_step": kernel_ms,
        "kernel_ms_source": (f"K1 (scan_ms) from the timed region, CUDA events around K1 only; the other kernels "
                             f"from {breakdown_steps} further steps with events around every kernel"
                             if breakdown_steps else "CUDA events around every kernel in the timed steps"),
        # per-op time (this rank's kernels) and algorithmic bytes, and the round
        # trip's algorithmic bytes per lane 2w + rho (3w + 2E) against the measured peak
        "ops": ops_view(kernel_ms, local_lanes, width, nnz_local, idx_local, body_local,
                        peaks.get("hbm_gbs", 6650.0), value, scanned_total, total_lanes, nnz_total,
                        idx_total),
        "roofline": {"kernel": "k_scan_tiles (K1)", "bound": "hbm",
                     "achieved": round(achieved, 1) if achieved else None,
                     "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4) if achieved else None,
                     "traffic": k1_traffic,
                     "traffic_source": "profiles/ncu_traffic.json (ncu dram__bytes_read+write.sum, one launch)"
                     if k1_traffic else None,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if "hbm_gbs" in peaks
                     else "fallback 6650 GB/s (B200_PROFILING.md)",
                     "algorithmic_bytes_per_launch": k1_bytes},
        # per rank and step: K1, K2 (tile prefixes + offset table), K4, K5 + A1-A4
        # (fixed-width indices: A1, A2f, A4f) [+ delta_assemble with --assembly nvlink]
        "gpu_launches": ((8 if args.index_codec == "leb128" else 7)
                         + (1 if world > 1 and nvasm is not None else 0)
                         + (2 if world > 1 and rasm is not None else 0)) * args.steps,
        "clocks": clk,
    }
    if k1_ms > 0:
        result["roofline"]["k1_share_of_step"] = round(k1_ms / ms_step, 4)
    if rank_view is not None:
        result["per_rank"] = rank_view
    if comm_info is not None:
        result["comm"] = comm_info
    result["config"]["host_sync"] = "end (steps enqueued back to back)" if pipelined else "every step"
    if world > 1:
        result["config"]["assembly"] = {
            "fused": "fused emit: K4/K5 store each rank's records at their global offsets in rank 0's buffer over "
                     "NVLink (CUDA IPC), sizes by one NCCL all-gather, 2 root buffers",
            "nvlink": "delta_assemble copy kernel over NVLink (CUDA IPC) on a comm stream, 2 body buffers",
            "nccl": "NCCL P2P batch", "none": "NONE (diagnostics: no S2/S3)"}[args.assembly]
        if rasm is not None:
            result["config"]["assembly"] = ("record sizes all-reduced (NCCL), delta_assemble_records copies every "
                                            "record to its global offset in rank 0's buffer over NVLink (CUDA IPC) "
                                            "on a comm stream, 2 body buffers")
        result["config"]["partition"] = args.partition
    if pipelined:  # the same steps with the host waiting for each one (latency view)
        ks = max(3, args.steps // 2)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ks):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_s = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_s = float(t.item())
        result["host_synced"] = {"steps": ks, "ms_per_step": round(ms_s / ks, 4),
                                 "value": round(scanned_total * ks / (ms_s / 1e3) / 1e9, 2)}

    # ---- e2e: the same step with inputs copied from pinned host memory every step
    if not args.no_e2e:
        # e2e: the shadow-resident trainer step (H2D of the new weights only), and beside it
        # every input from the host (H2D of old and new)
        result["e2e_full_inputs"] = e2e(args, step, olds, news, body_local, dev, scanned_total, world)
        torch.cuda.synchronize()
        result["e2e"] = e2e_shadow(args, sd, [specs[k].name for k in mine], mine, specs, olds, news, targets,
                                   dev, scanned_total, world, rho, pattern, dtype)
    # ---- CPU oracle beside it (rank 0, N=1 only)
    if not args.no_cpu_baseline and world == 1:
        smp = OracleSample(specs, rho, pattern, args.seed, dtype, args.cpu_seconds, args.index_codec)
        v1, secs1 = smp.run()
        cores = host_cores()
        vp, secsp = smp.run(cores) if cores > 1 else (v1, secs1)
        if vp < v1:  # e.g. a single-tensor sample: the pool cannot help, report one core
            vp, secsp, cores = v1, secs1, 1
        result["cpu_baseline"] = {"value": round(vp, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
                                  "sample": smp.sample + (f"; {cores} worker processes (one tensor per task)"
                                                          if cores > 1 else "; one process"),
                                  "seconds": round(secsp, 2), "host_cpus": os.cpu_count(),
                                  "single_core": {"value": round(v1, 4), "seconds": round(secs1, 2)},
                                  "host": host_info()}
        if args.config == "M1":  # the pure-Python definition on configs[0]
            result["cpu_baseline"]["brute_force"] = brute_m1(smp)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if nvasm is not None:  # drop the CUDA IPC mapping of rank 0's buffer before rank 0 exits
        nvasm.close()
    if rasm is not None:
        rasm.close()
    if fuasm is not None:
        fuasm.close()
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def e2e(args, step, olds, news, body_cap, dev, scanned_total, world):
    """Same metric through the public API with host buffers: every step copies old and new
    from pinned host memory (H2D), runs the step and reads the packed body back (D2H), on
    the same stream as the kernels; CUDA events around the whole step, max over ranks."""
    import torch
    import torch.distributed as dist
    stream = torch.cuda.current_stream()
    h_old = [o.cpu().pin_memory() for o in olds]
    h_new = [w.cpu().pin_memory() for w in news]
    h_body = torch.empty(body_cap + body_cap // 8 + 4096, dtype=torch.uint8).pin_memory()
    h2d = sum(o.numel() * o.element_size() * 2 for o in olds)
    d2h = 0

    def one():
        nonlocal d2h
        for o, w, ho, hw in zip(olds, news, h_old, h_new):
            o.copy_(ho, non_blocking=True)
            w.copy_(hw, non_blocking=True)
        body, _ = step()
        h_body[:body.numel()].copy_(body, non_blocking=True)
        d2h = body.numel()
    one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.e2e_steps):
        one()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": round(scanned_total * args.e2e_steps / (ms / 1e3) / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
            "ms_per_step": round(ms / args.e2e_steps, 3),
            "note": "bytes per rank; old+new H2D from pinned host, body D2H, apply on device"}


def e2e_shadow(args, sd, names, ks, specs, olds, news, targets, dev, scanned_total, world, rho, pattern, dtype):
    """The trainer's view of e2e: W_t stays resident on the device as the extract-and-advance
    shadow (DELTA_OPT_ADVANCE: the compare leaves old == new), so each step's input from the
    host is only the new weights.  Every step: H2D of W_{t+1} from pinned host memory, extract
    (advancing the shadow), apply to the actor copy, D2H of the body; versions alternate
    V1, V2, V1, ... where V2 = V1 XOR the change pattern of a second seeded pair, so each
    step changes the configured share of lanes.  Public API only; CUDA events around the
    whole step, max over ranks."""
    import torch
    import torch.distributed as dist
    from workload import generate_pair
    stream = torch.cuda.current_stream()
    lt = torch.int16 if news[0].element_size() == 2 else torch.int32
    h_v = [[], []]
    for k, w in zip(ks, news):
        o2, w2 = generate_pair(specs[k], k, args.seed + 1, rho=rho, pattern=pattern, dtype=dtype, device=dev)
        x = o2.view(lt) ^ w2.view(lt)
        del o2, w2
        h_v[0].append(w.cpu().pin_memory())
        h_v[1].append((w.view(lt) ^ x).view(w.dtype).cpu().pin_memory())
        del x
    # two device copies of the new weights (and of the body): step s+1's H2D (copy stream)
    # runs while step s extracts and applies (compute stream) and step s-1's body goes D2H
    # (a third stream; PCIe is full duplex).  One context per buffer set, both advancing the
    # same shadow, in stream order.
    news2 = [torch.empty_like(w) for w in news]
    bufs = [news, news2]
    ctxs, tls = [], []
    for nb in bufs:
        cx = sd.DeltaContext(dev)
        cx.set_option(9, 2)  # DELTA_OPT_ADVANCE
        ctxs.append(cx)
        tls.append(sd.TensorList([(n, o, w) for n, o, w in zip(names, olds, nb)]))
    tg = sd.TargetList([(n, t) for n, t in zip(names, targets)])
    for o, t in zip(olds, targets):  # shadow and actor copy start at the same version
        t.copy_(o)
    cap = ctxs[0].delta_size(tls[0])  # compaction cached for the first extract below
    outs = [torch.empty(4 * cap + 4096, dtype=torch.uint8, device=dev) for _ in range(2)]
    h_bodies = [torch.empty(o.numel(), dtype=torch.uint8).pin_memory() for o in outs]
    cps, dhs = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    loaded = [torch.cuda.Event() for _ in range(2)]
    free = [None, None]      # compute-stream event: the extract reading buffer i is done
    out_free = [None, None]  # D2H-stream event: body buffer i has reached the host
    d2h = [0]
    state = {"s": 0}

    def one():
        s = state["s"]
        state["s"] += 1
        i = s % 2
        with torch.cuda.stream(cps):  # H2D of this step's W_{t+1} into buffer i
            if free[i] is not None:
                cps.wait_event(free[i])
            for w, hw in zip(bufs[i], h_v[i]):
                w.copy_(hw, non_blocking=True)
            loaded[i].record(cps)
        stream.wait_event(loaded[i])
        if out_free[i] is not None:
            stream.wait_event(out_free[i])
        body, table = ctxs[i].delta_extract(tls[i], out=outs[i], table="device")
        ev = torch.cuda.Event()
        ev.record(stream)
        free[i] = ev
        ctxs[i].delta_apply(tg, body, table=table)
        dhs.wait_stream(stream)
        with torch.cuda.stream(dhs):
            h_bodies[i][:body.numel()].copy_(body, non_blocking=True)
            ev2 = torch.cuda.Event()
            ev2.record(dhs)
            out_free[i] = ev2
        d2h[0] = body.numel()
    for _ in range(2):
        one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.e2e_steps):
        one()
    stream.wait_stream(cps)
    stream.wait_stream(dhs)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    last = bufs[(state["s"] - 1) % 2]
    ok = all(torch.equal(t.view(lt), w.view(lt)) and torch.equal(o.view(lt), w.view(lt))
             for t, o, w in zip(targets, olds, last))
    if not ok:
        raise SystemExit("bench: e2e (shadow) round trip mismatch")
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    for cx in ctxs:
        cx.close()
    del news2, bufs
    h2d = sum(w.numel() * w.element_size() for w in news)
    return {"value": round(scanned_total * args.e2e_steps / (ms / 1e3) / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h[0], "steps": args.e2e_steps,
            "ms_per_step": round(ms / args.e2e_steps, 3),
            "note": ("bytes per rank; W_{t+1} H2D from pinned host (W_t resident as the extract-and-advance "
                     "shadow), body D2H, apply on device; the compare still scans old+new; step s+1's H2D "
                     "overlaps step s's kernels and step s-1's D2H (two device buffers)")}


if __name__ == "__main__":
    sys.exit(main())
