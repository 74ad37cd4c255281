"""Thin Python binding of the C ABI (include/sparsedelta.h): argument marshalling only.

Every step of the path runs in the CUDA kernels behind ``libsparsedelta.so``; this module
turns torch tensors into descriptor arrays (pointers + sizes), passes the current CUDA
stream, and turns status codes into exceptions.  PyTorch supplies device memory and
streams only.
"""

import ctypes
from ctypes import byref, c_uint64, c_void_p

import torch

from . import _abi
from ._abi import RecordInfo, Span, Target, Tensor

_ELEM = {2: _abi.DELTA_ELEM16, 4: _abi.DELTA_ELEM32}
TABLE_FIELDS = ("record_offset", "element_count", "nnz", "index_offset", "index_bytes",
                "values_offset", "record_bytes")


class Table:
    """Offset-table rows of one extract (TABLE_FIELDS order), kept as the ctypes array the
    library filled, so it can be handed back to delta_apply as a hint without conversion.
    Indexing / iteration yield plain tuples."""

    __slots__ = ("arr", "n")

    def __init__(self, arr, n):
        self.arr, self.n = arr, n

    def __len__(self):
        return self.n

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(self.n))]
        if k < 0:
            k += self.n
        if not 0 <= k < self.n:
            raise IndexError(k)
        r = self.arr[k]
        return (r.record_offset, r.element_count, r.nnz, r.index_offset, r.index_bytes,
                r.values_offset, r.record_bytes)

    def __iter__(self):
        return (self[k] for k in range(self.n))

    def __eq__(self, other):
        return list(self) == list(other)


class DeviceTable:
    """The offset table of the last extract on ``ctx``, left in device memory (no host
    round trip); valid until the next extract on that context.  Pass it to delta_apply."""

    __slots__ = ("ptr", "n", "ctx")

    def __init__(self, ptr, n, ctx):
        self.ptr, self.n, self.ctx = ptr, n, ctx

    def __len__(self):
        return self.n


class DeltaError(RuntimeError):
    """A non-OK status from the library; ``status``/``detail`` are the C codes and
    ``kind`` the DELTA_D_* name (e.g. "truncated", "name") when there is one."""

    def __init__(self, status, detail, msg):
        self.status, self.detail = status, detail
        self.kind = _abi.DETAIL_NAMES.get(detail)
        super().__init__(f"{_abi.STATUS_NAMES.get(status, status)}: {msg}")


def _stream_handle(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return c_void_p(s.cuda_stream)


def _width(t: torch.Tensor) -> int:
    w = t.element_size()
    if w not in (2, 4):
        raise ValueError(f"lanes must be 2 or 4 bytes wide, got {t.dtype}")
    return w


class TensorList:
    """Descriptor array for a list of logical tensors, built once and reusable.

    ``tensors``: sequence of ``(name, old, new)`` where old/new are CUDA tensors (one
    span) or equal-length sequences of CUDA tensors (the spans of a fused tensor, in
    fusion order — PAPER.md:383).  Tensors must stay alive while this object is used."""

    def __init__(self, tensors):
        self.names = []
        self._keep = []
        n = len(tensors)
        self.arr = (Tensor * max(n, 1))()
        self.n = n
        self.width = None
        self.numel = []
        self.device = None
        for k, (name, old, new) in enumerate(tensors):
            olds = [old] if isinstance(old, torch.Tensor) else list(old)
            news = [new] if isinstance(new, torch.Tensor) else list(new)
            if len(olds) != len(news) or not olds:
                raise ValueError(f"tensor {name!r}: old/new span lists differ")
            spans = (Span * len(olds))()
            tot = 0
            for s, (o, w) in enumerate(zip(olds, news)):
                if not (o.is_cuda and w.is_cuda):
                    raise ValueError(f"tensor {name!r}: spans must be CUDA tensors")
                if o.numel() != w.numel() or o.element_size() != w.element_size():
                    raise ValueError(f"tensor {name!r} span {s}: old/new shape or width differ")
                if not (o.is_contiguous() and w.is_contiguous()):
                    raise ValueError(f"tensor {name!r} span {s}: spans must be contiguous")
                ww = _width(o)
                if self.width is None:
                    self.width = ww
                elif self.width != ww:
                    raise ValueError("all tensors must have the same lane width (SPEC.md:34)")
                if o.device != w.device or (self.device is not None and o.device != self.device):
                    raise ValueError(f"tensor {name!r} span {s}: all spans must be on one device")
                self.device = o.device
                spans[s].old_dev = o.data_ptr()
                spans[s].new_dev = w.data_ptr()
                spans[s].numel = o.numel()
                tot += o.numel()
            nb = name.encode("utf-8")
            self.arr[k].name = nb
            self.arr[k].name_len = len(nb)
            self.arr[k].n_spans = len(olds)
            self.arr[k].spans = spans
            self._keep += [nb, spans, olds, news]
            self.names.append(name)
            self.numel.append(tot)
        if self.width is None:
            self.width = 2


class TargetList:
    """Descriptor array for apply targets: sequence of ``(name, w)`` with ``w`` the
    resident fused parameter (contiguous CUDA tensor)."""

    def __init__(self, targets):
        n = len(targets)
        self.arr = (Target * max(n, 1))()
        self.n = n
        self._keep = []
        self.width = None
        self.device = None
        for k, (name, w) in enumerate(targets):
            if not w.is_cuda or not w.is_contiguous():
                raise ValueError(f"target {name!r} must be a contiguous CUDA tensor")
            if self.device is not None and w.device != self.device:
                raise ValueError(f"target {name!r}: all targets must be on one device")
            self.device = w.device
            ww = _width(w)
            if self.width is None:
                self.width = ww
            elif self.width != ww:
                raise ValueError("all targets must have the same lane width")
            nb = name.encode("utf-8")
            self.arr[k].w_dev = w.data_ptr()
            self.arr[k].numel = w.numel()
            self.arr[k].name = nb
            self.arr[k].name_len = len(nb)
            self._keep += [nb, w]
        if self.width is None:
            self.width = 2


class DeltaContext:
    """One ``delta_ctx`` (device workspace + cached plan) bound to a CUDA device."""

    def __init__(self, device=None):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.device = dev
        self._lib = _abi.lib()
        h = c_void_p()
        rc = self._lib.delta_ctx_create(byref(h), dev.index)
        if rc != 0:
            raise DeltaError(rc, 0, f"delta_ctx_create(device={dev.index}) failed")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            torch.cuda.synchronize(self.device)
            self._lib.delta_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            msg = self._lib.delta_last_error(self._h).decode(errors="replace")
            raise DeltaError(rc, self._lib.delta_last_detail(self._h), msg)

    def set_option(self, option: int, value: int):
        """DELTA_OPT_* launch-shape option (performance only)."""
        self._check(self._lib.delta_set_option(self._h, option, value))

    def set_profiling(self, enable):
        """Per-kernel CUDA-event timing inside the library: True / 1 = last calls
        (last_timing), 2 = accumulated over calls without host waits (timing_totals), 3 = as 2
        for the compare kernel K1 only."""
        mode = 1 if enable is True else (0 if enable is False else int(enable))
        self._check(self._lib.delta_set_profiling(self._h, mode))

    def timing_totals(self):
        """Profiling modes 2 / 3: (per-kernel totals in ms since the last call, extract scans
        covered); resets the totals."""
        t = _abi.Timing()
        calls = ctypes.c_uint32()
        self._check(self._lib.delta_timing_totals(self._h, byref(t), byref(calls)))
        return {f: getattr(t, f) for f, _ in _abi.Timing._fields_}, calls.value

    def last_timing(self) -> dict:
        t = _abi.Timing()
        self._check(self._lib.delta_last_timing(self._h, byref(t)))
        return {f: getattr(t, f) for f, _ in _abi.Timing._fields_}

    def _tensors(self, tensors) -> "TensorList":
        tl = tensors if isinstance(tensors, TensorList) else TensorList(tensors)
        if tl.device is not None and tl.device != self.device:
            raise ValueError(f"tensors are on {tl.device}, the context on {self.device}")
        return tl

    def _targets(self, targets) -> "TargetList":
        tg = targets if isinstance(targets, TargetList) else TargetList(targets)
        if tg.device is not None and tg.device != self.device:
            raise ValueError(f"targets are on {tg.device}, the context on {self.device}")
        return tg

    # --------------------------------------------------------------- C-ABI mirrors
    def delta_size(self, tensors, stream=None) -> int:
        """Body size in bytes (runs and caches the compare + compaction)."""
        tl = self._tensors(tensors)
        out = c_uint64()
        self._check(self._lib.delta_size(self._h, tl.arr, tl.n, _ELEM[tl.width],
                                         _stream_handle(stream), byref(out)))
        return out.value

    def size_table(self, n: int, stream=None) -> "Table":
        """Offset-table rows of the compaction the last ``delta_size`` left cached (host
        Table, no body written; the cache stays valid for a following ``delta_extract``)."""
        rows = (RecordInfo * max(n, 1))()
        self._check(self._lib.delta_size_table(self._h, n, rows, _stream_handle(stream)))
        return Table(rows, n)

    def compute_rho(self, tensors, stream=None):
        """SPEC.md:116-119 ``compute_rho`` / PAPER.md:294-297 Eq. 1 (delta_compute_rho):
        rho = sum_k nnz_k / sum_k N_k, nnz_k = lanes whose bits differ (reading R2).
        Returns ``(rho, nnz)``: the ratio and the per-tensor counts (descriptor order), both
        computed by the library.  Refused (DeltaError EINVAL) on an extract-and-advance
        context: its compare overwrites old."""
        tl = self._tensors(tensors)
        nnz = (c_uint64 * max(tl.n, 1))()
        tot, numel, rho = c_uint64(), c_uint64(), ctypes.c_double()
        self._check(self._lib.delta_compute_rho(self._h, tl.arr, tl.n, _ELEM[tl.width], _stream_handle(stream),
                                                nnz, byref(tot), byref(numel), byref(rho)))
        return rho.value, list(nnz[:tl.n])

    def delta_extract(self, tensors, out=None, stream=None, table=True):
        """Pack the delta.  Returns ``(body, table)``: ``body`` a uint8 CUDA tensor view of
        exactly the body bytes (``out``'s prefix if ``out`` is given); ``table``: True -> a
        host Table of offset-table rows (TABLE_FIELDS order; one extra synchronisation),
        "device" -> a DeviceTable (no extra synchronisation), False -> None."""
        tl = self._tensors(tensors)
        st = _stream_handle(stream)
        nbytes = c_uint64()
        rows = (RecordInfo * max(tl.n, 1))() if table is True else None
        if out is None:
            self._check(self._lib.delta_size(self._h, tl.arr, tl.n, _ELEM[tl.width], st, byref(nbytes)))
            out = torch.empty(max(nbytes.value, 1), dtype=torch.uint8, device=tl.device or self.device)
        if out.dtype != torch.uint8 or not out.is_contiguous() or not out.is_cuda:
            raise ValueError("out must be a contiguous uint8 CUDA tensor")
        self._check(self._lib.delta_extract(self._h, tl.arr, tl.n, _ELEM[tl.width], out.data_ptr(),
                                            out.numel(), rows, st, byref(nbytes)))
        body = out[:nbytes.value]
        if table == "device":
            return body, DeviceTable(self._lib.delta_table_dev(self._h), tl.n, self)
        if rows is None:
            return body, None
        return body, Table(rows, tl.n)

    def delta_extract_async(self, tensors, out, size, stream=None) -> "DeviceTable":
        """Enqueue the extraction into ``out`` (uint8 CUDA tensor, its numel the capacity)
        with no host synchronisation; ``size`` (int64 CUDA tensor, 1 element) receives the
        body size on the device (or -1 = UINT64_MAX if nothing was written).  Returns the
        device-resident offset table.  Pair with ``extract_wait``."""
        tl = self._tensors(tensors)
        if out.dtype != torch.uint8 or not out.is_contiguous() or not out.is_cuda:
            raise ValueError("out must be a contiguous uint8 CUDA tensor")
        if size.dtype != torch.int64 or not size.is_cuda or size.numel() != 1:
            raise ValueError("size must be a one-element int64 CUDA tensor")
        self._check(self._lib.delta_extract_async(self._h, tl.arr, tl.n, _ELEM[tl.width], out.data_ptr(),
                                                  out.numel(), c_void_p(size.data_ptr()), _stream_handle(stream)))
        return DeviceTable(self._lib.delta_table_dev(self._h), tl.n, self)

    def delta_extract_scan_async(self, tensors, size, stream=None):
        """Phase 1 of the async extract (compare, compaction, offset table): ``size`` (int64
        CUDA tensor, 1 element) receives this rank's body size on the device (-1 if a tile
        overflowed).  Follow with ``delta_extract_emit_async``."""
        tl = self._tensors(tensors)
        self._ntensors_last = tl.n
        if size is not None and (size.dtype != torch.int64 or not size.is_cuda or size.numel() != 1):
            raise ValueError("size must be a one-element int64 CUDA tensor")
        self._check(self._lib.delta_extract_scan_async(self._h, tl.arr, tl.n, _ELEM[tl.width],
                                                       c_void_p(size.data_ptr() if size is not None else 0),
                                                       _stream_handle(stream)))

    def delta_extract_emit_async(self, out, size, peer=None, sizes=None, rank: int = 0, stream=None) -> "DeviceTable":
        """Phase 2: the body into ``out`` (uint8 CUDA tensor) and, with ``peer`` (uint8 CUDA
        tensor, e.g. the root's buffer mapped by CUDA IPC), the same bytes into ``peer`` at
        sum(sizes[:rank]) — the fused emit + assembly.  ``sizes``: int64 CUDA tensor of every
        rank's size.  ``size`` receives the body size.  Pair with ``extract_wait``."""
        if out.dtype != torch.uint8 or not out.is_contiguous() or not out.is_cuda:
            raise ValueError("out must be a contiguous uint8 CUDA tensor")
        pp = c_void_p(peer.data_ptr()) if peer is not None else c_void_p(0)
        self._check(self._lib.delta_extract_emit_async(
            self._h, out.data_ptr(), out.numel(), c_void_p(size.data_ptr() if size is not None else 0), pp,
            peer.numel() if peer is not None else 0, c_void_p(sizes.data_ptr() if sizes is not None else 0),
            sizes.numel() if sizes is not None else 0, rank, _stream_handle(stream)))
        return DeviceTable(self._lib.delta_table_dev(self._h), self._ntensors_last, self)

    def extract_wait(self) -> int:
        """Wait for the last delta_extract_async; returns the body size.  Raises DeltaError
        with status EAGAIN after a slot overflow (workspace grown: issue the extract, and
        whatever was chained on it, again) or ECAPACITY."""
        nbytes = c_uint64()
        self._check(self._lib.delta_extract_wait(self._h, byref(nbytes)))
        return nbytes.value

    def round_trip(self, tensors, targets, out, size, stream=None, before_apply=None, wait=True, extract=None):
        """extract(tensors) -> apply into ``targets`` as one stream of kernels: the apply
        reads the body size and offset table on the device (delta_apply_async_chain), so
        the host waits once, at the end.  ``before_apply(out, size)`` may enqueue work
        between the two (e.g. the multi-GPU body assembly).  ``extract(tensors, out, size,
        stream) -> DeviceTable`` replaces the plain async extract (e.g. the fused multi-GPU
        emit, dist.FusedAssembler).  A first call at a higher density that overflows the tile
        slots (EAGAIN) is re-issued once.  Returns the body size.  ``wait=False``: enqueue
        only and return None — the host never waits, an overflow leaves the apply's gate
        closed (targets untouched) and is reported by the next extract_wait / apply_wait
        (steady-state loops after a first waited call)."""
        ex = extract or (lambda tl, o, sz, st: self.delta_extract_async(tl, o, sz, st))
        if not wait:  # enqueue only; errors surface at the next extract_wait / apply_wait
            table = ex(tensors, out, size, stream)
            if before_apply is not None:
                before_apply(out, size)
            self.delta_apply(targets, out, table=table, size=size, stream=stream, wait=False)
            return None
        for attempt in range(2):
            table = ex(tensors, out, size, stream)
            if before_apply is not None:
                before_apply(out, size)
            self.delta_apply(targets, out, table=table, size=size, stream=stream, wait=False)
            try:
                n = self.extract_wait()
            except DeltaError as e:
                if e.status != _abi.DELTA_EAGAIN or attempt:
                    raise
                try:  # the chained apply refused to run (gate closed): clear its status
                    self.apply_wait(stream)
                except DeltaError:
                    pass
                continue
            self.apply_wait(stream)
            return n
        raise AssertionError("unreachable")

    def delta_apply(self, targets, body, table=None, stream=None, wait=True, size=None):
        """Validate ``body`` fully, then scatter its values into ``targets`` in place
        (all-or-nothing).  ``table``: optional offset-table rows from delta_extract.
        ``wait=False`` enqueues only (delta_apply_async); call ``apply_wait`` later."""
        tg = self._targets(targets)
        if body.dtype != torch.uint8 or not body.is_contiguous() or not body.is_cuda:
            raise ValueError("body must be a contiguous uint8 CUDA tensor")
        hint = None
        if size is not None:  # chained: size (int64 CUDA tensor) and table on the device
            if not isinstance(table, DeviceTable):
                raise ValueError("a device-resident size needs a DeviceTable")
            self._check(self._lib.delta_apply_async_chain(self._h, tg.arr, tg.n, _ELEM[tg.width], body.data_ptr(),
                                                          body.numel(), c_void_p(size.data_ptr()),
                                                          c_void_p(table.ptr), _stream_handle(stream)))
            if wait:
                self.apply_wait(stream)
            return
        if isinstance(table, DeviceTable):
            self._check(self._lib.delta_apply_async_dev(self._h, tg.arr, tg.n, _ELEM[tg.width], body.data_ptr(),
                                                        body.numel(), c_void_p(table.ptr), _stream_handle(stream)))
            if wait:
                self.apply_wait(stream)
            return
        if table is not None:
            if isinstance(table, Table):
                hint = table.arr
            elif isinstance(table, ctypes.Array):
                hint = table
            else:
                hint = _rows_to_ctypes(table)
        fn = self._lib.delta_apply if wait else self._lib.delta_apply_async
        self._check(fn(self._h, tg.arr, tg.n, _ELEM[tg.width], body.data_ptr(), body.numel(), hint,
                       _stream_handle(stream)))

    def assemble(self, src, dst_peer, sizes, rank, stream=None):
        """Copy this rank's body ``src`` (uint8 CUDA tensor) into ``dst_peer`` (the root's
        assembled-body tensor mapped into this process) at the offset given by the device
        tensor ``sizes`` (int64, one per rank); see delta_assemble."""
        self._check(self._lib.delta_assemble(self._h, c_void_p(src.data_ptr() if src.numel() else 0),
                                             c_void_p(dst_peer.data_ptr()), dst_peer.numel(),
                                             c_void_p(sizes.data_ptr()), sizes.numel(), rank,
                                             _stream_handle(stream)))

    def table_dev_ptr(self) -> int:
        """Device pointer of this context's offset table (delta_table_dev): valid after an
        extract until the next one on the same context."""
        return self._lib.delta_table_dev(self._h) or 0

    def record_sizes(self, table_ptr: int, n_local: int, gidx, sizes, stream=None):
        """This rank's record sizes into the global-order int64 CUDA tensor ``sizes`` (zeros
        elsewhere); ``table_ptr``: device offset table (DeviceTable.ptr), ``gidx``: int32
        CUDA tensor of the local records' global indices (delta_record_sizes)."""
        self._check(self._lib.delta_record_sizes(self._h, c_void_p(table_ptr), n_local, c_void_p(gidx.data_ptr()),
                                                 c_void_p(sizes.data_ptr()), sizes.numel(), _stream_handle(stream)))

    def assemble_records(self, src, gidx, sizes, dst, stream=None):
        """Copy this rank's body ``src`` record by record to the global offsets in ``dst``
        (the root's buffer, local or IPC-mapped) from the summed global ``sizes``
        (delta_assemble_records)."""
        self._check(self._lib.delta_assemble_records(self._h, c_void_p(src.data_ptr() if src.numel() else 0),
                                                     c_void_p(gidx.data_ptr()), gidx.numel(),
                                                     c_void_p(sizes.data_ptr()), sizes.numel(),
                                                     c_void_p(dst.data_ptr()), dst.numel(), _stream_handle(stream)))

    def digest(self, body, stream=None) -> bytes:
        """BLAKE3-256 of a uint8 CUDA tensor, computed on the GPU (delta_digest)."""
        out = ctypes.create_string_buffer(32)
        self._check(self._lib.delta_digest(self._h, c_void_p(body.data_ptr() if body.numel() else 0),
                                           body.numel(), out, _stream_handle(stream)))
        return out.raw

    def delta_merge(self, body_a, body_b, n: int, width: int = 2, out=None, stream=None):
        """The body equivalent to applying ``body_a`` then ``body_b`` (both uint8 CUDA
        tensors holding n records each; reading R19).  Returns a uint8 CUDA tensor view of
        exactly the merged bytes (``out``'s prefix if given)."""
        st = _stream_handle(stream)
        nbytes = c_uint64()
        elem = _ELEM[width]

        def call(o, cap):
            return self._lib.delta_merge(self._h, n, elem, c_void_p(body_a.data_ptr() if body_a.numel() else 0),
                                         body_a.numel(), c_void_p(body_b.data_ptr() if body_b.numel() else 0),
                                         body_b.numel(), c_void_p(o.data_ptr() if o is not None else 0), cap, st,
                                         byref(nbytes))
        if out is None:  # the merge is never longer than the two bodies together
            out = torch.empty(max(body_a.numel() + body_b.numel(), 1), dtype=torch.uint8, device=body_b.device)
        self._check(call(out, out.numel()))
        return out[:nbytes.value]

    def container_header(self, body, version: int, base_version: int, width: int, n_tensors: int, out,
                         index_codec: str = "leb128", stream=None):
        """delta_container_header: the 67-byte SPDC header of ``body`` (uint8 CUDA tensor),
        digest included, written on the device into ``out`` (uint8 CUDA tensor, first 67
        bytes)."""
        self._check(self._lib.delta_container_header(
            self._h, c_void_p(body.data_ptr() if body.numel() else 0), body.numel(), version, base_version,
            _ELEM[width], n_tensors, {"leb128": 1, "fixed": 2}[index_codec], c_void_p(out.data_ptr()),
            _stream_handle(stream)))

    def assemble_wait(self, stream=None):
        self._check(self._lib.delta_assemble_wait(self._h, _stream_handle(stream)))

    def apply_wait(self, stream=None):
        """Synchronise and raise the first error of the async applies since the last wait."""
        self._check(self._lib.delta_apply_wait(self._h, _stream_handle(stream)))


def rebase(rows, offset: int) -> "Table":
    """Offset-table rows of a body placed ``offset`` bytes into a larger body (the library's
    delta_table_rebase; host only).  ``rows``: a Table or a sequence of TABLE_FIELDS tuples;
    returns a new Table."""
    src = rows.arr if isinstance(rows, Table) else _rows_to_ctypes(rows)
    n = len(rows)
    arr = (RecordInfo * max(n, 1))()
    ctypes.memmove(arr, src, ctypes.sizeof(RecordInfo) * n)
    rc = _abi.lib().delta_table_rebase(arr, n, offset)
    if rc != 0:
        raise DeltaError(rc, 0, f"delta_table_rebase(offset={offset}) failed")
    return Table(arr, n)


def _rows_to_ctypes(rows):
    arr = (RecordInfo * max(len(rows), 1))()
    for k, r in enumerate(rows):
        for f, v in zip(TABLE_FIELDS, r):
            setattr(arr[k], f, int(v))
    return arr


_default = {}


def context(device=None) -> DeltaContext:
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    if dev not in _default:
        _default[dev] = DeltaContext(torch.device("cuda", dev))
    return _default[dev]


def delta_size(tensors, stream=None) -> int:
    return context().delta_size(tensors, stream=stream)


def compute_rho(tensors, stream=None):
    return context().compute_rho(tensors, stream=stream)


def delta_extract(tensors, out=None, stream=None, table=True):
    return context().delta_extract(tensors, out=out, stream=stream, table=table)


def delta_apply(targets, body, table=None, stream=None):
    return context().delta_apply(targets, body, table=table, stream=stream)


def version() -> str:
    return _abi.lib().delta_version().decode()
