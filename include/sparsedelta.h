/*
 * sparsedelta.h — C ABI of the B200 sparse-delta codec (SparrowRL, arXiv 2602.11456).
 *
 * The operation (§3 Eq. 1; §5.1 "Sparse encoding",
 * "Lossless precision"): given K parameter tensors before (W_t) and after (W_{t+1}) one
 * RL step, the trainer "flattens each tensor's delta into a one-dimensional index space
 * and stores the non-zeros as two 1D arrays, idx and val", encodes idx by
 * "delta encoding" — first index as-is, then differences — written as
 * unsigned LEB128; Actors "apply the update with a flat scatter-add
 * over the parameter's storage" so they hold "exactly the same update as
 * the Trainer".
 *
 * Readings fixed at this boundary:
 *   R1 replace mode: values are the NEW lane bits; apply is a scatter-STORE (bit-exact).
 *   R2 "changed" = bitwise lane inequality (-0.0 vs +0.0 changes; equal NaN bits do not).
 *   R3 the first index is stored as its absolute value, also LEB128.
 *   R4 one index space per logical (fused) tensor; the gap chain restarts per record.
 *   R5 a fused tensor's lanes are its spans concatenated in the order given (Q,K,V; Gate,Up).
 *
 * Body layout (little-endian), one record per tensor in descriptor order,
 * also when nothing changed:
 *     u16 name_len | name | u64 element_count | u64 nnz | u64 index_bytes |
 *     index_stream[index_bytes] | values[nnz * w] | u8 mode (= 0, replace)
 * record_bytes = 27 + name_len + index_bytes + w * nnz.
 *
 * Conventions
 *   - Pointers named *_dev are CUDA global memory on the context's device; everything
 *     else is host memory.  `stream` is a cudaStream_t passed as void* (NULL = legacy
 *     default stream).  All device work is ordered on `stream`.
 *   - The caller owns every buffer and descriptor array; they are read only during the
 *     call (device buffers: until the stream work of the call has completed).
 *   - The context owns a grow-only device workspace reused across calls; no device
 *     allocation happens in steady state.  One context per (host thread, stream); a
 *     context is not thread-safe.
 *   - Every call returns DELTA_OK (0) or a negative status; delta_last_error() then
 *     describes it.  Nothing aborts the process.
 *   - There is no CPU fallback: without a usable CUDA device every call that needs one
 *     returns DELTA_ECUDA.
 */
#ifndef SPARSEDELTA_H
#define SPARSEDELTA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. */
enum {
    DELTA_OK = 0,
    DELTA_EINVAL = -1,    /* NULL pointer, n_spans == 0, name_len > 65535, bad elem, misaligned target */
    DELTA_ESHAPE = -2,    /* old/new span structure mismatch */
    DELTA_ECAPACITY = -3, /* out_capacity too small; *body_bytes holds the size needed */
    DELTA_ECORRUPT = -4,  /* malformed body; see delta_last_detail() */
    DELTA_ENAME = -5,     /* record name / element count does not match its target */
    DELTA_ECUDA = -6,     /* CUDA runtime error or no device */
    DELTA_ENOMEM = -7,    /* device workspace allocation failed */
    DELTA_EAGAIN = -8     /* delta_extract_wait: tile slots overflowed at a new density; the
                             workspace has been grown, nothing was written — issue again */
};

/* Detail of a DELTA_ECORRUPT / DELTA_ENAME status (delta_last_detail). */
enum {
    DELTA_D_NONE = 0,
    DELTA_D_TRUNCATED = 1,     /* index stream ends inside a varint */
    DELTA_D_OVERLONG = 2,      /* non-minimal varint, e.g. 80 00 */
    DELTA_D_OVERFLOW = 3,      /* varint exceeds 64 bits */
    DELTA_D_NONINCREASING = 4, /* zero gap after the first index */
    DELTA_D_RANGE = 5,         /* decoded index >= element_count */
    DELTA_D_COUNT = 6,         /* number of varints != nnz */
    DELTA_D_NAME = 7,          /* record name != target name */
    DELTA_D_NUMEL = 8,         /* record element_count != target numel */
    DELTA_D_MODE = 9,          /* mode byte not in {0 (replace), 1 (additive)}; delta_merge: not 0 */
    DELTA_D_LAYOUT = 10        /* record past the body end, trailing bytes, record count != n */
};

/* Element lane widths (SPEC.md:147 element-type codes). */
enum { DELTA_ELEM16 = 0, /* bf16 / fp16: 2-byte lanes */
       DELTA_ELEM32 = 1  /* fp32: 4-byte lanes */ };

/* One contiguous block of a logical tensor (e.g. the q_proj block of qkv_proj).
 * old_dev / new_dev: numel lanes each, any alignment (16-byte aligned pairs take the
 * vectorised path, others a lane-by-lane path of the same kernel). */
typedef struct {
    const void *old_dev;
    const void *new_dev;
    uint64_t numel;
} delta_span;

/* One logical (fused) tensor: the concatenation of n_spans spans (reading R5).
 * name: name_len UTF-8 bytes (not NUL-terminated, <= 65535), host memory. */
typedef struct {
    const char *name;
    uint32_t name_len;
    uint32_t n_spans;
    const delta_span *spans;
} delta_tensor;

/* One apply target: the resident fused parameter, numel lanes, lane-aligned. */
typedef struct {
    void *w_dev;
    uint64_t numel;
    const char *name;
    uint32_t name_len;
} delta_target;

/* Per-record offset table row (north_star "per-tensor offset tables"); byte offsets are
 * relative to the start of the body. */
typedef struct {
    uint64_t record_offset;
    uint64_t element_count;
    uint64_t nnz;
    uint64_t index_offset;  /* = record_offset + 2 + name_len + 24 */
    uint64_t index_bytes;
    uint64_t values_offset; /* = index_offset + index_bytes */
    uint64_t record_bytes;  /* = 27 + name_len + index_bytes + w * nnz */
} delta_record_info;

typedef struct delta_ctx delta_ctx; /* opaque: device, workspace, cached plan + scan */

/* Create a context bound to CUDA device `device` (makes it current on this thread).
 * *ctx is NULL on failure: DELTA_ECUDA if the device is unusable. */
int delta_ctx_create(delta_ctx **ctx, int device);

/* Free the context and its workspace.  Waits for no stream; the caller must make sure
 * no call's device work on this context is still pending.  NULL is a no-op. */
void delta_ctx_destroy(delta_ctx *ctx);

/* Message for the last non-OK status on this context ("" if none).  Owned by ctx. */
const char *delta_last_error(const delta_ctx *ctx);

/* DELTA_D_* detail of the last DELTA_ECORRUPT / DELTA_ENAME status. */
int delta_last_detail(const delta_ctx *ctx);

/* Library build string (compile flags, target arch). */
const char *delta_version(void);

/* delta_size — size of the packed body for `tensors` (E1-E3 + size readback E7).
 *
 * Runs the bitwise compare + ordered compaction over all n tensors (one grouped launch),
 * the LEB128 length pass and the offset-table pass, then synchronises `stream` once and
 * writes the body size in bytes to *body_bytes (host).  The compaction is cached on ctx:
 * a following delta_extract with identical descriptors (same pointers, sizes, names,
 * elem) reuses it without re-reading old/new — the caller must not modify old/new in
 * between (two-phase, as CUB's temp-storage query).
 * With DELTA_OPT_ADVANCE the compare also overwrites old with new: call delta_size at most
 * once per step (a second call compares old against itself and finds nothing) and follow it
 * with delta_extract, which consumes the cached compaction — also after a DELTA_ECAPACITY
 * return, so the retry with a larger buffer emits the same body.
 *   tensors: n descriptors (host); elem: DELTA_ELEM16 or DELTA_ELEM32.
 * Errors: DELTA_EINVAL, DELTA_ESHAPE (a span with numel but NULL pointers), DELTA_ECUDA,
 * DELTA_ENOMEM. */
int delta_size(delta_ctx *ctx, const delta_tensor *tensors, uint32_t n, int elem,
               void *stream, uint64_t *body_bytes);

/* delta_size_table — the offset table of the compaction the last delta_size on ctx left
 * cached, without writing a body (E6 table rows, E7 per-tensor readback).
 *
 * Rows (host, n entries, descriptor order) carry element_count N_k and nnz_k = ||ΔW^(k)||_0
 * under the bitwise-inequality reading (Eq. 1
 * compute_rho: rho = Σ nnz_k / Σ N_k), plus the offsets the body would have.  Synchronises
 * `stream` once.  The cached compaction stays valid for a following delta_extract.
 *   n: must equal the tensor count of that delta_size call.
 * Errors: DELTA_EINVAL (no cached delta_size result — e.g. a delta_extract consumed it —,
 * n mismatch, NULL table with n > 0), DELTA_ECUDA. */
int delta_size_table(delta_ctx *ctx, uint32_t n, delta_record_info *table, void *stream);

/* delta_compute_rho — SPEC.md:116-119 compute_rho, Eq. 1:
 *     rho = sum_k ||dW^(k)||_0 / sum_k N_k,
 * with ||dW^(k)||_0 = nnz_k, the lanes of tensor k whose bits differ (reading R2).  Runs the
 * compare + compaction of delta_size (cached on ctx for a following delta_extract) and sums
 * the offset-table rows on the host side of the library.  Synchronises `stream` twice.
 *   nnz:         host array of n uint64 (per-tensor nnz_k, descriptor order) or NULL;
 *   nnz_total, numel_total, rho: host, required (rho = 0 when numel_total == 0).
 * Errors: as delta_size; DELTA_EINVAL on a context with DELTA_OPT_ADVANCE set (the advancing
 * compare would overwrite old — compute_rho is a pure function). */
int delta_compute_rho(delta_ctx *ctx, const delta_tensor *tensors, uint32_t n, int elem, void *stream,
                      uint64_t *nnz, uint64_t *nnz_total, uint64_t *numel_total, double *rho);

/* delta_table_rebase — host-only (no device, no context): shift n offset-table rows (host) of a
 * body that is placed `offset` bytes into a larger body, e.g. a group's or a rank's records
 * after the earlier ones (R15): record_offset, index_offset and values_offset += offset.
 * DELTA_EINVAL for NULL rows with n > 0 or an offset that overflows 64 bits (rows untouched
 * from the failing row on). */
int delta_table_rebase(delta_record_info *rows, uint32_t n, uint64_t offset);

/* delta_extract — write the packed body (records in descriptor order) to out_dev.
 *
 * If the previous call on ctx was delta_size with identical descriptors, its cached
 * compaction is consumed; otherwise the whole extraction runs here.  Synchronises
 * `stream` once (size readback) and, if `table` is non-NULL, a second time to copy the
 * n offset-table rows to `table` (host, n entries).  *body_bytes (host, required)
 * receives the body size.
 *   out_dev: device buffer of out_capacity bytes, any alignment.
 * Errors: as delta_size, plus DELTA_ECAPACITY (nothing written; *body_bytes = needed). */
int delta_extract(delta_ctx *ctx, const delta_tensor *tensors, uint32_t n, int elem,
                  void *out_dev, uint64_t out_capacity, delta_record_info *table,
                  void *stream, uint64_t *body_bytes);

/* delta_extract_async — delta_extract as enqueue-only work: no host synchronisation
 * (except the one-time plan upload when the descriptors change).  The same K1-K5
 * kernels run on `stream`; K4/K5 write the body only if every tile's changes fitted the
 * context's tile slots and the body fits out_capacity (the "emit gate"), and write the
 * body size — or UINT64_MAX when the gate is closed — to body_bytes_dev (device, 8-byte
 * aligned u64, may be NULL).  The offset table is left on the device (delta_table_dev).
 * Pair every call with delta_extract_wait.  Work chained after it on the same stream
 * (delta_apply_async_chain) reads the size and table on the device.
 * Errors (immediate): as delta_size. */
int delta_extract_async(delta_ctx *ctx, const delta_tensor *tensors, uint32_t n, int elem,
                        void *out_dev, uint64_t out_capacity, uint64_t *body_bytes_dev,
                        void *stream);

/* delta_extract_scan_async + delta_extract_emit_async — delta_extract_async in its two
 * phases, for the fused multi-GPU emit + assembly (the
 * in-box analog of the paper's cut-through emission).
 *
 * delta_extract_scan_async: compare, compaction and offset table (K1-K3) on `stream`; writes
 * this rank's body size to size_dev (device, 8-byte aligned u64; UINT64_MAX if a tile
 * overflowed its slot; may be NULL).  No host synchronisation.  Must be followed by exactly
 * one delta_extract_emit_async on the same ctx and stream (DELTA_EINVAL otherwise).
 *
 * delta_extract_emit_async: writes the body to out_dev (out_capacity bytes) and, if peer_dev
 * is not NULL, the same bytes to peer_dev (peer_capacity bytes; e.g. the root's assembled-body
 * buffer mapped into this process with CUDA IPC, so the stores go over NVLink) at byte offset
 * sum(sizes_dev[q], q < rank) — every record lands at its global offset straight from the
 * compaction, with no separate copy of the body.  sizes_dev: n_ranks u64 on this device (e.g. an
 * NCCL all-gather of every rank's size_dev); rank < n_ranks.  body_bytes_dev (may be NULL)
 * receives the size, or UINT64_MAX if the local gate is closed.  The local body is written iff
 * the scan fitted and the body fits out_capacity; the peer copy iff, in addition, no size is
 * UINT64_MAX and the records fit peer_capacity.  delta_extract_wait reports the outcome of both:
 * DELTA_EAGAIN (a tile overflowed here, or another rank's size was UINT64_MAX: nothing was
 * assembled), DELTA_ECAPACITY (out or peer too small).  The caller orders the peer stores
 * before the root's readers (e.g. an NCCL all-reduce on this stream after the call).
 * Errors (immediate): as delta_size; DELTA_EINVAL for a missing scan phase, misaligned size
 * pointers, NULL sizes_dev with a peer, or rank >= n_ranks. */
int delta_extract_scan_async(delta_ctx *ctx, const delta_tensor *tensors, uint32_t n, int elem,
                             uint64_t *size_dev, void *stream);
int delta_extract_emit_async(delta_ctx *ctx, void *out_dev, uint64_t out_capacity, uint64_t *body_bytes_dev,
                             void *peer_dev, uint64_t peer_capacity, const uint64_t *sizes_dev, uint32_t n_ranks,
                             uint32_t rank, void *stream);

/* delta_extract_wait — wait for the last delta_extract_async on ctx (an event, not the
 * whole stream) and report the outcome of EVERY delta_extract_async since the previous wait
 * (a closed emit gate in any of them is reported, not only in the last); *body_bytes (host,
 * may be NULL) = the last body's size (on DELTA_ECAPACITY: the largest size needed).
 * DELTA_EAGAIN: a tile held more changes than the slots (first call at a higher density);
 * the slots have been grown, no body was written, repeat the extract (and anything
 * chained on it, which refused to run: see delta_apply_async_chain).  DELTA_ECAPACITY:
 * body larger than out_capacity, nothing written, *body_bytes = size needed. */
int delta_extract_wait(delta_ctx *ctx, uint64_t *body_bytes);

/* delta_apply — validate the whole body, then scatter-store its values into the targets
 * (A1-A4; "validate fully before mutating").
 *
 * targets: n descriptors (host), one per record in body order; each w_dev is lane-aligned.
 * body_dev: device, body_bytes bytes, any alignment.
 * table_hint: optional host array of n rows as produced by delta_extract.  With it the
 *   record headers are located in one parallel pass and every field is re-verified
 *   against the body; a hint that does not match the body is ignored (the headers are
 *   then walked sequentially), so a wrong hint can cost time but never correctness.
 * All-or-nothing: on any non-OK status the targets are bitwise unchanged.  The call
 * synchronises `stream` once at the end to read the device status word.
 * Errors: DELTA_EINVAL, DELTA_ECORRUPT, DELTA_ENAME (detail via delta_last_detail),
 * DELTA_ECUDA, DELTA_ENOMEM. */
int delta_apply(delta_ctx *ctx, const delta_target *targets, uint32_t n, int elem,
                const void *body_dev, uint64_t body_bytes,
                const delta_record_info *table_hint, void *stream);

/* delta_apply_async — delta_apply without the final synchronisation: validates and
 * scatters on `stream` (same all-or-nothing gate per call) and returns once the work is
 * enqueued.  Errors found on the device are kept in a sticky status word read by
 * delta_apply_wait.  Host-side argument errors are returned immediately.  Several calls
 * may be enqueued on one stream (each call's targets/body must stay valid until the
 * matching wait); do not mix streams on one ctx. */
int delta_apply_async(delta_ctx *ctx, const delta_target *targets, uint32_t n, int elem,
                      const void *body_dev, uint64_t body_bytes,
                      const delta_record_info *table_hint, void *stream);

/* delta_apply_async_dev — delta_apply_async with the table hint in DEVICE memory (same
 * layout as delta_record_info, n rows), e.g. delta_table_dev() of the context that
 * extracted the body, so no host round trip is needed between extract and apply.  The
 * hint must stay valid until the stream work is done; it is verified like the host hint. */
int delta_apply_async_dev(delta_ctx *ctx, const delta_target *targets, uint32_t n, int elem,
                          const void *body_dev, uint64_t body_bytes,
                          const delta_record_info *table_hint_dev, void *stream);

/* delta_apply_async_chain — delta_apply_async_dev with the body SIZE in device memory as
 * well: body_bytes_dev (u64, 8-byte aligned) as written by delta_extract_async, body_dev
 * a buffer of body_capacity bytes.  A size above body_capacity (UINT64_MAX: the extract's
 * emit gate was closed) fails the call's gate with detail DELTA_D_LAYOUT and mutates
 * nothing.  With delta_extract_async this makes extract -> apply one stream of kernels
 * with no host round trip between them. */
int delta_apply_async_chain(delta_ctx *ctx, const delta_target *targets, uint32_t n, int elem,
                            const void *body_dev, uint64_t body_capacity, const uint64_t *body_bytes_dev,
                            const delta_record_info *table_hint_dev, void *stream);

/* Device address of the offset table written by the last delta_size/delta_extract on ctx
 * (n rows; NULL if none).  Valid until the next extract call on ctx. */
const delta_record_info *delta_table_dev(const delta_ctx *ctx);

/* delta_apply_wait — synchronise `stream` and return the first device-side error of the
 * delta_apply_async calls since the previous wait (DELTA_OK if none), then clear it. */
int delta_apply_wait(delta_ctx *ctx, void *stream);

/* delta_assemble — S3 of the multi-GPU path as one kernel over NVLink peer memory: copy
 * this rank's body (src_dev, sizes_dev[rank] bytes; this GPU, 16-byte aligned) into the
 * assembled body on the root GPU, dst_peer_dev (the root's buffer mapped into this process
 * with CUDA IPC, dst_capacity bytes), at offset sum(sizes_dev[0..rank-1]).  sizes_dev: the
 * n_ranks body sizes in device memory (e.g. an NCCL all-gather); the offset is computed on
 * the device, so no host round trip is needed.  Asynchronous on `stream`; a destination
 * overflow is reported by delta_assemble_wait.  The caller orders the copy against the
 * root's readers (e.g. an NCCL all-reduce on the same stream after it). */
int delta_assemble(delta_ctx *ctx, const void *src_dev, void *dst_peer_dev, uint64_t dst_capacity,
                   const uint64_t *sizes_dev, uint32_t n_ranks, uint32_t rank, void *stream);

/* Record-granular assembly, for any tensor partition (LPT balances the
 * shards better than contiguous ranges, but then a rank's records are not one byte range of
 * the global body).  Global record order is the descriptor order of the whole list (R15).
 *
 * delta_record_sizes — write this rank's record sizes into sizes_dev (n_global uint64, device,
 * global order; every other entry set to 0): sizes_dev[gidx_dev[j]] = table_dev[j].record_bytes
 * for the n_local rows of table_dev (this rank's device offset table, e.g. delta_table_dev,
 * rows in this rank's order) and gidx_dev (n_local uint32, device: global index of local
 * record j, ascending).  Asynchronous on `stream`.  Summing sizes_dev over the ranks (one
 * NCCL all-reduce) gives every record's size on every rank.
 *
 * delta_assemble_records — copy this rank's body (src_dev: its records back to back in local
 * order) record by record into dst_dev (the root's assembled-body buffer, this GPU's own
 * memory or a CUDA IPC peer mapping over NVLink, dst_capacity bytes): record j goes to the
 * global offset sum(sizes_dev[0 .. gidx_dev[j] - 1]), computed on the device from the summed
 * sizes_dev.  Asynchronous on `stream`; a total larger than dst_capacity (or a ~0 size from a
 * closed extract gate) writes nothing and is reported by delta_assemble_wait.  The caller
 * orders the copies against the root's readers (e.g. an all-reduce after them). */
int delta_record_sizes(delta_ctx *ctx, const delta_record_info *table_dev, uint32_t n_local,
                       const uint32_t *gidx_dev, uint64_t *sizes_dev, uint32_t n_global, void *stream);
int delta_assemble_records(delta_ctx *ctx, const void *src_dev, const uint32_t *gidx_dev, uint32_t n_local,
                           const uint64_t *sizes_dev, uint32_t n_global, void *dst_dev, uint64_t dst_capacity,
                           void *stream);

/* Synchronise `stream`; DELTA_ECAPACITY if a delta_assemble since the last wait would have
 * overflowed its destination (nothing was written by that copy), else DELTA_OK. */
int delta_assemble_wait(delta_ctx *ctx, void *stream);

/* delta_digest — BLAKE3-256 of body_dev[0..bytes) computed on the GPU (NEXT f1: the delta
 * checkpoint's integrity hash; reading R10: BLAKE3 over exactly the
 * body bytes).  Writes the 32-byte digest to out32 (host) after synchronising
 * `stream` once. */
int delta_digest(delta_ctx *ctx, const void *body_dev, uint64_t bytes, uint8_t *out32, void *stream);

/* delta_container_header — the SPDC container header written on the device (NEXT f1;
 * PAPER.md:368-370 "versioned, immutable ... integrity hash"):
 *     "SPDC" | u16 format_version | u64 version | u64 base_version | u8 element code
 *     (0 = 16-bit lanes, 1 = 32-bit) | u32 n_tensors | u64 body length | BLAKE3-256(body)
 * = 67 bytes, little-endian, to out_dev (device, any alignment; e.g. the 67 bytes ahead of the
 * body in one buffer, so the container never passes through host memory).  The digest covers
 * exactly the body bytes (reading R10); format_version = index_codec: 1 LEB128, 2 fixed-width
 * (reading R18).  Asynchronous on `stream` (no host synchronisation).
 * Errors: DELTA_EINVAL (NULL pointers, elem, index_codec not 1/2, version != base_version + 1),
 * DELTA_ECUDA, DELTA_ENOMEM. */
int delta_container_header(delta_ctx *ctx, const void *body_dev, uint64_t body_bytes, uint64_t version,
                           uint64_t base_version, int elem, uint32_t n_tensors, int index_codec, void *out_dev,
                           void *stream);

/* ---------------------------------------------------------------------------------------
 * delta_merge — NEXT f4 (reading R19): two consecutive bodies D_a (version v-1 ->
 * v) and D_b (v -> v+1) over the same n tensors become ONE body (v-1 -> v+1) that a laggard
 * applies instead of replaying both ("laggards catch up asynchronously";
 * SPEC.md:476 leaves merging open).  Per record: the index set is the union of the two, the
 * value is D_b's where D_b has the index and D_a's otherwise, so
 * delta_apply(merge) == delta_apply(D_a) then delta_apply(D_b) for any base weights.  The
 * merged body is canonical (sorted unique indices, minimal LEB128), in D_b's record order
 * and names.
 *   body_a_dev / body_b_dev  device, a_bytes / b_bytes long, read only; LEB128 index streams
 *                            (DELTA_OPT_INDEX_CODEC = 1 on ctx, else DELTA_EINVAL);
 *   n                        records expected in each body;
 *   out_dev                  device, out_capacity bytes, receives the merged body;
 *   *out_bytes (host)        the merged size (also on DELTA_ECAPACITY, nothing written).
 * Both bodies are validated fully before anything is written: layout / record count, mode
 * byte != 0 (replace only) -> DELTA_ECORRUPT (detail LAYOUT / MODE); names or element counts
 * that differ between the bodies -> DELTA_ENAME (detail NAME / NUMEL); every decode check of
 * delta_apply (TRUNCATED, OVERLONG, OVERFLOW, NONINCREASING, RANGE, COUNT) -> DELTA_ECORRUPT.
 * Stream-ordered on `stream`; synchronises with the host four times (intermediate sizes);
 * the emit is asynchronous (synchronise the stream before reading out_dev). */
int delta_merge(delta_ctx *ctx, uint32_t n, int elem, const void *body_a_dev, uint64_t a_bytes,
                const void *body_b_dev, uint64_t b_bytes, void *out_dev, uint64_t out_capacity, void *stream,
                uint64_t *out_bytes);

/* Per-kernel device times of the last delta_size/delta_extract/delta_apply on this ctx,
 * in milliseconds, measured with CUDA events recorded on the call's stream around each
 * kernel (only while profiling is enabled; zero otherwise).  A field is the time of the
 * most recent launch of that kernel; *_count fields say how many launches it covers. */
typedef struct {
    float scan_ms;      /* K1 compare + ordered compaction (reads old and new) */
    float lens_ms;      /* K2 gap LEB128 lengths */
    float finalize_ms;  /* K3 offset table */
    float emit_ms;      /* K4 index bytes + values */
    float headers_ms;   /* K5 record headers */
    float locate_ms;    /* A1 record headers located + verified */
    float decode_ms;    /* A2 LEB128 decode + validation */
    float apply_scan_ms;/* A3 per-record scans + count/range checks */
    float scatter_ms;   /* A4 gated scatter-store */
} delta_timing;

/* Launch-shape options (performance only; results never depend on them). */
enum {
    DELTA_OPT_APPLY_CTAS_PER_SM = 1, /* grid of the apply decode kernel, CTAs per SM (default 64 CTAs of 128
                                        threads: many short CTAs, scheduled as slots free up, balance
                                        the chunks; measured 0.080 ms at 32, 0.076 at 64) */
    DELTA_OPT_EMIT_CTAS_PER_SM = 2,  /* grid of the extract emit kernel, CTAs per SM (default 24: ~5 resident,
                                        the rest scheduled as slots free; measured 0.164 ms at 8, 0.153 at 24) */
    DELTA_OPT_SCAN_KERNEL = 3,       /* compare+compaction kernel: 1 = one CTA per tile, 16-byte
                                        vectors, bitmap compaction (the only form; the retired
                                        variants 2-5 — TMA pipeline, 128-byte runs, 512 x 4,
                                        persistent — were measured slower): DELTA_EINVAL */
    DELTA_OPT_SCATTER_CTAS_PER_SM = 4, /* grid of the apply scatter kernel, CTAs per SM (default 96: ~19
                                        waves of 5 resident CTAs; measured 2.44 ms at 5, 2.30 at 96) */
    DELTA_OPT_PREFETCH_TILES = 5,     /* 1 + distance, in tiles, of the L2 bulk prefetch issued by
                                         the default compare kernel (1 = off; default: one wave of
                                         resident tiles, 3 x SMs) */
    DELTA_OPT_SCATTER_ORDER = 6,      /* 1 = each thread stores the entries it decoded,
                                         2 = entry-major: thread i stores entries i, i+256, ...
                                         (default for 16-bit lanes) */
    DELTA_OPT_MODE = 7,               /* records written by extract: 1 = replace (default; values
                                         are the new lanes, apply stores them, bit-exact),
                                         2 = additive (values are new - old and apply adds them,
                                         SPEC.md:99, 135: 16-bit lanes read as bf16, 32-bit as
                                         fp32, fp32 arithmetic rounded to nearest even — lossy,
                                         for fidelity experiments).  delta_apply follows each
                                         record's mode byte. */
    DELTA_OPT_INDEX_CODEC = 8,        /* index stream of the records, for delta_extract* AND
                                         delta_apply* on this ctx (the body does not say which;
                                         the SPDC container's format_version does: 1 / 2):
                                         1 = LEB128 gaps (default);
                                         2 = the naive fixed-width encoding the paper compares
                                         against ("int32 or int64 (depending on tensor
                                         size)"): nnz absolute indices, little-endian,
                                         4 bytes if element_count - 1 <= 2^31 - 1 else 8, so
                                         index_bytes = nnz x width (reading R18).  Apply
                                         of a fixed-width body: index_bytes not a multiple of the
                                         width -> DELTA_D_TRUNCATED, != nnz indices -> DELTA_D_COUNT,
                                         not strictly increasing -> DELTA_D_NONINCREASING, an index
                                         >= element_count -> DELTA_D_RANGE (all-or-nothing as ever). */
    DELTA_OPT_ASSEMBLE_CTAS = 10,     /* grid (CTAs, total) of delta_assemble / delta_assemble_records
                                         (default 32): fewer CTAs take fewer SM slots from the
                                         kernels the copy overlaps */
    DELTA_OPT_ADVANCE = 9             /* extract-and-advance (NEXT f3; the trainer keeps W_t only to
                                         diff it against W_{t+1}): 2 = the
                                         compare kernel also stores every changed lane of new into
                                         old, so after delta_size / delta_extract every old_dev span
                                         equals its new_dev span bitwise (old_dev must then be
                                         writable; a lane is only ever overwritten with its own new
                                         value: 32-byte sectors holding a change are rewritten
                                         whole).  The body is
                                         unchanged.  1 = off (default).  Replace mode only
                                         (DELTA_EINVAL with DELTA_OPT_MODE = 2); delta_extract_async
                                         returns DELTA_EINVAL while it is on (a slot-overflow retry
                                         needs the host).  A second extract of the same pair after
                                         an advance sees no change (all records empty). */
};

/* Set a DELTA_OPT_* option on ctx.  DELTA_EINVAL for an unknown option or a value < 1. */
int delta_set_option(delta_ctx *ctx, int option, int64_t value);

/* Per-kernel event timing on ctx: 0 = off (default); 1 = the timings of the last calls,
 * read with delta_last_timing (the synchronising calls fill them); 2 = accumulate over calls
 * without any extra host synchronisation (each call records into the next set of a ring of 8
 * event sets; a set is folded into the running totals when it is reused), read and reset
 * with delta_timing_totals — for timing loops that never wait on the host between calls;
 * 3 = as 2 but around the compare kernel K1 only (scan_ms; two events per extract, none on
 * the other kernels, so a timed loop carries almost no profiling work).
 * Changing the mode synchronises the device and resets all timings.  DELTA_EINVAL for other
 * values. */
int delta_set_profiling(delta_ctx *ctx, int enable);

/* Copy the timings of the last calls (see delta_timing) to *out (host).  Mode 1 only (all
 * zero in mode 2). */
int delta_last_timing(const delta_ctx *ctx, delta_timing *out);

/* Modes 2 and 3: waits for the recorded events, writes the per-kernel totals since the last
 * call (or since delta_set_profiling) to *out and the number of extract scans they cover to
 * *calls (host), then resets them.  DELTA_EINVAL unless profiling mode is 2 or 3. */
int delta_timing_totals(delta_ctx *ctx, delta_timing *out, uint32_t *calls);

#ifdef __cplusplus
}
#endif
#endif
