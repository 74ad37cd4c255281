// api.cu — the C ABI of include/sparsedelta.h: context, workspace, extract plan (tile
// table) cache, descriptor validation, kernel launches, size readback and error reporting.
// Host code compiled by nvcc into libsparsedelta.so (static cudart).  Product code.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/sparsedelta.h"
#include "sd_internal.cuh"

using namespace sd;

namespace {

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    int grow(size_t bytes) {  // grow-only; contents are not preserved
        if (bytes <= cap) return DELTA_OK;
        if (p) {
            cudaDeviceSynchronize();  // async work (delta_apply_async) may still read it
            cudaFree(p);
        }
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(bytes, 256);
        if (cudaMalloc(&p, want) != cudaSuccess) {
            cudaGetLastError();
            return DELTA_ENOMEM;
        }
        cap = want;
        return DELTA_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T> T *as() const { return static_cast<T *>(p); }
};

uint64_t fnv(uint64_t h, const void *data, size_t n) {
    const uint8_t *b = static_cast<const uint8_t *>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 1099511628211ull;
    }
    return h;
}

}  // namespace

struct delta_ctx {
    int device = 0;
    int sm_count = 148;
    std::string err;
    int detail = DELTA_D_NONE;

    // ---- extract plan (rebuilt only when the descriptor key changes)
    uint64_t plan_key = 0;
    bool plan_valid = false;
    uint32_t ntiles = 0, ntensors = 0;
    int width = 2;
    unsigned long long total_lanes = 0;
    DevBuf tiles, name_len, name_off, names, numel, tensor_first_tile;
    // ---- extract workspace
    DevBuf slot_bytes, slot_val, meta, tile_plan, lb_slots, tensor_bases, entry_begin, tensor_byte_begin, table,
        summary, sticky;
    uint32_t slot_cap = 0;          // entries per tile slot (grows on overflow)
    bool scan_cached = false;       // K1-K3 results valid for plan_key (delta_size)
    // delta_extract_async: readback of the summary lands in h_summary when ev_extract fires
    bool async_pending = false;
    unsigned long long async_cap = 0;
    cudaEvent_t ev_extract = nullptr;
    ExtractSummary *h_summary = nullptr;  // pinned
    ExtractSticky *h_sticky = nullptr;    // pinned: outcome of every async extract since the last wait
    cudaStream_t async_stream = nullptr;
    bool scan_phase = false;  // a delta_extract_scan_async awaits its emit

    // ---- apply workspace
    DevBuf a_upload, a_recs, a_rcb, a_crec, a_cnt, a_sum, a_ord, a_idx, a_state, asm_status, asm_off, dg_ws;
    uint32_t *h_asm = nullptr;  // pinned
    ApplyState *h_state = nullptr;  // pinned
    // ---- delta_merge workspace
    DevBuf m_bstat, m_ha, m_hb, m_targets, m_name_len, m_name_off, m_numel, m_ea, m_eb, m_eu, m_status, m_ia, m_ib, m_va, m_vb, m_lb,
        m_dup, m_ds, m_u, m_uv, m_len, m_lo, m_blk, m_table, m_size;
    // pinned staging ring for the per-call apply uploads (targets, hint, names): with a
    // pinned source cudaMemcpyAsync does not wait for earlier work on the stream, so
    // delta_apply_async never blocks the host on a previous scatter.
    static constexpr int kRing = 8;
    void *ring[kRing] = {};
    size_t ring_cap[kRing] = {};
    cudaEvent_t ring_ev[kRing] = {};
    int ring_next = 0;

    // ---- launch options
    uint32_t lb_epoch = 0;  // K2 look-back launch epoch
    int apply_ctas_per_sm = 64, emit_ctas_per_sm = 24, scatter_ctas_per_sm = 96, scan_kernel = 0;
    int prefetch_tiles = -1;  // K1 L2 prefetch distance in tiles (-1: one wave = 3 x SMs)
    int assemble_ctas = 32;   // grid of the NVLink assembly kernels (peer stores; 32: measured best at N=4, round 2)
    bool entry_major = true;
    int mode = 0;  // records written by extract: 0 replace, 1 additive
    int index_codec = 0;  // 0 LEB128 gaps, 1 fixed-width absolute indices (extract and apply)
    bool advance = false;  // extract-and-advance: old_dev is overwritten with new (synchronous extract only)

    // ---- optional per-kernel event timing
    int profiling = 0;  // 0 off, 1 timings of the last calls, 2 accumulate over calls (ring of event
                        // sets), 3 accumulate the compare kernel K1 only (two events per call)
    cudaEvent_t ev_scan[4] = {}, ev_emit[3] = {}, ev_apply[5] = {};
    static constexpr int kProfRing = 8;
    cudaEvent_t rs_scan[kProfRing][4] = {}, rs_emit[kProfRing][3] = {}, rs_apply[kProfRing][5] = {};
    bool ru_scan[kProfRing] = {}, ru_emit[kProfRing] = {}, ru_apply[kProfRing] = {};
    unsigned ri_scan = 0, ri_emit = 0, ri_apply = 0;
    delta_timing acc = {};
    uint32_t acc_calls = 0;
    delta_timing timing = {};
};

static float ev_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
        cudaGetLastError();
        return 0.f;
    }
    return ms;
}

static int fail(delta_ctx *c, int code, int detail, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) {
        c->err = buf;
        c->detail = detail;
    }
    return code;
}

static int cuda_fail(delta_ctx *c, cudaError_t e, const char *where) {
    return fail(c, DELTA_ECUDA, DELTA_D_NONE, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(call, where)                                       \
    do {                                                      \
        cudaError_t e_ = (call);                              \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, where); \
    } while (0)

#define GROW(buf, bytes)                                                                  \
    do {                                                                                  \
        if ((buf).grow(bytes) != DELTA_OK)                                                \
            return fail(ctx, DELTA_ENOMEM, DELTA_D_NONE, "device allocation of %zu bytes failed", \
                        (size_t)(bytes));                                                 \
    } while (0)

extern "C" {

const char *delta_version(void) {
    return "sparsedelta 2 (sm_100a; K1 tile-slot compaction, tile scans, half-warp-per-tile LEB128 emit, gated scatter with dense-window vector rewrite)";
}

int delta_ctx_create(delta_ctx **out, int device) {
    if (!out) return DELTA_EINVAL;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        return DELTA_ECUDA;
    }
    if (cudaSetDevice(device) != cudaSuccess) return DELTA_ECUDA;
    delta_ctx *c = new delta_ctx();
    c->device = device;
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (cudaMallocHost(&c->h_summary, sizeof(ExtractSummary)) != cudaSuccess ||
        cudaMallocHost(&c->h_sticky, sizeof(ExtractSticky)) != cudaSuccess ||
        cudaMallocHost(&c->h_state, sizeof(ApplyState)) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return DELTA_ECUDA;
    }
    *out = c;
    return DELTA_OK;
}

void delta_ctx_destroy(delta_ctx *c) {
    if (c && c->ev_extract) cudaEventDestroy(c->ev_extract);
    if (!c) return;
    cudaSetDevice(c->device);
    DevBuf *mbufs[] = {&c->m_bstat, &c->m_ha, &c->m_hb, &c->m_targets, &c->m_name_len, &c->m_name_off, &c->m_numel, &c->m_ea, &c->m_eb, &c->m_eu,
                       &c->m_status, &c->m_ia, &c->m_ib, &c->m_va, &c->m_vb, &c->m_lb, &c->m_dup, &c->m_ds,
                       &c->m_u, &c->m_uv, &c->m_len, &c->m_lo, &c->m_blk, &c->m_table, &c->m_size};
    for (DevBuf *b : mbufs) b->release();
    DevBuf *bufs[] = {&c->tiles, &c->name_len, &c->name_off, &c->names, &c->numel,
                      &c->tensor_first_tile, &c->slot_bytes, &c->slot_val, &c->meta,
                      &c->tile_plan, &c->lb_slots, &c->tensor_bases, &c->entry_begin, &c->tensor_byte_begin, &c->table,
                      &c->summary, &c->sticky, &c->a_upload, &c->a_recs, &c->a_rcb, &c->a_crec, &c->asm_status, &c->asm_off, &c->dg_ws, &c->a_cnt, &c->a_sum,
                      &c->a_ord, &c->a_idx, &c->a_state};
    for (DevBuf *b : bufs) b->release();
    if (c->profiling) {
        for (auto &e : c->ev_scan) cudaEventDestroy(e);
        for (auto &e : c->ev_emit) cudaEventDestroy(e);
        for (auto &e : c->ev_apply) cudaEventDestroy(e);
        for (int j = 0; j < delta_ctx::kProfRing; ++j) {
            for (auto &e : c->rs_scan[j]) cudaEventDestroy(e);
            for (auto &e : c->rs_emit[j]) cudaEventDestroy(e);
            for (auto &e : c->rs_apply[j]) cudaEventDestroy(e);
        }
    }
    if (c->h_summary) cudaFreeHost(c->h_summary);
    if (c->h_sticky) cudaFreeHost(c->h_sticky);
    if (c->h_state) cudaFreeHost(c->h_state);
    if (c->h_asm) cudaFreeHost(c->h_asm);
    for (int i = 0; i < delta_ctx::kRing; ++i) {
        if (c->ring[i]) cudaFreeHost(c->ring[i]);
        if (c->ring_ev[i]) cudaEventDestroy(c->ring_ev[i]);
    }
    delete c;
}

const char *delta_last_error(const delta_ctx *c) { return c ? c->err.c_str() : "no context"; }

int delta_last_detail(const delta_ctx *c) { return c ? c->detail : DELTA_D_NONE; }

int delta_set_option(delta_ctx *c, int option, int64_t value) {
    if (!c || value < 1 || value > (1 << 20)) return DELTA_EINVAL;
    if (option == DELTA_OPT_APPLY_CTAS_PER_SM) c->apply_ctas_per_sm = (int)value;
    else if (option == DELTA_OPT_EMIT_CTAS_PER_SM) c->emit_ctas_per_sm = (int)value;
    else if (option == DELTA_OPT_SCAN_KERNEL) {
        if (value != 1) return DELTA_EINVAL;  // 2-5: retired variants (measured slower)
        c->scan_kernel = 0;
    }
    else if (option == DELTA_OPT_SCATTER_CTAS_PER_SM) c->scatter_ctas_per_sm = (int)value;
    else if (option == DELTA_OPT_PREFETCH_TILES) c->prefetch_tiles = (int)value - 1;
    else if (option == DELTA_OPT_SCATTER_ORDER) c->entry_major = value == 2;
    else if (option == DELTA_OPT_MODE) {
        if (value > 2 || (value == 2 && c->advance)) return DELTA_EINVAL;
        if (c->mode != (int)value - 1) c->scan_cached = false;
        c->mode = (int)value - 1;
    }
    else if (option == DELTA_OPT_ASSEMBLE_CTAS) c->assemble_ctas = (int)value;
    else if (option == DELTA_OPT_ADVANCE) {
        if (value > 2) return DELTA_EINVAL;
        if (value == 2 && c->mode != 0) return DELTA_EINVAL;  // replace mode only
        c->advance = value == 2;
        c->scan_cached = false;
    }
    else if (option == DELTA_OPT_INDEX_CODEC) {
        if (value > 2) return DELTA_EINVAL;
        if (c->index_codec != (int)value - 1) c->scan_cached = false;
        c->index_codec = (int)value - 1;
    }
    else return DELTA_EINVAL;
    return DELTA_OK;
}

int delta_set_profiling(delta_ctx *c, int enable) {
    if (!c || enable < 0 || enable > 3) return DELTA_EINVAL;
    if (cudaSetDevice(c->device) != cudaSuccess) return DELTA_ECUDA;
    if (enable && !c->profiling) {
        for (auto &e : c->ev_scan) cudaEventCreate(&e);
        for (auto &e : c->ev_emit) cudaEventCreate(&e);
        for (auto &e : c->ev_apply) cudaEventCreate(&e);
        for (int j = 0; j < delta_ctx::kProfRing; ++j) {
            for (auto &e : c->rs_scan[j]) cudaEventCreate(&e);
            for (auto &e : c->rs_emit[j]) cudaEventCreate(&e);
            for (auto &e : c->rs_apply[j]) cudaEventCreate(&e);
        }
        if (cudaGetLastError() != cudaSuccess) return DELTA_ECUDA;
    } else if (!enable && c->profiling) {
        cudaDeviceSynchronize();
        for (auto &e : c->ev_scan) cudaEventDestroy(e);
        for (auto &e : c->ev_emit) cudaEventDestroy(e);
        for (auto &e : c->ev_apply) cudaEventDestroy(e);
        for (int j = 0; j < delta_ctx::kProfRing; ++j) {
            for (auto &e : c->rs_scan[j]) cudaEventDestroy(e);
            for (auto &e : c->rs_emit[j]) cudaEventDestroy(e);
            for (auto &e : c->rs_apply[j]) cudaEventDestroy(e);
        }
    }
    if (enable) cudaDeviceSynchronize();
    c->profiling = enable;
    c->timing = delta_timing{};
    c->acc = delta_timing{};
    c->acc_calls = 0;
    for (int j = 0; j < delta_ctx::kProfRing; ++j) c->ru_scan[j] = c->ru_emit[j] = c->ru_apply[j] = false;
    return DELTA_OK;
}

int delta_last_timing(const delta_ctx *c, delta_timing *out) {
    if (!c || !out) return DELTA_EINVAL;
    *out = c->timing;
    return DELTA_OK;
}

}  // extern "C"

// Accumulating profiling (mode 2): each call records into the next event set of a ring;
// a set is folded into the totals when it is reused (it is kProfRing calls old, so its
// events have long completed) or by delta_timing_totals.
static void fold_scan(delta_ctx *c, int j) {
    if (!c->ru_scan[j]) return;
    if (c->profiling == 3) {  // K1 only
        cudaEventSynchronize(c->rs_scan[j][1]);
        c->acc.scan_ms += ev_ms(c->rs_scan[j][0], c->rs_scan[j][1]);
        c->acc_calls += 1;
        c->ru_scan[j] = false;
        return;
    }
    cudaEventSynchronize(c->rs_scan[j][3]);
    c->acc.scan_ms += ev_ms(c->rs_scan[j][0], c->rs_scan[j][1]);
    c->acc.lens_ms += ev_ms(c->rs_scan[j][1], c->rs_scan[j][2]);
    c->acc.finalize_ms += ev_ms(c->rs_scan[j][2], c->rs_scan[j][3]);
    c->acc_calls += 1;
    c->ru_scan[j] = false;
}
static void fold_emit(delta_ctx *c, int j) {
    if (!c->ru_emit[j]) return;
    cudaEventSynchronize(c->rs_emit[j][2]);
    c->acc.emit_ms += ev_ms(c->rs_emit[j][0], c->rs_emit[j][1]);
    c->acc.headers_ms += ev_ms(c->rs_emit[j][1], c->rs_emit[j][2]);
    c->ru_emit[j] = false;
}
static void fold_apply(delta_ctx *c, int j) {
    if (!c->ru_apply[j]) return;
    cudaEventSynchronize(c->rs_apply[j][4]);
    c->acc.locate_ms += ev_ms(c->rs_apply[j][0], c->rs_apply[j][1]);
    c->acc.decode_ms += ev_ms(c->rs_apply[j][1], c->rs_apply[j][2]);
    c->acc.apply_scan_ms += ev_ms(c->rs_apply[j][2], c->rs_apply[j][3]);
    c->acc.scatter_ms += ev_ms(c->rs_apply[j][3], c->rs_apply[j][4]);
    c->ru_apply[j] = false;
}
static cudaEvent_t *prof_scan(delta_ctx *c) {
    if (c->profiling < 2) return c->profiling ? c->ev_scan : nullptr;
    const int j = (int)(c->ri_scan++ % delta_ctx::kProfRing);
    fold_scan(c, j);
    c->ru_scan[j] = true;
    return c->rs_scan[j];
}
static cudaEvent_t *prof_emit(delta_ctx *c) {
    if (c->profiling == 3) return nullptr;
    if (c->profiling != 2) return c->profiling ? c->ev_emit : nullptr;
    const int j = (int)(c->ri_emit++ % delta_ctx::kProfRing);
    fold_emit(c, j);
    c->ru_emit[j] = true;
    return c->rs_emit[j];
}
static cudaEvent_t *prof_apply(delta_ctx *c) {
    if (c->profiling == 3) return nullptr;
    if (c->profiling != 2) return c->profiling ? c->ev_apply : nullptr;
    const int j = (int)(c->ri_apply++ % delta_ctx::kProfRing);
    fold_apply(c, j);
    c->ru_apply[j] = true;
    return c->rs_apply[j];
}

extern "C" {

int delta_timing_totals(delta_ctx *c, delta_timing *out, uint32_t *calls) {
    if (!c || !out || !calls) return DELTA_EINVAL;
    if (c->profiling < 2) return DELTA_EINVAL;
    if (cudaSetDevice(c->device) != cudaSuccess) return DELTA_ECUDA;
    for (int j = 0; j < delta_ctx::kProfRing; ++j) {
        fold_scan(c, j);
        fold_emit(c, j);
        fold_apply(c, j);
    }
    *out = c->acc;
    *calls = c->acc_calls;
    c->acc = delta_timing{};
    c->acc_calls = 0;
    return DELTA_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------- extract
static int elem_width(int elem) { return elem == DELTA_ELEM16 ? 2 : (elem == DELTA_ELEM32 ? 4 : 0); }

static int validate_tensors(delta_ctx *ctx, const delta_tensor *t, uint32_t n, int w) {
    if (n && !t) return fail(ctx, DELTA_EINVAL, 0, "tensors is NULL");
    if (n >= (1u << 30)) return fail(ctx, DELTA_EINVAL, 0, "too many tensors (%u)", n);
    for (uint32_t k = 0; k < n; ++k) {
        if (t[k].name_len > 0xFFFF)
            return fail(ctx, DELTA_EINVAL, 0, "tensor %u: name_len %u exceeds u16 (SPEC.md:148)", k,
                        t[k].name_len);
        if (t[k].name_len && !t[k].name) return fail(ctx, DELTA_EINVAL, 0, "tensor %u: name is NULL", k);
        if (t[k].n_spans == 0 || !t[k].spans)
            return fail(ctx, DELTA_EINVAL, 0, "tensor %u: no spans", k);
        for (uint32_t s = 0; s < t[k].n_spans; ++s) {
            const delta_span &sp = t[k].spans[s];
            if (sp.numel && (!sp.old_dev || !sp.new_dev))
                return fail(ctx, DELTA_ESHAPE, 0, "tensor %u span %u: NULL old/new with numel %llu", k, s,
                            (unsigned long long)sp.numel);
            if ((reinterpret_cast<uintptr_t>(sp.old_dev) | reinterpret_cast<uintptr_t>(sp.new_dev)) % w)
                return fail(ctx, DELTA_EINVAL, 0, "tensor %u span %u: pointers not %d-byte aligned", k, s, w);
        }
    }
    return DELTA_OK;
}

static uint64_t plan_key_of(const delta_tensor *t, uint32_t n, int w) {
    uint64_t h = 1469598103934665603ull;
    h = fnv(h, &w, sizeof w);
    h = fnv(h, &n, sizeof n);
    for (uint32_t k = 0; k < n; ++k) {
        h = fnv(h, &t[k].name_len, sizeof t[k].name_len);
        h = fnv(h, t[k].name, t[k].name_len);
        h = fnv(h, &t[k].n_spans, sizeof t[k].n_spans);
        h = fnv(h, t[k].spans, sizeof(delta_span) * t[k].n_spans);
    }
    return h;
}

static int build_plan(delta_ctx *ctx, const delta_tensor *t, uint32_t n, int w, cudaStream_t s) {
    const uint64_t key = plan_key_of(t, n, w);
    if (ctx->plan_valid && ctx->plan_key == key) return DELTA_OK;
    ctx->plan_valid = false;
    ctx->scan_cached = false;
    const uint32_t lanes_per_tile = kTileBytes / w;
    std::vector<TileDesc> tiles;
    std::vector<uint32_t> nlen(n), noff(n);
    std::vector<unsigned long long> numel(n);
    std::vector<uint32_t> first_tile(n);
    std::string blob;
    unsigned long long total = 0;
    for (uint32_t k = 0; k < n; ++k) {
        nlen[k] = t[k].name_len;
        noff[k] = (uint32_t)blob.size();
        blob.append(t[k].name ? t[k].name : "", t[k].name_len);
        unsigned long long base = 0;
        bool first = true;
        first_tile[k] = (uint32_t)tiles.size();
        for (uint32_t sidx = 0; sidx < t[k].n_spans; ++sidx) {
            const delta_span &sp = t[k].spans[sidx];
            const bool aligned = ((reinterpret_cast<uintptr_t>(sp.old_dev) |
                                   reinterpret_cast<uintptr_t>(sp.new_dev)) % 16) == 0;
            for (unsigned long long off = 0; off < sp.numel; off += lanes_per_tile) {
                TileDesc d;
                d.old_p = static_cast<const uint8_t *>(sp.old_dev) + off * w;
                d.new_p = static_cast<const uint8_t *>(sp.new_dev) + off * w;
                d.lane_base = base + off;
                d.nlanes = (uint32_t)std::min<unsigned long long>(lanes_per_tile, sp.numel - off);
                d.flags_tensor = k | (first ? kTileFirstOfTensor : 0u) | (aligned ? kTileAligned : 0u);
                first = false;
                tiles.push_back(d);
            }
            base += sp.numel;
        }
        if (first) {  // empty tensor: a placeholder tile records its entry offset E_k
            TileDesc d{};
            d.flags_tensor = k | kTileFirstOfTensor;
            tiles.push_back(d);
        }
        numel[k] = base;
        total += base;
    }
    if (tiles.empty()) {  // n == 0: one placeholder so K1 still writes M = 0
        TileDesc d{};
        tiles.push_back(d);
    }
    if (tiles.size() >= 0x7FFFFFFFull) return fail(ctx, DELTA_EINVAL, 0, "too many tiles");
    GROW(ctx->tiles, tiles.size() * sizeof(TileDesc));
    GROW(ctx->name_len, std::max<size_t>(n, 1) * 4);
    GROW(ctx->name_off, std::max<size_t>(n, 1) * 4);
    GROW(ctx->names, std::max<size_t>(blob.size(), 1));
    GROW(ctx->numel, std::max<size_t>(n, 1) * 8);
    GROW(ctx->tensor_first_tile, std::max<size_t>(n, 1) * 4);
    CK(cudaMemcpyAsync(ctx->tiles.p, tiles.data(), tiles.size() * sizeof(TileDesc), cudaMemcpyHostToDevice, s), "upload tiles");
    if (n) {
        CK(cudaMemcpyAsync(ctx->name_len.p, nlen.data(), n * 4, cudaMemcpyHostToDevice, s), "upload");
        CK(cudaMemcpyAsync(ctx->name_off.p, noff.data(), n * 4, cudaMemcpyHostToDevice, s), "upload");
        CK(cudaMemcpyAsync(ctx->numel.p, numel.data(), n * 8, cudaMemcpyHostToDevice, s), "upload");
        CK(cudaMemcpyAsync(ctx->tensor_first_tile.p, first_tile.data(), n * 4, cudaMemcpyHostToDevice, s), "upload");
    }
    if (!blob.empty()) CK(cudaMemcpyAsync(ctx->names.p, blob.data(), blob.size(), cudaMemcpyHostToDevice, s), "upload");
    // the host vectors die at return: make the pageable copies complete first
    CK(cudaStreamSynchronize(s), "plan upload");
    ctx->ntiles = (uint32_t)tiles.size();
    ctx->ntensors = n;
    ctx->width = w;
    ctx->total_lanes = total;
    ctx->plan_key = key;
    ctx->plan_valid = true;
    return DELTA_OK;
}

static ExtractArgs extract_args(delta_ctx *ctx) {
    ExtractArgs a;
    a.tiles = ctx->tiles.as<TileDesc>();
    a.ntiles = ctx->ntiles;
    a.ntensors = ctx->ntensors;
    a.slot_cap = ctx->slot_cap;
    a.slot_bytes = ctx->slot_bytes.as<uint8_t>();
    a.slot_val = ctx->slot_val.p;
    a.meta = ctx->meta.as<TileMeta>();
    a.plan = ctx->tile_plan.as<TileEmit>();
    a.lb = ctx->lb_slots.as<LbSlot>();
    if (++ctx->lb_epoch >= (1u << 30)) {  // the status words hold 30 epoch bits: start over
        cudaMemset(ctx->lb_slots.p, 0, ctx->lb_slots.cap);
        ctx->lb_epoch = 1;
    }
    a.epoch = ctx->lb_epoch;
    a.bases = ctx->tensor_bases.as<TensorBase>();
    a.tensor_first_tile = ctx->tensor_first_tile.as<uint32_t>();
    a.entry_begin = ctx->entry_begin.as<unsigned long long>();
    a.tensor_byte_begin = ctx->tensor_byte_begin.as<unsigned long long>();
    a.table = ctx->table.as<RecordRow>();
    a.name_len = ctx->name_len.as<uint32_t>();
    a.name_off = ctx->name_off.as<uint32_t>();
    a.names = ctx->names.as<uint8_t>();
    a.numel = ctx->numel.as<unsigned long long>();
    a.summary = ctx->summary.as<ExtractSummary>();
    a.width = ctx->width;
    a.persist_ctas = ctx->sm_count * ctx->emit_ctas_per_sm;
    a.sm_count = ctx->sm_count;
    a.prefetch_dist = (uint32_t)(ctx->prefetch_tiles < 0 ? ctx->sm_count * 3 : ctx->prefetch_tiles);
    a.mode = ctx->mode;
    a.index_codec = ctx->index_codec;
    a.advance = ctx->advance;
    return a;
}

static int reserve_slots(delta_ctx *ctx, uint32_t cap) {
    GROW(ctx->slot_bytes, (size_t)ctx->ntiles * cap * 2 + 64);
    GROW(ctx->slot_val, (size_t)ctx->ntiles * cap * ctx->width + 64);
    ctx->slot_cap = cap;
    return DELTA_OK;
}

// K1-K3 + the single size readback; on slot overflow grows the slots to the largest
// per-tile count seen and runs again (first call at a new density only).
static int prepare_scan(delta_ctx *ctx) {
    const uint32_t T = ctx->ntensors, nt = ctx->ntiles;
    const uint32_t nblk = (nt + kTileBlock - 1) / kTileBlock;
    const uint32_t lanes_per_tile = kTileBytes / ctx->width;
    GROW(ctx->meta, (size_t)nt * sizeof(TileMeta));
    GROW(ctx->tile_plan, (size_t)nt * sizeof(TileEmit));
    {
        void *old = ctx->lb_slots.p;
        GROW(ctx->lb_slots, (size_t)std::max<uint32_t>(nblk, 1) * sizeof(LbSlot));
        if (ctx->lb_slots.p != old) {  // fresh slots: no status word may carry a live epoch
            CK(cudaMemset(ctx->lb_slots.p, 0, ctx->lb_slots.cap), "memset");
            ctx->lb_epoch = 0;
        }
    }
    GROW(ctx->tensor_bases, (size_t)std::max<uint32_t>(T, 1) * sizeof(TensorBase));
    GROW(ctx->entry_begin, (size_t)(T + 1) * 8);
    GROW(ctx->tensor_byte_begin, (size_t)(T + 1) * 8);
    GROW(ctx->table, (size_t)std::max<uint32_t>(T, 1) * sizeof(RecordRow));
    GROW(ctx->summary, sizeof(ExtractSummary));
    // slots: start at 1/16 of a tile (6.25% density); grown to the exact need on overflow
    uint32_t cap = std::max<uint32_t>(ctx->slot_cap, lanes_per_tile / 16);
    if (cap > lanes_per_tile) cap = lanes_per_tile;
    if (cap != ctx->slot_cap || ctx->slot_bytes.cap < (size_t)nt * cap * 2 + 64) {
        int rc = reserve_slots(ctx, cap);
        if (rc) return rc;
    }
    return DELTA_OK;
}

static int run_scan(delta_ctx *ctx, cudaStream_t s) {
    const uint32_t lanes_per_tile = kTileBytes / ctx->width;
    int rc0 = prepare_scan(ctx);
    if (rc0) return rc0;
    uint32_t redo_cap = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        CK(cudaMemsetAsync(ctx->summary.p, 0, sizeof(ExtractSummary), s), "memset");
        ExtractArgs a = extract_args(ctx);
        a.redo_cap = redo_cap;
        a.prof_k1_only = ctx->profiling == 3;
        CK(launch_extract_scan(a, s, prof_scan(ctx)), "extract scan launch");
        CK(cudaMemcpyAsync(ctx->h_summary, ctx->summary.p, sizeof(ExtractSummary), cudaMemcpyDeviceToHost, s), "readback");
        CK(cudaStreamSynchronize(s), "extract scan");
        if (ctx->profiling == 1) {
            ctx->timing.scan_ms = ev_ms(ctx->ev_scan[0], ctx->ev_scan[1]);
            ctx->timing.lens_ms = ev_ms(ctx->ev_scan[1], ctx->ev_scan[2]);
            ctx->timing.finalize_ms = ev_ms(ctx->ev_scan[2], ctx->ev_scan[3]);
        }
        if (!ctx->h_summary->overflow) {
            ctx->scan_cached = true;
            return DELTA_OK;
        }
        uint32_t need = 2;
        while (need < ctx->h_summary->max_count) need <<= 1;
        need = std::min(need, lanes_per_tile);
        if (ctx->advance) {
            // the tiles that fitted were compacted AND advanced (old == new there now): keep
            // their slots, move them into the larger layout, and redo only the overflowed tiles
            DevBuf nb, nv;
            if (nb.grow((size_t)ctx->ntiles * need * 2 + 64) || nv.grow((size_t)ctx->ntiles * need * ctx->width + 64)) {
                nb.release();
                nv.release();
                return fail(ctx, DELTA_ENOMEM, 0, "slot regrowth allocation failed");
            }
            CK(launch_slots_regrow(ctx->meta.as<TileMeta>(), ctx->ntiles, ctx->width, ctx->slot_cap, ctx->slot_bytes.p,
                                   ctx->slot_val.p, need, nb.p, nv.p, ctx->sm_count * 8, s), "slot regrowth");
            CK(cudaStreamSynchronize(s), "slot regrowth");
            ctx->slot_bytes.release();
            ctx->slot_val.release();
            ctx->slot_bytes = nb;
            ctx->slot_val = nv;
            redo_cap = ctx->slot_cap;
            ctx->slot_cap = need;
            continue;
        }
        int rc = reserve_slots(ctx, need);
        if (rc) return rc;
    }
    return fail(ctx, DELTA_ENOMEM, 0, "tile slot overflow after resize");
}

extern "C" int delta_size(delta_ctx *ctx, const delta_tensor *t, uint32_t n, int elem, void *stream,
                          uint64_t *body_bytes) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    const int w = elem_width(elem);
    if (!w) return fail(ctx, DELTA_EINVAL, 0, "unknown elem %d", elem);
    if (!body_bytes) return fail(ctx, DELTA_EINVAL, 0, "body_bytes is NULL");
    int rc = validate_tensors(ctx, t, n, w);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    rc = build_plan(ctx, t, n, w, s);
    if (rc) return rc;
    rc = run_scan(ctx, s);
    if (rc) return rc;
    *body_bytes = ctx->h_summary->body_bytes;
    return DELTA_OK;
}

// The offset table of the compaction the last delta_size left cached (K3 wrote it on the
// device), copied to the host without emitting a body; the cache stays valid.
extern "C" int delta_size_table(delta_ctx *ctx, uint32_t n, delta_record_info *table, void *stream) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    if (!ctx->scan_cached || !ctx->plan_valid)
        return fail(ctx, DELTA_EINVAL, 0, "no cached delta_size result on this context");
    if (n != ctx->ntensors) return fail(ctx, DELTA_EINVAL, 0, "n = %u but delta_size ran on %u tensors", n, ctx->ntensors);
    if (n && !table) return fail(ctx, DELTA_EINVAL, 0, "table is NULL");
    if (!n) return DELTA_OK;
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaMemcpyAsync(table, ctx->table.p, (size_t)n * sizeof(RecordRow), cudaMemcpyDeviceToHost, s), "table readback");
    CK(cudaStreamSynchronize(s), "table readback");
    return DELTA_OK;
}

// compute_rho (Eq. 1): rho = sum_k nnz_k / sum_k N_k with
// nnz_k the changed lanes under the bitwise reading R2.  One compare + compaction (cached for a
// following delta_extract, like delta_size); the sums are taken over the offset-table rows.
extern "C" int delta_compute_rho(delta_ctx *ctx, const delta_tensor *t, uint32_t n, int elem, void *stream,
                                 uint64_t *nnz, uint64_t *nnz_total, uint64_t *numel_total, double *rho) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    if (!nnz_total || !numel_total || !rho) return fail(ctx, DELTA_EINVAL, 0, "NULL result pointer");
    if (ctx->advance)  // the advancing compare overwrites old: compute_rho is a pure function
        return fail(ctx, DELTA_EINVAL, 0, "compute_rho on a context with DELTA_OPT_ADVANCE set");
    uint64_t body = 0;
    int rc = delta_size(ctx, t, n, elem, stream, &body);
    if (rc) return rc;
    std::vector<delta_record_info> rows(std::max<uint32_t>(n, 1));
    if (n) {
        rc = delta_size_table(ctx, n, rows.data(), stream);
        if (rc) return rc;
    }
    uint64_t sn = 0, sN = 0;
    for (uint32_t k = 0; k < n; ++k) {
        if (nnz) nnz[k] = rows[k].nnz;
        sn += rows[k].nnz;
        sN += rows[k].element_count;
    }
    *nnz_total = sn;
    *numel_total = sN;
    *rho = sN ? (double)sn / (double)sN : 0.0;
    return DELTA_OK;
}

// Host-only: offset-table rows of a body that starts `offset` bytes into a larger body
// (a group's or a rank's records placed after the earlier ones, reading R15).
extern "C" int delta_table_rebase(delta_record_info *rows, uint32_t n, uint64_t offset) {
    if (n && !rows) return DELTA_EINVAL;
    for (uint32_t k = 0; k < n; ++k) {
        if (rows[k].record_offset + rows[k].record_bytes > UINT64_MAX - offset) return DELTA_EINVAL;
        rows[k].record_offset += offset;
        rows[k].index_offset += offset;
        rows[k].values_offset += offset;
    }
    return DELTA_OK;
}

extern "C" int delta_extract(delta_ctx *ctx, const delta_tensor *t, uint32_t n, int elem, void *out,
                             uint64_t cap, delta_record_info *table, void *stream,
                             uint64_t *body_bytes) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    const int w = elem_width(elem);
    if (!w) return fail(ctx, DELTA_EINVAL, 0, "unknown elem %d", elem);
    if (!body_bytes) return fail(ctx, DELTA_EINVAL, 0, "body_bytes is NULL");
    int rc = validate_tensors(ctx, t, n, w);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t key = plan_key_of(t, n, w);
    const bool reuse = ctx->scan_cached && ctx->plan_valid && ctx->plan_key == key;
    if (!reuse) {
        rc = build_plan(ctx, t, n, w, s);
        if (rc) return rc;
        rc = run_scan(ctx, s);
        if (rc) return rc;
    }
    // The compaction stays cached across DELTA_ECAPACITY / a NULL out_dev: with
    // extract-and-advance, old already equals new, so a retry with a larger buffer must
    // emit from this scan rather than compare again (it would find nothing).
    ctx->scan_cached = true;
    const unsigned long long need = ctx->h_summary->body_bytes;
    *body_bytes = need;
    if (need > cap)
        return fail(ctx, DELTA_ECAPACITY, 0, "output capacity %llu < body size %llu",
                    (unsigned long long)cap, need);
    if (need && !out) return fail(ctx, DELTA_EINVAL, 0, "out_dev is NULL");
    ctx->scan_cached = false;  // consumed
    if (n)
        CK(launch_extract_emit(extract_args(ctx), static_cast<uint8_t *>(out), s,
                               prof_emit(ctx)),
           "extract emit launch");
    if (table && n) {
        CK(cudaMemcpyAsync(table, ctx->table.p, (size_t)n * sizeof(RecordRow), cudaMemcpyDeviceToHost, s), "table readback");
    }
    if ((table && n) || (ctx->profiling == 1 && n)) CK(cudaStreamSynchronize(s), "extract emit");
    if (ctx->profiling == 1 && n) {
        ctx->timing.emit_ms = ev_ms(ctx->ev_emit[0], ctx->ev_emit[1]);
        ctx->timing.headers_ms = ev_ms(ctx->ev_emit[1], ctx->ev_emit[2]);
    }
    return DELTA_OK;
}

// Enqueue-only extract (no host synchronisation when the plan is cached): K1-K5 run
// back to back; K4/K5 write the body only if the scan fitted its tile slots and the body
// fits `cap`, and write the size (or ~0) to body_bytes_dev.  delta_extract_wait reports
// the outcome.
// Enqueue-only extract in two phases (no host synchronisation when the plan is cached).
// Phase 1 (scan, K1-K3) on the context's cached plan; phase 2 (emit, K4-K5) writes the body
// only if the scan fitted its tile slots and the body fits `cap` (and, fused assembly, the
// peer copy only if every rank's size is known and the records fit the peer buffer).
static int extract_scan_async(delta_ctx *ctx, const delta_tensor *t, uint32_t n, int elem,
                              uint64_t *size_dev, cudaStream_t s) {
    const int w = elem_width(elem);
    if (!w) return fail(ctx, DELTA_EINVAL, 0, "unknown elem %d", elem);
    if (ctx->advance)  // an overflow retry needs the host: extract-and-advance is synchronous only
        return fail(ctx, DELTA_EINVAL, 0, "DELTA_OPT_ADVANCE needs delta_size / delta_extract");
    if (reinterpret_cast<uintptr_t>(size_dev) % 8) return fail(ctx, DELTA_EINVAL, 0, "size not 8-byte aligned");
    int rc = validate_tensors(ctx, t, n, w);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    rc = build_plan(ctx, t, n, w, s);
    if (rc) return rc;
    rc = prepare_scan(ctx);
    if (rc) return rc;
    ctx->scan_cached = false;
    if (!ctx->ev_extract) CK(cudaEventCreateWithFlags(&ctx->ev_extract, cudaEventDisableTiming), "event");
    GROW(ctx->sticky, sizeof(ExtractSticky));
    if (!ctx->async_pending) CK(cudaMemsetAsync(ctx->sticky.p, 0, sizeof(ExtractSticky), s), "memset");
    CK(cudaMemsetAsync(ctx->summary.p, 0, sizeof(ExtractSummary), s), "memset");
    ExtractArgs a = extract_args(ctx);
    a.scan_size_out = reinterpret_cast<unsigned long long *>(size_dev);
    a.prof_k1_only = ctx->profiling == 3;
    CK(launch_extract_scan(a, s, prof_scan(ctx)), "extract scan launch");
    if (!n && size_dev) CK(cudaMemsetAsync(size_dev, 0, 8, s), "memset");
    ctx->scan_phase = true;
    return DELTA_OK;
}

static int extract_emit_async(delta_ctx *ctx, void *out, uint64_t cap, uint64_t *body_bytes_dev, void *peer,
                              uint64_t peer_cap, const uint64_t *sizes_dev, uint32_t n_ranks, uint32_t rank,
                              cudaStream_t s) {
    if (!ctx->scan_phase) return fail(ctx, DELTA_EINVAL, 0, "no delta_extract_scan_async to emit");
    if (cap && !out) return fail(ctx, DELTA_EINVAL, 0, "out_dev is NULL");
    if (reinterpret_cast<uintptr_t>(body_bytes_dev) % 8)
        return fail(ctx, DELTA_EINVAL, 0, "body_bytes_dev not 8-byte aligned");
    if (peer && (!sizes_dev || rank >= n_ranks))
        return fail(ctx, DELTA_EINVAL, 0, "peer destination needs sizes_dev and rank < n_ranks");
    ctx->scan_phase = false;
    ExtractArgs a = extract_args(ctx);
    a.out_cap = cap;
    a.size_out = reinterpret_cast<unsigned long long *>(body_bytes_dev);
    a.sticky = ctx->sticky.as<ExtractSticky>();
    if (peer) {
        a.peer.base = static_cast<uint8_t *>(peer);
        a.peer.cap = peer_cap;
        a.peer.sizes = reinterpret_cast<const unsigned long long *>(sizes_dev);
        a.peer.n_ranks = n_ranks;
        a.peer.rank = rank;
    }
    if (ctx->ntensors) {
        CK(launch_extract_emit(a, static_cast<uint8_t *>(out), s, prof_emit(ctx)), "extract emit launch");
    } else if (body_bytes_dev) {
        CK(cudaMemsetAsync(body_bytes_dev, 0, 8, s), "memset");
    }
    CK(cudaMemcpyAsync(ctx->h_summary, ctx->summary.p, sizeof(ExtractSummary), cudaMemcpyDeviceToHost, s), "readback");
    CK(cudaMemcpyAsync(ctx->h_sticky, ctx->sticky.p, sizeof(ExtractSticky), cudaMemcpyDeviceToHost, s), "readback");
    CK(cudaEventRecord(ctx->ev_extract, s), "event");
    ctx->async_pending = true;
    ctx->async_stream = s;
    ctx->async_cap = cap;
    return DELTA_OK;
}

extern "C" int delta_extract_async(delta_ctx *ctx, const delta_tensor *t, uint32_t n, int elem, void *out,
                                   uint64_t cap, uint64_t *body_bytes_dev, void *stream) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    if (cap && !out) return fail(ctx, DELTA_EINVAL, 0, "out_dev is NULL");
    if (reinterpret_cast<uintptr_t>(body_bytes_dev) % 8)
        return fail(ctx, DELTA_EINVAL, 0, "body_bytes_dev not 8-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int rc = extract_scan_async(ctx, t, n, elem, nullptr, s);
    if (rc) return rc;
    return extract_emit_async(ctx, out, cap, body_bytes_dev, nullptr, 0, nullptr, 0, 0, s);
}

extern "C" int delta_extract_scan_async(delta_ctx *ctx, const delta_tensor *t, uint32_t n, int elem,
                                        uint64_t *size_dev, void *stream) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    return extract_scan_async(ctx, t, n, elem, size_dev, static_cast<cudaStream_t>(stream));
}

extern "C" int delta_extract_emit_async(delta_ctx *ctx, void *out, uint64_t cap, uint64_t *body_bytes_dev,
                                        void *peer, uint64_t peer_cap, const uint64_t *sizes_dev, uint32_t n_ranks,
                                        uint32_t rank, void *stream) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    return extract_emit_async(ctx, out, cap, body_bytes_dev, peer, peer_cap, sizes_dev, n_ranks, rank,
                              static_cast<cudaStream_t>(stream));
}

extern "C" int delta_extract_wait(delta_ctx *ctx, uint64_t *body_bytes) {
    if (!ctx) return DELTA_EINVAL;
    if (!ctx->async_pending) return fail(ctx, DELTA_EINVAL, 0, "no delta_extract_async pending");
    ctx->async_pending = false;
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(cudaEventSynchronize(ctx->ev_extract), "extract");
    if (ctx->profiling == 1) {
        ctx->timing.scan_ms = ev_ms(ctx->ev_scan[0], ctx->ev_scan[1]);
        ctx->timing.lens_ms = ev_ms(ctx->ev_scan[1], ctx->ev_scan[2]);
        ctx->timing.finalize_ms = ev_ms(ctx->ev_scan[2], ctx->ev_scan[3]);
        if (ctx->ntensors) {
            ctx->timing.emit_ms = ev_ms(ctx->ev_emit[0], ctx->ev_emit[1]);
            ctx->timing.headers_ms = ev_ms(ctx->ev_emit[1], ctx->ev_emit[2]);
        }
    }
    // the sticky record covers every async extract since the last wait (the summary only
    // the last one): an earlier call's closed gate is reported here, not lost
    const ExtractSummary &sm = *ctx->h_summary;
    const ExtractSticky sk = *ctx->h_sticky;
    if (sk.overflow) {
        const uint32_t lanes_per_tile = kTileBytes / ctx->width;
        uint32_t need = 2;
        while (need < sk.max_count) need <<= 1;
        int rc = reserve_slots(ctx, std::min(need, lanes_per_tile));
        if (rc) return rc;
        return fail(ctx, DELTA_EAGAIN, 0,
                    "tile slots overflowed (largest tile count %llu); workspace grown, issue the call again",
                    (unsigned long long)sk.max_count);
    }
    if (body_bytes) *body_bytes = sk.over_cap ? sk.need : sm.body_bytes;
    if (sk.over_cap)
        return fail(ctx, DELTA_ECAPACITY, 0, "output capacity %llu < body size %llu",
                    (unsigned long long)ctx->async_cap, (unsigned long long)sk.need);
    if (sk.peer_fail == 1)
        return fail(ctx, DELTA_EAGAIN, 0, "fused assembly skipped: a rank's extract did not complete (size ~0)");
    if (sk.peer_fail == 2)
        return fail(ctx, DELTA_ECAPACITY, 0, "fused assembly skipped: the records do not fit the peer buffer");
    return DELTA_OK;
}

// --------------------------------------------------------------------------- apply
static const int kDetailToStatus[] = {
    DELTA_OK,        DELTA_ECORRUPT, DELTA_ECORRUPT, DELTA_ECORRUPT, DELTA_ECORRUPT, DELTA_ECORRUPT,
    DELTA_ECORRUPT,  DELTA_ENAME,    DELTA_ENAME,    DELTA_ECORRUPT, DELTA_ECORRUPT};
static const char *kDetailName[] = {"ok", "truncated varint", "overlong varint", "varint exceeds 64 bits",
                                    "non-increasing index", "index >= element_count", "index count != nnz",
                                    "record name != target name", "record element_count != target numel",
                                    "mode byte not in {0, 1}", "record layout"};

static int apply_enqueue(delta_ctx *ctx, const delta_target *tg, uint32_t n, int elem, const void *body,
                         uint64_t body_bytes, const delta_record_info *hint, cudaStream_t s,
                         const delta_record_info *hint_dev = nullptr,
                         const uint64_t *body_bytes_dev = nullptr) {
    ctx->err.clear();
    ctx->detail = 0;
    const int w = elem_width(elem);
    if (!w) return fail(ctx, DELTA_EINVAL, 0, "unknown elem %d", elem);
    if (n && !tg) return fail(ctx, DELTA_EINVAL, 0, "targets is NULL");
    if (body_bytes && !body) return fail(ctx, DELTA_EINVAL, 0, "body_dev is NULL");
    std::vector<TargetDesc> td(n);
    std::string blob;
    for (uint32_t k = 0; k < n; ++k) {
        if (tg[k].name_len > 0xFFFF || (tg[k].name_len && !tg[k].name))
            return fail(ctx, DELTA_EINVAL, 0, "target %u: bad name", k);
        if (tg[k].numel && !tg[k].w_dev) return fail(ctx, DELTA_EINVAL, 0, "target %u: NULL w_dev", k);
        if (reinterpret_cast<uintptr_t>(tg[k].w_dev) % w)
            return fail(ctx, DELTA_EINVAL, 0, "target %u: w_dev not %d-byte aligned", k, w);
        td[k].w = static_cast<uint8_t *>(tg[k].w_dev);
        td[k].numel = tg[k].numel;
        td[k].name_off = blob.size();
        td[k].name_len = tg[k].name_len;
        blob.append(tg[k].name ? tg[k].name : "", tg[k].name_len);
    }
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    const size_t nn = std::max<uint32_t>(n, 1);
    // one upload per call: [TargetDesc x n | RecordRow x n (hint) | names]
    const size_t off_hint = (n * sizeof(TargetDesc) + 63) & ~size_t(63);
    const size_t off_names = off_hint + ((hint ? n * sizeof(RecordRow) : 0) + 63 & ~size_t(63));
    const size_t up_bytes = off_names + blob.size();
    GROW(ctx->a_upload, std::max<size_t>(up_bytes, 64));
    GROW(ctx->a_recs, nn * sizeof(ApplyRec));
    GROW(ctx->a_rcb, (nn + 1) * 8);
    if (!ctx->a_state.p) {
        GROW(ctx->a_state, sizeof(ApplyState));
        CK(cudaMemsetAsync(ctx->a_state.p, 0, sizeof(ApplyState), s), "memset");
    }
    const size_t nch = body_bytes / kByteChunk + n + 2;
    GROW(ctx->a_cnt, nch * 4);
    GROW(ctx->a_crec, nch * 4);
    GROW(ctx->a_sum, nch * 8);
    GROW(ctx->a_ord, nch * 8);
    GROW(ctx->a_idx, nch * 8);
    {
        const int r = ctx->ring_next;
        ctx->ring_next = (r + 1) % delta_ctx::kRing;
        if (ctx->ring_ev[r]) CK(cudaEventSynchronize(ctx->ring_ev[r]), "ring");  // its last copy is done
        else CK(cudaEventCreateWithFlags(&ctx->ring_ev[r], cudaEventDisableTiming), "ring event");
        if (ctx->ring_cap[r] < up_bytes) {
            if (ctx->ring[r]) cudaFreeHost(ctx->ring[r]);
            ctx->ring[r] = nullptr;
            ctx->ring_cap[r] = 0;
            CK(cudaMallocHost(&ctx->ring[r], std::max<size_t>(up_bytes, 4096)), "pinned ring");
            ctx->ring_cap[r] = std::max<size_t>(up_bytes, 4096);
        }
        uint8_t *h = static_cast<uint8_t *>(ctx->ring[r]);
        if (n) memcpy(h, td.data(), n * sizeof(TargetDesc));
        if (hint && n) memcpy(h + off_hint, hint, n * sizeof(RecordRow));
        if (!blob.empty()) memcpy(h + off_names, blob.data(), blob.size());
        if (up_bytes) CK(cudaMemcpyAsync(ctx->a_upload.p, h, up_bytes, cudaMemcpyHostToDevice, s), "upload");
        CK(cudaEventRecord(ctx->ring_ev[r], s), "ring event");
    }
    CK(cudaMemsetAsync(ctx->a_state.p, 0, sizeof(uint32_t), s), "memset");  // this call's gate
    ApplyArgs a;
    a.body = static_cast<const uint8_t *>(body);
    a.body_bytes = body_bytes;
    a.body_bytes_dev = reinterpret_cast<const unsigned long long *>(body_bytes_dev);
    a.targets = ctx->a_upload.as<TargetDesc>();
    a.n = n;
    a.names = ctx->a_upload.as<uint8_t>() + off_names;
    a.hint = (hint && n) ? reinterpret_cast<const RecordRow *>(ctx->a_upload.as<uint8_t>() + off_hint) : nullptr;
    if (hint_dev && n) a.hint = reinterpret_cast<const RecordRow *>(hint_dev);
    a.recs = ctx->a_recs.as<ApplyRec>();
    a.rec_chunk_begin = ctx->a_rcb.as<unsigned long long>();
    a.chunk_rec = ctx->a_crec.as<uint32_t>();
    a.chunk_count = ctx->a_cnt.as<unsigned int>();
    a.chunk_sum = ctx->a_sum.as<unsigned long long>();
    a.chunk_ord_base = ctx->a_ord.as<unsigned long long>();
    a.chunk_idx_base = ctx->a_idx.as<unsigned long long>();
    a.chunk_cap = nch;
    a.state = ctx->a_state.as<ApplyState>();
    a.width = w;
    a.persist_ctas = ctx->sm_count * ctx->apply_ctas_per_sm;
    a.scatter_ctas = ctx->sm_count * ctx->scatter_ctas_per_sm;
    a.entry_major = ctx->entry_major;
    a.index_codec = ctx->index_codec;
    {  // launch-shape hint only (any value is correct): body bytes per target lane, from the
       // host size or the capacity of a device-sized body
        unsigned long long lanes = 0;
        for (uint32_t k = 0; k < n; ++k) lanes += tg[k].numel;
        a.dense_hint = (double)body_bytes > 0.125 * (double)w * (double)lanes;
    }
    CK(launch_apply(a, s, prof_apply(ctx)), "apply launch");
    return DELTA_OK;
}

extern "C" int delta_apply_async(delta_ctx *ctx, const delta_target *tg, uint32_t n, int elem,
                                 const void *body, uint64_t body_bytes, const delta_record_info *hint,
                                 void *stream) {
    if (!ctx) return DELTA_EINVAL;
    return apply_enqueue(ctx, tg, n, elem, body, body_bytes, hint, static_cast<cudaStream_t>(stream));
}

extern "C" int delta_apply_async_dev(delta_ctx *ctx, const delta_target *tg, uint32_t n, int elem,
                                     const void *body, uint64_t body_bytes,
                                     const delta_record_info *table_hint_dev, void *stream) {
    if (!ctx) return DELTA_EINVAL;
    return apply_enqueue(ctx, tg, n, elem, body, body_bytes, nullptr, static_cast<cudaStream_t>(stream),
                         table_hint_dev);
}

extern "C" int delta_apply_async_chain(delta_ctx *ctx, const delta_target *tg, uint32_t n, int elem,
                                       const void *body, uint64_t body_cap, const uint64_t *body_bytes_dev,
                                       const delta_record_info *table_hint_dev, void *stream) {
    if (!ctx) return DELTA_EINVAL;
    if (!body_bytes_dev || reinterpret_cast<uintptr_t>(body_bytes_dev) % 8)
        return fail(ctx, DELTA_EINVAL, 0, "body_bytes_dev NULL or not 8-byte aligned");
    return apply_enqueue(ctx, tg, n, elem, body, body_cap, nullptr, static_cast<cudaStream_t>(stream),
                         table_hint_dev, body_bytes_dev);
}

extern "C" const delta_record_info *delta_table_dev(const delta_ctx *ctx) {
    if (!ctx || !ctx->table.p || ctx->ntensors == 0) return nullptr;
    return static_cast<const delta_record_info *>(ctx->table.p);
}

extern "C" int delta_apply_wait(delta_ctx *ctx, void *stream) {
    if (!ctx) return DELTA_EINVAL;
    if (!ctx->a_state.p) return DELTA_OK;  // nothing was ever enqueued
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(cudaMemcpyAsync(ctx->h_state, ctx->a_state.p, sizeof(ApplyState), cudaMemcpyDeviceToHost, s), "status readback");
    CK(cudaStreamSynchronize(s), "apply");
    CK(cudaMemsetAsync(static_cast<uint8_t *>(ctx->a_state.p) + offsetof(ApplyState, first_error), 0,
                       sizeof(uint32_t), s), "memset");
    if (ctx->profiling == 1) {
        ctx->timing.locate_ms = ev_ms(ctx->ev_apply[0], ctx->ev_apply[1]);
        ctx->timing.decode_ms = ev_ms(ctx->ev_apply[1], ctx->ev_apply[2]);
        ctx->timing.apply_scan_ms = ev_ms(ctx->ev_apply[2], ctx->ev_apply[3]);
        ctx->timing.scatter_ms = ev_ms(ctx->ev_apply[3], ctx->ev_apply[4]);
    }
    const uint32_t st = ctx->h_state->first_error;
    if (st == 0) return DELTA_OK;
    if (st > 10) return fail(ctx, DELTA_ECORRUPT, (int)st, "unknown status %u", st);
    return fail(ctx, kDetailToStatus[st], (int)st, "delta_apply: %s", kDetailName[st]);
}

extern "C" int delta_apply(delta_ctx *ctx, const delta_target *tg, uint32_t n, int elem,
                           const void *body, uint64_t body_bytes, const delta_record_info *hint,
                           void *stream) {
    if (!ctx) return DELTA_EINVAL;
    int rc = apply_enqueue(ctx, tg, n, elem, body, body_bytes, hint, static_cast<cudaStream_t>(stream));
    if (rc) return rc;
    return delta_apply_wait(ctx, stream);
}

extern "C" int delta_assemble(delta_ctx *ctx, const void *src, void *dst, uint64_t cap, const uint64_t *sizes,
                              uint32_t n_ranks, uint32_t rank, void *stream) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    if (!sizes || rank >= n_ranks || (!src && rank != 0) || !dst)
        return fail(ctx, DELTA_EINVAL, 0, "delta_assemble: bad arguments");
    if (reinterpret_cast<uintptr_t>(src) % 16) return fail(ctx, DELTA_EINVAL, 0, "delta_assemble: src not 16-byte aligned");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!ctx->asm_status.p) {
        GROW(ctx->asm_status, 16);
        CK(cudaMemsetAsync(ctx->asm_status.p, 0, 16, s), "memset");
    }
    CK(launch_assemble(static_cast<const uint8_t *>(src), static_cast<uint8_t *>(dst), cap,
                       reinterpret_cast<const unsigned long long *>(sizes), rank, ctx->asm_status.as<uint32_t>(),
                       ctx->assemble_ctas, s),
       "assemble launch");
    return DELTA_OK;
}




extern "C" int delta_record_sizes(delta_ctx *ctx, const delta_record_info *table_dev, uint32_t n_local,
                                  const uint32_t *gidx_dev, uint64_t *sizes_dev, uint32_t n_global, void *stream) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    if (!sizes_dev || (n_local && (!table_dev || !gidx_dev)) || n_local > n_global)
        return fail(ctx, DELTA_EINVAL, 0, "delta_record_sizes: bad arguments");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(launch_record_sizes(reinterpret_cast<const RecordRow *>(table_dev), n_local, gidx_dev,
                           reinterpret_cast<unsigned long long *>(sizes_dev), n_global,
                           static_cast<cudaStream_t>(stream)),
       "record sizes launch");
    return DELTA_OK;
}

extern "C" int delta_assemble_records(delta_ctx *ctx, const void *src_dev, const uint32_t *gidx_dev, uint32_t n_local,
                                      const uint64_t *sizes_dev, uint32_t n_global, void *dst_dev, uint64_t dst_capacity,
                                      void *stream) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    if (!sizes_dev || !dst_dev || (n_local && (!src_dev || !gidx_dev)) || n_local > n_global)
        return fail(ctx, DELTA_EINVAL, 0, "delta_assemble_records: bad arguments");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!ctx->asm_status.p) {
        GROW(ctx->asm_status, 16);
        CK(cudaMemsetAsync(ctx->asm_status.p, 0, 16, s), "memset");
    }
    GROW(ctx->asm_off, ((size_t)n_global + 1 + n_local + 1) * 8);
    unsigned long long *goff = ctx->asm_off.as<unsigned long long>();
    CK(launch_assemble_records(static_cast<const uint8_t *>(src_dev), static_cast<uint8_t *>(dst_dev), dst_capacity,
                               reinterpret_cast<const unsigned long long *>(sizes_dev), gidx_dev, n_local, n_global,
                               goff, goff + n_global + 1, ctx->asm_status.as<uint32_t>(), ctx->assemble_ctas, s),
       "assemble records launch");
    return DELTA_OK;
}

extern "C" int delta_assemble_wait(delta_ctx *ctx, void *stream) {
    if (!ctx) return DELTA_EINVAL;
    if (!ctx->asm_status.p) return DELTA_OK;
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!ctx->h_asm) CK(cudaMallocHost(&ctx->h_asm, 64), "pinned");
    CK(cudaMemcpyAsync(ctx->h_asm, ctx->asm_status.p, 4, cudaMemcpyDeviceToHost, s), "readback");
    CK(cudaStreamSynchronize(s), "assemble");
    CK(cudaMemsetAsync(ctx->asm_status.p, 0, 16, s), "memset");
    if (*ctx->h_asm) return fail(ctx, DELTA_ECAPACITY, 0, "delta_assemble: destination too small");
    return DELTA_OK;
}

extern "C" int delta_digest(delta_ctx *ctx, const void *body, uint64_t bytes, uint8_t *out32, void *stream) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    if (!out32 || (bytes && !body)) return fail(ctx, DELTA_EINVAL, 0, "delta_digest: bad arguments");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const unsigned long long nch = bytes == 0 ? 1 : (bytes + 1023) / 1024;
    GROW(ctx->dg_ws, (size_t)(2 * nch * 32 + 64));
    uint32_t *ws = ctx->dg_ws.as<uint32_t>();
    uint32_t *dout = ws + 2 * nch * 8;
    CK(launch_blake3(static_cast<const uint8_t *>(body), bytes, ws, dout, s), "digest launch");
    if (!ctx->h_asm) CK(cudaMallocHost(&ctx->h_asm, 64), "pinned");
    CK(cudaMemcpyAsync(ctx->h_asm, dout, 32, cudaMemcpyDeviceToHost, s), "digest readback");
    CK(cudaStreamSynchronize(s), "digest");
    memcpy(out32, ctx->h_asm, 32);
    return DELTA_OK;
}

// SPDC container header on the device (NEXT f1): the BLAKE3-256 of exactly
// the body (reading R10) and the 67 header bytes, written to out_dev — e.g. the 67 bytes just
// ahead of the body in one buffer, so a container never passes through host memory.
extern "C" int delta_container_header(delta_ctx *ctx, const void *body_dev, uint64_t body_bytes, uint64_t version,
                                      uint64_t base_version, int elem, uint32_t n_tensors, int index_codec,
                                      void *out_dev, void *stream) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    const int w = elem_width(elem);
    if (!w) return fail(ctx, DELTA_EINVAL, 0, "unknown elem %d", elem);
    if (!out_dev || (body_bytes && !body_dev)) return fail(ctx, DELTA_EINVAL, 0, "delta_container_header: NULL pointer");
    if (index_codec != 1 && index_codec != 2) return fail(ctx, DELTA_EINVAL, 0, "index_codec must be 1 or 2");
    if (version != base_version + 1) return fail(ctx, DELTA_EINVAL, 0, "version must be base_version + 1 (SPEC.md:46)");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const unsigned long long nch = body_bytes == 0 ? 1 : (body_bytes + 1023) / 1024;
    GROW(ctx->dg_ws, (size_t)(2 * nch * 32 + 64));
    uint32_t *ws = ctx->dg_ws.as<uint32_t>();
    uint32_t *dout = ws + 2 * nch * 8;
    CK(launch_blake3(static_cast<const uint8_t *>(body_dev), body_bytes, ws, dout, s), "digest launch");
    CK(launch_spdc_header(static_cast<uint8_t *>(out_dev), dout, (uint32_t)index_codec, version, base_version,
                          w == 2 ? 0u : 1u, n_tensors, body_bytes, s),
       "header launch");
    return DELTA_OK;
}

// --------------------------------------------------------------------------- merge
// DELTA_MERGE_TIMING=1: host wall time of each delta_merge phase (each ends in a stream
// synchronisation) printed to stderr — diagnostics for scripts/merge_bench.py.
struct MergeTimer {
    bool on;
    std::chrono::steady_clock::time_point t;
    explicit MergeTimer(cudaStream_t s) : on(getenv("DELTA_MERGE_TIMING") != nullptr) {
        if (on) {
            cudaStreamSynchronize(s);
            t = std::chrono::steady_clock::now();
        }
    }
    void mark(const char *what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "delta_merge %-42s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// delta_merge (NEXT f4, reading R19): validate both bodies (layout, pairwise names and
// element counts, replace mode, full LEB128 decode with the apply's checks), decode them to
// (record, index) keys + values, merge the two key arrays by merge path, re-encode.  Four
// host syncs (sizes of the intermediate arrays and of the result).
extern "C" int delta_merge(delta_ctx *ctx, uint32_t n, int elem, const void *body_a, uint64_t a_bytes,
                           const void *body_b, uint64_t b_bytes, void *out, uint64_t out_capacity, void *stream,
                           uint64_t *out_bytes) {
    if (!ctx) return DELTA_EINVAL;
    ctx->err.clear();
    ctx->detail = 0;
    const int w = elem_width(elem);
    if (!w) return fail(ctx, DELTA_EINVAL, 0, "unknown elem %d", elem);
    if (!out_bytes) return fail(ctx, DELTA_EINVAL, 0, "out_bytes is NULL");
    if ((a_bytes && !body_a) || (b_bytes && !body_b)) return fail(ctx, DELTA_EINVAL, 0, "body is NULL");
    if (out_capacity && !out) return fail(ctx, DELTA_EINVAL, 0, "out_dev is NULL");
    if (ctx->index_codec != 0) return fail(ctx, DELTA_EINVAL, 0, "delta_merge reads LEB128 bodies only");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t nn = std::max<uint32_t>(n, 1);
    GROW(ctx->m_targets, nn * sizeof(TargetDesc));
    GROW(ctx->m_ha, nn * sizeof(RecordRow));
    GROW(ctx->m_hb, nn * sizeof(RecordRow));
    GROW(ctx->m_name_len, nn * 4);
    GROW(ctx->m_name_off, nn * 8);
    GROW(ctx->m_numel, nn * 8);
    GROW(ctx->m_ea, (nn + 1) * 8);
    GROW(ctx->m_eb, (nn + 1) * 8);
    GROW(ctx->m_eu, (nn + 1) * 8);
    GROW(ctx->m_status, 64);
    GROW(ctx->m_table, nn * sizeof(RecordRow));
    GROW(ctx->m_size, 64);
    MergeArgs m{};
    m.a = static_cast<const uint8_t *>(body_a);
    m.b = static_cast<const uint8_t *>(body_b);
    m.a_bytes = a_bytes;
    m.b_bytes = b_bytes;
    m.n = n;
    m.width = w;
    m.targets = ctx->m_targets.as<TargetDesc>();
    m.ha = ctx->m_ha.as<RecordRow>();
    m.hb = ctx->m_hb.as<RecordRow>();
    m.name_len = ctx->m_name_len.as<uint32_t>();
    m.name_off = ctx->m_name_off.as<unsigned long long>();
    m.numel = ctx->m_numel.as<unsigned long long>();
    m.ea = ctx->m_ea.as<unsigned long long>();
    m.eb = ctx->m_eb.as<unsigned long long>();
    m.eu = ctx->m_eu.as<unsigned long long>();
    m.status = ctx->m_status.as<uint32_t>();
    m.table = ctx->m_table.as<RecordRow>();
    m.body_size = ctx->m_size.as<unsigned long long>();
    MergeTimer mt(s);
    CK(launch_merge_walk(m, s), "merge walk");
    unsigned long long h[3];
    uint32_t st = 0;
    CK(cudaMemcpyAsync(&st, m.status, 4, cudaMemcpyDeviceToHost, s), "readback");
    CK(cudaMemcpyAsync(&h[0], m.ea + n, 8, cudaMemcpyDeviceToHost, s), "readback");
    CK(cudaMemcpyAsync(&h[1], m.eb + n, 8, cudaMemcpyDeviceToHost, s), "readback");
    CK(cudaStreamSynchronize(s), "merge walk");
    mt.mark("walk+check");
    if (st == kMergeTooLarge)
        return fail(ctx, DELTA_EINVAL, 0, "delta_merge: element_count >= 2^40 is not supported");
    if (st != kOk)
        return fail(ctx, st <= 10 ? kDetailToStatus[st] : DELTA_ECORRUPT, (int)st, "delta_merge: %s",
                    st <= 10 ? kDetailName[st] : "?");
    m.ma = h[0];
    m.mb = h[1];
    GROW(ctx->m_ia, std::max<size_t>(m.ma, 1) * 8);
    GROW(ctx->m_ib, std::max<size_t>(m.mb, 1) * 8);
    GROW(ctx->m_va, std::max<size_t>(m.ma, 1) * w);
    GROW(ctx->m_vb, std::max<size_t>(m.mb, 1) * w);
    m.ia = ctx->m_ia.as<unsigned long long>();
    m.ib = ctx->m_ib.as<unsigned long long>();
    m.va = ctx->m_va.p;
    m.vb = ctx->m_vb.p;
    // decode both bodies with the apply's validation (A1-A3), targets = the walk's
    if (!ctx->a_state.p) {
        GROW(ctx->a_state, sizeof(ApplyState));
        CK(cudaMemsetAsync(ctx->a_state.p, 0, sizeof(ApplyState), s), "memset");
    }
    GROW(ctx->a_recs, nn * sizeof(ApplyRec));
    GROW(ctx->a_rcb, (nn + 1) * 8);
    const size_t nch = std::max(a_bytes, b_bytes) / kByteChunk + n + 2;
    GROW(ctx->a_cnt, nch * 4);
    GROW(ctx->a_crec, nch * 4);
    GROW(ctx->a_sum, nch * 8);
    GROW(ctx->a_ord, nch * 8);
    GROW(ctx->a_idx, nch * 8);
    uint32_t dst[2] = {0, 0};
    for (int x = 0; x < 2; ++x) {
        CK(cudaMemsetAsync(ctx->a_state.p, 0, sizeof(uint32_t), s), "memset");  // this pass's gate
        ApplyArgs a;
        a.body = x ? m.b : m.a;
        a.body_bytes = x ? b_bytes : a_bytes;
        a.targets = m.targets;
        a.n = n;
        a.names = m.b;
        a.hint = x ? m.hb : m.ha;  // the walk's rows: A1 verifies all records in parallel
        a.recs = ctx->a_recs.as<ApplyRec>();
        a.rec_chunk_begin = ctx->a_rcb.as<unsigned long long>();
        a.chunk_rec = ctx->a_crec.as<uint32_t>();
        a.chunk_count = ctx->a_cnt.as<unsigned int>();
        a.chunk_sum = ctx->a_sum.as<unsigned long long>();
        a.chunk_ord_base = ctx->a_ord.as<unsigned long long>();
        a.chunk_idx_base = ctx->a_idx.as<unsigned long long>();
        a.chunk_cap = nch;
        a.state = ctx->a_state.as<ApplyState>();
        a.width = w;
        a.persist_ctas = ctx->sm_count * ctx->apply_ctas_per_sm;
        a.scatter_ctas = ctx->sm_count * ctx->scatter_ctas_per_sm;
        a.entry_major = false;
        a.index_codec = 0;
        CK(launch_decode_only(a, x ? m.ib : m.ia, x ? m.vb : m.va, x ? m.eb : m.ea, s), "merge decode");
        CK(cudaMemcpyAsync(&dst[x], ctx->a_state.p, 4, cudaMemcpyDeviceToHost, s), "readback");
    }
    CK(cudaStreamSynchronize(s), "merge decode");
    mt.mark("decode a+b");
    for (int x = 0; x < 2; ++x)
        if (dst[x] != kOk)
            return fail(ctx, dst[x] <= 10 ? kDetailToStatus[dst[x]] : DELTA_ECORRUPT, (int)dst[x],
                        "delta_merge: body %c: %s", x ? 'b' : 'a', dst[x] <= 10 ? kDetailName[dst[x]] : "?");
    m.ntiles = (m.ma + m.mb + 2047) / 2048;
    const size_t mx = std::max<size_t>(m.ma + m.mb, 1);  // the union is at most a + b entries
    GROW(ctx->m_dup, std::max<size_t>(m.ntiles, 2) * 4);
    GROW(ctx->m_ds, (m.ntiles + 1) * 8);
    GROW(ctx->m_blk, ((mx + 4095) / 4096 + 1) * 8);
    GROW(ctx->m_lb, (m.ntiles + 1) * 8);
    GROW(ctx->m_bstat, (m.ntiles + 1) * 8);
    m.bstat = ctx->m_bstat.as<unsigned long long>();
    GROW(ctx->m_u, mx * 8);
    GROW(ctx->m_uv, mx * w);
    GROW(ctx->m_len, mx * 4);
    GROW(ctx->m_lo, (mx + 1) * 8);
    m.split = ctx->m_lb.as<unsigned long long>();
    m.tile_cnt = ctx->m_dup.as<uint32_t>();
    m.tile_off = ctx->m_ds.as<unsigned long long>();
    m.blk = ctx->m_blk.as<unsigned long long>();
    m.u = ctx->m_u.as<unsigned long long>();
    m.uv = ctx->m_uv.p;
    m.len = ctx->m_len.as<uint32_t>();
    m.lo = ctx->m_lo.as<unsigned long long>();
    CK(launch_merge_count(m, s), "merge path");
    CK(cudaMemcpyAsync(&h[2], m.tile_off + m.ntiles, 8, cudaMemcpyDeviceToHost, s), "readback");
    CK(cudaStreamSynchronize(s), "merge path");
    mt.mark("merge path (one pass, look-back offsets)");
    m.mu = m.ntiles ? h[2] : 0;
    CK(launch_merge_place(m, s), "merge place");
    unsigned long long size = 0;
    CK(cudaMemcpyAsync(&size, m.body_size, 8, cudaMemcpyDeviceToHost, s), "readback");
    CK(cudaStreamSynchronize(s), "merge place");
    mt.mark("record bounds + table");
    *out_bytes = size;
    if (size > out_capacity)
        return fail(ctx, DELTA_ECAPACITY, 0, "output capacity %llu < merged body size %llu",
                    (unsigned long long)out_capacity, size);
    CK(launch_merge_emit(m, static_cast<uint8_t *>(out), s), "merge emit");
    if (mt.on) {
        CK(cudaStreamSynchronize(s), "merge emit");
        mt.mark("emit + headers");
    }
    return DELTA_OK;
}

