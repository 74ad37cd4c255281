// extract.cu — sm_100a kernels for delta extraction.
//
//   K1 k_scan_compact   E2+E3: bitwise compare of old/new (16-byte streaming loads),
//                       per-vector lane masks, packed block scan of counts, decoupled
//                       look-back across tiles (ticket-ordered), ordered write of the
//                       compacted (index, value) entries.  The only kernel that reads the
//                       2W bytes of weights: it bounds the whole path (HBM roofline).
//   K2 k_entry_lens     E4+E5 lengths: gap of every entry (first index of a tensor as-is,
//                       PAPER.md:389), LEB128 length, per-chunk byte sums and the partial
//                       sums at tensor starts.
//   K3 k_finalize       E6: scan of chunk sums, per-tensor index-stream lengths, record
//                       sizes and offsets (the offset table), body size.
//   K4 k_emit           E5+E6: LEB128 bytes and raw values written to their final offsets.
//   K5 k_headers        E6: record headers (name_len, name, N, nnz, index_bytes) + mode.
//
// Every kernel here is product code written for this library; none shares code with
// oracle/.  Semantics: DESIGN.md §3 readings R1-R5, R12-R15.
#include <cstdint>
#include <cuda_runtime.h>

#include "sd_device.cuh"
#include "sd_internal.cuh"

namespace sd {

template <int W> struct LaneOf;
template <> struct LaneOf<2> { using T = uint16_t; };
template <> struct LaneOf<4> { using T = uint32_t; };

__device__ __forceinline__ uint32_t word_of(const uint4 &v, int w) {
    return w == 0 ? v.x : (w == 1 ? v.y : (w == 2 ? v.z : v.w));
}

// Lane j of a 16-byte vector (little-endian lane order).
template <int W>
__device__ __forceinline__ uint32_t lane_of(const uint4 &v, int j) {
    if constexpr (W == 2) {
        return (word_of(v, j >> 1) >> ((j & 1) * 16)) & 0xFFFFu;
    } else {
        return word_of(v, j);
    }
}

template <int W>
__device__ __forceinline__ void set_lane(uint4 &v, int j, uint32_t x) {
    if constexpr (W == 2) {
        const int w = j >> 1, sh = (j & 1) * 16;
        uint32_t m = 0xFFFFu << sh, y = (x & 0xFFFFu) << sh;
        if (w == 0) v.x = (v.x & ~m) | y;
        else if (w == 1) v.y = (v.y & ~m) | y;
        else if (w == 2) v.z = (v.z & ~m) | y;
        else v.w = (v.w & ~m) | y;
    } else {
        if (j == 0) v.x = x;
        else if (j == 1) v.y = x;
        else if (j == 2) v.z = x;
        else v.w = x;
    }
}

// Bit j set iff lane j of the two vectors differs as an unsigned integer (reading R2).
template <int W>
__device__ __forceinline__ uint32_t diff_mask(const uint4 &a, const uint4 &b) {
    const uint32_t x0 = a.x ^ b.x, x1 = a.y ^ b.y, x2 = a.z ^ b.z, x3 = a.w ^ b.w;
    if constexpr (W == 2) {
        return (uint32_t)((x0 & 0xFFFFu) != 0) | ((uint32_t)((x0 >> 16) != 0) << 1) |
               ((uint32_t)((x1 & 0xFFFFu) != 0) << 2) | ((uint32_t)((x1 >> 16) != 0) << 3) |
               ((uint32_t)((x2 & 0xFFFFu) != 0) << 4) | ((uint32_t)((x2 >> 16) != 0) << 5) |
               ((uint32_t)((x3 & 0xFFFFu) != 0) << 6) | ((uint32_t)((x3 >> 16) != 0) << 7);
    } else {
        return (uint32_t)(x0 != 0) | ((uint32_t)(x1 != 0) << 1) | ((uint32_t)(x2 != 0) << 2) |
               ((uint32_t)(x3 != 0) << 3);
    }
}

// ------------------------------------------------------------------------------ K1
template <int W, typename IdxT>
__global__ void __launch_bounds__(kScanThreads)
k_scan_compact(const TileDesc *__restrict__ tiles, uint32_t ntiles, uint32_t ntensors,
               unsigned long long *tile_state, unsigned int *ticket,
               IdxT *__restrict__ ws_idx, typename LaneOf<W>::T *__restrict__ ws_val,
               unsigned long long ws_cap, unsigned long long *__restrict__ entry_begin,
               ExtractSummary *summary) {
    using LT = typename LaneOf<W>::T;
    constexpr int LPV = 16 / W;  // lanes per 16-byte vector
    static_assert(kScanVecs == 8, "count packing assumes 8 vectors per thread");
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_warp[kScanThreads / 32][4];
    __shared__ unsigned long long s_excl;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // Ticket order = look-back order: every tile with a smaller id belongs to a CTA that
    // is already running, so the look-back below always makes progress.
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    const TileDesc d = tiles[t];
    const uint32_t nl = d.nlanes;

    uint4 vo[kScanVecs], vn[kScanVecs];
    if (d.flags_tensor & kTileAligned) {
#pragma unroll
        for (int r = 0; r < kScanVecs; ++r) {
            const uint32_t v = r * kScanThreads + tid;
            if ((v + 1) * LPV <= nl) {
                vo[r] = ld_stream_v4(d.old_p + (size_t)v * 16);
                vn[r] = ld_stream_v4(d.new_p + (size_t)v * 16);
            } else {
                vo[r] = make_uint4(0, 0, 0, 0);
                vn[r] = vo[r];
                if (v * LPV < nl) {
                    for (int j = 0; j < LPV && v * LPV + j < nl; ++j) {
                        set_lane<W>(vo[r], j, reinterpret_cast<const LT *>(d.old_p)[v * LPV + j]);
                        set_lane<W>(vn[r], j, reinterpret_cast<const LT *>(d.new_p)[v * LPV + j]);
                    }
                }
            }
        }
    } else {  // span not 16-byte aligned: same lane order, lane-by-lane loads
#pragma unroll
        for (int r = 0; r < kScanVecs; ++r) {
            const uint32_t v = r * kScanThreads + tid;
            vo[r] = make_uint4(0, 0, 0, 0);
            vn[r] = vo[r];
            for (int j = 0; j < LPV && v * LPV + j < nl; ++j) {
                set_lane<W>(vo[r], j, __ldg(reinterpret_cast<const LT *>(d.old_p) + v * LPV + j));
                set_lane<W>(vn[r], j, __ldg(reinterpret_cast<const LT *>(d.new_p) + v * LPV + j));
            }
        }
    }

    // Per-vector change masks and counts; 8 counts (<= LPV each) packed as 16-bit
    // fields into 4 words so one block scan yields all 8 per-vector prefixes.
    uint32_t m[kScanVecs];
    uint32_t pk[4];
#pragma unroll
    for (int r = 0; r < kScanVecs; ++r) m[r] = diff_mask<W>(vo[r], vn[r]);
#pragma unroll
    for (int q = 0; q < 4; ++q) pk[q] = __popc(m[2 * q]) | (__popc(m[2 * q + 1]) << 16);

    uint32_t inc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) inc[q] = warp_inclusive_sum(pk[q]);
    if (lane == 31) {
#pragma unroll
        for (int q = 0; q < 4; ++q) s_warp[warp][q] = inc[q];
    }
    __syncthreads();
    uint32_t pre[4] = {0, 0, 0, 0}, tot[4] = {0, 0, 0, 0};
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t x = s_warp[w][q];
            if (w < warp) pre[q] += x;
            tot[q] += x;
        }
    }
    uint32_t agg = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) agg += (tot[q] & 0xFFFFu) + (tot[q] >> 16);

    // Decoupled look-back (warp 0): publish the aggregate, then sum predecessors until an
    // inclusive prefix is found, then publish our inclusive prefix.
    if (warp == 0) {
        unsigned long long excl = 0;
        if (t == 0) {
            if (lane == 0) st_release_u64(&tile_state[0], kFlagIncl | agg);
        } else {
            if (lane == 0) st_release_u64(&tile_state[t], kFlagAgg | agg);
            long long pred = (long long)t - 1;
            while (true) {
                const long long i = pred - lane;
                unsigned long long s = kFlagIncl;  // before tile 0: inclusive prefix 0
                if (i >= 0) {
                    do {
                        s = ld_acquire_u64(&tile_state[i]);
                    } while ((s >> 62) == 0);
                }
                const unsigned incl = __ballot_sync(0xffffffffu, (s >> 62) == 2);
                unsigned long long v = s & kValMask;
                if (incl) {
                    const int k = __ffs(incl) - 1;
                    if (lane > k) v = 0;
                    excl += warp_sum(v);
                    break;
                }
                excl += warp_sum(v);
                pred -= 32;
            }
            if (lane == 0) st_release_u64(&tile_state[t], kFlagIncl | (excl + agg));
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    const unsigned long long base = s_excl;

    if (tid == 0) {
        if (d.flags_tensor & kTileFirstOfTensor)
            entry_begin[d.flags_tensor & kTileTensorMask] = base;
        if (t == ntiles - 1) {
            summary->M = base + agg;
            entry_begin[ntensors] = base + agg;
        }
    }
    if (base + agg > ws_cap) {
        if (tid == 0) summary->overflow = 1;
        return;
    }
    // Ordered write: entry (r, tid, j) goes to base + sum_{r'<r} tot_r' + prefix_r(tid) + rank_j.
    unsigned long long rbase = base;
#pragma unroll
    for (int r = 0; r < kScanVecs; ++r) {
        const int q = r >> 1, sh = (r & 1) * 16;
        unsigned long long pos = rbase + (((pre[q] + inc[q] - pk[q]) >> sh) & 0xFFFFu);
        uint32_t mm = m[r];
        while (mm) {
            const int j = __ffs(mm) - 1;
            mm &= mm - 1;
            const uint64_t li = (uint64_t)(r * kScanThreads + tid) * LPV + j;
            ws_idx[pos] = (IdxT)(d.lane_base + li);
            ws_val[pos] = (LT)lane_of<W>(vn[r], j);
            ++pos;
        }
        rbase += (tot[q] >> sh) & 0xFFFFu;
    }
}

// ---------------------------------------------------------------- entry helpers (K2, K4)
// Largest k in [0, T] with E[k] <= i (E nondecreasing, E[0] = 0).
__device__ __forceinline__ uint32_t tensor_of(const unsigned long long *E, uint32_t T,
                                              unsigned long long i) {
    uint32_t lo = 0, hi = T;  // invariant: E[lo] <= i
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (__ldg(E + mid) <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

template <typename IdxT>
__device__ __forceinline__ void load_entries(const IdxT *ws_idx, unsigned long long i0,
                                             unsigned long long M, IdxT (&v)[kEntryPerThread]) {
    if (i0 + kEntryPerThread <= M) {
        const uint4 *p = reinterpret_cast<const uint4 *>(ws_idx + i0);
        constexpr int NV = kEntryPerThread * sizeof(IdxT) / 16;
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            uint4 x = __ldg(p + q);
            IdxT *dst = reinterpret_cast<IdxT *>(&x);
#pragma unroll
            for (int e = 0; e < (int)(16 / sizeof(IdxT)); ++e) v[q * (16 / sizeof(IdxT)) + e] = dst[e];
        }
    } else {
#pragma unroll
        for (int e = 0; e < kEntryPerThread; ++e) v[e] = (i0 + e < M) ? __ldg(ws_idx + i0 + e) : 0;
    }
}

template <int NW, typename T>
__device__ __forceinline__ T block_excl_scan(T v, T *s_warp, T &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const T inc = warp_inclusive_sum(v);
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    T pre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const T x = s_warp[w];
        if (w < warp) pre += x;
        tot += x;
    }
    __syncthreads();
    total = tot;
    return pre + inc - v;
}

// ------------------------------------------------------------------------------ K2
template <typename IdxT>
__global__ void __launch_bounds__(256)
k_entry_lens(const IdxT *__restrict__ ws_idx, const unsigned long long *__restrict__ E,
             uint32_t T, const ExtractSummary *summary, unsigned int *__restrict__ chunk_bytes,
             unsigned long long *__restrict__ tstart_partial) {
    if (summary->overflow) return;
    const unsigned long long M = summary->M;
    const unsigned long long nchunks = (M + kEntryChunk - 1) / kEntryChunk;
    __shared__ uint32_t s_warp[8];
    for (unsigned long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const unsigned long long i0 = c * kEntryChunk + (unsigned long long)threadIdx.x * kEntryPerThread;
        IdxT v[kEntryPerThread];
        load_entries<IdxT>(ws_idx, i0, M, v);
        uint32_t k = tensor_of(E, T, i0 < M ? i0 : M);
        unsigned long long prev = (i0 > 0 && i0 < M) ? (unsigned long long)__ldg(ws_idx + i0 - 1) : 0;
        uint32_t lens[kEntryPerThread];
        uint32_t S = 0;
        bool has_start = false;
#pragma unroll
        for (int e = 0; e < kEntryPerThread; ++e) {
            const unsigned long long i = i0 + e;
            uint32_t L = 0;
            if (i < M) {
                while (__ldg(E + k + 1) <= i) ++k;
                const bool first = (i == __ldg(E + k));
                has_start |= first;
                const unsigned long long g = (unsigned long long)v[e] - (first ? 0ull : prev);
                L = leb_len(g);
                prev = v[e];
            }
            lens[e] = L;
            S += L;
        }
        uint32_t total;
        const uint32_t P = block_excl_scan<8, uint32_t>(S, s_warp, total);
        if (threadIdx.x == 0) chunk_bytes[c] = total;
        if (has_start) {  // byte offset (within the chunk) of every tensor start we hold
            uint32_t acc = P;
            k = tensor_of(E, T, i0);
            for (int e = 0; e < kEntryPerThread; ++e) {
                const unsigned long long i = i0 + e;
                if (i >= M) break;
                while (__ldg(E + k + 1) <= i) ++k;
                if (i == __ldg(E + k)) {
                    // tensor k starts here, and so do any empty tensors just before it
                    for (int kk = (int)k; kk >= 0 && __ldg(E + kk) == i; --kk) tstart_partial[kk] = acc;
                }
                acc += lens[e];
            }
        }
    }
}

// ------------------------------------------------------------------------------ K3
__global__ void __launch_bounds__(1024)
k_finalize(const unsigned long long *__restrict__ E, uint32_t T, const uint32_t *__restrict__ name_len,
           const unsigned int *__restrict__ chunk_bytes, unsigned long long *__restrict__ chunk_prefix,
           const unsigned long long *__restrict__ tstart_partial,
           unsigned long long *__restrict__ Bk, RecordRow *__restrict__ table, int width,
           const unsigned long long *__restrict__ numel, ExtractSummary *summary) {
    if (summary->overflow) return;
    __shared__ unsigned long long s_warp[32];
    const unsigned long long M = summary->M;
    const unsigned long long nchunks = (M + kEntryChunk - 1) / kEntryChunk;
    unsigned long long carry = 0;
    for (unsigned long long b = 0; b < nchunks; b += 1024) {
        const unsigned long long c = b + threadIdx.x;
        const unsigned long long x = c < nchunks ? chunk_bytes[c] : 0;
        unsigned long long tot;
        const unsigned long long ex = block_excl_scan<32, unsigned long long>(x, s_warp, tot);
        if (c < nchunks) chunk_prefix[c] = carry + ex;
        carry += tot;
    }
    const unsigned long long total_idx = carry;
    __syncthreads();
    for (uint32_t k = threadIdx.x; k <= T; k += 1024) {
        const unsigned long long e = E[k];
        Bk[k] = (e >= M) ? total_idx : chunk_prefix[e / kEntryChunk] + tstart_partial[k];
    }
    __syncthreads();
    carry = 0;
    for (uint32_t b = 0; b < T; b += 1024) {
        const uint32_t k = b + threadIdx.x;
        unsigned long long rb = 0, nnz = 0, ilen = 0;
        if (k < T) {
            nnz = E[k + 1] - E[k];
            ilen = Bk[k + 1] - Bk[k];
            rb = 27ull + name_len[k] + ilen + (unsigned long long)width * nnz;
        }
        unsigned long long tot;
        const unsigned long long ex = block_excl_scan<32, unsigned long long>(rb, s_warp, tot);
        if (k < T) {
            RecordRow r;
            r.record_offset = carry + ex;
            r.element_count = numel[k];
            r.nnz = nnz;
            r.index_offset = r.record_offset + 2 + name_len[k] + 24;
            r.index_bytes = ilen;
            r.values_offset = r.index_offset + ilen;
            r.record_bytes = rb;
            table[k] = r;
        }
        carry += tot;
    }
    if (threadIdx.x == 0) {
        summary->idx_bytes = total_idx;
        summary->body_bytes = carry;
    }
}

// ------------------------------------------------------------------------------ K4
template <int W, typename IdxT>
__global__ void __launch_bounds__(256)
k_emit(const IdxT *__restrict__ ws_idx, const typename LaneOf<W>::T *__restrict__ ws_val,
       const unsigned long long *__restrict__ E, uint32_t T, const ExtractSummary *summary,
       const unsigned long long *__restrict__ chunk_prefix, const unsigned long long *__restrict__ Bk,
       const RecordRow *__restrict__ table, uint8_t *__restrict__ out) {
    using LT = typename LaneOf<W>::T;
    const unsigned long long M = summary->M;
    const unsigned long long nchunks = (M + kEntryChunk - 1) / kEntryChunk;
    __shared__ uint32_t s_warp[8];
    for (unsigned long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const unsigned long long i0 = c * kEntryChunk + (unsigned long long)threadIdx.x * kEntryPerThread;
        IdxT v[kEntryPerThread];
        load_entries<IdxT>(ws_idx, i0, M, v);
        const uint32_t k0 = tensor_of(E, T, i0 < M ? i0 : M);
        const unsigned long long prev0 = (i0 > 0 && i0 < M) ? (unsigned long long)__ldg(ws_idx + i0 - 1) : 0;
        uint32_t k = k0;
        unsigned long long prev = prev0;
        uint32_t S = 0;
#pragma unroll
        for (int e = 0; e < kEntryPerThread; ++e) {
            const unsigned long long i = i0 + e;
            if (i < M) {
                while (__ldg(E + k + 1) <= i) ++k;
                const bool first = (i == __ldg(E + k));
                S += leb_len((unsigned long long)v[e] - (first ? 0ull : prev));
                prev = v[e];
            }
        }
        uint32_t total;
        const uint32_t P = block_excl_scan<8, uint32_t>(S, s_warp, total);
        unsigned long long pos = chunk_prefix[c] + P;  // position in the concatenated streams
        k = k0;
        prev = prev0;
        for (int e = 0; e < kEntryPerThread; ++e) {
            const unsigned long long i = i0 + e;
            if (i >= M) break;
            while (__ldg(E + k + 1) <= i) ++k;
            const unsigned long long Ek = __ldg(E + k);
            const bool first = (i == Ek);
            unsigned long long g = (unsigned long long)v[e] - (first ? 0ull : prev);
            prev = v[e];
            const RecordRow &row = table[k];
            uint8_t *dst = out + __ldg(&row.index_offset) + (pos - __ldg(Bk + k));
            uint32_t n = 0;
            while (g >= 0x80) {
                dst[n++] = (uint8_t)(g | 0x80);
                g >>= 7;
            }
            dst[n++] = (uint8_t)g;
            pos += n;
            const LT val = __ldg(ws_val + i);
            uint8_t *vd = out + __ldg(&row.values_offset) + (i - Ek) * W;
#pragma unroll
            for (int b = 0; b < W; ++b) vd[b] = (uint8_t)(val >> (8 * b));
        }
    }
}

// ------------------------------------------------------------------------------ K5
__device__ __forceinline__ void put_u64(uint8_t *p, unsigned long long x) {
#pragma unroll
    for (int b = 0; b < 8; ++b) p[b] = (uint8_t)(x >> (8 * b));
}

__global__ void __launch_bounds__(128)
k_headers(const RecordRow *__restrict__ table, uint32_t T, const uint32_t *__restrict__ name_len,
          const uint32_t *__restrict__ name_off, const uint8_t *__restrict__ names,
          uint8_t *__restrict__ out) {
    for (uint32_t k = blockIdx.x; k < T; k += gridDim.x) {
        const RecordRow r = table[k];
        uint8_t *o = out + r.record_offset;
        const uint32_t nl = name_len[k];
        for (uint32_t b = threadIdx.x; b < nl; b += blockDim.x) o[2 + b] = names[name_off[k] + b];
        if (threadIdx.x == 0) {
            o[0] = (uint8_t)nl;
            o[1] = (uint8_t)(nl >> 8);
            put_u64(o + 2 + nl, r.element_count);
            put_u64(o + 2 + nl + 8, r.nnz);
            put_u64(o + 2 + nl + 16, r.index_bytes);
            o[r.record_bytes - 1] = 0;  // mode: replace (reading R1/R9)
        }
    }
}

// ------------------------------------------------------------------------------ launchers
template <int W, typename IdxT>
static cudaError_t scan_impl(const ExtractArgs &a, cudaStream_t s, cudaEvent_t *ev) {
    using LT = typename LaneOf<W>::T;
    if (ev) cudaEventRecord(ev[0], s);
    k_scan_compact<W, IdxT><<<a.ntiles, kScanThreads, 0, s>>>(
        a.tiles, a.ntiles, a.ntensors, a.tile_state, a.ticket, static_cast<IdxT *>(a.ws_idx),
        static_cast<LT *>(a.ws_val), a.ws_cap, a.entry_begin, a.summary);
    if (ev) cudaEventRecord(ev[1], s);
    k_entry_lens<IdxT><<<a.persist_ctas, 256, 0, s>>>(static_cast<const IdxT *>(a.ws_idx),
                                                      a.entry_begin, a.ntensors, a.summary,
                                                      a.chunk_bytes, a.tstart_partial);
    if (ev) cudaEventRecord(ev[2], s);
    k_finalize<<<1, 1024, 0, s>>>(a.entry_begin, a.ntensors, a.name_len, a.chunk_bytes,
                                  a.chunk_prefix, a.tstart_partial, a.tensor_byte_begin, a.table,
                                  a.width, a.numel, a.summary);
    if (ev) cudaEventRecord(ev[3], s);
    return cudaGetLastError();
}

template <int W, typename IdxT>
static cudaError_t emit_impl(const ExtractArgs &a, uint8_t *out, cudaStream_t s, cudaEvent_t *ev) {
    using LT = typename LaneOf<W>::T;
    if (ev) cudaEventRecord(ev[0], s);
    k_emit<W, IdxT><<<a.persist_ctas, 256, 0, s>>>(
        static_cast<const IdxT *>(a.ws_idx), static_cast<const LT *>(a.ws_val), a.entry_begin,
        a.ntensors, a.summary, a.chunk_prefix, a.tensor_byte_begin, a.table, out);
    if (ev) cudaEventRecord(ev[1], s);
    const uint32_t hb = a.ntensors < 65535u ? (a.ntensors ? a.ntensors : 1u) : 65535u;
    k_headers<<<hb, 128, 0, s>>>(a.table, a.ntensors, a.name_len, a.name_off, a.names, out);
    if (ev) cudaEventRecord(ev[2], s);
    return cudaGetLastError();
}

cudaError_t launch_extract_scan(const ExtractArgs &a, cudaStream_t s, cudaEvent_t *ev) {
    if (a.width == 2) return a.idx64 ? scan_impl<2, uint64_t>(a, s, ev) : scan_impl<2, uint32_t>(a, s, ev);
    return a.idx64 ? scan_impl<4, uint64_t>(a, s, ev) : scan_impl<4, uint32_t>(a, s, ev);
}

cudaError_t launch_extract_emit(const ExtractArgs &a, uint8_t *out, cudaStream_t s, cudaEvent_t *ev) {
    if (a.width == 2) return a.idx64 ? emit_impl<2, uint64_t>(a, out, s, ev) : emit_impl<2, uint32_t>(a, out, s, ev);
    return a.idx64 ? emit_impl<4, uint64_t>(a, out, s, ev) : emit_impl<4, uint32_t>(a, out, s, ev);
}

}  // namespace sd
