// merge.cu — sm_100a kernels for delta_merge (NEXT f4, reading R19): the delta
// D_a (v-1 -> v) followed by D_b (v -> v+1) as ONE delta (v-1 -> v+1) for a laggard's
// catch-up ("laggards catch up asynchronously"; SPEC.md:476 leaves merging
// open).  Per tensor: the union of the two index sets, D_b's value where D_b has the
// index, else D_a's — applying the merge equals applying D_a then D_b.
//
//   M1 k_merge_walk     one thread follows both bodies' chains of record offsets (layout,
//                       entry prefixes E_a, E_b, table rows); k_merge_check per record in
//                       parallel: mode byte (replace only), names and element counts equal
//                       pairwise; apply targets (B's names) and table hints for the decodes.
//   (decode)            each body through A1-A3 + k_decode_write (apply.cu): validated,
//                       absolute indices + values per entry.
//   M2 k_merge_path     merge path over the two key arrays (keys = record << 40 | index
//                       ascend over a whole body): 2048 merged positions per tile, tile
//                       splits by one binary search per boundary (k_merge_splits, all in
//                       parallel), tiles staged in shared memory, 8 positions per thread (a
//                       second binary search in shared memory); an a-entry is dropped when
//                       the b head equals it (b's value wins).  One pass: tiles are
//                       claimed in order from a ticket; each finds the offset of its kept
//                       entries and of their LEB128 bytes by decoupled look-back over its
//                       predecessors, marks record starts and writes keys, values and byte
//                       offsets coalesced (via shared memory).
//   M3 k_merge_bounds_fill / k_merge_table: empty records, the offset table, body size.
//   M4 k_merge_emit     LEB128 bytes + values per entry; k_merge_headers per record.
//
// Product code; shares nothing with oracle/.
#include <cstdint>
#include <cuda_runtime.h>

#include "sd_device.cuh"
#include "sd_internal.cuh"

namespace sd {

namespace {

template <int W> struct Lane;
template <> struct Lane<2> { using T = uint16_t; };
template <> struct Lane<4> { using T = uint32_t; };

__device__ __forceinline__ unsigned long long rd_u(const uint8_t *p, int nbytes) {
    unsigned long long x = 0;
    for (int b = 0; b < nbytes; ++b) x |= (unsigned long long)p[b] << (8 * b);
    return x;
}

constexpr unsigned long long kIdxMask = (1ull << kKeyShift) - 1;

// ---------------------------------------------------------------- block-wide exclusive scan (u64)

__device__ __forceinline__ unsigned long long block_scan_excl(unsigned long long v, unsigned long long *s_w,
                                                              unsigned long long &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    unsigned long long pre = 0, tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        if (w < warp) pre += s_w[w];
        tot += s_w[w];
    }
    __syncthreads();
    total = tot;
    return pre + inc - v;
}

// ---------------------------------------------------------------- M1
// Record geometry of one body at offset ro (bounds-checked: the bodies are untrusted).
// Returns false on a layout fault.
__device__ __forceinline__ bool header_at(const uint8_t *B, unsigned long long sz, unsigned long long ro,
                                          int width, RecordRow &r) {
    if (ro > sz || sz - ro < 2) return false;
    const unsigned long long nl = rd_u(B + ro, 2);
    if (sz - ro - 2 < nl + 24) return false;
    const unsigned long long q = ro + 2 + nl;
    const unsigned long long N = rd_u(B + q, 8), nnz = rd_u(B + q + 8, 8), il = rd_u(B + q + 16, 8);
    const unsigned long long rem = sz - q - 24;
    if (il > rem || nnz > (rem - il) / (unsigned long long)width || rem - il - nnz * width < 1) return false;
    r.record_offset = ro;
    r.element_count = N;
    r.nnz = nnz;
    r.index_offset = q + 24;
    r.index_bytes = il;
    r.values_offset = q + 24 + il;
    r.record_bytes = 2 + nl + 24 + il + nnz * width + 1;
    return true;
}

// One thread follows the chain of record offsets of both bodies (the only sequential part:
// two dependent header loads per record, the two bodies interleaved); everything else is
// checked per record in parallel by k_merge_check.  The rows double as the decodes' table
// hints (A1 then verifies all records in parallel).
__global__ void k_merge_walk(MergeArgs m) {
    if (blockIdx.x || threadIdx.x) return;
    unsigned long long pa = 0, pb = 0, ea = 0, eb = 0;
    uint32_t st = kOk;
    for (uint32_t k = 0; k < m.n; ++k) {
        RecordRow ra, rb;
        const bool oa = header_at(m.a, m.a_bytes, pa, m.width, ra);
        const bool ob = header_at(m.b, m.b_bytes, pb, m.width, rb);
        if (!oa || !ob) {
            st = kLayout;
            break;
        }
        m.ha[k] = ra;
        m.hb[k] = rb;
        m.ea[k] = ea;
        m.eb[k] = eb;
        ea += ra.nnz;
        eb += rb.nnz;
        pa += ra.record_bytes;
        pb += rb.record_bytes;
    }
    if (st == kOk && (pa != m.a_bytes || pb != m.b_bytes)) st = kLayout;
    m.ea[m.n] = ea;
    m.eb[m.n] = eb;
    *m.status = st;
}

// Per record (parallel): replace-mode bytes, equal names and element counts, the element
// count within the 40-bit index field of the merge keys; apply targets for the decodes.
__global__ void __launch_bounds__(256) k_merge_check(MergeArgs m) {
    if (*m.status != kOk) return;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < m.n; k += gridDim.x * blockDim.x) {
        const RecordRow ra = m.ha[k], rb = m.hb[k];
        uint32_t e = kOk;
        if (m.a[ra.record_offset + ra.record_bytes - 1] != 0 || m.b[rb.record_offset + rb.record_bytes - 1] != 0) {
            e = kMode;  // replace-mode records only
        } else {
            const unsigned long long nla = ra.index_offset - 24 - 2 - ra.record_offset;
            const unsigned long long nlb = rb.index_offset - 24 - 2 - rb.record_offset;
            uint32_t diff = nla != nlb;
            for (unsigned long long j = 0; j < nlb && !diff; j += 16) {
                const unsigned long long jn = min(nlb, j + 16);
                for (unsigned long long x = j; x < jn; ++x)
                    diff |= m.a[ra.record_offset + 2 + x] ^ m.b[rb.record_offset + 2 + x];
            }
            if (diff) e = kName;
            else if (ra.element_count != rb.element_count) e = kNumel;
            else if (rb.element_count > kIdxMask + 1) e = kMergeTooLarge;
            m.targets[k] = TargetDesc{nullptr, rb.element_count, rb.record_offset + 2, nlb};
            m.name_len[k] = (uint32_t)nlb;
            m.name_off[k] = rb.record_offset + 2;
            m.numel[k] = rb.element_count;
        }
        if (e != kOk) atomicCAS(m.status, (uint32_t)kOk, e);
    }
}

// ---------------------------------------------------------------- M2
constexpr int kMpTile = 2048;  // merged positions per tile (256 threads x 8)

// number of A elements among the first d positions of merge(A, B), A first on ties
template <typename T>
__device__ __forceinline__ unsigned long long mp_split(const T *A, unsigned long long na, const T *B,
                                                       unsigned long long nb, unsigned long long d) {
    unsigned long long lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
    while (lo < hi) {
        const unsigned long long mid = (lo + hi) >> 1;
        if (A[mid] <= B[d - mid - 1]) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// split[t] = A elements among the first t * kMpTile merged positions (t = 0 .. ntiles)
__global__ void __launch_bounds__(256) k_merge_splits(MergeArgs m) {
    const unsigned long long total = m.ma + m.mb;
    for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t <= m.ntiles;
         t += (unsigned long long)gridDim.x * blockDim.x)
        m.split[t] = mp_split(m.ia, m.ma, m.ib, m.mb, min(t * kMpTile, total));
}

// One tile of 2048 merged positions per iteration: the tile's a and b runs staged in
// shared memory, 8 positions per thread (split by a binary search in shared memory),
// pass 1 counts the kept entries, pass 2 stages them in shared memory (keys, and the source
// position of each value) and writes them out coalesced.
template <int W, bool WRITE>
__global__ void __launch_bounds__(256) k_merge_path(MergeArgs m) {
    using LT = typename Lane<W>::T;
    __shared__ unsigned long long sa[kMpTile + 1], sb[kMpTile + 1];
    __shared__ uint32_t s_src[WRITE ? kMpTile : 1];  // kept entry -> source (bit 31: from b)
    __shared__ uint32_t s_w[8];
    __shared__ unsigned long long s_prev;
    __shared__ unsigned long long s_t, s_base, s_bbase;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // WRITE: one pass — tiles are claimed in order from a ticket and each finds its output
    // offset by decoupled look-back over its predecessors' published counts (tile_off is
    // the status array, zeroed: flag 1 = the tile's own count, 2 = inclusive prefix)
    for (unsigned long long t0 = blockIdx.x;; t0 += gridDim.x) {
        if constexpr (WRITE) {
            if (tid == 0) s_t = atomicAdd(reinterpret_cast<unsigned long long *>(m.tile_cnt), 1ull);
            __syncthreads();
        }
        const unsigned long long t = WRITE ? s_t : t0;
        if (t >= m.ntiles) break;
        const unsigned long long d0 = t * kMpTile, d1 = min(d0 + kMpTile, m.ma + m.mb);
        const unsigned long long i0 = m.split[t], j0 = d0 - i0;
        const uint32_t na = (uint32_t)(m.split[t + 1] - i0), nb = (uint32_t)(d1 - m.split[t + 1] - j0);
        for (uint32_t x = tid; x < na; x += blockDim.x) sa[x] = m.ia[i0 + x];
        for (uint32_t x = tid; x < nb; x += blockDim.x) sb[x] = m.ib[j0 + x];
        if (tid == 0) {  // the heads just past the tile (a b head there can equal our last a)
            sa[na] = i0 + na < m.ma ? m.ia[i0 + na] : ~0ull;
            sb[nb] = j0 + nb < m.mb ? m.ib[j0 + nb] : ~0ull;
        }
        __syncthreads();
        const uint32_t n = na + nb, e0 = min((uint32_t)tid * 8u, n), e1 = min(e0 + 8u, n);
        const uint32_t i_start = (uint32_t)mp_split(sa, na, sb, nb, e0);
        uint32_t keep = 0;
        {
            uint32_t i = i_start, j = e0 - i_start;
            for (uint32_t e = e0; e < e1; ++e) {
                if (j >= nb || (i < na && sa[i] <= sb[j])) {
                    keep += sa[i] != sb[j];
                    ++i;
                } else {
                    ++keep;
                    ++j;
                }
            }
        }
        uint32_t inc = keep;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) s_w[warp] = inc;
        __syncthreads();
        uint32_t pre = 0, tot = 0;
        for (int w = 0; w < 8; ++w) {
            if (w < warp) pre += s_w[w];
            tot += s_w[w];
        }
        if constexpr (!WRITE) {
            if (tid == 0) m.tile_cnt[t] = tot;
        } else {
            if (tid == 0) {
                constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = (1ull << 62) - 1;
                unsigned long long excl = 0;
                if (t == 0) {
                    st_release_u64(m.tile_off, kInc | tot);
                } else {
                    st_release_u64(m.tile_off + t, kAgg | tot);
                    for (unsigned long long q = t - 1;; --q) {
                        unsigned long long v;
                        while (((v = ld_acquire_u64(m.tile_off + q)) >> 62) == 0) {
                        }
                        excl += v & kVal;
                        if ((v >> 62) == 2) break;
                    }
                    st_release_u64(m.tile_off + t, kInc | (excl + tot));
                }
                if (t == m.ntiles - 1) m.tile_off[m.ntiles] = excl + tot;  // the union's size
                s_base = excl;
            }
            uint32_t q = pre + inc - keep;
            uint32_t i = i_start, j = e0 - i_start;
            for (uint32_t e = e0; e < e1; ++e) {
                if (j >= nb || (i < na && sa[i] <= sb[j])) {
                    if (sa[i] != sb[j]) s_src[q++] = i;
                    ++i;
                } else {
                    s_src[q++] = 0x80000000u | j;
                    ++j;
                }
            }
            if (tid == 0) {  // the union's entry just before this tile (none: ~0)
                const unsigned long long ap = i0 > 0 ? m.ia[i0 - 1] : ~0ull;
                const unsigned long long bp = j0 > 0 ? m.ib[j0 - 1] : ~0ull;
                // an a-entry equal to the b head at this tile's start (sb[0]: the tile's first b
                // or the one just past it) was dropped: its b twin comes later
                const unsigned long long aprev =
                    (ap != ~0ull && ap == sb[0]) ? (i0 > 1 ? m.ia[i0 - 2] : ~0ull) : ap;
                s_prev = aprev == ~0ull ? bp : (bp == ~0ull ? aprev : max(aprev, bp));
            }
            __syncthreads();
            const LT *va = static_cast<const LT *>(m.va), *vb = static_cast<const LT *>(m.vb);
            LT *uv = static_cast<LT *>(m.uv);
            const unsigned long long base = s_base;
            uint32_t lens[kMpTile / 256];
#pragma unroll
            for (int r = 0; r < kMpTile / 256; ++r) {
                const uint32_t x = tid + 256u * r;
                lens[r] = 0;
                if (x >= tot) continue;
                const uint32_t src = s_src[x], k = src & 0x7FFFFFFFu;
                const bool fb = src >> 31;
                const unsigned long long key = fb ? sb[k] : sa[k];
                m.u[base + x] = key;
                uv[base + x] = fb ? vb[j0 + k] : va[i0 + k];
                // fused M3: record start and the LEB128 length of the entry's gap
                unsigned long long prev = s_prev;
                if (x > 0) {
                    const uint32_t ps = s_src[x - 1], pk = ps & 0x7FFFFFFFu;
                    prev = (ps >> 31) ? sb[pk] : sa[pk];
                }
                const bool first = prev == ~0ull || (prev >> kKeyShift) != (key >> kKeyShift);
                if (first) m.eu[key >> kKeyShift] = base + x;
                lens[r] = leb_len(first ? (key & kIdxMask) : key - prev);
            }
            // the entries' byte offsets: block scan of the lengths (in sa's space, free now)
            // plus the tile's byte base from a second look-back; no separate scan pass
            __syncthreads();
            uint32_t *sl = reinterpret_cast<uint32_t *>(sa);
#pragma unroll
            for (int r = 0; r < kMpTile / 256; ++r) sl[tid + 256u * r] = lens[r];
            __syncthreads();
            uint32_t loc[8], run = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                loc[e] = run;
                run += sl[tid * 8 + e];
            }
            uint32_t binc = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, binc, o);
                if (lane >= o) binc += y;
            }
            __syncthreads();
            if (lane == 31) s_w[warp] = binc;
            __syncthreads();
            uint32_t bpre = 0, btot = 0;
            for (int w = 0; w < 8; ++w) {
                if (w < warp) bpre += s_w[w];
                btot += s_w[w];
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) sl[tid * 8 + e] = bpre + binc - run + loc[e];
            if (tid == 0) {
                constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = (1ull << 62) - 1;
                unsigned long long excl = 0;
                if (t == 0) {
                    st_release_u64(m.bstat, kInc | btot);
                } else {
                    st_release_u64(m.bstat + t, kAgg | btot);
                    for (unsigned long long q = t - 1;; --q) {
                        unsigned long long v;
                        while (((v = ld_acquire_u64(m.bstat + q)) >> 62) == 0) {
                        }
                        excl += v & kVal;
                        if ((v >> 62) == 2) break;
                    }
                    st_release_u64(m.bstat + t, kInc | (excl + btot));
                }
                if (t == m.ntiles - 1) m.lo[base + tot] = excl + btot;  // lo[union size] = total bytes
                s_bbase = excl;
            }
            __syncthreads();
            const unsigned long long bbase = s_bbase;
            for (uint32_t x = tid; x < tot; x += blockDim.x) m.lo[base + x] = bbase + sl[x];
        }
        __syncthreads();  // shared staging reused by the next tile
    }
}

// ---------------------------------------------------------------- M3
__global__ void k_merge_bounds_fill(MergeArgs m) {  // records without entries start where the next one does
    if (blockIdx.x || threadIdx.x) return;
    m.eu[m.n] = m.mu;
    for (uint32_t k = m.n; k-- > 0;)
        if (m.eu[k] == ~0ull) m.eu[k] = m.eu[k + 1];
}

// offset table + body size (one block)
__global__ void __launch_bounds__(1024) k_merge_table(MergeArgs m) {
    __shared__ unsigned long long s_w[32];
    unsigned long long carry = 0;
    for (uint32_t b = 0; b < m.n; b += 1024) {
        const uint32_t k = b + threadIdx.x;
        unsigned long long rb = 0, nnz = 0, il = 0;
        if (k < m.n) {
            nnz = m.eu[k + 1] - m.eu[k];
            il = m.lo[m.eu[k + 1]] - m.lo[m.eu[k]];
            rb = 27ull + m.name_len[k] + il + (unsigned long long)m.width * nnz;
        }
        unsigned long long tot;
        const unsigned long long ex = block_scan_excl(rb, s_w, tot);
        if (k < m.n) {
            RecordRow r;
            r.record_offset = carry + ex;
            r.element_count = m.numel[k];
            r.nnz = nnz;
            r.index_offset = r.record_offset + 2 + m.name_len[k] + 24;
            r.index_bytes = il;
            r.values_offset = r.index_offset + il;
            r.record_bytes = rb;
            m.table[k] = r;
        }
        carry += tot;
    }
    if (threadIdx.x == 0) *m.body_size = carry;
}

// ---------------------------------------------------------------- M4
template <int W>
__global__ void __launch_bounds__(256) k_merge_emit(MergeArgs m, uint8_t *__restrict__ out) {
    using LT = typename Lane<W>::T;
    const LT *uv = static_cast<const LT *>(m.uv);
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long p = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; p < m.mu; p += stride) {
        const unsigned long long k = m.u[p] >> kKeyShift, x = m.u[p] & kIdxMask;
        const RecordRow r = m.table[k];
        const unsigned long long e0 = m.eu[k];
        unsigned long long g = p == e0 ? x : x - (m.u[p - 1] & kIdxMask);
        uint8_t *q = out + r.index_offset + (m.lo[p] - m.lo[e0]);
        const uint32_t L = leb_len(g);
        for (uint32_t j = 0; j + 1 < L; ++j) {
            q[j] = (uint8_t)(g | 0x80);
            g >>= 7;
        }
        q[L - 1] = (uint8_t)g;
        const uint32_t v = uv[p];
        uint8_t *o = out + r.values_offset + (p - e0) * W;
#pragma unroll
        for (int b = 0; b < W; ++b) o[b] = (uint8_t)(v >> (8 * b));
    }
}

__global__ void __launch_bounds__(128) k_merge_headers(MergeArgs m, uint8_t *__restrict__ out) {
    for (uint32_t k = blockIdx.x; k < m.n; k += gridDim.x) {
        const RecordRow r = m.table[k];
        uint8_t *o = out + r.record_offset;
        const uint32_t nl = m.name_len[k];
        for (uint32_t b = threadIdx.x; b < nl; b += blockDim.x) o[2 + b] = m.b[m.name_off[k] + b];
        if (threadIdx.x == 0) {
            o[0] = (uint8_t)nl;
            o[1] = (uint8_t)(nl >> 8);
            for (int b = 0; b < 8; ++b) {
                o[2 + nl + b] = (uint8_t)(r.element_count >> (8 * b));
                o[2 + nl + 8 + b] = (uint8_t)(r.nnz >> (8 * b));
                o[2 + nl + 16 + b] = (uint8_t)(r.index_bytes >> (8 * b));
            }
            o[r.record_bytes - 1] = 0;  // replace mode
        }
    }
}

uint32_t grid_for(unsigned long long m) {
    const unsigned long long g = (m + 255) / 256;
    return (uint32_t)(g < 148ull * 16 ? (g ? g : 1) : 148ull * 16);
}

}  // namespace

cudaError_t launch_merge_walk(const MergeArgs &m, cudaStream_t s) {
    k_merge_walk<<<1, 32, 0, s>>>(m);
    if (m.n) k_merge_check<<<(m.n + 255) / 256, 256, 0, s>>>(m);
    return cudaGetLastError();
}

cudaError_t launch_merge_count(const MergeArgs &m, cudaStream_t s) {
    // splits, then the single merge-path pass (look-back offsets); tile_off[ntiles] = the
    // union's size.  tile_cnt[0..1] is the tile ticket, tile_off the look-back status.
    k_merge_splits<<<(uint32_t)((m.ntiles + 1 + 255) / 256), 256, 0, s>>>(m);
    cudaError_t e = cudaMemsetAsync(m.tile_off, 0, (size_t)(m.ntiles + 1) * 8, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(m.bstat, 0, (size_t)(m.ntiles + 1) * 8, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(m.tile_cnt, 0, 8, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(m.eu, 0xFF, (size_t)(m.n + 1) * 8, s);  // record starts
    if (e != cudaSuccess) return e;
    if (m.ntiles) {
        const uint32_t g = (uint32_t)(m.ntiles < 148ull * 8 ? m.ntiles : 148ull * 8);
        if (m.width == 2) k_merge_path<2, true><<<g, 256, 0, s>>>(m);
        else k_merge_path<4, true><<<g, 256, 0, s>>>(m);
    }
    return cudaGetLastError();
}

cudaError_t launch_merge_place(const MergeArgs &m, cudaStream_t s) {
    if (m.mu == 0) {  // no entry at all: lo[0] = 0 bytes
        cudaError_t e = cudaMemsetAsync(m.lo, 0, 8, s);
        if (e != cudaSuccess) return e;
    }
    k_merge_bounds_fill<<<1, 32, 0, s>>>(m);
    k_merge_table<<<1, 1024, 0, s>>>(m);
    return cudaGetLastError();
}

cudaError_t launch_merge_emit(const MergeArgs &m, uint8_t *out, cudaStream_t s) {
    if (m.mu) {
        if (m.width == 2) k_merge_emit<2><<<grid_for(m.mu), 256, 0, s>>>(m, out);
        else k_merge_emit<4><<<grid_for(m.mu), 256, 0, s>>>(m, out);
    }
    if (m.n) k_merge_headers<<<m.n < 65535u ? m.n : 65535u, 128, 0, s>>>(m, out);
    return cudaGetLastError();
}

}  // namespace sd
