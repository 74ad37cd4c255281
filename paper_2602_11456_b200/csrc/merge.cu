// merge.cu — sm_100a kernels for delta_merge (NEXT f4, reading R19): the delta
// D_a (v-1 -> v) followed by D_b (v -> v+1) as ONE delta (v-1 -> v+1) for a laggard's
// catch-up ("laggards catch up asynchronously"; SPEC.md:476 leaves merging
// open).  Per tensor: the union of the two index sets, D_b's value where D_b has the
// index, else D_a's — applying the merge equals applying D_a then D_b.
//
//   M1 k_merge_walk     one thread walks both bodies' record headers in order: layout,
//                       mode byte (replace only), names and element counts equal pairwise;
//                       entry prefixes E_a, E_b; apply targets (B's names) for the decodes.
//   (decode)            each body through A1-A3 + k_decode_write (apply.cu): validated,
//                       absolute indices + values per entry.
//   M2 k_merge_rank     per a-entry: lower bound in its b-segment and duplicate flag;
//                       exclusive scan of the flags; per-record union sizes E_u.
//   M3 k_merge_place    rank-based merge: a-entry i (not a duplicate) lands at
//                       E_u + i' + lb(i) - dups before i; b-entry j at E_u + j' + lb_a(b_j) -
//                       dups among a-entries below b_j.  Then LEB128 lengths of the union's
//                       gaps, their exclusive scan, the offset table and the body size.
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

// largest k in [0, n) with e[k] <= i (e ascending, e[0] = 0 <= i)
__device__ __forceinline__ uint32_t record_of(const unsigned long long *e, uint32_t n, unsigned long long i) {
    uint32_t lo = 0, hi = n;  // e[lo] <= i < e[hi] (e[n] = total > i)
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (e[mid] <= i) lo = mid;
        else hi = mid;
    }
    return lo;
}

// number of elements of the ascending array s[0, n) that are < x
__device__ __forceinline__ unsigned long long lower_bound(const unsigned long long *s, unsigned long long n,
                                                          unsigned long long x) {
    unsigned long long lo = 0, hi = n;
    while (lo < hi) {
        const unsigned long long mid = (lo + hi) >> 1;
        if (s[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------- exclusive scan u32 -> u64
constexpr int kScanPer = 4096;  // elements per block (1024 threads x 4)

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

__global__ void __launch_bounds__(1024) k_scan_reduce(const uint32_t *__restrict__ x, unsigned long long m,
                                                      unsigned long long *__restrict__ blk) {
    __shared__ unsigned long long s_w[32];
    const unsigned long long i0 = (unsigned long long)blockIdx.x * kScanPer + threadIdx.x * 4;
    unsigned long long v = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if (i0 + e < m) v += x[i0 + e];
    unsigned long long tot;
    block_scan_excl(v, s_w, tot);
    if (threadIdx.x == 0) blk[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_blocks(unsigned long long *__restrict__ blk, uint32_t nblk) {
    __shared__ unsigned long long s_w[32];
    unsigned long long carry = 0;
    for (uint32_t b = 0; b < nblk; b += 1024) {
        const uint32_t i = b + threadIdx.x;
        const unsigned long long v = i < nblk ? blk[i] : 0;
        unsigned long long tot;
        const unsigned long long ex = block_scan_excl(v, s_w, tot);
        if (i < nblk) blk[i] = carry + ex;
        carry += tot;
    }
}

__global__ void __launch_bounds__(1024) k_scan_down(const uint32_t *__restrict__ x, unsigned long long m,
                                                    const unsigned long long *__restrict__ blk,
                                                    unsigned long long *__restrict__ y) {
    __shared__ unsigned long long s_w[32];
    const unsigned long long i0 = (unsigned long long)blockIdx.x * kScanPer + threadIdx.x * 4;
    uint32_t v[4];
    unsigned long long mine = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        v[e] = i0 + e < m ? x[i0 + e] : 0u;
        mine += v[e];
    }
    unsigned long long tot;
    unsigned long long ex = block_scan_excl(mine, s_w, tot) + blk[blockIdx.x];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (i0 + e < m) y[i0 + e] = ex;
        if (i0 + e == m - 1) y[m] = ex + v[e];
        ex += v[e];
    }
}

cudaError_t scan_u32(const uint32_t *x, unsigned long long m, unsigned long long *y, unsigned long long *blk,
                     cudaStream_t s) {
    if (m == 0) return cudaMemsetAsync(y, 0, 8, s);
    const uint32_t nblk = (uint32_t)((m + kScanPer - 1) / kScanPer);
    k_scan_reduce<<<nblk, 1024, 0, s>>>(x, m, blk);
    k_scan_blocks<<<1, 1024, 0, s>>>(blk, nblk);
    k_scan_down<<<nblk, 1024, 0, s>>>(x, m, blk, y);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- M1
// One thread: both bodies' record headers in order (the bodies are untrusted: every read
// is bounds-checked).  Decoding errors are left to the decode passes.
__global__ void k_merge_walk(MergeArgs m) {
    if (blockIdx.x || threadIdx.x) return;
    unsigned long long pa = 0, pb = 0, ea = 0, eb = 0;
    uint32_t st = kOk;
    for (uint32_t k = 0; k < m.n && st == kOk; ++k) {
        unsigned long long hdr[2][5];  // name_len, N, nnz, ilen, end
        const uint8_t *bodies[2] = {m.a, m.b};
        const unsigned long long sizes[2] = {m.a_bytes, m.b_bytes}, pos[2] = {pa, pb};
        for (int x = 0; x < 2 && st == kOk; ++x) {
            const uint8_t *B = bodies[x];
            const unsigned long long sz = sizes[x], ro = pos[x];
            if (ro > sz || sz - ro < 2) { st = kLayout; break; }
            const unsigned long long nl = rd_u(B + ro, 2);
            if (sz - ro - 2 < nl + 24) { st = kLayout; break; }
            const unsigned long long q = ro + 2 + nl;
            const unsigned long long N = rd_u(B + q, 8), nnz = rd_u(B + q + 8, 8), il = rd_u(B + q + 16, 8);
            const unsigned long long rem = sz - q - 24;
            if (il > rem || nnz > (rem - il) / (unsigned long long)m.width || rem - il - nnz * m.width < 1) {
                st = kLayout;
                break;
            }
            const unsigned long long end = q + 24 + il + nnz * m.width + 1;
            if (B[end - 1] != 0) { st = kMode; break; }  // replace-mode records only
            hdr[x][0] = nl; hdr[x][1] = N; hdr[x][2] = nnz; hdr[x][3] = il; hdr[x][4] = end;
        }
        if (st != kOk) break;
        if (hdr[0][0] != hdr[1][0]) { st = kName; break; }
        for (unsigned long long j = 0; j < hdr[0][0]; ++j)
            if (m.a[pa + 2 + j] != m.b[pb + 2 + j]) { st = kName; break; }
        if (st != kOk) break;
        if (hdr[0][1] != hdr[1][1]) { st = kNumel; break; }
        m.targets[k] = TargetDesc{nullptr, hdr[1][1], pb + 2, hdr[1][0]};
        m.name_len[k] = (uint32_t)hdr[1][0];
        m.name_off[k] = pb + 2;
        m.numel[k] = hdr[1][1];
        m.ea[k] = ea;
        m.eb[k] = eb;
        ea += hdr[0][2];
        eb += hdr[1][2];
        pa = hdr[0][4];
        pb = hdr[1][4];
    }
    if (st == kOk && (pa != m.a_bytes || pb != m.b_bytes)) st = kLayout;
    m.ea[m.n] = ea;
    m.eb[m.n] = eb;
    *m.status = st;
}

// ---------------------------------------------------------------- M2
__global__ void __launch_bounds__(256) k_merge_rank(MergeArgs m) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m.ma; i += stride) {
        const uint32_t k = record_of(m.ea, m.n, i);
        const unsigned long long a = m.ia[i], b0 = m.eb[k], nb = m.eb[k + 1] - b0;
        const unsigned long long l = lower_bound(m.ib + b0, nb, a);
        m.lb[i] = l;
        m.dup[i] = (l < nb && m.ib[b0 + l] == a) ? 1u : 0u;
    }
}

// per record: union size (one block; the record count is small)
__global__ void __launch_bounds__(1024) k_merge_union(MergeArgs m) {
    __shared__ unsigned long long s_w[32];
    unsigned long long carry = 0;
    for (uint32_t b = 0; b < m.n; b += 1024) {
        const uint32_t k = b + threadIdx.x;
        unsigned long long nu = 0;
        if (k < m.n) {
            const unsigned long long dups = m.ds[m.ea[k + 1]] - m.ds[m.ea[k]];
            nu = (m.ea[k + 1] - m.ea[k]) + (m.eb[k + 1] - m.eb[k]) - dups;
        }
        unsigned long long tot;
        const unsigned long long ex = block_scan_excl(nu, s_w, tot);
        if (k < m.n) m.eu[k] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) m.eu[m.n] = carry;
}

// ---------------------------------------------------------------- M3
template <int W>
__global__ void __launch_bounds__(256) k_merge_place(MergeArgs m) {
    using LT = typename Lane<W>::T;
    const LT *va = static_cast<const LT *>(m.va), *vb = static_cast<const LT *>(m.vb);
    LT *uv = static_cast<LT *>(m.uv);
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long t0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (unsigned long long i = t0; i < m.ma; i += stride) {
        if (m.dup[i]) continue;  // b's value wins
        const uint32_t k = record_of(m.ea, m.n, i);
        const unsigned long long a0 = m.ea[k];
        const unsigned long long p = m.eu[k] + (i - a0) + m.lb[i] - (m.ds[i] - m.ds[a0]);
        m.u[p] = m.ia[i];
        uv[p] = va[i];
    }
    for (unsigned long long j = t0; j < m.mb; j += stride) {
        const uint32_t k = record_of(m.eb, m.n, j);
        const unsigned long long a0 = m.ea[k], na = m.ea[k + 1] - a0, b = m.ib[j];
        const unsigned long long l = lower_bound(m.ia + a0, na, b);
        const unsigned long long p = m.eu[k] + (j - m.eb[k]) + l - (m.ds[a0 + l] - m.ds[a0]);
        m.u[p] = b;
        uv[p] = vb[j];
    }
}

// LEB128 length of every union entry's gap (first entry of a record: the index itself)
__global__ void __launch_bounds__(256) k_merge_len(MergeArgs m) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long p = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; p < m.mu; p += stride) {
        const uint32_t k = record_of(m.eu, m.n, p);
        const unsigned long long g = p == m.eu[k] ? m.u[p] : m.u[p] - m.u[p - 1];
        m.len[p] = leb_len(g);
    }
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
        const uint32_t k = record_of(m.eu, m.n, p);
        const RecordRow r = m.table[k];
        const unsigned long long e0 = m.eu[k];
        unsigned long long g = p == e0 ? m.u[p] : m.u[p] - m.u[p - 1];
        uint8_t *q = out + r.index_offset + (m.lo[p] - m.lo[e0]);
        const uint32_t L = m.len[p];
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
    return cudaGetLastError();
}

cudaError_t launch_merge_rank(const MergeArgs &m, cudaStream_t s) {
    if (m.ma) k_merge_rank<<<grid_for(m.ma), 256, 0, s>>>(m);
    cudaError_t e = scan_u32(m.dup, m.ma, m.ds, m.blk, s);
    if (e != cudaSuccess) return e;
    k_merge_union<<<1, 1024, 0, s>>>(m);
    return cudaGetLastError();
}

cudaError_t launch_merge_place(const MergeArgs &m, cudaStream_t s) {
    const unsigned long long mx = m.ma > m.mb ? m.ma : m.mb;
    if (mx) {
        if (m.width == 2) k_merge_place<2><<<grid_for(mx), 256, 0, s>>>(m);
        else k_merge_place<4><<<grid_for(mx), 256, 0, s>>>(m);
    }
    if (m.mu) k_merge_len<<<grid_for(m.mu), 256, 0, s>>>(m);
    cudaError_t e = scan_u32(m.len, m.mu, m.lo, m.blk, s);
    if (e != cudaSuccess) return e;
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
