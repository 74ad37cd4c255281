// membench.cu — microbenchmarks that calibrate the design (not part of the product):
//   read      : streaming 16-byte loads of a large buffer (XOR-reduced), the read roofline
//   scatter_* : sorted random 2-byte stores at density rho into a large buffer, variants:
//       plain    one thread per entry, st.global.u16
//       pf       prefetch.global.L2 of a batch of targets, then the stores
//       sector   read the full 32-byte sector, merge the lanes, write the full sector
// Built by scripts/membench.py with nvcc -arch sm_100a into scripts/libmembench.so.
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_read(const uint4 *__restrict__ p, size_t n16, unsigned long long *out) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 a, b, c, d;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(p + i));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p + i + stride));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "l"(p + i + 2 * stride));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(d.x), "=r"(d.y), "=r"(d.z), "=r"(d.w) : "l"(p + i + 3 * stride));
        acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
    }
    for (; i < n16; i += stride) {
        uint4 a = p[i];
        acc ^= a.x ^ a.y ^ a.z ^ a.w;
    }
    if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

__global__ void k_scatter_plain(uint16_t *w, const unsigned long long *pos, const uint16_t *val, size_t n) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) w[pos[i]] = val[i];
}

// each thread handles a run of 16 consecutive entries: prefetch all 16 targets, then store
__global__ void k_scatter_pf(uint16_t *w, const unsigned long long *pos, const uint16_t *val, size_t n) {
    const size_t nt = (n + 15) / 16;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += stride) {
        const size_t b = t * 16, e = b + 16 < n ? b + 16 : n;
        for (size_t i = b; i < e; ++i) asm volatile("prefetch.global.L2 [%0];" ::"l"(w + pos[i]));
        for (size_t i = b; i < e; ++i) w[pos[i]] = val[i];
    }
}

// sector merge: one thread per entry run; entries sharing a 32-byte sector are merged
__global__ void k_scatter_sector(uint16_t *w, const unsigned long long *pos, const uint16_t *val, size_t n) {
    const size_t nt = (n + 15) / 16;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += stride) {
        const size_t b = t * 16, e = b + 16 < n ? b + 16 : n;
        size_t i = b;
        while (i < e) {
            const unsigned long long sec = pos[i] >> 4;  // 16 lanes per 32-byte sector
            uint4 *sp = reinterpret_cast<uint4 *>(w + (sec << 4));
            uint4 lo = sp[0], hi = sp[1];
            uint16_t *l = reinterpret_cast<uint16_t *>(&lo);
            uint16_t *h = reinterpret_cast<uint16_t *>(&hi);
            while (i < e && (pos[i] >> 4) == sec) {
                const int j = (int)(pos[i] & 15);
                if (j < 8) l[j] = val[i];
                else h[j - 8] = val[i];
                ++i;
            }
            sp[0] = lo;
            sp[1] = hi;
        }
    }
}

// v3 warp-batched sector read-modify-write: a warp takes 256 consecutive entries, loads
// every 32-byte sector they touch with lane-pair 16-byte loads (several in flight), merges
// the lanes in shared memory and writes the sectors back whole (lane pairs: full-sector
// writes, no L2 fill).  The run's first / last sectors may be shared with the neighbouring
// runs: those entries are stored lane-wise.  HINT 1: loads evict_first / stores evict_first.
template <int HINT>
__global__ void __launch_bounds__(128) k_scatter_batch(uint16_t *w, const unsigned long long *pos, const uint16_t *val, size_t n) {
    __shared__ uint4 s_sec[4][256][2];
    __shared__ unsigned long long s_addr[4][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t nrun = (n + 255) / 256;
    const size_t nw = (size_t)gridDim.x * 4;
    const uint32_t le = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
    for (size_t r = (size_t)blockIdx.x * 4 + warp; r < nrun; r += nw) {
        const size_t b = r * 256, e = b + 256 < n ? b + 256 : n;
        const unsigned long long fs = pos[b] >> 4, ls = pos[e - 1] >> 4;
        unsigned long long sec[8];
        uint16_t v[8];
        uint32_t rank[8];
        uint32_t off[8];
        bool inter[8];
        uint32_t base = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const size_t i = b + 32 * j + lane;
            const bool act = i < e;
            const unsigned long long p = act ? pos[i] : ~0ull;
            v[j] = act ? val[i] : 0;
            sec[j] = p >> 4;
            off[j] = (uint32_t)(p & 15);
            unsigned long long ps = __shfl_up_sync(0xffffffffu, sec[j], 1);
            const unsigned long long carry = __shfl_sync(0xffffffffu, sec[j ? j - 1 : 0], 31);
            if (lane == 0) ps = j ? carry : ~0ull;
            inter[j] = act && sec[j] != fs && sec[j] != ls;
            const bool lead = inter[j] && sec[j] != ps;
            const uint32_t bal = __ballot_sync(0xffffffffu, lead);
            rank[j] = base + __popc(bal & le) - 1;
            if (lead) s_addr[warp][rank[j]] = sec[j];
            base += __popc(bal);
            if (act && !inter[j]) w[p] = v[j];
        }
        __syncwarp();
        const uint32_t nl = base;
        for (uint32_t q0 = 0; q0 < nl; q0 += 64) {
            uint4 t[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t q = q0 + 16 * k + (lane >> 1);
                if (q < nl) {
                    const uint4 *src = reinterpret_cast<const uint4 *>(w + (s_addr[warp][q] << 4)) + (lane & 1);
                    if (HINT) asm volatile("ld.global.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(t[k].x), "=r"(t[k].y), "=r"(t[k].z), "=r"(t[k].w) : "l"(src));
                    else t[k] = *src;
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t q = q0 + 16 * k + (lane >> 1);
                if (q < nl) s_sec[warp][q][lane & 1] = t[k];
            }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (inter[j]) reinterpret_cast<uint16_t *>(&s_sec[warp][rank[j]][0])[off[j]] = v[j];
        __syncwarp();
        for (uint32_t q = lane >> 1; q < nl; q += 16)
            reinterpret_cast<uint4 *>(w + (s_addr[warp][q] << 4))[lane & 1] = s_sec[warp][q][lane & 1];
        __syncwarp();
    }
}

// v5/v6: plain one-thread-per-entry stores with an L2 eviction-priority policy
template <int POL>
__global__ void k_scatter_hint(uint16_t *w, const unsigned long long *pos, const uint16_t *val, size_t n) {
    unsigned long long pol;
    if (POL == 0) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const unsigned short x = val[i];
        asm volatile("st.global.L2::cache_hint.u16 [%0], %1, %2;" ::"l"(w + pos[i]), "h"(x), "l"(pol) : "memory");
    }
}

// v7: plain, one warp per 32 consecutive entries but the grid sweeps the entries in narrow
// windows: CTA b handles entries [k*S + b*256, ...) for k = 0.. (S = grid*256) — same as plain
// with a grid of 148 CTAs (small window in flight)

// v7: windowed plain stores — the whole grid sweeps the entries together: warp w of W handles
// entries [(k W + w) 32, +32) at iteration k, so the stores in flight span ~W x 32 entries of
// address space (the DRAM row-locality window); UNROLL iterations' loads are issued first.
template <int UNROLL>
__global__ void __launch_bounds__(256) k_scatter_window(uint16_t *w, const unsigned long long *pos, const uint16_t *val, size_t n) {
    const int lane = threadIdx.x & 31;
    const size_t W = (size_t)gridDim.x * (blockDim.x >> 5);
    const size_t wid = (size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (size_t k = 0;; k += UNROLL) {
        unsigned long long p[UNROLL];
        uint16_t v[UNROLL];
        bool any = false;
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const size_t i = ((k + u) * W + wid) * 32 + lane;
            p[u] = i < n ? pos[i] : ~0ull;
            v[u] = i < n ? val[i] : 0;
            any |= ((k + u) * W + wid) * 32 < n;
        }
        if (!__any_sync(0xffffffffu, any)) break;
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
            if (p[u] != ~0ull) w[p[u]] = v[u];
    }
}

// v8: read-only gather of the same lanes (the L2 fills alone): XOR of w[pos[i]]
__global__ void __launch_bounds__(256) k_gather(const uint16_t *w, const unsigned long long *pos, size_t n, unsigned long long *out) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) acc ^= w[pos[i]];
    if (acc == 0x12345u) atomicAdd(out, 1ull);
}

// v9: full 32-byte sector writes of every touched sector (the write-backs alone, no fill):
// thread pair (2j, 2j+1) writes the two 16-byte halves of sector sec[j]
__global__ void __launch_bounds__(256) k_sector_write(uint16_t *w, const unsigned long long *sec, size_t ns) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < 2 * ns; t += stride) {
        uint4 *p = reinterpret_cast<uint4 *>(w + (sec[t >> 1] << 4)) + (t & 1);
        *p = make_uint4((uint32_t)t, 1u, 2u, 3u);
    }
}

// v10: full 32-byte sector read of every touched sector (the fills as whole-sector loads)
__global__ void __launch_bounds__(256) k_sector_read(const uint16_t *w, const unsigned long long *sec, size_t ns, unsigned long long *out) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < 2 * ns; t += stride) {
        const uint4 x = *(reinterpret_cast<const uint4 *>(w + (sec[t >> 1] << 4)) + (t & 1));
        acc ^= x.x ^ x.y ^ x.z ^ x.w;
    }
    if (acc == 0x12345u) atomicAdd(out, 1ull);
}

extern "C" {
int mb_read(const void *p, size_t bytes, void *out, int grid, int block, cudaStream_t s) {
    k_read<<<grid, block, 0, s>>>(static_cast<const uint4 *>(p), bytes / 16, static_cast<unsigned long long *>(out));
    return (int)cudaGetLastError();
}
int mb_scatter(int variant, void *w, const void *pos, const void *val, size_t n, int grid, int block, cudaStream_t s) {
    auto W = static_cast<uint16_t *>(w);
    auto P = static_cast<const unsigned long long *>(pos);
    auto V = static_cast<const uint16_t *>(val);
    if (variant == 0) k_scatter_plain<<<grid, block, 0, s>>>(W, P, V, n);
    else if (variant == 1) k_scatter_pf<<<grid, block, 0, s>>>(W, P, V, n);
    else if (variant == 2) k_scatter_sector<<<grid, block, 0, s>>>(W, P, V, n);
    else if (variant == 3) k_scatter_batch<0><<<grid, 128, 0, s>>>(W, P, V, n);
    else if (variant == 4) k_scatter_batch<1><<<grid, 128, 0, s>>>(W, P, V, n);
    else if (variant == 5) k_scatter_hint<0><<<grid, block, 0, s>>>(W, P, V, n);
    else if (variant == 6) k_scatter_hint<1><<<grid, block, 0, s>>>(W, P, V, n);
    else if (variant == 7) k_scatter_window<4><<<grid, block, 0, s>>>(W, P, V, n);
    else if (variant == 8) k_scatter_window<1><<<grid, block, 0, s>>>(W, P, V, n);
    return (int)cudaGetLastError();
}

int mb_gather(const void *w, const void *pos, size_t n, void *out, int grid, int block, cudaStream_t s) {
    k_gather<<<grid, block, 0, s>>>(static_cast<const uint16_t *>(w), static_cast<const unsigned long long *>(pos), n,
                                    static_cast<unsigned long long *>(out));
    return (int)cudaGetLastError();
}
int mb_sector(int write, void *w, const void *sec, size_t ns, void *out, int grid, int block, cudaStream_t s) {
    if (write) k_sector_write<<<grid, block, 0, s>>>(static_cast<uint16_t *>(w), static_cast<const unsigned long long *>(sec), ns);
    else k_sector_read<<<grid, block, 0, s>>>(static_cast<const uint16_t *>(w), static_cast<const unsigned long long *>(sec), ns,
                                             static_cast<unsigned long long *>(out));
    return (int)cudaGetLastError();
}
}
