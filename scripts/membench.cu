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
    else k_scatter_sector<<<grid, block, 0, s>>>(W, P, V, n);
    return (int)cudaGetLastError();
}
}
