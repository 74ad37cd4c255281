// sd_device.cuh — small sm_100a device helpers (memory-order loads/stores, streaming loads,
// LEB128 length).  Product code.
#pragma once
#include <cstdint>

namespace sd {

// Streaming 128-bit load of data read exactly once: non-coherent path, no L1 allocation.
__device__ __forceinline__ uint4 ld_stream_v4(const void *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// Coherent 128-bit load without L1 allocation, for data the same kernel later writes
// (the extract-and-advance compare kernel stores new lanes into the old buffer).
__device__ __forceinline__ uint4 ld_noalloc_v4(const void *p) {
    uint4 v;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Number of bytes of the unsigned LEB128 encoding of g: 1 + #{t in 7,14,..,63 : g >= 2^t}.
__device__ __forceinline__ uint32_t leb_len(unsigned long long g) {
    // bits needed (at least 1), then ceil(bits / 7)
    uint32_t bits = 64 - __clzll(g | 1ull);
    return (bits + 6) / 7;
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ unsigned long long sat_add(unsigned long long a, unsigned long long b) {
    unsigned long long s = a + b;
    return s < a ? ~0ull : s;
}

}  // namespace sd

// ---------------------------------------------------------------- additive-mode lane arithmetic
// (R17): 16-bit lanes are bf16, 32-bit lanes fp32; arithmetic in
// fp32 (IEEE, round to nearest even), bf16 results rounded to nearest even, NaN results
// canonical (0x7FC0 / 0x7FC00000).
namespace sd {

__device__ __forceinline__ uint32_t f32_to_bf16_rne(float f) {
    const uint32_t b = __float_as_uint(f);
    if ((b & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FC0u;
    return (b + 0x7FFFu + ((b >> 16) & 1u)) >> 16;
}

template <int W>
__device__ __forceinline__ uint32_t lane_combine(uint32_t a, uint32_t b, bool subtract) {
    if constexpr (W == 2) {
        const float fa = __uint_as_float(a << 16), fb = __uint_as_float(b << 16);
        return f32_to_bf16_rne(subtract ? __fsub_rn(fa, fb) : __fadd_rn(fa, fb));
    } else {
        const float r = subtract ? __fsub_rn(__uint_as_float(a), __uint_as_float(b))
                                 : __fadd_rn(__uint_as_float(a), __uint_as_float(b));
        return (__float_as_uint(r) & 0x7FFFFFFFu) > 0x7F800000u ? 0x7FC00000u : __float_as_uint(r);
    }
}

}  // namespace sd

// ---------------------------------------------------------------- bulk L2 prefetch (TMA engine)
namespace sd {

// Bulk prefetch of [src, src + bytes) into L2 (TMA engine; no registers, no shared
// memory, no completion to wait for).  src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

}  // namespace sd
