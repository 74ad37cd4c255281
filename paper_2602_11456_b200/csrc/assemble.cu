// assemble.cu — S3 of SURVEY.md §8(e) as one kernel over NVLink peer memory.
//
//   k_assemble   copies this rank's packed body into the assembled body on the root GPU
//                with stores to the root's memory (CUDA IPC mapping over NVLink/NVSwitch).
//                The destination offset — the sum of the body sizes of the lower ranks — is
//                read on the device from the all-gathered sizes, so no host round trip sits
//                between the size exchange and the transfer.  Records are self-contained
//                and in list order (R4, R15): the concatenation of the rank bodies
//                in rank order IS the body of the whole tensor list.
//
// Product code; shares nothing with the test oracle.
#include <cstdint>
#include <cuda_runtime.h>

#include "sd_device.cuh"
#include "sd_internal.cuh"

namespace sd {

// Grid-wide copy of the body: 16-byte destination-aligned stores assembled from funnel-
// shifted 16-byte-aligned source words (the source is this rank's body, 16-byte aligned).
__global__ void __launch_bounds__(256)
k_assemble(const uint8_t *__restrict__ src, uint8_t *__restrict__ dst_base, unsigned long long capacity,
           const unsigned long long *__restrict__ sizes, uint32_t rank, uint32_t *status) {
    unsigned long long off = 0;
    bool bad = false;
    for (uint32_t q = 0; q < rank; ++q) {  // each size <= capacity: the sum cannot wrap
        bad |= sizes[q] > capacity;
        off += bad ? 0ull : sizes[q];
    }
    const unsigned long long n = sizes[rank];
    if (bad || n > capacity || off + n > capacity) {  // incl. ~0 sizes from a closed extract gate
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(status, 1u);
        return;
    }
    uint8_t *dst = dst_base + off;
    const unsigned long long gtid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
    const uint32_t head = (uint32_t)min(n, (unsigned long long)((16u - ((uintptr_t)dst & 15u)) & 15u));
    if (gtid < head) dst[gtid] = src[gtid];
    const unsigned long long rest = n - head, nv = rest >> 4;
    uint4 *d16 = reinterpret_cast<uint4 *>(dst + head);
    const uint32_t *s32 = reinterpret_cast<const uint32_t *>(src);
    const uint32_t q0 = head >> 2, sh = 8u * (head & 3u);
    for (unsigned long long j = gtid; j < nv; j += nthreads) {
        const unsigned long long q = q0 + 4 * j;
        const uint32_t a0 = __ldg(s32 + q), a1 = __ldg(s32 + q + 1), a2 = __ldg(s32 + q + 2),
                       a3 = __ldg(s32 + q + 3), a4 = __ldg(s32 + q + 4);
        uint4 o;
        o.x = __funnelshift_r(a0, a1, sh);
        o.y = __funnelshift_r(a1, a2, sh);
        o.z = __funnelshift_r(a2, a3, sh);
        o.w = __funnelshift_r(a3, a4, sh);
        d16[j] = o;
    }
    for (unsigned long long b = (nv << 4) + gtid; b < rest; b += nthreads) dst[head + b] = src[head + b];
}

cudaError_t launch_assemble(const uint8_t *src, uint8_t *dst, unsigned long long capacity,
                            const unsigned long long *sizes, uint32_t rank, uint32_t *status, int ctas,
                            cudaStream_t s) {
    k_assemble<<<ctas, 256, 0, s>>>(src, dst, capacity, sizes, rank, status);
    return cudaGetLastError();
}

}  // namespace sd
