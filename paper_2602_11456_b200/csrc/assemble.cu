// assemble.cu — S3 of SURVEY.md §8(e) as one kernel over NVLink peer memory.
//
//   k_assemble   copies this rank's packed body into the assembled body on the root GPU
//                with stores to the root's memory (CUDA IPC mapping over NVLink/NVSwitch).
//                The destination offset — the sum of the body sizes of the lower ranks — is
//                read on the device from the all-gathered sizes, so no host round trip sits
//                between the size exchange and the transfer.  Records are self-contained
//                and in list order (R4, R15): the concatenation of the rank bodies
//                in rank order IS the body of the whole tensor list.
//   k_record_sizes / k_record_offsets / k_assemble_records
//                the same for any tensor partition (LPT): each record to its own global
//                offset, computed on the device from the all-reduced record sizes.
// The default multi-GPU path no longer runs a separate copy: K4/K5 store each rank's records
// at their global offsets directly (delta_extract_emit_async with a peer destination).
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

// ---------------------------------------------------------------- record-granular assembly
// With a non-contiguous partition (LPT) a rank's records are not one
// byte range of the global body: every record goes to its own global offset.  Protocol:
// k_record_sizes scatters this rank's record sizes (its offset table) into a global-order
// array (zeros elsewhere) on the extract's stream; the caller sums that array over the
// ranks (one NCCL all-reduce); k_record_offsets turns it into global offsets (and this
// rank's local offsets); k_assemble_records copies each local record to its global offset.
__global__ void __launch_bounds__(256)
k_record_sizes(const RecordRow *__restrict__ table, uint32_t n_local, const uint32_t *__restrict__ gidx,
               unsigned long long *__restrict__ sizes, uint32_t n_global) {
    for (uint32_t k = threadIdx.x; k < n_global; k += blockDim.x) sizes[k] = 0;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < n_local; j += blockDim.x) sizes[gidx[j]] = table[j].record_bytes;
}

// One block: exclusive scans of the global sizes (global offsets, total at [n_global]) and
// of this rank's record sizes in local order (local body offsets).
__global__ void __launch_bounds__(1024)
k_record_offsets(const unsigned long long *__restrict__ sizes, uint32_t n_global, const uint32_t *__restrict__ gidx,
                 uint32_t n_local, unsigned long long *__restrict__ goff, unsigned long long *__restrict__ loff) {
    __shared__ unsigned long long s_w[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int pass = 0; pass < 2; ++pass) {
        const uint32_t n = pass ? n_local : n_global;
        unsigned long long *out = pass ? loff : goff;
        unsigned long long carry = 0;
        for (uint32_t b = 0; b < n; b += 1024) {
            const uint32_t i = b + threadIdx.x;
            const unsigned long long v = i < n ? sizes[pass ? gidx[i] : i] : 0ull;
            unsigned long long inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) s_w[warp] = inc;
            __syncthreads();
            unsigned long long pre = 0, tot = 0;
            for (int w = 0; w < 32; ++w) {
                if (w < warp) pre += s_w[w];
                tot += s_w[w];
            }
            __syncthreads();
            if (i < n) out[i] = carry + pre + inc - v;
            carry += tot;
        }
        if (threadIdx.x == 0) out[n] = carry;
        __syncthreads();
    }
}

// Every CTA takes its grid-stride share of every local record: 16-byte destination-aligned
// stores assembled from funnel-shifted 4-byte source words (any source alignment; reads at
// most 3 bytes before and 4 bytes after a record, inside the padded body buffer).
__global__ void __launch_bounds__(256)
k_assemble_records(const uint8_t *__restrict__ src, uint8_t *__restrict__ dst, unsigned long long capacity,
                   const unsigned long long *__restrict__ sizes, const uint32_t *__restrict__ gidx, uint32_t n_local,
                   uint32_t n_global, const unsigned long long *__restrict__ goff,
                   const unsigned long long *__restrict__ loff, uint32_t *status) {
    if (goff[n_global] > capacity) {  // incl. ~0 sizes from a closed extract gate
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(status, 1u);
        return;
    }
    const unsigned long long gtid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
    for (uint32_t j = 0; j < n_local; ++j) {
        const uint32_t k = gidx[j];
        const unsigned long long n = sizes[k];
        const uint8_t *s = src + loff[j];
        uint8_t *d = dst + goff[k];
        const uint32_t head = (uint32_t)min(n, (unsigned long long)((16u - ((uintptr_t)d & 15u)) & 15u));
        if (gtid < head) d[gtid] = s[gtid];
        const unsigned long long rest = n - head, nv = rest >> 4;
        const uint8_t *sh0 = s + head;
        const uint32_t *w = reinterpret_cast<const uint32_t *>(reinterpret_cast<uintptr_t>(sh0) & ~uintptr_t(3));
        const uint32_t sh = 8u * (uint32_t)(reinterpret_cast<uintptr_t>(sh0) & 3u);
        uint4 *d16 = reinterpret_cast<uint4 *>(d + head);
        for (unsigned long long v = gtid; v < nv; v += nthreads) {
            const uint32_t *q = w + 4 * v;
            const uint32_t a0 = __ldg(q), a1 = __ldg(q + 1), a2 = __ldg(q + 2), a3 = __ldg(q + 3), a4 = __ldg(q + 4);
            uint4 o;
            o.x = __funnelshift_r(a0, a1, sh);
            o.y = __funnelshift_r(a1, a2, sh);
            o.z = __funnelshift_r(a2, a3, sh);
            o.w = __funnelshift_r(a3, a4, sh);
            d16[v] = o;
        }
        for (unsigned long long b = (nv << 4) + gtid; b < rest; b += nthreads) d[head + b] = sh0[b];
    }
}

cudaError_t launch_record_sizes(const RecordRow *table, uint32_t n_local, const uint32_t *gidx,
                                unsigned long long *sizes, uint32_t n_global, cudaStream_t s) {
    k_record_sizes<<<1, 256, 0, s>>>(table, n_local, gidx, sizes, n_global);
    return cudaGetLastError();
}

cudaError_t launch_assemble_records(const uint8_t *src, uint8_t *dst, unsigned long long capacity,
                                    const unsigned long long *sizes, const uint32_t *gidx, uint32_t n_local,
                                    uint32_t n_global, unsigned long long *goff, unsigned long long *loff,
                                    uint32_t *status, int ctas, cudaStream_t s) {
    k_record_offsets<<<1, 1024, 0, s>>>(sizes, n_global, gidx, n_local, goff, loff);
    k_assemble_records<<<ctas, 256, 0, s>>>(src, dst, capacity, sizes, gidx, n_local, n_global, goff, loff, status);
    return cudaGetLastError();
}

cudaError_t launch_assemble(const uint8_t *src, uint8_t *dst, unsigned long long capacity,
                            const unsigned long long *sizes, uint32_t rank, uint32_t *status, int ctas,
                            cudaStream_t s) {
    k_assemble<<<ctas, 256, 0, s>>>(src, dst, capacity, sizes, rank, status);
    return cudaGetLastError();
}

}  // namespace sd
