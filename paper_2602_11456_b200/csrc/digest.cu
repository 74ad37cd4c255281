// digest.cu — BLAKE3-256 of the packed body on the GPU (NEXT f1; reading R10:
// the delta checkpoint's "integrity hash" is BLAKE3-256 of exactly the body
// bytes).
//
//   k_b3_chunks   one thread per 1 KiB chunk: up to 16 64-byte block compressions with the
//                 chunk counter, CHUNK_START / CHUNK_END flags -> the chunk's chaining value
//                 (ROOT on the last block when the whole input is one chunk).
//   k_b3_parents  one tree level: pairs of chaining values -> parent compressions (PARENT,
//                 ROOT for the final pair); an odd last value is carried up, which yields
//                 BLAKE3's left-balanced tree.
//
// BLAKE3 constants and the G / round structure are the public specification's; product
// code, shares nothing with the test oracle (which calls the `blake3` package).
#include <cstdint>
#include <cuda_runtime.h>

namespace sd {

__constant__ uint32_t kB3IV[8] = {0x6A09E667u, 0xBB67AE85u, 0x3C6EF372u, 0xA54FF53Au,
                                  0x510E527Fu, 0x9B05688Cu, 0x1F83D9ABu, 0x5BE0CD19u};
constexpr uint32_t kChunkStart = 1, kChunkEnd = 2, kParent = 4, kRoot = 8;

__device__ __forceinline__ uint32_t rotr(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

__device__ __forceinline__ void b3_g(uint32_t *s, int a, int b, int c, int d, uint32_t x, uint32_t y) {
    s[a] = s[a] + s[b] + x;
    s[d] = rotr(s[d] ^ s[a], 16);
    s[c] = s[c] + s[d];
    s[b] = rotr(s[b] ^ s[c], 12);
    s[a] = s[a] + s[b] + y;
    s[d] = rotr(s[d] ^ s[a], 8);
    s[c] = s[c] + s[d];
    s[b] = rotr(s[b] ^ s[c], 7);
}

// Compression: cv (8 words) x block (16 words) -> the first 8 output words (new cv).
__device__ __forceinline__ void b3_compress(const uint32_t *cv, const uint32_t *m_in, unsigned long long counter,
                                            uint32_t block_len, uint32_t flags, uint32_t *out) {
    uint32_t s[16] = {cv[0], cv[1], cv[2], cv[3], cv[4], cv[5], cv[6], cv[7],
                      kB3IV[0], kB3IV[1], kB3IV[2], kB3IV[3],
                      (uint32_t)counter, (uint32_t)(counter >> 32), block_len, flags};
    uint32_t m[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) m[i] = m_in[i];
#pragma unroll
    for (int r = 0; r < 7; ++r) {
        b3_g(s, 0, 4, 8, 12, m[0], m[1]);
        b3_g(s, 1, 5, 9, 13, m[2], m[3]);
        b3_g(s, 2, 6, 10, 14, m[4], m[5]);
        b3_g(s, 3, 7, 11, 15, m[6], m[7]);
        b3_g(s, 0, 5, 10, 15, m[8], m[9]);
        b3_g(s, 1, 6, 11, 12, m[10], m[11]);
        b3_g(s, 2, 7, 8, 13, m[12], m[13]);
        b3_g(s, 3, 4, 9, 14, m[14], m[15]);
        if (r < 6) {  // message permutation
            const uint32_t t[16] = {m[2], m[6], m[3], m[10], m[7], m[0], m[4], m[13],
                                    m[1], m[11], m[12], m[5], m[9], m[14], m[15], m[8]};
#pragma unroll
            for (int i = 0; i < 16; ++i) m[i] = t[i];
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) out[i] = s[i] ^ s[i + 8];
}

__global__ void __launch_bounds__(128)
k_b3_chunks(const uint8_t *__restrict__ in, unsigned long long n, unsigned long long nchunks,
            uint32_t *__restrict__ cvs) {
    const unsigned long long c = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    const unsigned long long base = c * 1024;
    const uint32_t len = (uint32_t)min(1024ull, n - min(n, base));
    const uint32_t nblocks = len == 0 ? 1 : (len + 63) / 64;
    uint32_t cv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) cv[i] = kB3IV[i];
    const bool aligned = ((reinterpret_cast<uintptr_t>(in) + base) & 3) == 0;
    for (uint32_t b = 0; b < nblocks; ++b) {
        const uint32_t off = b * 64;
        const uint32_t blen = min(64u, len - off);
        uint32_t m[16];
        if (aligned && blen == 64) {
            const uint32_t *p = reinterpret_cast<const uint32_t *>(in + base + off);
#pragma unroll
            for (int i = 0; i < 16; ++i) m[i] = __ldg(p + i);
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                uint32_t w = 0;
                for (int k = 0; k < 4; ++k) {
                    const uint32_t j = 4 * i + k;
                    if (j < blen) w |= (uint32_t)__ldg(in + base + off + j) << (8 * k);
                }
                m[i] = w;
            }
        }
        uint32_t flags = (b == 0 ? kChunkStart : 0u) | (b == nblocks - 1 ? kChunkEnd : 0u);
        if (b == nblocks - 1 && nchunks == 1) flags |= kRoot;
        b3_compress(cv, m, c, blen, flags, cv);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) cvs[c * 8 + i] = cv[i];
}

__global__ void __launch_bounds__(128)
k_b3_parents(const uint32_t *__restrict__ in, unsigned long long n, uint32_t *__restrict__ out) {
    const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long nout = (n + 1) / 2;
    if (i >= nout) return;
    if (2 * i + 1 < n) {
        uint32_t m[16], cv[8];
#pragma unroll
        for (int k = 0; k < 16; ++k) m[k] = in[2 * i * 8 + k];  // left cv || right cv
#pragma unroll
        for (int k = 0; k < 8; ++k) cv[k] = kB3IV[k];
        const uint32_t flags = kParent | (n == 2 ? kRoot : 0u);
        b3_compress(cv, m, 0, 64, flags, cv);
#pragma unroll
        for (int k = 0; k < 8; ++k) out[i * 8 + k] = cv[k];
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) out[i * 8 + k] = in[2 * i * 8 + k];  // odd value carried up
    }
}

// BLAKE3-256 of in[0..n) into out32 (device, 8 words, little-endian bytes); ws: 2 x
// ceil(n / 1024) x 32 bytes of scratch.
cudaError_t launch_blake3(const uint8_t *in, unsigned long long n, uint32_t *ws, uint32_t *out32,
                          cudaStream_t s) {
    const unsigned long long nch = n == 0 ? 1 : (n + 1023) / 1024;
    uint32_t *a = ws, *b = ws + nch * 8;
    k_b3_chunks<<<(unsigned)((nch + 127) / 128), 128, 0, s>>>(in, n, nch, a);
    unsigned long long m = nch;
    while (m > 1) {
        const unsigned long long nout = (m + 1) / 2;
        k_b3_parents<<<(unsigned)((nout + 127) / 128), 128, 0, s>>>(a, m, b);
        uint32_t *t = a;
        a = b;
        b = t;
        m = nout;
    }
    return cudaMemcpyAsync(out32, a, 32, cudaMemcpyDeviceToDevice, s);
}

// SPDC header (readings R9, R10, R18), written on the device from the digest the
// tree above left in `digest` (device, 32 bytes): "SPDC" | u16 format_version | u64 version |
// u64 base_version | u8 element code | u32 tensor count | u64 body length | 32-byte BLAKE3.
// 67 bytes, little-endian, to `out` (any alignment).
__global__ void k_spdc_header(uint8_t *out, const uint32_t *digest, uint32_t format_version,
                              unsigned long long version, unsigned long long base_version, uint32_t elem_code,
                              uint32_t n_tensors, unsigned long long body_bytes) {
    const int i = threadIdx.x;
    if (i >= 67) return;
    uint8_t b;
    auto le = [](unsigned long long x, int k) { return (uint8_t)(x >> (8 * k)); };
    if (i < 4) b = (uint8_t)"SPDC"[i];
    else if (i < 6) b = le(format_version, i - 4);
    else if (i < 14) b = le(version, i - 6);
    else if (i < 22) b = le(base_version, i - 14);
    else if (i < 23) b = (uint8_t)elem_code;
    else if (i < 27) b = le(n_tensors, i - 23);
    else if (i < 35) b = le(body_bytes, i - 27);
    else b = (uint8_t)(digest[(i - 35) >> 2] >> (8 * ((i - 35) & 3)));
    out[i] = b;
}

cudaError_t launch_spdc_header(uint8_t *out, const uint32_t *digest, uint32_t format_version,
                               unsigned long long version, unsigned long long base_version, uint32_t elem_code,
                               uint32_t n_tensors, unsigned long long body_bytes, cudaStream_t s) {
    k_spdc_header<<<1, 96, 0, s>>>(out, digest, format_version, version, base_version, elem_code, n_tensors,
                                   body_bytes);
    return cudaGetLastError();
}

}  // namespace sd
