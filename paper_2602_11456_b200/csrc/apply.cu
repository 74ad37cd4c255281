// apply.cu — sm_100a kernels for delta application.
//
//   A1 k_locate        header walk: find every record, check it fits the body, its mode
//                      byte, its name and element count against the target.
//                      With a table hint all records are verified in one parallel pass;
//                      otherwise (or if any hint field disagrees with the body) one thread
//                      walks the records in order.
//   A2 k_decode_count  parallel LEB128 decode of 4 KiB index-stream chunks: terminator
//                      bytes (MSB clear) end an entry; each entry is decoded by reading
//                      back from its terminator; strict checks (truncated, overlong,
//                      > 64-bit, zero gap after the first, gap >= N); per-chunk entry count
//                      and gap sum.
//   A3 k_apply_scan    per record: scan of chunk (count, gap sum) -> each chunk's ordinal
//                      and index base; count == nnz and last index < N.
//   A4 k_scatter       gated on the device status word (all-or-nothing):
//                      decode again, absolute index = base + running gap sum, value read
//                      from the record's value array, W[index] = value (replace mode, R1);
//                      dense chunks rewrite whole 16-byte vectors of the chunk's window.
//
// Product code; shares nothing with oracle/.
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "sd_device.cuh"
#include "sd_internal.cuh"

namespace sd {

__device__ __forceinline__ void set_status(ApplyState *st, uint32_t code) {
    atomicCAS(&st->status, 0u, code);
}

__device__ __forceinline__ unsigned long long rd_le(const uint8_t *p, int nbytes) {
    unsigned long long x = 0;
    if (nbytes == 8) {  // all eight loads in flight at once
        uint8_t b[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) b[i] = p[i];
#pragma unroll
        for (int i = 0; i < 8; ++i) x |= (unsigned long long)b[i] << (8 * i);
        return x;
    }
    for (int b = 0; b < nbytes; ++b) x |= (unsigned long long)p[b] << (8 * b);
    return x;
}

// ------------------------------------------------------------------------------ A1
// Checks one record header at `ro` against target k; returns a status code and the
// record's geometry.  Bounds are checked before every read (the body is untrusted).
__device__ uint32_t check_record(const uint8_t *body, unsigned long long body_bytes,
                                 unsigned long long ro, const TargetDesc &tg,
                                 const uint8_t *names, int width, int fixed, ApplyRec &rec,
                                 unsigned long long &end) {
    if (ro > body_bytes || body_bytes - ro < 2) return kLayout;
    const unsigned long long nl = rd_le(body + ro, 2);
    if (body_bytes - ro - 2 < nl + 24) return kLayout;
    const unsigned long long p = ro + 2 + nl;
    const unsigned long long N = rd_le(body + p, 8);
    const unsigned long long nnz = rd_le(body + p + 8, 8);
    const unsigned long long ilen = rd_le(body + p + 16, 8);
    const unsigned long long q = p + 24;
    const unsigned long long rem = body_bytes - q;
    if (ilen > rem || nnz > (rem - ilen) / (unsigned long long)width) return kLayout;
    end = q + ilen + nnz * width + 1;
    if (end > body_bytes) return kLayout;
    const uint8_t mode = body[end - 1];
    if (mode > 1) return kMode;  // 0 replace, 1 additive
    if (nl != tg.name_len) return kName;
    uint32_t diff = 0;  // no early exit: the byte loads are independent (4 in flight per step)
    unsigned long long b = 0;
    for (; b + 4 <= nl; b += 4) {
        const uint8_t *x = body + ro + 2 + b, *y = names + tg.name_off + b;
        diff |= (x[0] ^ y[0]) | (x[1] ^ y[1]) | (x[2] ^ y[2]) | (x[3] ^ y[3]);
    }
    for (; b < nl; ++b) diff |= body[ro + 2 + b] ^ names[tg.name_off + b];
    if (diff) return kName;
    if (N != tg.numel) return kNumel;
    if (fixed) {  // reading R18: a whole number of fixed-width indices, one per entry
        const uint32_t iw = fixed_index_width(N);
        if (ilen % iw) return kTruncated;
        if (ilen / iw != nnz) return kCount;
    }
    rec.idx_off = q;
    rec.idx_len = ilen;
    rec.val_off = q + ilen;
    rec.nnz = nnz;
    rec.numel = N;
    rec.w = tg.w;
    rec.mode = mode;
    return kOk;
}

constexpr int kLocateThreads = 512;  // one round of record checks for up to 512 records
__global__ void __launch_bounds__(kLocateThreads)
k_locate(const uint8_t *__restrict__ body, unsigned long long body_bytes,
         const unsigned long long *__restrict__ body_bytes_dev,
         const TargetDesc *__restrict__ tg, uint32_t n, const uint8_t *__restrict__ names,
         const RecordRow *__restrict__ hint, ApplyRec *__restrict__ recs,
         unsigned long long *__restrict__ rec_chunk_begin, uint32_t *__restrict__ chunk_rec, ApplyState *st,
         int width, int fixed) {
    if (body_bytes_dev != nullptr) {  // chained after delta_extract_async: size on the device
        const unsigned long long b = *body_bytes_dev;
        if (b > body_bytes) {  // ~0: the extract's gate was closed (no body was written)
            if (threadIdx.x == 0) {
                set_status(st, kLayout);
                rec_chunk_begin[n] = 0;
                st->n_chunks = 0;
            }
            return;
        }
        body_bytes = b;
    }
    bool ok = hint != nullptr;
    if (hint != nullptr) {
        for (uint32_t k = threadIdx.x; k < n && ok; k += blockDim.x) {
            const RecordRow h = hint[k];
            const unsigned long long expect_ro =
                k == 0 ? 0ull : hint[k - 1].record_offset + hint[k - 1].record_bytes;
            ApplyRec r;
            unsigned long long end = 0;
            if (h.record_offset != expect_ro ||
                check_record(body, body_bytes, h.record_offset, tg[k], names, width, fixed, r, end) != kOk ||
                end - h.record_offset != h.record_bytes || r.idx_off != h.index_offset ||
                r.idx_len != h.index_bytes || r.nnz != h.nnz || r.val_off != h.values_offset ||
                (k == n - 1 && end != body_bytes)) {
                ok = false;
            } else {
                recs[k] = r;
            }
        }
    }
    ok = __syncthreads_and(ok) && (n > 0 || body_bytes == 0);
    if (!ok) {  // authoritative walk: thread 0 follows the chain of record offsets (two
                // dependent header loads per record), then every record is checked in parallel
        if (threadIdx.x == 0) {
            unsigned long long pos = 0;
            uint32_t code = kOk;
            for (uint32_t k = 0; k < n; ++k) {
                if (pos > body_bytes || body_bytes - pos < 2) { code = kLayout; break; }
                const unsigned long long nl = rd_le(body + pos, 2);
                if (body_bytes - pos - 2 < nl + 24) { code = kLayout; break; }
                const unsigned long long q = pos + 2 + nl;
                const unsigned long long nnz = rd_le(body + q + 8, 8), il = rd_le(body + q + 16, 8);
                const unsigned long long rem = body_bytes - q - 24;
                if (il > rem || nnz > (rem - il) / (unsigned long long)width || rem - il - nnz * width < 1) {
                    code = kLayout;
                    break;
                }
                recs[k].idx_off = pos;  // the record's offset, re-checked in full below
                pos = q + 24 + il + nnz * width + 1;
            }
            if (code == kOk && pos != body_bytes) code = kLayout;
            if (code != kOk) set_status(st, code);
        }
        __syncthreads();
        if (st->status == kOk) {
            for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) {
                ApplyRec r;
                unsigned long long end = 0;
                const uint32_t c = check_record(body, body_bytes, recs[k].idx_off, tg[k], names, width, fixed, r, end);
                if (c != kOk) set_status(st, c);
                else recs[k] = r;
            }
        }
    }
    __syncthreads();
    {   // chunk prefix over the records: block-wide exclusive scan, 256 records per round
        __shared__ unsigned long long s_w[kLocateThreads / 32];
        const bool okst = st->status == kOk;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        unsigned long long carry = 0;
        for (uint32_t b = 0; b < n; b += blockDim.x) {
            const uint32_t k = b + threadIdx.x;
            const unsigned long long x = (okst && k < n) ? (recs[k].idx_len + kByteChunk - 1) / kByteChunk : 0ull;
            const unsigned long long inc = warp_inclusive_sum(x);
            if (lane == 31) s_w[warp] = inc;
            __syncthreads();
            unsigned long long pre = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < kLocateThreads / 32; ++w) {
                const unsigned long long y = s_w[w];
                if (w < warp) pre += y;
                tot += y;
            }
            if (k < n) rec_chunk_begin[k] = carry + pre + inc - x;
            carry += tot;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            rec_chunk_begin[n] = carry;
            st->n_chunks = carry;
        }
    }
    __syncthreads();
    // chunk -> record map (one load per chunk in A2/A4 instead of a binary search)
    if (st->status == kOk) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (uint32_t k = warp; k < n; k += blockDim.x >> 5) {
            const unsigned long long c0 = rec_chunk_begin[k], c1 = rec_chunk_begin[k + 1];
            for (unsigned long long c = c0 + lane; c < c1; c += 32) chunk_rec[c] = k;
        }
    }
}

// ---------------------------------------------------------------- chunk staging (A2, A4)
struct ChunkView {
    unsigned long long cs;   // chunk start within the record's index stream
    uint32_t len;            // bytes in this chunk
    bool last;               // chunk holds the stream's final byte
    const uint8_t *b;        // b[p] = stream byte cs + p, valid for -min(cs, kHalo) <= p < len
};

// Bytes [src, src + n) into shared memory with 16-byte loads of the aligned superset (one
// or two per thread for a 4 KiB chunk); returns p with p[i] = src[i].  buf is 16-byte
// aligned with room for n + 32 bytes.  The over-read stays inside the 16-byte aligned
// vectors that hold the range (never across an allocation granule).
__device__ __forceinline__ const uint8_t *stage_bytes(uint8_t *buf, const uint8_t *src, uint32_t n) {
    const uint4 *a = reinterpret_cast<const uint4 *>(reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15));
    const uint32_t o = (uint32_t)(reinterpret_cast<uintptr_t>(src) & 15);
    const uint32_t nv = (o + n + 15) / 16;
    for (uint32_t j = threadIdx.x; j < nv; j += blockDim.x) reinterpret_cast<uint4 *>(buf)[j] = __ldg(a + j);
    return buf + o;
}

constexpr int kStagePad = 16;  // bytes below the staged data that validate_fast may read (never used)
constexpr int kStageBytes = kStagePad + kHalo + kByteChunk + 32;

// Stage bytes [cs - halo, cs + len) of the record's stream.  The caller synchronises
// before reading.
__device__ __forceinline__ ChunkView stage_chunk(const uint8_t *body, const ApplyRec &R,
                                                 unsigned long long j, uint8_t *buf) {
    ChunkView v;
    v.cs = j * kByteChunk;
    const unsigned long long ce = min(R.idx_len, v.cs + kByteChunk);
    v.len = (uint32_t)(ce - v.cs);
    v.last = (ce == R.idx_len);
    const uint32_t hs = (uint32_t)min(v.cs, (unsigned long long)kHalo);
    v.b = stage_bytes(buf, body + R.idx_off + v.cs - hs, hs + v.len) + hs;
    return v;
}

// Walk back from the thread's first byte p0 over continuation bytes (at most 10) to the
// first byte of the varint that straddles into this thread's 16 bytes; returns its start q
// (p0 if the previous byte ends a varint) and sets `longrun` if 10 continuation bytes
// precede p0 (the varint is already longer than 10 bytes).
__device__ __forceinline__ int varint_start(const ChunkView &v, int p0, bool &longrun) {
    int q = p0, back = 0;
    while ((long long)v.cs + q > 0 && (v.b[q - 1] & 0x80) && back < 10) {
        --q;
        ++back;
    }
    longrun = back == 10 && (long long)v.cs + q > 0 && (v.b[q - 1] & 0x80);
    return q;
}

// Forward LEB128 decode of the varints whose terminator byte lies in this thread's 16
// bytes; f(value) is called per varint in stream order.  Only used after validation.
template <typename F>
__device__ __forceinline__ void decode_thread(const ChunkView &v, F &&f) {
    const int p0 = threadIdx.x * 16;
    const int p1 = min(p0 + 16, (int)v.len);
    if (p0 >= p1) return;
    bool longrun;
    const int q = varint_start(v, p0, longrun);
    unsigned long long acc = 0;
    int d = 0;
    for (int p = q; p < p1; ++p) {
        const uint32_t b = v.b[p];
        if (d < 10) acc |= (unsigned long long)(b & 0x7F) << (7 * d);
        if (b & 0x80) {
            ++d;
        } else {
            if (p >= p0) f(acc);
            acc = 0;
            d = 0;
        }
    }
}

// A2's per-thread pass: count and (saturating) sum of the varints ending in this thread's
// bytes, and the first decode error (zero gap after the first index):
//   > 10 bytes, or a 10th byte carrying more than bit 63  -> overflow
//   a 0x00 byte ending a multi-byte varint                -> overlong
//   a lone 0x00 byte (gap 0) that is not the record's first -> non-increasing
// Indices >= N are caught by A3 (last index = total sum, gaps >= 1).
// Fast path of validate_thread for a full 16-byte window whose varints are all 1-3 bytes
// long and contain no 0x00 byte (the common case at any density), SIMD within 32-bit words:
// with C the continuation bits (byte MSBs), a byte's position d in its varint is >= 1 iff the
// byte before it continues, >= 2 iff the two before it do, so the window's sum of varint
// values is  S_all + 127 S_1 + 16256 S_2  (S_j: payload bytes with d >= j, each a dp4a of the
// payloads masked by those funnel-shifted bits).  Bytes after the window's last terminator
// belong to the next window's varint; the continuation run just before p0 (at most two bytes)
// belongs to this window's first varint.  Returns false if the window needs the byte loop.
__device__ __forceinline__ bool validate_fast(const ChunkView &v, int p0, uint32_t &cnt,
                                              unsigned long long &sum, bool *ones = nullptr) {
    const uint8_t *ptr = v.b + p0 - 4;  // 4 bytes before the window: the straddling varint
    const uint32_t *a4 = reinterpret_cast<const uint32_t *>(reinterpret_cast<uintptr_t>(ptr) & ~uintptr_t(3));
    const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(ptr) & 3) * 8;
    uint32_t W[6], w[5];  // w[0] = bytes p0-4 .. p0-1, w[1..4] = the window
#pragma unroll
    for (int j = 0; j < 6; ++j) W[j] = a4[j];
#pragma unroll
    for (int k = 0; k < 5; ++k) w[k] = sh ? __funnelshift_r(W[k], W[k + 1], sh) : W[k];
    if ((long long)v.cs + p0 == 0) w[0] = 0;  // the stream's first byte: nothing before it
    // 16 one-byte varints (no continuation bit in the window or just before it; the dense
    // regime's common case): count 16, sum = the byte sum; a 0x00 byte goes to the byte loop
    if (((w[1] | w[2] | w[3] | w[4]) & 0x80808080u) == 0u && !(w[0] & 0x80000000u)) {
        uint32_t z = 0;
#pragma unroll
        for (int k = 1; k < 5; ++k) z |= ~(((w[k] & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w[k]) & 0x80808080u;
        if (z) return false;
        const uint32_t s16 = __dp4a(w[1], 0x01010101u, __dp4a(w[2], 0x01010101u, __dp4a(w[3], 0x01010101u, __dp4a(w[4], 0x01010101u, 0u))));
        if (ones) *ones = true;
        cnt += 16;
        sum = sat_add(sum, (unsigned long long)s16);
        return true;
    }
    uint32_t C[5], t[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        C[k] = w[k] & 0x80808080u;
        t[k] = C[k] ^ 0x80808080u;  // terminators
    }
    const uint32_t n = __popc(t[1]) + __popc(t[2]) + __popc(t[3]) + __popc(t[4]);
    if (n == 0) return true;  // no varint ends in this window (a long one is its owner's concern)
    // valid bytes: up to and including the last terminator
    const int kl = t[4] ? 4 : t[3] ? 3 : t[2] ? 2 : 1;
    const uint32_t lastmask = 0xFFFFFFFFu >> __clz(t[kl]);  // bits up to the terminator's MSB
    uint32_t V[5];
    // bytes before p0 that belong to the first varint: the continuation run ending at p0-1
    V[0] = (C[0] & 0x80000000u) ? ((C[0] & 0x00800000u) ? 0xFFFF0000u : 0xFF000000u) : 0u;
#pragma unroll
    for (int k = 1; k < 5; ++k) V[k] = k < kl ? 0xFFFFFFFFu : (k == kl ? lastmask : 0u);
    uint32_t s_all = 0, s1 = 0, s2 = 0, bad = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const uint32_t Cp = k ? C[k - 1] : 0u;
        const uint32_t P1 = __funnelshift_l(Cp, C[k], 8), P2 = __funnelshift_l(Cp, C[k], 16),
                       P3 = __funnelshift_l(Cp, C[k], 24);
        const uint32_t M2 = P1 & P2;
        if (k) {  // > 3-byte varint, or a 0x00 byte (overlong / zero gap / a first index of 0)
            // bit 7 of byte i of nz is set iff byte i of w is nonzero (exact, no borrows)
            const uint32_t nz = ((w[k] & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w[k];
            bad |= ((M2 & P3) | (~nz & 0x80808080u)) & V[k];
        }
        const uint32_t pw = w[k] & 0x7F7F7F7Fu & V[k];
        s_all = __dp4a(pw, 0x01010101u, s_all);
        s1 = __dp4a(pw & ((P1 >> 7) * 0xFFu), 0x01010101u, s1);
        s2 = __dp4a(pw & ((M2 >> 7) * 0xFFu), 0x01010101u, s2);
    }
    if (bad) return false;
    if (V[0] == 0xFFFF0000u && (C[0] & 0x00008000u)) return false;  // > 3 bytes into the window
    if (ones) *ones = (n == 16 && V[0] == 0);  // 16 one-byte varints
    cnt += n;
    sum = sat_add(sum, (unsigned long long)s_all + 127ull * s1 + 16256ull * s2);
    return true;
}

__device__ __forceinline__ void validate_thread(const ChunkView &v, int p0, uint32_t &cnt,
                                                unsigned long long &sum, uint32_t &err) {
    const int p1 = min(p0 + 16, (int)v.len);
    if (p0 >= p1) return;
    if (p1 - p0 == 16 && validate_fast(v, p0, cnt, sum)) return;
    bool longrun;
    const int q = varint_start(v, p0, longrun);
    bool first = ((long long)v.cs + q == 0);
    unsigned long long acc = 0;
    int d = longrun ? 11 : 0;
    for (int p = q; p < p1; ++p) {
        const uint32_t b = v.b[p];
        if (d < 10) acc |= (unsigned long long)(b & 0x7F) << (7 * d);
        if (b & 0x80) {
            d = d < 11 ? d + 1 : 11;
            continue;
        }
        if (p >= p0) {
            uint32_t e = kOk;
            if (d >= 10 || (d == 9 && b > 1)) e = kOverflow;
            else if (b == 0 && d > 0) e = kOverlong;
            else if (b == 0 && !first) e = kNonIncreasing;
            if (e != kOk && err == kOk) err = e;
            ++cnt;
            sum = sat_add(sum, acc);
        }
        acc = 0;
        d = 0;
        first = false;
    }
}

// ------------------------------------------------------------------------------ A2
// 128 threads per 4 KiB chunk, two 16-byte windows each (windows t and t + 128): half the
// per-chunk staging / reduction instructions of one window per thread
constexpr int kDecodeThreads = 128, kDecodeWin = kByteChunk / 16 / kDecodeThreads;
__global__ void __launch_bounds__(kDecodeThreads)
k_decode_count(const uint8_t *__restrict__ body, const ApplyRec *__restrict__ recs, uint32_t n,
               const unsigned long long *__restrict__ rcb, const uint32_t *__restrict__ chunk_rec,
               unsigned int *__restrict__ chunk_count,
               unsigned long long *__restrict__ chunk_sum, ApplyState *st) {
    if (st->status != kOk) return;
    const unsigned long long nch = st->n_chunks;
    __shared__ __align__(16) uint8_t sb[kStageBytes];
    __shared__ uint32_t s_cnt[8];
    __shared__ unsigned long long s_sum[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (unsigned long long c = blockIdx.x; c < nch; c += gridDim.x) {
        const uint32_t k = __ldg(chunk_rec + c);
        const ApplyRec R = recs[k];
        const ChunkView v = stage_chunk(body, R, c - __ldg(rcb + k), sb + kStagePad);
        __syncthreads();
        uint32_t cnt = 0, err = kOk;
        unsigned long long sum = 0;
        const int pl = (int)v.len - 1;  // the stream's last byte must end a varint
#pragma unroll
        for (int h = 0; h < kDecodeWin; ++h) {
            const int p0 = (threadIdx.x + h * kDecodeThreads) * 16;
            validate_thread(v, p0, cnt, sum, err);
            if (v.last && pl >= p0 && pl < p0 + 16 && (v.b[pl] & 0x80)) err = err ? err : kTruncated;
        }
        if (err != kOk) set_status(st, err);
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        if (__all_sync(0xffffffffu, sum < (1ull << 26))) {  // 32 lanes x 2^26 < 2^32: no overflow
            sum = __reduce_add_sync(0xffffffffu, (uint32_t)sum);
        } else {  // saturating (a malformed stream can decode to gaps up to 2^64 - 1)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum = sat_add(sum, __shfl_xor_sync(0xffffffffu, sum, o));
        }
        if (lane == 0) {
            s_cnt[warp] = cnt;
            s_sum[warp] = sum;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tc = 0;
            unsigned long long ts = 0;
#pragma unroll
            for (int w = 0; w < kDecodeThreads / 32; ++w) {
                tc += s_cnt[w];
                ts = sat_add(ts, s_sum[w]);
            }
            chunk_count[c] = tc;
            chunk_sum[c] = ts;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------ A3
// One CTA per record: exclusive scan of its chunks' (count, gap sum) -> ordinal and index
// base of every chunk; count == nnz and last index (= total gap sum) < N.
constexpr int kApplyScanThreads = 256;  // most records span one or a few 4 KiB chunks
__global__ void __launch_bounds__(kApplyScanThreads)
k_apply_scan(const ApplyRec *__restrict__ recs, uint32_t n, const unsigned long long *__restrict__ rcb,
             const unsigned int *__restrict__ chunk_count, const unsigned long long *__restrict__ chunk_sum,
             unsigned long long *__restrict__ ord_base, unsigned long long *__restrict__ idx_base,
             ApplyState *st) {
    if (st->status != kOk) return;
    constexpr int NW = kApplyScanThreads / 32;
    __shared__ unsigned long long s_c[NW], s_s[NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t k = blockIdx.x; k < n; k += gridDim.x) {
        const unsigned long long c0 = rcb[k], c1 = rcb[k + 1];
        unsigned long long cc = 0, cs = 0;
        for (unsigned long long b = c0; b < c1; b += kApplyScanThreads) {
            const unsigned long long c = b + threadIdx.x;
            unsigned long long x = c < c1 ? chunk_count[c] : 0;
            unsigned long long y = c < c1 ? chunk_sum[c] : 0;
            const unsigned long long x0 = x, y0 = y;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long xx = __shfl_up_sync(0xffffffffu, x, o);
                const unsigned long long yy = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) {
                    x += xx;
                    y = sat_add(y, yy);
                }
            }
            if (lane == 31) {
                s_c[warp] = x;
                s_s[warp] = y;
            }
            __syncthreads();
            unsigned long long pc = 0, ps = 0, tc = 0, ts = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                if (w < warp) {
                    pc += s_c[w];
                    ps = sat_add(ps, s_s[w]);
                }
                tc += s_c[w];
                ts = sat_add(ts, s_s[w]);
            }
            __syncthreads();
            // exclusive = prefix of earlier warps + inclusive within warp - own
            // (the gap sum is saturating: recompute the exclusive part via a shuffle)
            unsigned long long ye = __shfl_up_sync(0xffffffffu, y, 1);
            if (lane == 0) ye = 0;
            if (c < c1) {
                ord_base[c] = cc + pc + (x - x0);
                idx_base[c] = sat_add(cs, sat_add(ps, ye));
            }
            (void)y0;
            cc += tc;
            cs = sat_add(cs, ts);
        }
        if (threadIdx.x == 0) {
            const ApplyRec R = recs[k];
            if (cc != R.nnz) set_status(st, kCount);
            else if (R.nnz > 0 && cs >= R.numel) set_status(st, kRange);
        }
    }
}

// ------------------------------------------------------------------------------ A4
// Dense chunk: >= 256 entries whose gap sum is < 4 per entry, so all its changes fall in a
// window of < 4 kByteChunk lanes: [wlo, whi] = (previous chunk's last index, own last
// index] (the record's first chunk: [0, last]).  No other chunk writes a lane of it (indices
// ascend), so every 16-byte vector of the target lying wholly inside the window can be
// rewritten whole: unchanged lanes keep the bits just loaded.  The chunk's changes go into a
// bitmap over the window's vectors; a changed lane's ordinal in the chunk is its rank there.
constexpr uint32_t kDenseWords = 768;  // bitmap words: >= (4 * kByteChunk + 16) / 32, 3 per thread

template <int W>
struct DenseLanes {
    static constexpr int LV = 16 / W;       // lanes per 16-byte vector
    static constexpr int VPW = 32 / LV;     // vectors per bitmap word
    static constexpr uint32_t ALL = (1u << LV) - 1u;
};

// Bytes [src, src + n) into shared memory realigned to buf (16-byte aligned): vector j of
// buf = source bytes 16 j .. 16 j + 15, funnel-shifted from the two aligned source vectors
// that hold them (the second only when it lies inside the aligned superset of the range), so
// the chunk's values are lane-aligned (one LDS per value instead of W byte loads).
__device__ __forceinline__ void stage_aligned(uint8_t *buf, const uint8_t *src, uint32_t n) {
    const uint4 *a = reinterpret_cast<const uint4 *>(reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15));
    const uint32_t o = (uint32_t)(reinterpret_cast<uintptr_t>(src) & 15);
    const uint32_t ns = (o + n + 15) / 16, nv = (n + 15) / 16;  // source / output vectors
    const uint32_t sh = (o & 3u) * 8u, q = o >> 2;
    for (uint32_t j = threadIdx.x; j < nv; j += blockDim.x) {
        const uint4 x = __ldg(a + j);
        const uint4 y = j + 1 < ns ? __ldg(a + j + 1) : make_uint4(0, 0, 0, 0);
        const uint32_t w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
        uint32_t r[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) r[i] = q == 0 ? w[i] : q == 1 ? w[i + 1] : q == 2 ? w[i + 2] : w[i + 3];
        reinterpret_cast<uint4 *>(buf)[j] = make_uint4(__funnelshift_r(r[0], r[1], sh), __funnelshift_r(r[1], r[2], sh),
                                                       __funnelshift_r(r[2], r[3], sh), __funnelshift_r(r[3], r[4], sh));
    }
}

// Gated scatter-store: decode again, absolute index = chunk base + running gap sum, value
// from the chunk's slice of the record's value array (staged in shared memory).
// MINB: CTAs per SM the registers are capped for — 5 (48 registers) for sparse deltas, where
// the scatter is bound by the HBM access rate; 6 (40 registers) for dense ones, where the
// merge is issue-bound (A/B r66: 1 % uniform 2.30 vs 2.32 ms with 5; 50 % 13.9 vs 15.6 with 6)
template <int W, bool ENTRY_MAJOR, int MINB>
__global__ void __launch_bounds__(256, MINB)
k_scatter(const uint8_t *__restrict__ body, const ApplyRec *__restrict__ recs, uint32_t n,
          const unsigned long long *__restrict__ rcb, const uint32_t *__restrict__ chunk_rec,
          const unsigned int *__restrict__ chunk_count, const unsigned long long *__restrict__ chunk_sum,
          const unsigned long long *__restrict__ ord_base, const unsigned long long *__restrict__ idx_base,
          ApplyState *st) {
    using LT = typename std::conditional<W == 2, uint16_t, uint32_t>::type;
    using D = DenseLanes<W>;
    const uint32_t gate = st->status;
    if (gate != kOk) {  // the gate: nothing is written unless all checks passed
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(&st->first_error, 0u, gate);
        return;
    }
    const unsigned long long nch = st->n_chunks;
    __shared__ __align__(16) uint8_t sb[kStageBytes];
    __shared__ __align__(16) uint8_t svb[kByteChunk * W + 32];  // at most one varint per byte
    __shared__ uint32_t s_cnt[8];
    __shared__ unsigned long long s_sum[8];
    __shared__ uint32_t s_wtot[8];
    // entry-major order (sparse chunks): the chunk's indices relative to idx_base[c], by
    // ordinal; stores are issued entry i by thread i mod 256 (a warp covers 32 consecutive
    // entries).  Dense chunks: the change bitmap over the window's vectors and its word prefixes.
    __shared__ union {
        uint32_t rel[ENTRY_MAJOR ? kByteChunk : 1];
        struct {
            uint32_t bm[kDenseWords];
            uint32_t pre[kDenseWords];
        } d;
    } su;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (unsigned long long c = blockIdx.x; c < nch; c += gridDim.x) {
        const uint32_t k = __ldg(chunk_rec + c);
        const ApplyRec R = recs[k];
        const unsigned long long j = c - __ldg(rcb + k);
        const ChunkView v = stage_chunk(body, R, j, sb + kStagePad);
        const unsigned long long ob = ord_base[c];
        const uint32_t cn = chunk_count[c];
        const unsigned long long csum = chunk_sum[c];
        const bool dense = cn >= 256 && csum < 4ull * cn;
        // this chunk's values (cn lanes, any alignment in the body): lane-aligned in svb for a
        // dense chunk (one LDS per value in the merge), the aligned superset otherwise
        const LT *sval = reinterpret_cast<const LT *>(svb);
        const uint8_t *vals = svb;
        if (dense) stage_aligned(svb, body + R.val_off + ob * W, cn * W);
        else vals = stage_bytes(svb, body + R.val_off + ob * W, cn * W);
        if (dense) {
#pragma unroll
            for (int i = 0; i < 3; ++i) su.d.bm[threadIdx.x * 3 + i] = 0u;
        }
        __syncthreads();
        uint32_t cnt = 0;
        unsigned long long sum = 0;
        const int p0 = threadIdx.x * 16;
        const bool full16 = p0 + 16 <= (int)v.len;
        bool ones = false;  // all 16 bytes are single-byte varints
        if (!(full16 && validate_fast(v, p0, cnt, sum, &ones))) {
            decode_thread(v, [&](unsigned long long x) {
                ++cnt;
                sum += x;
            });
        }
        const uint32_t ci = warp_inclusive_sum(cnt);
        const unsigned long long si = warp_inclusive_sum(sum);
        if (lane == 31) {
            s_cnt[warp] = ci;
            s_sum[warp] = si;
        }
        __syncthreads();
        uint32_t cpre = 0;
        unsigned long long spre = 0;
        for (int w = 0; w < warp; ++w) {
            cpre += s_cnt[w];
            spre += s_sum[w];
        }
        uint32_t ord = cpre + ci - cnt;
        const unsigned long long base = idx_base[c];
        unsigned long long idx = base + spre + si - sum;
        LT *w = reinterpret_cast<LT *>(R.w);
        const bool add = R.mode == 1;  // additive record: scatter-add
        auto value = [&](uint32_t o) -> LT {  // sparse chunks
            if constexpr (W == 2) return (LT)(vals[2 * o] | (vals[2 * o + 1] << 8));
            else return (LT)vals[4 * o] | ((LT)vals[4 * o + 1] << 8) | ((LT)vals[4 * o + 2] << 16) | ((LT)vals[4 * o + 3] << 24);
        };
        if (dense) {
            const unsigned long long wlo = j == 0 ? base : base + 1, whi = base + csum;
            // vector-aligned lane base of the window (targets are lane-aligned)
            // (signed: below lane 0 when the target itself is not 16-byte aligned)
            const long long abase = (long long)wlo - (long long)((reinterpret_cast<uintptr_t>(w + wlo) & 15u) / W);
            if (ones) {
                uint32_t r = (uint32_t)(idx - abase);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    r += v.b[p0 + q];
                    atomicOr(&su.d.bm[r >> 5], 1u << (r & 31u));
                }
            } else {
                decode_thread(v, [&](unsigned long long x) {
                    idx += x;
                    const uint32_t r = (uint32_t)(idx - abase);
                    atomicOr(&su.d.bm[r >> 5], 1u << (r & 31u));
                });
            }
            __syncthreads();
            // ranks: exclusive prefix of the words' popcounts (3 words per thread)
            uint32_t pc[3], tot = 0;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                pc[i] = __popc(su.d.bm[threadIdx.x * 3 + i]);
                tot += pc[i];
            }
            const uint32_t ti = warp_inclusive_sum(tot);
            if (lane == 31) s_wtot[warp] = ti;
            __syncthreads();
            uint32_t wp = ti - tot;
            for (int w2 = 0; w2 < warp; ++w2) wp += s_wtot[w2];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                su.d.pre[threadIdx.x * 3 + i] = wp;
                wp += pc[i];
            }
            __syncthreads();
            // every vector holding a change: 4 per thread in flight (loads, then stores)
            const uint32_t nvec = (uint32_t)(((long long)whi - abase) / D::LV) + 1;
            uint4 *gv = reinterpret_cast<uint4 *>(w + abase);
            for (uint32_t v0 = threadIdx.x; v0 < nvec; v0 += 4 * blockDim.x) {
                uint32_t m[4];
                bool whole[4];
                uint4 old[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t vi = v0 + u * blockDim.x;
                    m[u] = vi < nvec ? (su.d.bm[vi / D::VPW] >> ((vi % D::VPW) * D::LV)) & D::ALL : 0u;
                    const long long l0 = abase + (long long)vi * D::LV;
                    whole[u] = l0 >= (long long)wlo && l0 + D::LV - 1 <= (long long)whi;
                    if (m[u] && whole[u] && (add || m[u] != D::ALL)) old[u] = gv[vi];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (!m[u]) continue;
                    const uint32_t vi = v0 + u * blockDim.x;
                    const uint32_t wd = vi / D::VPW, sh = (vi % D::VPW) * D::LV;
                    uint32_t o = su.d.pre[wd] + __popc(su.d.bm[wd] & ((1u << sh) - 1u));  // first change's ordinal
                    if (whole[u] && !add && m[u] == D::ALL) {  // every lane replaced: 4 (or 5) LDS.32
                        const uint32_t *s32 = reinterpret_cast<const uint32_t *>(sval) + (o * W >> 2);
                        uint32_t x[5];
#pragma unroll
                        for (int i = 0; i < 5; ++i) x[i] = s32[i];
                        const uint32_t sh = (o * W & 3u) * 8u;
                        gv[vi] = make_uint4(__funnelshift_r(x[0], x[1], sh), __funnelshift_r(x[1], x[2], sh),
                                            __funnelshift_r(x[2], x[3], sh), __funnelshift_r(x[3], x[4], sh));
                    } else if (whole[u]) {
                        uint32_t ow[4] = {old[u].x, old[u].y, old[u].z, old[u].w};
                        // lanes unrolled: the k-th changed lane takes value o + k (one LDS each)
#pragma unroll
                        for (int l = 0; l < D::LV; ++l) {
                            if (!((m[u] >> l) & 1u)) continue;
                            uint32_t nv = sval[o++];
                            if constexpr (W == 2) {
                                if (add) nv = lane_combine<2>((ow[l >> 1] >> ((l & 1) * 16)) & 0xFFFFu, nv, false);
                                ow[l >> 1] = __byte_perm(ow[l >> 1], nv, (l & 1) ? 0x5410 : 0x3254);
                            } else {
                                if (add) nv = lane_combine<4>(ow[l], nv, false);
                                ow[l] = nv;
                            }
                        }
                        gv[vi] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
                    } else {  // a vector across the window's edge: its changed lanes only
#pragma unroll
                        for (int l = 0; l < D::LV; ++l) {
                            if (!((m[u] >> l) & 1u)) continue;
                            LT &t = w[abase + (long long)vi * D::LV + l];
                            const LT nv = sval[o++];
                            t = add ? (LT)lane_combine<W>(t, nv, false) : nv;
                        }
                    }
                }
            }
        } else if (ENTRY_MAJOR && csum < 0xFFFFFFFFull) {  // needs 32-bit relative indices
            if (ones) {  // 16 one-byte gaps: no continuation handling
                uint32_t r = (uint32_t)(idx - base);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    r += v.b[p0 + q];
                    su.rel[ord + q] = r;
                }
            } else {
                decode_thread(v, [&](unsigned long long x) {
                    idx += x;
                    su.rel[ord++] = (uint32_t)(idx - base);
                });
            }
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < cn; i += blockDim.x) {
                LT &t = w[base + su.rel[i]];
                t = add ? (LT)lane_combine<W>(t, value(i), false) : value(i);
            }
        } else {
            decode_thread(v, [&](unsigned long long x) {
                idx += x;
                w[idx] = add ? (LT)lane_combine<W>(w[idx], value(ord), false) : value(ord);
                ++ord;
            });
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------ decode-only
// delta_merge's decode of a validated body (gated like A4): entry `ord` of record k gets
// the key (k << kKeyShift) | index and its value written at entry_base[k] + ord — keys
// ascend over the whole body, so the two bodies merge as two sorted arrays.
template <int W>
__global__ void __launch_bounds__(256)
k_decode_write(const uint8_t *__restrict__ body, const ApplyRec *__restrict__ recs,
               const unsigned long long *__restrict__ rcb, const uint32_t *__restrict__ chunk_rec,
               const unsigned int *__restrict__ chunk_count, const unsigned long long *__restrict__ chunk_sum,
               const unsigned long long *__restrict__ ord_base,
               const unsigned long long *__restrict__ idx_base, const unsigned long long *__restrict__ entry_base,
               unsigned long long *__restrict__ idx_out, typename std::conditional<W == 2, uint16_t, uint32_t>::type *val_out,
               ApplyState *st) {
    using LT = typename std::conditional<W == 2, uint16_t, uint32_t>::type;
    if (st->status != kOk) return;
    const unsigned long long nch = st->n_chunks;
    __shared__ __align__(16) uint8_t sb[kStageBytes];
    __shared__ __align__(16) uint8_t svb[kByteChunk * W + 32];
    __shared__ uint32_t s_cnt[8];
    __shared__ unsigned long long s_sum[8];
    __shared__ uint32_t s_rel[kByteChunk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (unsigned long long c = blockIdx.x; c < nch; c += gridDim.x) {
        const uint32_t k = __ldg(chunk_rec + c);
        const ApplyRec R = recs[k];
        const ChunkView v = stage_chunk(body, R, c - __ldg(rcb + k), sb + kStagePad);
        const unsigned long long ob = ord_base[c];
        const uint32_t cn = chunk_count[c];
        const uint8_t *vals = stage_bytes(svb, body + R.val_off + ob * W, cn * W);
        __syncthreads();
        uint32_t cnt = 0;
        unsigned long long sum = 0;
        decode_thread(v, [&](unsigned long long x) {
            ++cnt;
            sum += x;
        });
        const uint32_t ci = warp_inclusive_sum(cnt);
        const unsigned long long si = warp_inclusive_sum(sum);
        if (lane == 31) {
            s_cnt[warp] = ci;
            s_sum[warp] = si;
        }
        __syncthreads();
        uint32_t cpre = 0;
        unsigned long long spre = 0;
        for (int w = 0; w < warp; ++w) {
            cpre += s_cnt[w];
            spre += s_sum[w];
        }
        uint32_t o = cpre + ci - cnt;
        const unsigned long long base = idx_base[c];
        unsigned long long idx = base + spre + si - sum;
        const unsigned long long e0 = entry_base[k] + ob;
        const unsigned long long key = (unsigned long long)k << kKeyShift;  // (record, index) keys
        auto value = [&](uint32_t x) -> LT {
            if constexpr (W == 2) return (LT)(vals[2 * x] | (vals[2 * x + 1] << 8));
            else return (LT)vals[4 * x] | ((LT)vals[4 * x + 1] << 8) | ((LT)vals[4 * x + 2] << 16) |
                        ((LT)vals[4 * x + 3] << 24);
        };
        if (chunk_sum[c] < 0xFFFFFFFFull) {  // indices relative to the chunk fit u32: stage, then
            decode_thread(v, [&](unsigned long long x) {  // write entry i from thread i % 256
                idx += x;
                s_rel[o++] = (uint32_t)(idx - base);
            });
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < cn; i += blockDim.x) {
                idx_out[e0 + i] = key | (base + s_rel[i]);
                val_out[e0 + i] = value(i);
            }
        } else {
            decode_thread(v, [&](unsigned long long x) {
                idx += x;
                idx_out[e0 + o] = key | idx;
                val_out[e0 + o] = value(o);
                ++o;
            });
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------ A2f / A4f
// Fixed-width index codec (reading R18): chunk c of a record holds entries
// [c * kByteChunk / iw, ...) of its absolute index array.  The chunk's indices (plus the
// previous entry's, for the strictly-increasing check across chunks) are staged in shared
// memory with 16-byte loads; the body gives no alignment.
template <int IW>
__device__ __forceinline__ unsigned long long fixed_at(const uint8_t *p) {
    unsigned long long x = 0;
#pragma unroll
    for (int b = 0; b < IW; ++b) x |= (unsigned long long)p[b] << (8 * b);
    return x;
}

__device__ __forceinline__ const uint8_t *stage_fixed_chunk(const uint8_t *body, const ApplyRec &R,
                                                            unsigned long long j, uint32_t iw, uint8_t *buf,
                                                            uint32_t &len, unsigned long long &cs) {
    cs = j * kByteChunk;
    const unsigned long long ce = min(R.idx_len, cs + kByteChunk);
    len = (uint32_t)(ce - cs);
    const uint32_t hs = cs ? iw : 0u;  // the previous entry
    return stage_bytes(buf, body + R.idx_off + cs - hs, hs + len) + hs;
}

// Validation: idx[e] > idx[e - 1] (e >= 1), idx[e] < N.
__global__ void __launch_bounds__(256)
k_fixed_validate(const uint8_t *__restrict__ body, const ApplyRec *__restrict__ recs,
                 const unsigned long long *__restrict__ rcb, const uint32_t *__restrict__ chunk_rec,
                 ApplyState *st) {
    if (st->status != kOk) return;
    const unsigned long long nch = st->n_chunks;
    __shared__ __align__(16) uint8_t sb[kByteChunk + 48];
    for (unsigned long long c = blockIdx.x; c < nch; c += gridDim.x) {
        const uint32_t k = __ldg(chunk_rec + c);
        const ApplyRec R = recs[k];
        const uint32_t iw = fixed_index_width(R.numel);
        uint32_t len;
        unsigned long long cs;
        const uint8_t *b = stage_fixed_chunk(body, R, c - __ldg(rcb + k), iw, sb, len, cs);
        __syncthreads();
        uint32_t err = kOk;
        for (uint32_t i = threadIdx.x; i < len / iw; i += blockDim.x) {
            const uint8_t *p = b + (size_t)i * iw;
            const unsigned long long x = iw == 4 ? fixed_at<4>(p) : fixed_at<8>(p);
            if (cs + i * iw > 0) {
                const unsigned long long y = iw == 4 ? fixed_at<4>(p - 4) : fixed_at<8>(p - 8);
                if (x <= y && err == kOk) err = kNonIncreasing;
            }
            if (x >= R.numel && err == kOk) err = kRange;
        }
        if (err != kOk) set_status(st, err);
        __syncthreads();
    }
}

// Gated scatter: W[idx[e]] = val[e] (replace) or W[idx[e]] += val[e] (additive record).
template <int W>
__global__ void __launch_bounds__(256)
k_fixed_scatter(const uint8_t *__restrict__ body, const ApplyRec *__restrict__ recs,
                const unsigned long long *__restrict__ rcb, const uint32_t *__restrict__ chunk_rec,
                ApplyState *st) {
    using LT = typename std::conditional<W == 2, uint16_t, uint32_t>::type;
    const uint32_t gate = st->status;
    if (gate != kOk) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(&st->first_error, 0u, gate);
        return;
    }
    const unsigned long long nch = st->n_chunks;
    __shared__ __align__(16) uint8_t sb[kByteChunk + 48];
    __shared__ __align__(16) uint8_t svb[kByteChunk / 4 * W + 32];
    for (unsigned long long c = blockIdx.x; c < nch; c += gridDim.x) {
        const uint32_t k = __ldg(chunk_rec + c);
        const ApplyRec R = recs[k];
        const uint32_t iw = fixed_index_width(R.numel);
        uint32_t len;
        unsigned long long cs;
        const uint8_t *b = stage_fixed_chunk(body, R, c - __ldg(rcb + k), iw, sb, len, cs);
        const uint32_t ne = len / iw;
        const uint8_t *vals = stage_bytes(svb, body + R.val_off + cs / iw * W, ne * W);
        __syncthreads();
        LT *w = reinterpret_cast<LT *>(R.w);
        for (uint32_t i = threadIdx.x; i < ne; i += blockDim.x) {
            const uint8_t *p = b + (size_t)i * iw;
            const unsigned long long x = iw == 4 ? fixed_at<4>(p) : fixed_at<8>(p);
            LT v;
            if constexpr (W == 2) v = (LT)(vals[2 * i] | (vals[2 * i + 1] << 8));
            else v = (LT)fixed_at<4>(vals + 4 * i);
            w[x] = R.mode == 1 ? (LT)lane_combine<W>(w[x], v, false) : v;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------ launchers
cudaError_t launch_apply(const ApplyArgs &a, cudaStream_t s, cudaEvent_t *ev) {
    if (ev) cudaEventRecord(ev[0], s);
    k_locate<<<1, kLocateThreads, 0, s>>>(a.body, a.body_bytes, a.body_bytes_dev, a.targets, a.n, a.names, a.hint, a.recs,
                               a.rec_chunk_begin, a.chunk_rec, a.state, a.width, a.index_codec);
    if (ev) cudaEventRecord(ev[1], s);
    if (a.index_codec) {  // fixed-width indices: validate, then the gated scatter (no scans)
        k_fixed_validate<<<a.persist_ctas, 256, 0, s>>>(a.body, a.recs, a.rec_chunk_begin, a.chunk_rec, a.state);
        if (ev) {
            cudaEventRecord(ev[2], s);
            cudaEventRecord(ev[3], s);
        }
        if (a.width == 2)
            k_fixed_scatter<2><<<a.scatter_ctas, 256, 0, s>>>(a.body, a.recs, a.rec_chunk_begin, a.chunk_rec, a.state);
        else
            k_fixed_scatter<4><<<a.scatter_ctas, 256, 0, s>>>(a.body, a.recs, a.rec_chunk_begin, a.chunk_rec, a.state);
        if (ev) cudaEventRecord(ev[4], s);
        return cudaGetLastError();
    }
    k_decode_count<<<a.persist_ctas, kDecodeThreads, 0, s>>>(a.body, a.recs, a.n, a.rec_chunk_begin, a.chunk_rec,
                                                  a.chunk_count, a.chunk_sum, a.state);
    if (ev) cudaEventRecord(ev[2], s);
    const uint32_t nb = a.n ? (a.n < 65535u ? a.n : 65535u) : 1u;
    k_apply_scan<<<nb, kApplyScanThreads, 0, s>>>(a.recs, a.n, a.rec_chunk_begin, a.chunk_count, a.chunk_sum,
                                     a.chunk_ord_base, a.chunk_idx_base, a.state);
    if (ev) cudaEventRecord(ev[3], s);
#define SCATTER(WW, EM)                                                                                 \
    (a.dense_hint ? k_scatter<WW, EM, 6> : k_scatter<WW, EM, 5>)<<<a.scatter_ctas, 256, 0, s>>>(      \
        a.body, a.recs, a.n, a.rec_chunk_begin, a.chunk_rec, a.chunk_count, a.chunk_sum, a.chunk_ord_base,    \
        a.chunk_idx_base, a.state)
    if (a.width == 2) {
        if (a.entry_major) SCATTER(2, true);
        else SCATTER(2, false);
    } else {
        SCATTER(4, false);  // entry-major's index staging would exceed 48 KB static smem at W = 4
        // (dense chunks take the bitmap path at either width)
    }
#undef SCATTER
    if (ev) cudaEventRecord(ev[4], s);
    return cudaGetLastError();
}

cudaError_t launch_decode_only(const ApplyArgs &a, unsigned long long *idx_out, void *val_out,
                               const unsigned long long *entry_base, cudaStream_t s) {
    k_locate<<<1, kLocateThreads, 0, s>>>(a.body, a.body_bytes, a.body_bytes_dev, a.targets, a.n, a.names, a.hint, a.recs,
                               a.rec_chunk_begin, a.chunk_rec, a.state, a.width, 0);
    k_decode_count<<<a.persist_ctas, kDecodeThreads, 0, s>>>(a.body, a.recs, a.n, a.rec_chunk_begin, a.chunk_rec,
                                                  a.chunk_count, a.chunk_sum, a.state);
    const uint32_t nb = a.n ? (a.n < 65535u ? a.n : 65535u) : 1u;
    k_apply_scan<<<nb, kApplyScanThreads, 0, s>>>(a.recs, a.n, a.rec_chunk_begin, a.chunk_count, a.chunk_sum,
                                     a.chunk_ord_base, a.chunk_idx_base, a.state);
    if (a.width == 2)
        k_decode_write<2><<<a.persist_ctas, 256, 0, s>>>(a.body, a.recs, a.rec_chunk_begin, a.chunk_rec, a.chunk_count,
                                                         a.chunk_sum, a.chunk_ord_base, a.chunk_idx_base, entry_base, idx_out,
                                                         static_cast<uint16_t *>(val_out), a.state);
    else
        k_decode_write<4><<<a.persist_ctas, 256, 0, s>>>(a.body, a.recs, a.rec_chunk_begin, a.chunk_rec, a.chunk_count,
                                                         a.chunk_sum, a.chunk_ord_base, a.chunk_idx_base, entry_base, idx_out,
                                                         static_cast<uint32_t *>(val_out), a.state);
    return cudaGetLastError();
}

}  // namespace sd
