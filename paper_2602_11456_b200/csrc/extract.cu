// extract.cu — sm_100a kernels for delta extraction.
//
//   K1  k_scan_tiles    E2+E3: the only kernel that reads the 2W bytes of weights.  One
//                       CTA per tile (16 Ki 16-bit lanes = 32 KiB of old + 32 KiB of new),
//                       16-byte streaming loads, bitwise lane compare, per-vector change
//                       masks, one packed block scan for the ranks, ordered compaction
//                       straight into the tile's workspace slot (u16 lane offsets + raw
//                       values) and the tile's change count.  No inter-CTA communication
//                       and no shared-memory staging: a pure streaming pass.
//                       From the tile's change bitmap (shared memory) K1 also derives the
//                       first / last changed lane and the LEB128 bytes of the gaps inside the
//                       tile (< 2^14 lanes: 1-2 bytes each).
//   K2  k_tiles_reduce / k_blocks_scan / k_tiles_bytes / k_tiles_place
//                       E3+E4+E5 sizes: scans over the (small) per-tile metadata — entry
//                       prefix, nearest earlier non-empty tile (its last change is the
//                       predecessor of the tile's first change), each tile's
//                       LEB128 bytes, byte prefix, per-tensor entry/byte begins.
//   K3  k_finalize      E6: record sizes and offsets (the offset table), body size.
//   K4  k_emit_tiles    E5+E6: one warp per tile writes the LEB128 bytes of the first gap
//                       and of the in-tile gaps (ballot-placed, 32 at a time) and copies the
//                       raw values to their final offsets (FIXED: absolute indices instead).
//   K5  k_headers       E6: record headers (name_len, name, N, nnz, index_bytes) + mode.
//
// Product code written for this library; none of it is shared with the test oracle.
// Semantics: DESIGN.md §3 readings R1-R5, R12-R15.
#include <cstdint>
#include <cstdlib>
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
// 16-bit lanes without compares: for x = a ^ b, ((x & 0x7FFF7FFF) + 0x7FFF7FFF) | x has
// bit 15 (31) set iff the low (high) half of x is nonzero; PRMT gathers those bytes and a
// multiply packs their top bits into lane order.
template <int W>
__device__ __forceinline__ uint32_t diff_mask(const uint4 &a, const uint4 &b) {
    const uint32_t x0 = a.x ^ b.x, x1 = a.y ^ b.y, x2 = a.z ^ b.z, x3 = a.w ^ b.w;
    if constexpr (W == 2) {
        const uint32_t f0 = ((x0 & 0x7FFF7FFFu) + 0x7FFF7FFFu) | x0;
        const uint32_t f1 = ((x1 & 0x7FFF7FFFu) + 0x7FFF7FFFu) | x1;
        const uint32_t f2 = ((x2 & 0x7FFF7FFFu) + 0x7FFF7FFFu) | x2;
        const uint32_t f3 = ((x3 & 0x7FFF7FFFu) + 0x7FFF7FFFu) | x3;
        const uint32_t u = (__byte_perm(f0, f1, 0x7531) >> 7) & 0x01010101u;  // lanes 0..3
        const uint32_t v = (__byte_perm(f2, f3, 0x7531) >> 7) & 0x01010101u;  // lanes 4..7
        return ((u * 0x01020408u) >> 24) | (((v * 0x01020408u) >> 20) & 0xF0u);
    } else {
        return (uint32_t)(x0 != 0) | ((uint32_t)(x1 != 0) << 1) | ((uint32_t)(x2 != 0) << 2) |
               ((uint32_t)(x3 != 0) << 3);
    }
}

// 16-bit lanes: two masks per vector, lanes 0-3 (words x, y) and lanes 4-7 (words z, w),
// lane k of a half at bit 8k + 7 — ascending bit order is lane order, and the pair of
// words holding the half is what PRMT extracts lane k from (selector 0x22 k + 0x10).
// f = ((x & 0x7FFF7FFF) + 0x7FFF7FFF) | x has bit 15 (31) set iff the low (high) 16-bit
// half of x = a ^ b is nonzero; PRMT gathers the four high bytes of a half.
__device__ __forceinline__ uint32_t nz16_hi(uint32_t a, uint32_t b) {
    uint32_t t, f;
    asm("lop3.b32 %0, %1, %2, 0x7FFF7FFF, 0x28;" : "=r"(t) : "r"(a), "r"(b));  // (a ^ b) & C
    t += 0x7FFF7FFFu;
    asm("lop3.b32 %0, %1, %2, %3, 0xF6;" : "=r"(f) : "r"(t), "r"(a), "r"(b));  // t | (a ^ b)
    return f;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
__device__ __forceinline__ void diff_mask16(const uint4 &a, const uint4 &b, uint32_t &lo, uint32_t &hi) {
    lo = __byte_perm(nz16_hi(a.x, b.x), nz16_hi(a.y, b.y), 0x7531) & 0x80808080u;
    hi = __byte_perm(nz16_hi(a.z, b.z), nz16_hi(a.w, b.w), 0x7531) & 0x80808080u;
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

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const T y = __shfl_xor_sync(0xffffffffu, v, o);
        v = y > v ? y : v;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_max(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o && y > v) v = y;
    }
    return v;
}

// ------------------------------------------------------------------------------ K1
// THREADS x VECS = 2048 16-byte vectors per operand per tile (32 KiB); instantiated as
// 256 x 8 (3 CTAs / SM) and 512 x 4 (2 CTAs / SM, more warps, fewer registers each).
// ADVANCE (extract-and-advance, NEXT f3): every changed lane of old is overwritten with the
// new lane while the tile's sectors are still in L2, so old == new afterwards (the trainer's
// shadow copy advances to the new version without a second pass).  Old is then read with
// coherent loads, and on a retry after slot regrowth (redo_cap != 0) only the tiles that
// overflowed a redo_cap-entry slot run again (the others were compacted AND advanced).
template <int W, int THREADS, int VECS, bool DENSE, bool ADDITIVE = false, bool ADVANCE = false>
__device__ __forceinline__ void
scan_tile(const uint32_t t, const TileDesc *__restrict__ tiles, uint32_t ntiles, uint32_t prefetch_dist,
          uint32_t slot_cap, uint8_t *__restrict__ slot_bytes,
          typename LaneOf<W>::T *__restrict__ slot_val, TileMeta *__restrict__ meta,
          ExtractSummary *summary, uint32_t redo_cap = 0) {
    using LT = typename LaneOf<W>::T;
    constexpr int LPV = 16 / W;                  // lanes per 16-byte vector
    constexpr int LANES = THREADS * VECS * LPV;  // lanes per tile
    constexpr int NWARP = THREADS / 32;
    constexpr int NQ = VECS / 2;                 // packed count words (two 16-bit fields each)
    static_assert(THREADS * VECS * 16 == kTileBytes, "tile geometry is fixed by the plan");
    static_assert(LANES <= 65536, "lane offsets are u16");
    static_assert(NWARP * NQ == 32, "warp-0 scan covers NWARP warps x NQ words");
    __shared__ uint32_t s_warp[NWARP][NQ];
    __shared__ uint32_t s_pre[NWARP][NQ];
    __shared__ uint32_t s_tot[NQ];
    // the tile's change bitmap in lane order (bit L & 63 of word L >> 6) and per-warp gap
    // statistics: K1 derives the tile's first / last change and the LEB128 bytes of its
    // in-tile gaps itself (no second pass over the slot offsets)
    constexpr int NWORDS = LANES / 64;
    __shared__ __align__(8) unsigned long long s_bits[NWORDS];
    __shared__ uint32_t s_big[NWARP], s_first[NWARP], s_last[NWARP];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if constexpr (ADVANCE) {
        if (redo_cap && meta[t].count <= redo_cap) return;  // done (and advanced) by the first pass
    }
    const TileDesc d = tiles[t];
    const uint32_t nl = d.nlanes;

    uint4 vo[VECS], vn[VECS];
    if (d.flags_tensor & kTileAligned) {
#pragma unroll
        for (int r = 0; r < VECS; ++r) {
            const uint32_t v = r * THREADS + tid;
            if ((v + 1) * LPV <= nl) {
                vo[r] = ADVANCE ? ld_noalloc_v4(d.old_p + (size_t)v * 16) : ld_stream_v4(d.old_p + (size_t)v * 16);
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
        for (int r = 0; r < VECS; ++r) {
            const uint32_t v = r * THREADS + tid;
            vo[r] = make_uint4(0, 0, 0, 0);
            vn[r] = vo[r];
            for (int j = 0; j < LPV && v * LPV + j < nl; ++j) {
                set_lane<W>(vo[r], j, ADVANCE ? reinterpret_cast<const LT *>(d.old_p)[v * LPV + j]
                                              : __ldg(reinterpret_cast<const LT *>(d.old_p) + v * LPV + j));
                set_lane<W>(vn[r], j, __ldg(reinterpret_cast<const LT *>(d.new_p) + v * LPV + j));
            }
        }
    }

    // (after this tile's loads are in flight) L2 prefetch of a tile about prefetch_dist tiles ahead (CTAs run roughly in blockIdx
    // order): the TMA engine keeps DRAM streaming while this CTA's loads hit L2.
    if (prefetch_dist && tid == 0 && t + prefetch_dist < ntiles) {
        const TileDesc p = tiles[t + prefetch_dist];
        if (p.flags_tensor & kTileAligned) {
            const uint32_t bytes = (p.nlanes * W) & ~15u;
            if (bytes) {
                bulk_prefetch_l2(p.old_p, bytes);
                bulk_prefetch_l2(p.new_p, bytes);
            }
        }
    }

    // Per-vector change masks; VECS counts (<= LPV each) packed as 16-bit fields into NQ
    // words so one block scan yields every vector's rank base.
    constexpr bool H16 = (W == 2);  // 16-bit lanes: lanes 0-3 at bits 8k+7, lanes 4-7 at bits 8k+3
    uint32_t m[VECS];
    uint32_t pk[NQ];
#pragma unroll
    for (int r = 0; r < VECS; ++r) {
        if constexpr (H16) {
            uint32_t lo, hi;
            diff_mask16(vo[r], vn[r], lo, hi);
            m[r] = lo | (hi >> 4);
        } else {
            m[r] = diff_mask<W>(vo[r], vn[r]);
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) pk[q] = __popc(m[2 * q]) | (__popc(m[2 * q + 1]) << 16);
    // bitmap: vector v = r THREADS + tid holds lanes [v LPV, v LPV + LPV) -> lane-order bits
    {
        uint8_t *sb8 = reinterpret_cast<uint8_t *>(s_bits);
#pragma unroll
        for (int r = 0; r < VECS; ++r) {
            const uint32_t v = r * THREADS + tid;
            if constexpr (H16) {  // lanes 0-3 at bits 8k+7, lanes 4-7 at bits 8k+3 -> one byte
                const uint32_t u = (m[r] >> 7) & 0x01010101u, w = (m[r] >> 3) & 0x01010101u;
                sb8[v] = (uint8_t)(((u * 0x01020408u) >> 24) | (((w * 0x01020408u) >> 20) & 0xF0u));
            } else {  // 4 lanes per vector: an even/odd thread pair shares one byte
                const uint32_t other = __shfl_xor_sync(0xffffffffu, m[r], 1);
                if (!(tid & 1)) sb8[v >> 1] = (uint8_t)(m[r] | (other << 4));
            }
        }
    }
    uint32_t inc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) inc[q] = warp_inclusive_sum(pk[q]);
    if (lane == 31) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) s_warp[warp][q] = inc[q];
    }
    __syncthreads();
    // In-tile gap statistics from the bitmap: thread i owns word i (64 lanes).  Only the
    // first change of a word can sit >= 64 lanes after its predecessor; it is a two-byte
    // (>= 128-lane) gap iff the previous word is empty and either the word before it is
    // empty too or 128 + b - (its highest lane) >= 128.  The tile's very first change also
    // passes that test (no change before it): it is subtracted once below — its gap to the
    // previous tile is K2's.
    {
        uint32_t big = 0, first = 0xFFFFFFFFu, last = 0;
        if (tid < NWORDS) {
            const unsigned long long X = s_bits[tid];
            if (X) {
                const unsigned long long p1 = tid >= 1 ? s_bits[tid - 1] : 0ull;
                const unsigned long long p2 = tid >= 2 ? s_bits[tid - 2] : 0ull;
                const uint32_t b = (uint32_t)__ffsll((long long)X) - 1u;
                big = p1 ? 0u : (p2 ? (uint32_t)(b + __clzll((long long)p2) >= 63) : 1u);
                first = 64u * tid + b;
                last = 64u * tid + 63u - (uint32_t)__clzll((long long)X);
            }
        }
        big = __reduce_add_sync(0xffffffffu, big);
        first = __reduce_min_sync(0xffffffffu, first);
        last = __reduce_max_sync(0xffffffffu, last);
        if (lane == 0) {
            s_big[warp] = big;
            s_first[warp] = first;
            s_last[warp] = last;
        }
    }
    // warp 0 scans the NWARP x NQ warp totals across warps (lane = NQ * warp + word)
    if (warp == 0) {
        const uint32_t x = s_warp[lane / NQ][lane % NQ];
        uint32_t y = x;
#pragma unroll
        for (int o = NQ; o < 32; o <<= 1) {
            const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        s_pre[lane / NQ][lane % NQ] = y - x;
        if (lane >= 32 - NQ) s_tot[lane % NQ] = y;
    }
    __syncthreads();
    uint32_t pre[NQ], tot[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        pre[q] = s_pre[warp][q];
        tot[q] = s_tot[q];
    }
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) c += (tot[q] & 0xFFFFu) + (tot[q] >> 16);

    // Ordered compaction: entry (r, tid, j) gets rank sum_{r'<r} tot_r' + prefix_r(tid) +
    // popc(mask below j) — lane order.  Values go straight from registers to the tile's
    // slot; lane offsets to shared memory (for the in-tile gaps below).
    const bool fits = c <= slot_cap;  // CTA-uniform; an overflowing tile is redone after regrowth
    if (tid == 0) {
        uint32_t big = 0, first = 0xFFFFFFFFu, last = 0;
#pragma unroll
        for (int w = 0; w < NWARP; ++w) {
            big += s_big[w];
            first = min(first, s_first[w]);
            last = max(last, s_last[w]);
        }
        // internal bytes = one per in-tile gap plus one more per gap >= 128 lanes (< 2^14 lanes:
        // at most two LEB128 bytes); `big` counted the tile's first change once
        meta[t] = c ? TileMeta{c, (uint16_t)first, (uint16_t)last, c - 1 + big - 1, 0} : TileMeta{0, 0, 0, 0, 0};
        if (!fits) {
            summary->overflow = 1;
            atomicMax(&summary->max_count, (unsigned long long)c);
        }
    }
    if (!fits) return;
    if constexpr (ADVANCE) {
        // old <- new where anything changed: a thread pair (tid, tid ^ 1) holds one 32-byte
        // sector; if either half changed both store their whole 16-byte vector (a full-sector
        // write needs no DRAM fill; unchanged lanes are rewritten with their own value).
        // Partial vectors at the end of a tile and unaligned tiles: changed lanes only.
        LT *op = const_cast<LT *>(reinterpret_cast<const LT *>(d.old_p));
        const bool aligned = d.flags_tensor & kTileAligned;
#pragma unroll
        for (int r = 0; r < VECS; ++r) {
            const uint32_t v = r * THREADS + tid;
            const bool any = (m[r] | __shfl_xor_sync(0xffffffffu, m[r], 1)) != 0;
            if (aligned && any && (v + 1) * LPV <= nl) {
                reinterpret_cast<uint4 *>(op)[v] = vn[r];
            } else if (m[r]) {
                for (int j = 0; j < LPV && v * LPV + j < nl; ++j) {
                    const uint32_t bit = (W == 2) ? (j < 4 ? 8 * j + 7 : 8 * (j - 4) + 3) : j;
                    if ((m[r] >> bit) & 1u) op[v * LPV + j] = (LT)lane_of<W>(vn[r], j);
                }
            }
        }
    }
    LT *sv = slot_val + (size_t)t * slot_cap;
    uint16_t *sg = reinterpret_cast<uint16_t *>(slot_bytes + (size_t)t * 2 * slot_cap);
    uint32_t rbase = 0;
#pragma unroll
    for (int r = 0; r < VECS; ++r) {
        const int q = r >> 1, sh = (r & 1) * 16;
        const uint32_t p0 = rbase + (((pre[q] + inc[q] - pk[q]) >> sh) & 0xFFFFu);
        rbase += (tot[q] >> sh) & 0xFFFFu;
        uint16_t *so = sg + p0;
        LT *vp = sv + p0;
        if constexpr (H16) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t mm = (h ? m[r] << 4 : m[r]) & 0x80808080u;
                const uint32_t na = h ? vn[r].z : vn[r].x, nb = h ? vn[r].w : vn[r].y;
                const uint32_t oa = h ? vo[r].z : vo[r].x, ob = h ? vo[r].w : vo[r].y;
                const uint32_t obase = (r * THREADS + tid) * LPV + 4 * h;
                auto put = [&](uint32_t k, uint32_t sel) {
                    *so++ = (uint16_t)(obase + k);
                    const uint32_t nv = prmt(na, nb, sel);
                    if constexpr (ADDITIVE)  // the arithmetic difference new - old
                        *vp++ = (LT)lane_combine<W>(nv & 0xFFFFu, prmt(oa, ob, sel) & 0xFFFFu, true);
                    else
                        *vp++ = (LT)nv;
                };
                if constexpr (DENSE) {  // four predicated steps, no divergent loop
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (mm & (0x80u << (8 * k))) put(k, 0x22u * k + 0x10u);
                } else {
                    // 32-bit slot indices off the slot bases (no 64-bit pointer chains)
                    uint32_t pos = (uint32_t)(so - sg);
                    so += __popc(mm);
                    vp += __popc(mm);
                    while (mm) {
                        const uint32_t b = (uint32_t)__ffs(mm) - 1;  // 8k + 7
                        mm &= mm - 1;
                        const uint32_t k = b >> 3;
                        const uint32_t sel = __funnelshift_r(0x76543210u, 0u, b - 7);
                        const uint32_t nv = prmt(na, nb, sel);
                        sg[pos] = (uint16_t)(obase + k);
                        if constexpr (ADDITIVE)
                            sv[pos] = (LT)lane_combine<W>(nv & 0xFFFFu, prmt(oa, ob, sel) & 0xFFFFu, true);
                        else
                            sv[pos] = (LT)nv;
                        ++pos;
                    }
                }
            }
        } else {
            uint32_t mm = m[r];
            uint32_t pos = (uint32_t)(so - sg);  // 32-bit slot indices (no pointer chains)
            while (mm) {
                const int j = __ffs(mm) - 1;
                mm &= mm - 1;
                sg[pos] = (uint16_t)((r * THREADS + tid) * LPV + j);
                if constexpr (ADDITIVE)
                    sv[pos] = (LT)lane_combine<W>(lane_of<W>(vn[r], j), lane_of<W>(vo[r], j), true);
                else
                    sv[pos] = (LT)lane_of<W>(vn[r], j);
                ++pos;
            }
        }
    }
}

template <int W, int THREADS, int VECS, int MINB, bool DENSE, bool ADDITIVE = false, bool ADVANCE = false>
__global__ void __launch_bounds__(THREADS, MINB)
k_scan_tiles(const TileDesc *__restrict__ tiles, uint32_t ntiles, uint32_t prefetch_dist,
             uint32_t slot_cap, uint8_t *__restrict__ slot_bytes,
             typename LaneOf<W>::T *__restrict__ slot_val, TileMeta *__restrict__ meta,
             ExtractSummary *summary, uint32_t redo_cap) {
    scan_tile<W, THREADS, VECS, DENSE, ADDITIVE, ADVANCE>(blockIdx.x, tiles, ntiles, prefetch_dist, slot_cap,
                                                          slot_bytes, slot_val, meta, summary, redo_cap);
}

// Slot regrowth that keeps the compaction of the tiles that fitted (extract-and-advance:
// those tiles were advanced and cannot be compared again): entries of tile t move from the
// old_cap-entry slot to the new_cap-entry slot.
template <int W>
__global__ void __launch_bounds__(256)
k_slots_regrow(const TileMeta *__restrict__ meta, uint32_t ntiles, uint32_t old_cap, const uint16_t *__restrict__ ob,
               const typename LaneOf<W>::T *__restrict__ ov, uint32_t new_cap, uint16_t *__restrict__ nb,
               typename LaneOf<W>::T *__restrict__ nv) {
    const int lane = threadIdx.x & 31;
    const uint32_t wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    for (uint32_t t = wg; t < ntiles; t += nw) {
        const uint32_t c = meta[t].count;
        if (c > old_cap) continue;  // overflowed: recomputed by the retry
        for (uint32_t i = lane; i < c; i += 32) {
            nb[(size_t)t * new_cap + i] = ob[(size_t)t * old_cap + i];
            nv[(size_t)t * new_cap + i] = ov[(size_t)t * old_cap + i];
        }
    }
}

cudaError_t launch_slots_regrow(const TileMeta *meta, uint32_t ntiles, int width, uint32_t old_cap,
                                const void *ob, const void *ov, uint32_t new_cap, void *nb, void *nv, int ctas,
                                cudaStream_t s) {
    if (width == 2)
        k_slots_regrow<2><<<ctas, 256, 0, s>>>(meta, ntiles, old_cap, static_cast<const uint16_t *>(ob),
                                               static_cast<const uint16_t *>(ov), new_cap, static_cast<uint16_t *>(nb),
                                               static_cast<uint16_t *>(nv));
    else
        k_slots_regrow<4><<<ctas, 256, 0, s>>>(meta, ntiles, old_cap, static_cast<const uint16_t *>(ob),
                                               static_cast<const uint32_t *>(ov), new_cap, static_cast<uint16_t *>(nb),
                                               static_cast<uint32_t *>(nv));
    return cudaGetLastError();
}

// Persistent form: 3 CTAs per SM loop over the tiles (t = CTA, CTA + grid, ...), no
// per-tile CTA launch.
template <int W>
__global__ void __launch_bounds__(256, 3)
k_scan_tiles_persist(const TileDesc *__restrict__ tiles, uint32_t ntiles, uint32_t prefetch_dist,
                     uint32_t slot_cap, uint8_t *__restrict__ slot_bytes,
                     typename LaneOf<W>::T *__restrict__ slot_val, TileMeta *__restrict__ meta,
                     ExtractSummary *summary) {
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        scan_tile<W, 256, 8, false>(t, tiles, ntiles, prefetch_dist, slot_cap, slot_bytes, slot_val, meta, summary);
        __syncthreads();  // shared scratch is reused by the next tile
    }
}

// ------------------------------------------------------------------------------ K2
// Tile-level scans over blocks of kTileBlock tiles (1024 threads x 4 tiles).
__global__ void __launch_bounds__(1024)
k_tiles_reduce(const TileMeta *__restrict__ meta, uint32_t ntiles, unsigned long long *__restrict__ blk_cnt,
               long long *__restrict__ blk_key, const ExtractSummary *summary) {
    if (summary->overflow) return;
    __shared__ unsigned long long s_c[32];
    __shared__ long long s_k[32];
    const uint32_t t0 = blockIdx.x * kTileBlock + threadIdx.x * 4;
    unsigned long long c = 0;
    long long key = -1;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const uint32_t t = t0 + e;
        if (t < ntiles) {
            const uint32_t n = meta[t].count;
            c += n;
            if (n) key = t;
        }
    }
    c = warp_sum(c);
    key = warp_max(key);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_c[warp] = c;
        s_k[warp] = key;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tc = 0;
        long long tk = -1;
        for (int w = 0; w < 32; ++w) {
            tc += s_c[w];
            tk = s_k[w] > tk ? s_k[w] : tk;
        }
        blk_cnt[blockIdx.x] = tc;
        blk_key[blockIdx.x] = tk;
    }
}

// One CTA: exclusive sum-scan of blk_a (in place) and, if blk_key != nullptr, exclusive
// max-scan of blk_key (in place, identity -1).
__global__ void __launch_bounds__(1024)
k_blocks_scan(unsigned long long *__restrict__ blk_a, long long *__restrict__ blk_key, uint32_t nblk,
              const ExtractSummary *summary) {
    if (summary->overflow) return;
    __shared__ unsigned long long s_w[32];
    __shared__ long long s_m[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long carry = 0;
    long long mcarry = -1;
    for (uint32_t b = 0; b < nblk; b += 1024) {
        const uint32_t i = b + threadIdx.x;
        const unsigned long long x = i < nblk ? blk_a[i] : 0;
        unsigned long long tot;
        const unsigned long long ex = block_excl_scan<32, unsigned long long>(x, s_w, tot);
        if (blk_key) {
            const long long k = i < nblk ? blk_key[i] : -1;
            const long long inc = warp_inclusive_max(k);
            if (lane == 31) s_m[warp] = inc;
            __syncthreads();
            long long pre = -1, all = -1;
            for (int w = 0; w < 32; ++w) {
                if (w < warp && s_m[w] > pre) pre = s_m[w];
                if (s_m[w] > all) all = s_m[w];
            }
            long long exm = __shfl_up_sync(0xffffffffu, inc, 1);
            if (lane == 0) exm = -1;
            if (pre > exm) exm = pre;
            if (mcarry > exm) exm = mcarry;
            __syncthreads();
            if (i < nblk) blk_key[i] = exm;
            if (all > mcarry) mcarry = all;
        }
        if (i < nblk) blk_a[i] = carry + ex;
        carry += tot;
    }
}

// Per tile: entry prefix E_t, predecessor of its first change, its LEB128 bytes.
__global__ void __launch_bounds__(1024)
k_tiles_bytes(const TileDesc *__restrict__ tiles, const TileMeta *__restrict__ meta, uint32_t ntiles,
              const unsigned long long *__restrict__ blk_cnt, const long long *__restrict__ blk_key,
              const uint32_t *__restrict__ tensor_first_tile, unsigned long long *__restrict__ tile_entry,
              unsigned long long *__restrict__ tile_pred, unsigned int *__restrict__ tile_bytes,
              unsigned long long *__restrict__ blk_bytes, const unsigned long long *__restrict__ numel,
              int fixed, const ExtractSummary *summary) {
    if (summary->overflow) return;
    __shared__ unsigned long long s_w[32];
    __shared__ long long s_m[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t t0 = blockIdx.x * kTileBlock + threadIdx.x * 4;
    TileMeta mt[4];
    unsigned long long c = 0;
    long long key = -1;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        mt[e] = t0 + e < ntiles ? meta[t0 + e] : TileMeta{0, 0, 0, 0, 0};
        c += mt[e].count;
        if (mt[e].count) key = t0 + e;
    }
    unsigned long long tot;
    unsigned long long cex = block_excl_scan<32, unsigned long long>(c, s_w, tot) + blk_cnt[blockIdx.x];
    const long long kinc = warp_inclusive_max(key);
    if (lane == 31) s_m[warp] = kinc;
    __syncthreads();
    long long kex = __shfl_up_sync(0xffffffffu, kinc, 1);
    if (lane == 0) kex = -1;
    for (int w = 0; w < warp; ++w)
        if (s_m[w] > kex) kex = s_m[w];
    if (blk_key[blockIdx.x] > kex) kex = blk_key[blockIdx.x];
    unsigned int mybytes = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const uint32_t t = t0 + e;
        if (t >= ntiles) break;
        unsigned long long pred = 0;
        unsigned int b = 0;
        if (mt[e].count) {
            const TileDesc d = tiles[t];
            const uint32_t k = d.flags_tensor & kTileTensorMask;
            if (kex >= 0 && (unsigned long long)kex >= tensor_first_tile[k]) {
                pred = tiles[kex].lane_base + meta[kex].last_off;  // last change before this tile
            }
            const unsigned long long first = d.lane_base + mt[e].first_off;
            b = fixed ? mt[e].count * fixed_index_width(numel[k])  // reading R18: absolute indices
                      : mt[e].internal_bytes + leb_len(first - pred);
            kex = t;
        }
        tile_entry[t] = cex;
        tile_pred[t] = pred;
        tile_bytes[t] = b;
        cex += mt[e].count;
        mybytes += b;
    }
    __syncthreads();  // s_w reuse
    unsigned long long bs = warp_sum((unsigned long long)mybytes);
    if (lane == 0) s_w[warp] = bs;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long x = 0;
        for (int w = 0; w < 32; ++w) x += s_w[w];
        blk_bytes[blockIdx.x] = x;
    }
}

// Per tile: byte prefix; per tensor: E_k and B_k at its first tile; totals.
__global__ void __launch_bounds__(1024)
k_tiles_place(const TileDesc *__restrict__ tiles, const TileMeta *__restrict__ meta, uint32_t ntiles,
              uint32_t ntensors, const unsigned long long *__restrict__ tile_entry,
              const unsigned int *__restrict__ tile_bytes, const unsigned long long *__restrict__ blk_bytes,
              unsigned long long *__restrict__ tile_byte, unsigned long long *__restrict__ entry_begin,
              unsigned long long *__restrict__ tensor_byte_begin, ExtractSummary *summary) {
    if (summary->overflow) return;
    __shared__ unsigned long long s_w[32];
    const uint32_t t0 = blockIdx.x * kTileBlock + threadIdx.x * 4;
    unsigned int b[4];
    unsigned long long mine = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        b[e] = t0 + e < ntiles ? tile_bytes[t0 + e] : 0;
        mine += b[e];
    }
    unsigned long long tot;
    unsigned long long ex = block_excl_scan<32, unsigned long long>(mine, s_w, tot) + blk_bytes[blockIdx.x];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const uint32_t t = t0 + e;
        if (t >= ntiles) break;
        tile_byte[t] = ex;
        const uint32_t f = tiles[t].flags_tensor;
        if (f & kTileFirstOfTensor) {
            entry_begin[f & kTileTensorMask] = tile_entry[t];
            tensor_byte_begin[f & kTileTensorMask] = ex;
        }
        if (t == ntiles - 1) {
            const unsigned long long M = tile_entry[t] + meta[t].count;
            entry_begin[ntensors] = M;
            tensor_byte_begin[ntensors] = ex + b[e];
            summary->M = M;
            summary->idx_bytes = ex + b[e];
        }
        ex += b[e];
    }
}

// ------------------------------------------------------------------------------ K3
__global__ void __launch_bounds__(1024)
k_finalize(const unsigned long long *__restrict__ E, const unsigned long long *__restrict__ Bk, uint32_t T,
           const uint32_t *__restrict__ name_len, const unsigned long long *__restrict__ numel,
           RecordRow *__restrict__ table, int width, ExtractSummary *summary) {
    if (summary->overflow) return;
    __shared__ unsigned long long s_warp[32];
    unsigned long long carry = 0;
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
    if (threadIdx.x == 0) summary->body_bytes = carry;
}

// ------------------------------------------------------------------------------ K4
// Warp-wide copy of n bytes from a 16-byte aligned source to any destination: byte head
// up to the destination's 16-byte boundary, 16-byte stores assembled from funnel-shifted
// source words, byte tail.  Reads at most 4 bytes past the source range (slots are padded).
template <bool GLOBAL_SRC = true>
__device__ __forceinline__ void warp_copy4(uint8_t *dst, const uint8_t *src, uint32_t n, int lane) {
    const uint32_t head = min(n, (uint32_t)((4u - ((uintptr_t)dst & 3u)) & 3u));
    if ((uint32_t)lane < head) dst[lane] = src[lane];
    const uint32_t rest = n - head, nw = rest >> 2;
    uint32_t *d32 = reinterpret_cast<uint32_t *>(dst + head);
    const uint32_t *s32 = reinterpret_cast<const uint32_t *>(src);
    const uint32_t sh = 8u * head;  // source byte offset of word j is head + 4j
    for (uint32_t j = lane; j < nw; j += 32) {
        const uint32_t w0 = GLOBAL_SRC ? __ldg(s32 + j) : s32[j], w1 = GLOBAL_SRC ? __ldg(s32 + j + 1) : s32[j + 1];
        d32[j] = sh ? __funnelshift_r(w0, w1, sh) : w0;
    }
    for (uint32_t b = (nw << 2) + lane; b < rest; b += 32) dst[head + b] = src[head + b];
}

__device__ __forceinline__ void warp_copy(uint8_t *dst, const uint8_t *src, uint32_t n, int lane) {
    if (n < 1024) {  // a few words per lane: the 4-byte path has the shorter critical path
        warp_copy4(dst, src, n, lane);
        return;
    }
    // byte head up to the destination's 16-byte boundary
    const uint32_t head = min(n, (uint32_t)((16u - ((uintptr_t)dst & 15u)) & 15u));
    if ((uint32_t)lane < head) dst[lane] = src[lane];
    const uint32_t rest = n - head, nv = rest >> 4;
    uint4 *d16 = reinterpret_cast<uint4 *>(dst + head);
    // source 16-byte aligned: output vector j = source bytes [head + 16j, head + 16j + 16),
    // i.e. words q .. q+4 of the source shifted right by 8 * (head % 4) bits, q = head/4 + 4j
    const uint32_t *s32 = reinterpret_cast<const uint32_t *>(src);
    const uint32_t q0 = head >> 2, sh = 8u * (head & 3u);
#pragma unroll 2
    for (uint32_t j = lane; j < nv; j += 32) {
        const uint32_t q = q0 + 4 * j;
        const uint32_t a0 = __ldg(s32 + q), a1 = __ldg(s32 + q + 1), a2 = __ldg(s32 + q + 2),
                       a3 = __ldg(s32 + q + 3), a4 = __ldg(s32 + q + 4);
        uint4 o;
        o.x = __funnelshift_r(a0, a1, sh);
        o.y = __funnelshift_r(a1, a2, sh);
        o.z = __funnelshift_r(a2, a3, sh);
        o.w = __funnelshift_r(a3, a4, sh);
        d16[j] = o;
    }
    for (uint32_t b = (nv << 4) + lane; b < rest; b += 32) dst[head + b] = src[head + b];
}

// K3b: per tile, the final body offsets of its index bytes and values and its first gap
// (one thread per tile; turns K4's chain of dependent loads into one 32-byte load).
template <int W>
__global__ void __launch_bounds__(256)
k_tiles_emitplan(const TileDesc *__restrict__ tiles, const TileMeta *__restrict__ meta, uint32_t ntiles,
                 const unsigned long long *__restrict__ tile_entry, const unsigned long long *__restrict__ tile_byte,
                 const unsigned long long *__restrict__ tile_pred, const unsigned long long *__restrict__ E,
                 const unsigned long long *__restrict__ Bk, const RecordRow *__restrict__ table,
                 TileEmit *__restrict__ plan, const unsigned long long *__restrict__ numel, int fixed,
                 const ExtractSummary *summary) {
    if (summary->overflow) return;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x) {
        const TileMeta m = meta[t];
        TileEmit e{0, 0, 0, m.count, m.internal_bytes};
        if (m.count) {
            const TileDesc d = tiles[t];
            const uint32_t k = d.flags_tensor & kTileTensorMask;
            e.ib = table[k].index_offset + (tile_byte[t] - Bk[k]);
            e.vb = table[k].values_offset + (tile_entry[t] - E[k]) * W;
            e.g0 = fixed ? d.lane_base : d.lane_base + m.first_off - tile_pred[t];
            if (fixed) e.internal_bytes = fixed_index_width(numel[k]);
        }
        plan[t] = e;
    }
}

// One warp per tile: the LEB128 bytes of the tile's first gap, then the in-tile gaps
// (differences of the slot's u16 lane offsets, < 2^14: one or two bytes each) encoded 32 at
// a time — byte positions from a ballot of the two-byte ones — and the raw values copied
// to their final offsets in the body.
// BATCHED (chosen on the host when some tile has > 1024 changes): every tile's gaps in
// batches of 256 with the offsets loaded up front; 40 registers at 6 CTAs per SM, where
// the sparse variant keeps 32 registers at 8 CTAs per SM.
template <int W, bool FIXED, bool BATCHED = false>
__global__ void __launch_bounds__(256, BATCHED ? 6 : 8)
k_emit_tiles(const TileEmit *__restrict__ plan, uint32_t ntiles, uint32_t slot_cap,
             const uint8_t *__restrict__ slot_bytes, const typename LaneOf<W>::T *__restrict__ slot_val,
             uint8_t *__restrict__ out, const ExtractSummary *summary, unsigned long long cap) {
    if (summary->overflow || summary->body_bytes > cap) return;  // emit gate (async extract)
    const int lane = threadIdx.x & 31;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const uint32_t wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    // FIXED: absolute indices staged per warp in shared memory, then copied to the body
    __shared__ __align__(16) unsigned long long s_fix[FIXED ? 8 * 256 + 2 : 1];
    for (uint32_t t = wg; t < ntiles; t += nw) {
        // sparse variant: the first 256 slot offsets are loaded before the plan entry arrives
        // (every tile's slot region holds slot_cap >= 512 entries, so the unguarded loads
        // stay inside it; entries past the count are never used)
        uint32_t o[8];
        if constexpr (!FIXED && !BATCHED) {
            const uint16_t *so0 = reinterpret_cast<const uint16_t *>(slot_bytes + (size_t)t * 2 * slot_cap);
#pragma unroll
            for (int r = 0; r < 8; ++r) o[r] = so0[r * 32 + lane];
        }
        const TileEmit e = plan[t];
        if (e.count == 0) continue;
        if constexpr (FIXED) {  // reading R18: lane_base + offset as u32 / u64, little-endian
            const uint32_t iw = e.internal_bytes;  // the index width (set by K3b for FIXED)
            const uint16_t *so = reinterpret_cast<const uint16_t *>(slot_bytes + (size_t)t * 2 * slot_cap);
            unsigned long long *buf = s_fix + 256 * (threadIdx.x >> 5);
            uint8_t *dst = out + e.ib;
            for (uint32_t b = 0; b < e.count; b += 256) {
                const uint32_t n = min(256u, e.count - b);
                for (uint32_t i = lane; i < n; i += 32) {
                    const unsigned long long x = e.g0 + so[b + i];
                    if (iw == 4) reinterpret_cast<uint32_t *>(buf)[i] = (uint32_t)x;
                    else buf[i] = x;
                }
                __syncwarp();
                warp_copy4<false>(dst, reinterpret_cast<const uint8_t *>(buf), n * iw, lane);
                __syncwarp();
                dst += (size_t)n * iw;
            }
            warp_copy(out + e.vb, reinterpret_cast<const uint8_t *>(slot_val + (size_t)t * slot_cap), e.count * W,
                      lane);
            continue;
        }
        uint8_t *ib = out + e.ib;
        unsigned long long g = e.g0;
        const uint32_t L0 = leb_len(g);
        if (lane == 0) {
            for (uint32_t n = 0; n + 1 < L0; ++n) {
                ib[n] = (uint8_t)(g | 0x80);
                g >>= 7;
            }
            ib[L0 - 1] = (uint8_t)g;
        }
        const uint16_t *so = reinterpret_cast<const uint16_t *>(slot_bytes + (size_t)t * 2 * slot_cap);
        uint8_t *p = ib + L0;
        const uint32_t c = e.count;
        if constexpr (BATCHED) {  // dense regime: the values first, then batches of 256 gaps
            warp_copy(out + e.vb, reinterpret_cast<const uint8_t *>(slot_val + (size_t)t * slot_cap), c * W, lane);
            uint32_t last = 0;  // offset of the entry before the batch
            for (uint32_t b0 = 0; b0 < c; b0 += 256) {
                uint32_t o[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const uint32_t i = b0 + r * 32 + lane;
                    o[r] = i < c ? (uint32_t)so[i] : 0u;
                }
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    if (b0 + (uint32_t)r * 32u >= c) break;
                    const uint32_t i = b0 + r * 32 + lane;
                    uint32_t prev = __shfl_up_sync(0xffffffffu, o[r], 1);
                    const uint32_t carry = r ? __shfl_sync(0xffffffffu, o[r ? r - 1 : 0], 31) : last;
                    if (lane == 0) prev = carry;
                    const bool act = i >= 1 && i < c;
                    const uint32_t gi = act ? o[r] - prev : 0u;
                    const uint32_t two = __ballot_sync(0xffffffffu, act && gi >= 128u);
                    const uint32_t skip = (b0 == 0 && r == 0) ? 1u : 0u;  // entry 0 has no in-tile gap
                    if (act) {
                        uint8_t *q = p + (lane - skip) + __popc(two & lt_mask);
                        if (gi < 128u) {
                            q[0] = (uint8_t)gi;
                        } else {
                            q[0] = (uint8_t)(gi | 0x80u);
                            q[1] = (uint8_t)(gi >> 7);
                        }
                    }
                    p += min(32u, c - b0 - r * 32u) - skip + __popc(two);
                }
                last = __shfl_sync(0xffffffffu, o[7], 31);
            }
            continue;
        }
        if (c <= 256) {  // ~all tiles up to a few % density: every load of the tile issued up front
            warp_copy(out + e.vb, reinterpret_cast<const uint8_t *>(slot_val + (size_t)t * slot_cap), c * W, lane);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if ((uint32_t)r * 32u >= c) break;
                const uint32_t i = r * 32 + lane;
                uint32_t prev = __shfl_up_sync(0xffffffffu, o[r], 1);
                const uint32_t carry = __shfl_sync(0xffffffffu, o[r ? r - 1 : 0], 31);
                if (lane == 0) prev = carry;
                const bool act = i >= 1 && i < c;
                const uint32_t gi = act ? o[r] - prev : 0u;
                const uint32_t two = __ballot_sync(0xffffffffu, act && gi >= 128u);
                if (act) {
                    uint8_t *q = p + (lane - (r == 0 ? 1 : 0)) + __popc(two & lt_mask);
                    if (gi < 128u) {
                        q[0] = (uint8_t)gi;
                    } else {
                        q[0] = (uint8_t)(gi | 0x80u);
                        q[1] = (uint8_t)(gi >> 7);
                    }
                }
                p += min(32u, c - r * 32u) - (r == 0 ? 1u : 0u) + __popc(two);
            }
            continue;
        }
        for (uint32_t i0 = 1; i0 < e.count; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool act = i < e.count;
            const uint32_t gi = act ? (uint32_t)(so[i] - so[i - 1]) : 0u;
            const uint32_t two = __ballot_sync(0xffffffffu, act && gi >= 128u);
            if (act) {
                uint8_t *q = p + lane + __popc(two & lt_mask);
                if (gi < 128u) {
                    q[0] = (uint8_t)gi;
                } else {
                    q[0] = (uint8_t)(gi | 0x80u);
                    q[1] = (uint8_t)(gi >> 7);
                }
            }
            p += min(32u, e.count - i0) + __popc(two);
        }
        warp_copy(out + e.vb, reinterpret_cast<const uint8_t *>(slot_val + (size_t)t * slot_cap), e.count * W, lane);
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
          uint8_t *__restrict__ out, int mode, const ExtractSummary *summary, unsigned long long cap,
          unsigned long long *size_out, ExtractSticky *sticky) {
    const bool open = !summary->overflow && summary->body_bytes <= cap;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (size_out != nullptr) *size_out = open ? summary->body_bytes : ~0ull;
        if (sticky != nullptr && !open) {  // delta_extract_wait reports every closed gate, not just the last
            if (summary->overflow) {
                sticky->overflow = 1;
                sticky->max_count = max(sticky->max_count, summary->max_count);
            } else {
                sticky->over_cap = 1;
                sticky->need = max(sticky->need, summary->body_bytes);
            }
        }
    }
    if (!open) return;
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
            o[r.record_bytes - 1] = (uint8_t)mode;  // 0 replace (reading R1/R9), 1 additive
        }
    }
}

// ------------------------------------------------------------------------------ launchers
template <int W>
static cudaError_t scan_impl(const ExtractArgs &a, cudaStream_t s, cudaEvent_t *ev) {
    using LT = typename LaneOf<W>::T;
    // The ffs loop beats four predicated steps per half-vector at every density measured
    // (check 56: 10 % K1 6.46 vs 7.80 ms, 50 % 19.99 vs 24.29 ms), so the predicated
    // (DENSE) compaction is only a diagnostic: DELTA_K1_DENSE=1.
    static const bool dense = [] {
        const char *e = getenv("DELTA_K1_DENSE");
        return e != nullptr && atoi(e) == 1;
    }();
    if (ev) cudaEventRecord(ev[0], s);
    const bool variant_ok = !a.advance && a.mode == 0;  // the variants implement plain replace extraction
    if (a.scan_kernel == 4 && variant_ok) {
        const uint32_t grid = a.ntiles < 3u * a.sm_count ? a.ntiles : 3u * a.sm_count;
        k_scan_tiles_persist<W><<<grid, 256, 0, s>>>(a.tiles, a.ntiles, a.prefetch_dist, a.slot_cap, a.slot_bytes,
                                                    static_cast<LT *>(a.slot_val), a.meta, a.summary);
    } else if (a.scan_kernel == 3 && variant_ok) {
        k_scan_tiles<W, 512, 4, 2, false><<<a.ntiles, 512, 0, s>>>(a.tiles, a.ntiles, a.prefetch_dist, a.slot_cap,
                                                                  a.slot_bytes, static_cast<LT *>(a.slot_val),
                                                                  a.meta, a.summary, 0u);
    } else {
        (a.advance ? (dense ? k_scan_tiles<W, 256, 8, 3, true, false, true> : k_scan_tiles<W, 256, 8, 3, false, false, true>)
         : a.mode == 1 ? (dense ? k_scan_tiles<W, 256, 8, 2, true, true> : k_scan_tiles<W, 256, 8, 2, false, true>)
                       : (dense ? k_scan_tiles<W, 256, 8, 3, true> : k_scan_tiles<W, 256, 8, 3, false>))
            <<<a.ntiles, 256, 0, s>>>(a.tiles, a.ntiles, a.prefetch_dist, a.slot_cap, a.slot_bytes,
                                      static_cast<LT *>(a.slot_val), a.meta, a.summary, a.redo_cap);
    }
    if (ev) cudaEventRecord(ev[1], s);
    const uint32_t nblk = (a.ntiles + kTileBlock - 1) / kTileBlock;
    k_tiles_reduce<<<nblk, 1024, 0, s>>>(a.meta, a.ntiles, a.blk_a, a.blk_key, a.summary);
    k_blocks_scan<<<1, 1024, 0, s>>>(a.blk_a, a.blk_key, nblk, a.summary);
    k_tiles_bytes<<<nblk, 1024, 0, s>>>(a.tiles, a.meta, a.ntiles, a.blk_a, a.blk_key, a.tensor_first_tile,
                                        a.tile_entry, a.tile_pred, a.tile_bytes_tmp, a.blk_a + nblk,
                                        a.numel, a.index_codec, a.summary);
    k_blocks_scan<<<1, 1024, 0, s>>>(a.blk_a + nblk, nullptr, nblk, a.summary);
    k_tiles_place<<<nblk, 1024, 0, s>>>(a.tiles, a.meta, a.ntiles, a.ntensors, a.tile_entry,
                                        a.tile_bytes_tmp, a.blk_a + nblk, a.tile_byte, a.entry_begin,
                                        a.tensor_byte_begin, a.summary);
    if (ev) cudaEventRecord(ev[2], s);
    k_finalize<<<1, 1024, 0, s>>>(a.entry_begin, a.tensor_byte_begin, a.ntensors, a.name_len, a.numel,
                                  a.table, a.width, a.summary);
    {
        const uint32_t g = (a.ntiles + 255) / 256;
        k_tiles_emitplan<W><<<g < 65535u ? g : 65535u, 256, 0, s>>>(a.tiles, a.meta, a.ntiles, a.tile_entry,
                                                                   a.tile_byte, a.tile_pred, a.entry_begin,
                                                                   a.tensor_byte_begin, a.table, a.plan,
                                                                   a.numel, a.index_codec, a.summary);
    }
    if (ev) cudaEventRecord(ev[3], s);
    return cudaGetLastError();
}

template <int W>
static cudaError_t emit_impl(const ExtractArgs &a, uint8_t *out, cudaStream_t s, cudaEvent_t *ev) {
    using LT = typename LaneOf<W>::T;
    if (ev) cudaEventRecord(ev[0], s);
    if (a.index_codec)
        k_emit_tiles<W, true><<<a.persist_ctas, 256, 0, s>>>(a.plan, a.ntiles, a.slot_cap, a.slot_bytes,
                                                            static_cast<const LT *>(a.slot_val), out, a.summary,
                                                            a.out_cap);
    else if (a.slot_cap > kDenseEmitSlot)  // some tile has > kDenseEmitSlot changes
        k_emit_tiles<W, false, true><<<a.sm_count * 6, 256, 0, s>>>(a.plan, a.ntiles, a.slot_cap, a.slot_bytes,
                                                                   static_cast<const LT *>(a.slot_val), out,
                                                                   a.summary, a.out_cap);
    else
        k_emit_tiles<W, false><<<a.persist_ctas, 256, 0, s>>>(a.plan, a.ntiles, a.slot_cap, a.slot_bytes,
                                                             static_cast<const LT *>(a.slot_val), out, a.summary,
                                                             a.out_cap);
    if (ev) cudaEventRecord(ev[1], s);
    const uint32_t hb = a.ntensors < 65535u ? (a.ntensors ? a.ntensors : 1u) : 65535u;
    k_headers<<<hb, 128, 0, s>>>(a.table, a.ntensors, a.name_len, a.name_off, a.names, out, a.mode, a.summary,
                                 a.out_cap, a.size_out, a.sticky);
    if (ev) cudaEventRecord(ev[2], s);
    return cudaGetLastError();
}

cudaError_t launch_extract_scan(const ExtractArgs &a, cudaStream_t s, cudaEvent_t *ev) {
    return a.width == 2 ? scan_impl<2>(a, s, ev) : scan_impl<4>(a, s, ev);
}

cudaError_t launch_extract_emit(const ExtractArgs &a, uint8_t *out, cudaStream_t s, cudaEvent_t *ev) {
    return a.width == 2 ? emit_impl<2>(a, out, s, ev) : emit_impl<4>(a, out, s, ev);
}

}  // namespace sd
