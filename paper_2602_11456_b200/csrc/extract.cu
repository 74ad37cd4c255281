// extract.cu — sm_100a kernels for delta extraction.
//
//   K1  k_scan_tiles    E2+E3(+E4/E5 inside a tile): the only kernel that reads the 2W bytes
//                       of weights.  One CTA per tile (16 Ki 16-bit lanes = 32 KiB of old +
//                       32 KiB of new), 16-byte streaming loads, bitwise lane compare, a change
//                       bitmap in shared memory, one packed block scan for the ranks, ordered
//                       compaction straight into the tile's workspace slot: the LEB128 bytes of
//                       the gaps inside the tile (< 2^14 lanes: 1-2 bytes each; FIXED: u16 lane
//                       offsets) and the raw new values; per tile its count, first / last
//                       changed lane and in-tile LEB128 bytes.
//   K2  k_tiles_scan    E3+E4+E5 sizes + E6 table, one launch: per block of 1024 tiles an
//                       aggregate, folded in order across blocks (published aggregates), then
//                       per tile its entry / byte prefix and first gap (the predecessor of the
//                       tile's first change is the last change before it in its tensor,
//                       PAPER.md:389) -> K4's plan; the last CTA writes the offset table (K3).
//   K4  k_emit_pair     E5+E6: one half-warp per tile (two tiles per warp step): the first
//                       gap's LEB128 bytes, then the in-tile bytes and the values copied from
//                       the slot to their final offsets through a cp.async shared-memory ring.
//                       k_emit_fixed: FIXED codec.
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

// f = ((x & 0x7FFF7FFF) + 0x7FFF7FFF) | x, x = a ^ b, has bit 15 (31) set iff the low (high)
// 16-bit half of x is nonzero, i.e. iff that bf16 lane differs bitwise (reading R2): two LOP3
// and an add, no compares.
__device__ __forceinline__ uint32_t nz16_hi(uint32_t a, uint32_t b) {
    uint32_t t, f;
    asm("lop3.b32 %0, %1, %2, 0x7FFF7FFF, 0x28;" : "=r"(t) : "r"(a), "r"(b));  // (a ^ b) & C
    t += 0x7FFF7FFFu;
    asm("lop3.b32 %0, %1, %2, %3, 0xF6;" : "=r"(f) : "r"(t), "r"(a), "r"(b));  // t | (a ^ b)
    return f;
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
// One CTA per tile: THREADS x VECS = 2048 16-byte vectors per operand (32 KiB of old + 32
// KiB of new), streaming loads into registers, then everything else from shared memory:
//   1. each thread turns its 8 vector pairs into lane-order change masks (bitwise lane
//      inequality, reading R2) and writes them into the tile's change bitmap (lane L is bit
//      L & 63 of word L >> 6), and stages the new vectors that hold a change;
//   2. thread i owns bitmap word i (64 consecutive lanes): one block scan of its change
//      count (packed with its "two-byte gap" flag) gives every change its rank in lane order
//      (the ordered compaction) and the tile's totals;
//   3. thread i emits its word's changes in order: u16 lane offset + value into the tile's
//      slot.  One loop per thread over set bits (instead of one per half-vector), so a warp
//      iterates about as often as its busiest word has changes.
// Gap statistics for the LEB128 byte count come from the same bitmap: only the first change
// of a word can sit >= 64 lanes after its predecessor, and it is a two-byte (>= 128-lane) gap
// iff the previous word is empty and the word before it is empty too or its highest change
// is far enough back.  The tile's very first change also passes that test (nothing before it
// in the tile): it is subtracted once — its gap to the previous tile is K2's.
// ADVANCE (extract-and-advance, NEXT f3): every 32-byte sector of old holding a change is
// rewritten with the new lanes while the tile is in registers, so old == new afterwards; a
// retry after slot regrowth (redo_cap != 0) re-runs only the tiles that overflowed.
// ADDITIVE (reading R17): the staged vectors hold new - old in the lane's float type.
template <int W>
__device__ __forceinline__ uint32_t lane_mask(const uint4 &a, const uint4 &b) {
    if constexpr (W == 2) {  // bit j (lane order) iff 16-bit lane j differs: nz16_hi marks
                             // nonzero halves in bits 15 / 31, PRMT gathers those bytes
        const uint32_t p = __byte_perm(nz16_hi(a.x, b.x), nz16_hi(a.y, b.y), 0x7531);  // lanes 0..3
        const uint32_t q = __byte_perm(nz16_hi(a.z, b.z), nz16_hi(a.w, b.w), 0x7531);  // lanes 4..7
        const uint32_t u = (p >> 7) & 0x01010101u, v = (q >> 7) & 0x01010101u;
        return ((u * 0x01020408u) >> 24) | (((v * 0x01020408u) >> 20) & 0xF0u);
    } else {
        return (uint32_t)(a.x != b.x) | ((uint32_t)(a.y != b.y) << 1) | ((uint32_t)(a.z != b.z) << 2) |
               ((uint32_t)(a.w != b.w) << 3);
    }
}

template <int W, bool ADDITIVE = false, bool ADVANCE = false, bool OFFSETS = false>
__global__ void __launch_bounds__(256, 3)
k_scan_tiles(const TileDesc *__restrict__ tiles, uint32_t ntiles, uint32_t prefetch_dist, uint32_t slot_cap,
             uint8_t *__restrict__ slot_bytes, typename LaneOf<W>::T *__restrict__ slot_val,
             TileMeta *__restrict__ meta, ExtractSummary *summary, uint32_t redo_cap, uint32_t dense_tile) {
    using LT = typename LaneOf<W>::T;
    constexpr int THREADS = 256, VECS = 8;
    constexpr int LPV = 16 / W;                  // lanes per 16-byte vector
    constexpr int LANES = THREADS * VECS * LPV;  // lanes per tile
    constexpr int NWARP = THREADS / 32;
    constexpr int NWORDS = LANES / 64;           // bitmap words = threads that emit
    static_assert(THREADS * VECS * 16 == kTileBytes, "tile geometry is fixed by the plan");
    static_assert(LANES <= 65536, "lane offsets are u16");
    __shared__ __align__(16) uint4 s_new[THREADS * VECS];  // changed vectors (new, or new - old)
    __shared__ __align__(8) unsigned long long s_bits[NWORDS];
    __shared__ uint32_t s_wsum[NWARP];
    __shared__ int s_wfirst[NWARP], s_wlast[NWARP];

    const uint32_t t = blockIdx.x;
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

    // (after this tile's loads are in flight) L2 prefetch of a tile about prefetch_dist tiles
    // ahead (CTAs run roughly in blockIdx order): the TMA engine keeps DRAM streaming while
    // this CTA's loads hit L2.
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

    // ---- 1. change masks -> bitmap; stage the vectors that hold a change
    uint32_t m[VECS];
    uint8_t *sb8 = reinterpret_cast<uint8_t *>(s_bits);
#pragma unroll
    for (int r = 0; r < VECS; ++r) {
        const uint32_t v = r * THREADS + tid;
        m[r] = lane_mask<W>(vo[r], vn[r]);
        if constexpr (W == 2) {
            sb8[v] = (uint8_t)m[r];
        } else {  // 4 lanes per vector: an even/odd thread pair shares one byte
            const uint32_t other = __shfl_xor_sync(0xffffffffu, m[r], 1);
            if (!(tid & 1)) sb8[v >> 1] = (uint8_t)(m[r] | (other << 4));
        }
        if (m[r]) {
            uint4 x = vn[r];
            if constexpr (ADDITIVE) {  // the arithmetic difference new - old, changed lanes
#pragma unroll
                for (int j = 0; j < LPV; ++j)
                    if ((m[r] >> j) & 1u) set_lane<W>(x, j, lane_combine<W>(lane_of<W>(vn[r], j), lane_of<W>(vo[r], j), true));
            }
            s_new[v] = x;
        }
    }
    __syncthreads();

    // ---- 2. word i: change count + two-byte-gap flag, block scan -> ranks and tile totals
    unsigned long long X = 0;
    uint32_t val = 0;
    if (tid < NWORDS) {
        X = s_bits[tid];
        if (X) {
            const unsigned long long p1 = tid >= 1 ? s_bits[tid - 1] : 0ull;
            const unsigned long long p2 = tid >= 2 ? s_bits[tid - 2] : 0ull;
            const uint32_t b = (uint32_t)__ffsll((long long)X) - 1u;
            const uint32_t big = p1 ? 0u : (p2 ? (uint32_t)(b + __clzll((long long)p2) >= 63) : 1u);
            val = (uint32_t)__popcll((long long)X) | (big << 16);  // counts <= 16384, flags <= 256
        }
    }
    const uint32_t inc = warp_inclusive_sum(val);
    const uint32_t bw = __ballot_sync(0xffffffffu, X != 0);
    if (lane == 31) s_wsum[warp] = inc;
    if (lane == 0) {
        s_wfirst[warp] = bw ? 32 * warp + __ffs(bw) - 1 : -1;
        s_wlast[warp] = bw ? 32 * warp + 31 - __clz(bw) : -1;
    }
    __syncthreads();
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) {
        const uint32_t y = s_wsum[w];
        pre += w < warp ? y : 0u;
        tot += y;
    }
    const uint32_t c = tot & 0xFFFFu;
    const bool fits = c <= slot_cap;  // CTA-uniform; an overflowing tile is redone after regrowth
    if (tid == 0) {
        TileMeta mt{0, 0, 0, 0, 0};
        if (c) {
            int fw = -1, lw = -1;
#pragma unroll
            for (int w = 0; w < NWARP; ++w) {
                if (fw < 0) fw = s_wfirst[w];
                if (s_wlast[w] >= 0) lw = s_wlast[w];
            }
            // internal bytes = one per in-tile gap, one more per gap >= 128 lanes (< 2^14
            // lanes: at most two LEB128 bytes); the flag total counted the first change once
            mt = TileMeta{c, (uint16_t)(64 * fw + __ffsll((long long)s_bits[fw]) - 1),
                          (uint16_t)(64 * lw + 63 - __clzll((long long)s_bits[lw])), c - 1 + (tot >> 16) - 1, 0};
        }
        meta[t] = mt;
        if (!fits) {
            summary->overflow = 1;
            atomicMax(&summary->max_count, (unsigned long long)c);
        }
    }
    if (!fits) return;
    if constexpr (ADVANCE) {
        // old <- new where anything changed (only for tiles that fit their slot: an overflowed
        // tile is compared again after the regrowth): a thread pair (tid, tid ^ 1) holds one 32-byte
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
                for (int j = 0; j < LPV && v * LPV + j < nl; ++j)
                    if ((m[r] >> j) & 1u) op[v * LPV + j] = (LT)lane_of<W>(vn[r], j);
            }
        }
    }

    // ---- 3'. dense tiles (>= dense_tile changes, default kDenseTile): emission in vector order.  The owner of
    // word w publishes its rank / two-byte-flag prefix and its first entry's predecessor; then
    // thread tid emits the changes of ITS vectors v = r THREADS + tid (r = 0..7), whose 8 lanes
    // are byte v & 7 of word v >> 3: a warp's lanes hold consecutive vectors, so each store
    // instruction writes 32 nearby slots (the per-word loop below would write 32 runs 64
    // entries apart).  Values come from the staged vectors, gap bytes at their stream positions.
    if (c >= dense_tile) {
        __shared__ uint32_t s_wex[NWORDS], s_wprv[NWORDS];
        if (tid < NWORDS) {
            s_wex[tid] = pre + inc - val;  // entries | two-byte flags before the word
            s_wprv[tid] = 0;  // bits 0-15: predecessor lane; 16: first gap takes two bytes; 17: has one
        }
        // the predecessor of each word's first entry (shuffles: all lanes take part)
        {
            const uint32_t mylast = X ? 64u * tid + 63u - (uint32_t)__clzll((long long)X) : 0u;
            const uint32_t lower = bw & ((1u << lane) - 1u);
            uint32_t prev = __shfl_sync(0xffffffffu, mylast, lower ? 31 - __clz(lower) : 0);
            bool has_prev = lower != 0;
            if (X && !lower) {
                int lw = -1;
#pragma unroll
                for (int w = 0; w < NWARP; ++w)
                    if (w < warp && s_wlast[w] >= 0) lw = s_wlast[w];
                if (lw >= 0) {
                    prev = 64u * lw + 63u - (uint32_t)__clzll((long long)s_bits[lw]);
                    has_prev = true;
                }
            }
            if (tid < NWORDS && X)
                s_wprv[tid] = (has_prev ? (prev | (1u << 17) | ((val >> 16) ? (1u << 16) : 0u)) : 0u);
        }
        __syncthreads();
        LT *sv = slot_val + (size_t)t * slot_cap;
        uint8_t *sb = slot_bytes + (size_t)t * 2 * slot_cap;
        if constexpr (!ADDITIVE && !OFFSETS) {
            // values from the registers (s_new is no longer read), compacted into s_new by
            // rank, then the index bytes behind them (or, when both do not fit its 32 KiB,
            // after the values have left): every store is a shared-memory store, and the slot
            // is written with 16-byte stores (whole sectors instead of 2- and 1-byte scatters)
            const uint32_t nb = c - 1u + (tot >> 16) - 1u;  // in-tile index bytes (as meta)
            const uint32_t vb = (c * W + 15u) & ~15u;
            const bool bsm = vb + nb + 16u <= (uint32_t)sizeof(s_new);
            uint8_t *sm = reinterpret_cast<uint8_t *>(s_new);
            LT *smv = reinterpret_cast<LT *>(s_new);
            auto copy_out = [&](uint8_t *dst, uint32_t from, uint32_t bytes) {
                const uint4 *src = reinterpret_cast<const uint4 *>(sm + from);
                for (uint32_t i = tid; i < (bytes + 15u) / 16u; i += THREADS) reinterpret_cast<uint4 *>(dst)[i] = src[i];
            };
            // pass V: change k of vector v goes to rank + k (lanes unrolled: static extraction)
#pragma unroll
            for (int r = 0; r < VECS; ++r) {
                const uint32_t v = r * THREADS + tid;
                const uint32_t w = v / (64 / LPV), sub = v % (64 / LPV);
                const unsigned long long Wb = s_bits[w];
                const uint32_t mb = (uint32_t)(Wb >> (sub * LPV)) & ((1u << LPV) - 1u);
                if (!mb) continue;
                const unsigned long long below = Wb & ((1ull << (sub * LPV)) - 1ull);
                const uint32_t rank = (s_wex[w] & 0xFFFFu) + (uint32_t)__popcll((long long)below);
#pragma unroll
                for (int j = 0; j < LPV; ++j)
                    if ((mb >> j) & 1u) smv[rank + (uint32_t)__popc(mb & ((1u << j) - 1u))] = (LT)lane_of<W>(vn[r], j);
            }
            if (!bsm) {
                __syncthreads();
                copy_out(reinterpret_cast<uint8_t *>(sv), 0, c * W);
                __syncthreads();
            }
            uint8_t *bd = sm + (bsm ? vb : 0u);
            // pass B: the vector's first change's gap (from prevL) takes two bytes iff it starts
            // its word and the word is flagged; the tile's first change has no in-tile gap (its
            // byte position, -1, is virtual: K4 writes the plan's first gap ahead of the stream);
            // a later change k of the vector: one byte (< LPV lanes) at bq + k - 1
#pragma unroll
            for (int r = 0; r < VECS; ++r) {
                const uint32_t v = r * THREADS + tid;
                const uint32_t w = v / (64 / LPV), sub = v % (64 / LPV);
                const unsigned long long Wb = s_bits[w];
                const uint32_t mb = (uint32_t)(Wb >> (sub * LPV)) & ((1u << LPV) - 1u);
                if (!mb) continue;
                const unsigned long long below = Wb & ((1ull << (sub * LPV)) - 1ull);
                const uint32_t ex = s_wex[w], pv = s_wprv[w];
                const uint32_t rank = (ex & 0xFFFFu) + (uint32_t)__popcll((long long)below);
                const bool hp_w = pv & (1u << 17);
                const uint32_t bigs = (ex >> 16) - ((hp_w && (ex >> 16)) ? 1u : 0u);
                const uint32_t bp = rank - 1u + bigs + (below && (pv & (1u << 16)) ? 1u : 0u);
                const bool has_prev = below ? true : hp_w;
                const uint32_t prevL = below ? 64u * w + 63u - (uint32_t)__clzll((long long)below) : (pv & 0xFFFFu);
                const bool two = has_prev && below == 0 && (pv & (1u << 16));
                const uint32_t bq = bp + (two ? 2u : 1u);
                const uint32_t f = (uint32_t)__ffs(mb) - 1u;  // the vector's first change
                if (has_prev) {
                    const uint32_t g = v * LPV + f - prevL;
                    if (two) {
                        bd[bp] = (uint8_t)(g | 0x80u);
                        bd[bp + 1] = (uint8_t)(g >> 7);
                    } else {
                        bd[bp] = (uint8_t)g;
                    }
                }
#pragma unroll
                for (int j = 1; j < LPV; ++j) {
                    const uint32_t low = mb & ((1u << j) - 1u);
                    if (((mb >> j) & 1u) && low)
                        bd[bq + (uint32_t)__popc(low) - 1u] = (uint8_t)(j - (31 - __clz(low)));
                }
            }
            __syncthreads();
            if (bsm) copy_out(reinterpret_cast<uint8_t *>(sv), 0, c * W);
            copy_out(sb, bsm ? vb : 0u, nb);
            return;
        }
        const LT *sn = reinterpret_cast<const LT *>(s_new);
#pragma unroll 1
        for (int r = 0; r < VECS; ++r) {
            const uint32_t v = r * THREADS + tid;
            const uint32_t w = v / (64 / LPV), sub = v % (64 / LPV);  // word, lane group in it
            const unsigned long long Wb = s_bits[w];
            uint32_t mb = (uint32_t)(Wb >> (sub * LPV)) & ((1u << LPV) - 1u);
            if (!mb) continue;
            const unsigned long long below = Wb & ((1ull << (sub * LPV)) - 1ull);
            const uint32_t ex = s_wex[w], pv = s_wprv[w];
            uint32_t rank = (ex & 0xFFFFu) + (uint32_t)__popcll((long long)below);
            const bool hp_w = pv & (1u << 17);
            const uint32_t bigs = (ex >> 16) - ((hp_w && (ex >> 16)) ? 1u : 0u);
            // byte position: one per earlier in-tile gap + the earlier two-byte ones
            uint32_t bp = rank - 1u + bigs + (below && (pv & (1u << 16)) ? 1u : 0u);
            bool word_first = below == 0;
            bool has_prev = below ? true : hp_w;
            uint32_t prevL = below ? 64u * w + 63u - (uint32_t)__clzll((long long)below) : (pv & 0xFFFFu);
            while (mb) {
                const uint32_t jb = (uint32_t)__ffs(mb) - 1u;
                mb &= mb - 1u;
                const uint32_t L = v * LPV + jb;
                sv[rank] = sn[L];
                if constexpr (OFFSETS) {
                    reinterpret_cast<uint16_t *>(sb)[rank] = (uint16_t)L;
                } else {
                    if (has_prev) {
                        const uint32_t g = L - prevL;
                        if (word_first && (pv & (1u << 16))) {
                            sb[bp] = (uint8_t)(g | 0x80u);
                            sb[bp + 1] = (uint8_t)(g >> 7);
                            bp += 2;
                        } else {
                            sb[bp] = (uint8_t)g;
                            bp += 1;
                        }
                    } else {
                        bp += 1;  // the tile's first entry: its gap is the plan's first gap (K2)
                    }
                }
                has_prev = true;
                word_first = false;
                prevL = L;
                ++rank;
            }
        }
        return;
    }

    // ---- 3. ordered emission of word tid's changes: the value at its rank; the gap to the
    // previous change as LEB128 bytes at its position in the tile's internal index stream
    // (OFFSETS, for the fixed-width codec: the u16 lane offset at its rank instead).
    // Entry e >= 1 of the tile starts at byte (e - 1) + #{two-byte gaps before e}; two-byte
    // gaps are first entries of flagged words other than the tile's first word fw.
    const uint32_t ex = pre + inc - val;
    uint32_t pos = ex & 0xFFFFu;
    LT *sv = slot_val + (size_t)t * slot_cap;
    const LT *sn = reinterpret_cast<const LT *>(s_new);
    if constexpr (OFFSETS) {
        uint16_t *sg = reinterpret_cast<uint16_t *>(slot_bytes + (size_t)t * 2 * slot_cap);
        while (X) {
            const uint32_t L = 64u * tid + (uint32_t)__ffsll((long long)X) - 1u;
            X &= X - 1;
            sg[pos] = (uint16_t)L;
            sv[pos] = sn[L];
            ++pos;
        }
    } else {
        // the last change before this word: in an earlier word of this warp (ballot + shuffle of
        // that word's last lane), else in the last non-empty word of an earlier warp
        const uint32_t mylast = X ? 64u * tid + 63u - (uint32_t)__clzll((long long)X) : 0u;
        const uint32_t lower = bw & ((1u << lane) - 1u);
        uint32_t prev = __shfl_sync(0xffffffffu, mylast, lower ? 31 - __clz(lower) : 0);
        bool has_prev = lower != 0;
        if (X && !lower) {
            int lw = -1;
#pragma unroll
            for (int w = 0; w < NWARP; ++w)
                if (w < warp && s_wlast[w] >= 0) lw = s_wlast[w];
            if (lw >= 0) {
                prev = 64u * lw + 63u - (uint32_t)__clzll((long long)s_bits[lw]);
                has_prev = true;
            }
        }
        uint8_t *sb = slot_bytes + (size_t)t * 2 * slot_cap;
        // two-byte flags before this word, without the tile's first word's (it has no gap)
        const uint32_t bigs = (ex >> 16) - (has_prev && (ex >> 16) ? 1u : 0u);
        const bool rbig = has_prev && (val >> 16);  // this word's first gap takes two bytes
        uint32_t bp = pos + bigs - 1u;               // byte position of this word's first gap
        bool first = true;
        while (X) {
            const uint32_t L = 64u * tid + (uint32_t)__ffsll((long long)X) - 1u;
            X &= X - 1;
            sv[pos] = sn[L];
            if (has_prev) {  // every entry but the tile's first has an in-tile gap
                const uint32_t g = L - prev;
                if (first && rbig) {
                    sb[bp] = (uint8_t)(g | 0x80u);
                    sb[bp + 1] = (uint8_t)(g >> 7);
                    bp += 2;
                } else {
                    sb[bp] = (uint8_t)g;
                    bp += 1;
                }
            } else {
                bp += 1;  // the tile's first entry: its gap is the plan's first gap (K2)
            }
            has_prev = true;
            first = false;
            prev = L;
            ++pos;
        }
    }
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

// ------------------------------------------------------------------------------ K2 / K3 helpers

// Absolute lane index (within its fused tensor) of the last change of non-empty tile p, if p
// is in tensor k; otherwise 0 — the tile after it then starts its tensor's gap chain with the
// first index as-is (reading R3/R4).
__device__ __forceinline__ unsigned long long pred_abs(const TileDesc *__restrict__ tiles,
                                                       const TileMeta *__restrict__ meta, long long p, uint32_t k) {
    if (p < 0) return 0;
    const TileDesc d = tiles[p];
    if ((d.flags_tensor & kTileTensorMask) != k) return 0;
    return d.lane_base + meta[p].last_off;
}

// LEB128 bytes of non-empty tile t given its predecessor tile p (-1: none): the first gap
// plus the in-tile gaps; fixed-width codec (reading R18): count x index width.  Also its
// first gap g0 (fixed: the tile's lane base, i.e. the absolute index base).
__device__ __forceinline__ unsigned long long tile_bytes(const TileDesc &d, const TileMeta &m, const TileDesc *tiles,
                                                         const TileMeta *meta, long long p,
                                                         const unsigned long long *numel, int fixed,
                                                         unsigned long long &g0) {
    const uint32_t k = d.flags_tensor & kTileTensorMask;
    if (fixed) {
        g0 = d.lane_base;
        return (unsigned long long)m.count * fixed_index_width(numel[k]);
    }
    g0 = d.lane_base + m.first_off - pred_abs(tiles, meta, p, k);
    return m.internal_bytes + leb_len(g0);
}

// Block-wide (kTileThreads threads) exclusive scans: sum of x, max of key (identity -1).
__device__ __forceinline__ void block_scan_sum_max(unsigned long long x, long long key, unsigned long long &xex,
                                                   unsigned long long &xtot, long long &kex, long long &ktot) {
    constexpr int NW = kTileThreads / 32;
    __shared__ unsigned long long s_x[NW];
    __shared__ long long s_k[NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned long long xi = warp_inclusive_sum(x);
    const long long ki = warp_inclusive_max(key);
    if (lane == 31) {
        s_x[warp] = xi;
        s_k[warp] = ki;
    }
    __syncthreads();
    unsigned long long px = 0, tx = 0;
    long long pk = -1, tk = -1;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const unsigned long long a = s_x[w];
        const long long b = s_k[w];
        if (w < warp) {
            px += a;
            pk = b > pk ? b : pk;
        }
        tx += a;
        tk = b > tk ? b : tk;
    }
    __syncthreads();
    long long ke = __shfl_up_sync(0xffffffffu, ki, 1);
    if (lane == 0) ke = -1;
    xex = px + xi - x;
    xtot = tx;
    kex = pk > ke ? pk : ke;
    ktot = tk;
}

// ------------------------------------------------------------------------------ K2 / K3
// The tile-level prefixes and the offset table in ONE launch.  Each block of kTileBlock tiles
// publishes its aggregate (entries, LEB128 bytes but its first tile's first gap, first / last
// change as (lane index, tensor)) with a status word, then runs a decoupled look-back: its 256
// threads read the 256 nearest predecessors' published values at once, fold them in age order
// (ordered shuffle trees, then the warps' partials) and stop at the nearest block that has
// published its inclusive prefix, else look 256 blocks further back; then the block publishes
// its own inclusive prefix.  Between two blocks the later block's first gap is the LEB128
// length of its distance to the earlier block's last change when they share a tensor, else of
// its lane index.  Every tile is then placed (entry and byte prefix, first gap
// g0: K4's plan), each tensor's E_k / B_k recorded at its first tile, and the last CTA to finish
// writes the offset table (K3: record sizes and offsets, PAPER.md:382 + SPEC.md:148) and the
// per-tensor emit bases.  Block ids come from a ticket, so a block only waits for blocks that
// started before it (no deadlock whatever the residency); status words carry the launch's
// epoch, so the slots are never cleared between launches.
__device__ __forceinline__ LbAgg lb_combine(const LbAgg &a, const LbAgg &b, int fixed) {
    if (!a.any) return LbAgg{a.cnt + b.cnt, a.bytes + b.bytes, b.fabs, b.labs, b.fk, b.lk, b.any, 0};
    if (!b.any) return LbAgg{a.cnt + b.cnt, a.bytes + b.bytes, a.fabs, a.labs, a.fk, a.lk, a.any, 0};
    const unsigned long long gap = b.fabs - (a.lk == b.fk ? a.labs : 0ull);
    return LbAgg{a.cnt + b.cnt, a.bytes + b.bytes + (fixed ? 0ull : (unsigned long long)leb_len(gap)), a.fabs, b.labs,
                 a.fk, b.lk, 1u, 0};
}
__device__ __forceinline__ uint32_t lb_status_relaxed(const LbSlot *s) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&s->status) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lb_status(const LbSlot *s) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&s->status) : "memory");
    return v;
}
__device__ __forceinline__ LbAgg lb_load(const LbSlot *s, bool inclusive) {
    const unsigned long long *q = reinterpret_cast<const unsigned long long *>(inclusive ? &s->inc : &s->agg);
    LbAgg x;
    unsigned long long *o = reinterpret_cast<unsigned long long *>(&x);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(LbAgg) / 8); ++i) o[i] = __ldcg(q + i);
    return x;
}
__device__ __forceinline__ LbAgg lb_shfl_down(const LbAgg &v, int off) {
    LbAgg x;
    const unsigned long long *i = reinterpret_cast<const unsigned long long *>(&v);
    unsigned long long *o = reinterpret_cast<unsigned long long *>(&x);
#pragma unroll
    for (int k = 0; k < (int)(sizeof(LbAgg) / 8); ++k) o[k] = __shfl_down_sync(0xffffffffu, i[k], off);
    return x;
}
// status kind 1: the block's aggregate is in agg; 2: its inclusive prefix is in inc
__device__ __forceinline__ void lb_publish(LbSlot *s, const LbAgg &x, bool inclusive, uint32_t epoch) {
    if (inclusive) s->inc = x;
    else s->agg = x;
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&s->status), "r"((epoch << 2) | (inclusive ? 2u : 1u))
                 : "memory");
}

__global__ void __launch_bounds__(kTileThreads, 4)
k_tiles_scan(const TileDesc *__restrict__ tiles, const TileMeta *__restrict__ meta, uint32_t ntiles, uint32_t nblk,
             LbSlot *__restrict__ lb, uint32_t epoch, TileEmit *__restrict__ plan, unsigned long long *__restrict__ E,
             unsigned long long *__restrict__ Bk, uint32_t T, const uint32_t *__restrict__ name_len,
             const unsigned long long *__restrict__ numel, RecordRow *__restrict__ table,
             TensorBase *__restrict__ bases, int width, int fixed, ExtractSummary *summary,
             unsigned long long *size_out) {
    if (summary->overflow) {
        if (size_out != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *size_out = ~0ull;
        return;
    }
    __shared__ uint32_t s_b;
    __shared__ LbAgg s_excl, s_agg;
    __shared__ unsigned long long s_labs[kTileThreads];  // per thread: its last change (lane index)
    __shared__ uint32_t s_lk[kTileThreads];              // ... and its tensor
    __shared__ unsigned long long s_fabs, s_bytes[kTileThreads / 32];
    __shared__ uint32_t s_fk;
    __shared__ bool s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_b = atomicAdd(&summary->lb_ticket, 1ull);
    __syncthreads();
    const uint32_t b = s_b;
    const uint32_t blk0 = b * kTileBlock, t0 = blk0 + threadIdx.x * 4;
    // the thread's 4 tiles: metadata and (lane base, tensor), all loads issued together
    TileMeta mt[4];
    unsigned long long lb0[4];
    uint32_t tk[4], tf[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const bool in = t0 + e < ntiles;
        mt[e] = in ? meta[t0 + e] : TileMeta{0, 0, 0, 0, 0};
        const uint4 q = in ? reinterpret_cast<const uint4 *>(tiles + t0 + e)[1] : make_uint4(0, 0, 0, 0);
        lb0[e] = (unsigned long long)q.x | ((unsigned long long)q.y << 32);
        tf[e] = q.w;
        tk[e] = q.w & kTileTensorMask;
    }
    unsigned long long c = 0;
    long long klast = -1;
    int elast = -1;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        c += mt[e].count;
        if (mt[e].count) {
            klast = t0 + e;
            elast = e;
        }
    }
    if (elast >= 0) {  // this thread's last change, for the thread after it
        s_labs[threadIdx.x] = lb0[elast] + mt[elast].last_off;
        s_lk[threadIdx.x] = tk[elast];
    }
    unsigned long long cex, ctot;
    long long kex, ktot;
    block_scan_sum_max(c, klast, cex, ctot, kex, ktot);  // its barriers also publish s_labs / s_lk
    // per tile: its first gap g0 and LEB128 bytes bt, from the last change before it inside the
    // block (an earlier tile of this thread, else the thread owning tile kex); the block's first
    // non-empty tile (kex < 0) gets its first gap after the fold
    bool has_pred = kex >= 0;
    unsigned long long pabs = has_pred ? s_labs[(kex - blk0) >> 2] : 0ull;
    uint32_t pk = has_pred ? s_lk[(kex - blk0) >> 2] : 0xFFFFFFFFu;
    unsigned long long bt[4], g0[4], bloc = 0;
    int efirst = -1;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        bt[e] = 0;
        g0[e] = 0;
        if (!mt[e].count) continue;
        if (fixed) {
            g0[e] = lb0[e];
            bt[e] = (unsigned long long)mt[e].count * fixed_index_width(numel[tk[e]]);
        } else if (has_pred) {
            g0[e] = lb0[e] + mt[e].first_off - (pk == tk[e] ? pabs : 0ull);
            bt[e] = mt[e].internal_bytes + leb_len(g0[e]);
        } else {
            efirst = e;  // the block's first non-empty tile
            bt[e] = mt[e].internal_bytes;
        }
        bloc += bt[e];
        has_pred = true;
        pabs = lb0[e] + mt[e].last_off;
        pk = tk[e];
    }
    if (efirst >= 0 && !fixed) {
        s_fabs = lb0[efirst] + mt[efirst].first_off;
        s_fk = tk[efirst];
    }
    const unsigned long long bsum = warp_sum(bloc);
    if (lane == 0) s_bytes[warp] = bsum;
    __syncthreads();
    // ---- publish the block's aggregate, then fold every predecessor's (all threads)
    if (threadIdx.x == 0) {
        LbAgg agg{ctot, 0, 0, 0, 0, 0, ctot ? 1u : 0u, 0};
#pragma unroll
        for (int w = 0; w < kTileThreads / 32; ++w) agg.bytes += s_bytes[w];
        if (ctot) {
            agg.fabs = fixed ? 0ull : s_fabs;
            agg.fk = fixed ? 0u : s_fk;
            agg.labs = s_labs[(ktot - blk0) >> 2];
            agg.lk = s_lk[(ktot - blk0) >> 2];
        }
        lb_publish(lb + b, agg, b == 0, epoch);  // block 0's aggregate is its inclusive prefix
        s_agg = agg;  // for this thread's inclusive publish below
    }
    // ---- decoupled look-back over windows of 256 predecessors (thread t polls block hi - t,
    // nearest first): the window's published values fold in age order (ordered shuffle trees,
    // then the warps' partials), stopping at the nearest inclusive prefix, else 256 blocks
    // further back; then this block publishes its inclusive prefix (status kind 2)
    {
        __shared__ uint32_t s_im[kTileThreads / 32];
        __shared__ LbAgg s_part[kTileThreads / 32];
        LbAgg excl{0, 0, 0, 0, 0, 0, 0, 0};
        long long hi = (long long)b - 1;
        while (hi >= 0) {
            const long long j = hi - threadIdx.x;
            uint32_t st = 0;
            if (j >= 0) {  // relaxed polls, one acquire once this launch's status is there
                for (uint32_t ns = 32; (lb_status_relaxed(lb + j) >> 2) != epoch; ns = min(2 * ns, 512u))
                    __nanosleep(ns);
                st = lb_status(lb + j);
            }
            const bool inc = j >= 0 && (st & 3u) == 2u;
            const uint32_t im = __ballot_sync(0xffffffffu, inc);
            if (lane == 0) s_im[warp] = im;
            __syncthreads();
            int p = (int)min((long long)kTileThreads - 1, hi);  // threads 0..p take part
            bool found = false;
#pragma unroll
            for (int w = kTileThreads / 32 - 1; w >= 0; --w)
                if (s_im[w]) {
                    p = w * 32 + __ffs(s_im[w]) - 1;
                    found = true;
                }
            LbAgg v = (j >= 0 && (int)threadIdx.x <= p) ? lb_load(lb + j, inc) : LbAgg{0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {  // lane l + off holds an older block
                const LbAgg o = lb_shfl_down(v, off);
                if (lane + off < 32) v = lb_combine(o, v, fixed);
            }
            if (lane == 0) s_part[warp] = v;
            __syncthreads();
            if (threadIdx.x == 0) {
                LbAgg wv = s_part[kTileThreads / 32 - 1];  // warp w + 1 holds older blocks than warp w
#pragma unroll
                for (int w = kTileThreads / 32 - 2; w >= 0; --w) wv = lb_combine(wv, s_part[w], fixed);
                excl = lb_combine(wv, excl, fixed);  // older than the windows folded so far
            }
            if (found || hi < kTileThreads) break;
            hi -= kTileThreads;
            __syncthreads();  // s_im / s_part reused
        }
        if (threadIdx.x == 0) {
            if (b > 0) lb_publish(lb + b, lb_combine(excl, s_agg, fixed), true, epoch);
            s_excl = excl;
        }
    }
    __syncthreads();
    const LbAgg ex = s_excl;
    // ---- place the block's tiles: the block's first non-empty tile's first gap is to the last
    // change before the block in its tensor (or its lane index: the first of its tensor)
    unsigned long long mine = bloc;
    if (efirst >= 0 && !fixed) {
        g0[efirst] = lb0[efirst] + mt[efirst].first_off - ((ex.any && ex.lk == tk[efirst]) ? ex.labs : 0ull);
        const uint32_t l = leb_len(g0[efirst]);
        bt[efirst] += l;
        mine += l;
    }
    unsigned long long bex, btot;
    long long d0, d1;
    block_scan_sum_max(mine, -1, bex, btot, d0, d1);
    unsigned long long ent = ex.cnt + cex;
    unsigned long long byt = (ex.any ? ex.bytes + (fixed ? 0ull : (unsigned long long)leb_len(ex.fabs)) : ex.bytes) + bex;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const uint32_t t = t0 + e;
        if (t >= ntiles) break;
        const uint32_t k = tk[e];
        plan[t] = TileEmit{byt, ent, g0[e], mt[e].count | (fixed ? fixed_index_width(numel[k]) : mt[e].internal_bytes) << 16, k};
        if (tf[e] & kTileFirstOfTensor) {
            E[k] = ent;
            Bk[k] = byt;
        }
        ent += mt[e].count;
        byt += bt[e];
        if (t == ntiles - 1) {
            E[T] = ent;
            Bk[T] = byt;
        }
    }
    // ---- K3, by the last CTA to finish: the offset table and the per-tensor emit bases
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&summary->blocks_done, 1ull) == nblk - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    unsigned long long carry = 0;
    for (uint32_t b0 = 0; b0 < T; b0 += kTileThreads) {
        const uint32_t k = b0 + threadIdx.x;
        unsigned long long rb = 0, nnz = 0, ilen = 0, ek = 0, bk = 0;
        if (k < T) {
            ek = __ldcg(E + k);
            bk = __ldcg(Bk + k);
            nnz = __ldcg(E + k + 1) - ek;
            ilen = __ldcg(Bk + k + 1) - bk;
            rb = 27ull + name_len[k] + ilen + (unsigned long long)width * nnz;
        }
        unsigned long long exs, tot;
        long long d2, d3;
        block_scan_sum_max(rb, -1, exs, tot, d2, d3);
        if (k < T) {
            RecordRow r;
            r.record_offset = carry + exs;
            r.element_count = numel[k];
            r.nnz = nnz;
            r.index_offset = r.record_offset + 2 + name_len[k] + 24;
            r.index_bytes = ilen;
            r.values_offset = r.index_offset + ilen;
            r.record_bytes = rb;
            table[k] = r;
            bases[k] = TensorBase{r.index_offset - bk, r.values_offset - ek * (unsigned long long)width};
        }
        carry += tot;
    }
    if (threadIdx.x == 0) {
        summary->M = __ldcg(E + T);
        summary->idx_bytes = __ldcg(Bk + T);
        summary->body_bytes = carry;
        if (size_out != nullptr) *size_out = carry;
    }
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

// Warp-wide copy of n bytes from a 16-byte aligned source to any destination with 16-byte
// stores: the < 16 head bytes (up to the destination's alignment) by lanes 0-15 and the < 16
// tail bytes by lanes 16-31, one byte store each; every aligned destination vector j is source
// bytes [head + 16 j, +16), i.e. 20 bytes of two aligned source vectors funnel-shifted by the
// (warp-uniform) misalignment.  Reads at most 16 bytes past the source range (slots are padded).
__device__ __forceinline__ void warp_copy16(uint8_t *dst, const uint8_t *src, uint32_t n, int lane) {
    const uint32_t head = min(n, (uint32_t)((16u - ((uintptr_t)dst & 15u)) & 15u));
    const uint32_t rest = n - head, nv = rest >> 4, tail = rest & 15u;
    if ((uint32_t)lane < head) dst[lane] = src[lane];
    const uint32_t tb = head + 16u * nv + (uint32_t)(lane - 16);
    if (lane >= 16 && (uint32_t)(lane - 16) < tail) dst[tb] = src[tb];
    uint4 *d16 = reinterpret_cast<uint4 *>(dst + head);
    const uint4 *s16 = reinterpret_cast<const uint4 *>(src);
    const uint32_t qv = head >> 2, sh = 8u * (head & 3u);  // word offset into the vector pair, bit shift
    for (uint32_t j = lane; j < nv; j += 32) {
        const uint4 a = __ldg(s16 + j), b = __ldg(s16 + j + 1);
        uint32_t w0, w1, w2, w3, w4;  // source words qv .. qv + 4 of the pair (a, b)
        if (qv == 0) { w0 = a.x; w1 = a.y; w2 = a.z; w3 = a.w; w4 = b.x; }
        else if (qv == 1) { w0 = a.y; w1 = a.z; w2 = a.w; w3 = b.x; w4 = b.y; }
        else if (qv == 2) { w0 = a.z; w1 = a.w; w2 = b.x; w3 = b.y; w4 = b.z; }
        else { w0 = a.w; w1 = b.x; w2 = b.y; w3 = b.z; w4 = b.w; }
        d16[j] = make_uint4(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh), __funnelshift_r(w2, w3, sh),
                            __funnelshift_r(w3, w4, sh));
    }
}

// Tiles whose in-tile bytes and values each fit kPref bytes go through K4's shared-memory ring.
constexpr uint32_t kPref = 496;

// The emit gate (K4/K5): the local body is written iff every tile fitted its slot and the body
// fits `cap`; the fused-assembly copy (peer.base) iff, in addition, no rank's size is ~0 (its
// extract did not complete) and this rank's records fit the peer buffer at sum(sizes[q < rank]).
struct EmitGate {
    bool local, peer;
    unsigned long long off;  // this rank's byte offset in the peer buffer
    unsigned long long fail; // ExtractSticky::peer_fail code when the peer copy is skipped
};
__device__ __forceinline__ EmitGate emit_gate(const ExtractSummary *summary, unsigned long long cap,
                                              const PeerDst &peer) {
    EmitGate g{!summary->overflow && summary->body_bytes <= cap, false, 0, 0};
    if (peer.base != nullptr && g.local) {
        bool ok = true;
        for (uint32_t q = 0; q < peer.n_ranks; ++q) {
            const unsigned long long z = peer.sizes[q];
            if (z == ~0ull) ok = false;
            else if (q < peer.rank) g.off += z;
        }
        if (!ok) g.fail = 1;
        else if (g.off > peer.cap || summary->body_bytes > peer.cap - g.off) g.fail = 2;
        g.peer = g.fail == 0;
    }
    return g;
}

// FIXED codec K4 (reading R18): one warp per tile, absolute indices lane_base + offset as u32 /
// u64 built in shared memory, then the values.
template <int W>
__global__ void __launch_bounds__(256, 3)
k_emit_fixed(const TileEmit *__restrict__ plan, const TensorBase *__restrict__ bases, uint32_t ntiles, uint32_t slot_cap,
             const uint8_t *__restrict__ slot_bytes, const typename LaneOf<W>::T *__restrict__ slot_val,
             uint8_t *__restrict__ out, const ExtractSummary *summary, unsigned long long cap, PeerDst peer) {
    const EmitGate gate = emit_gate(summary, cap, peer);
    if (!gate.local) return;  // emit gate (async extract)
    uint8_t *const pout = gate.peer ? peer.base + gate.off : nullptr;  // fused assembly: the same bytes there too
    const int lane = threadIdx.x & 31;
    const uint32_t wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    {
        __shared__ __align__(16) unsigned long long s_fix[8 * 256 + 2];
        for (uint32_t t = wg; t < ntiles; t += nw) {
            const TileEmit pe = plan[t];
            const uint32_t count = pe.count_internal & 0xFFFFu;
            if (count == 0) continue;
            const TensorBase tb = bases[pe.k];
            uint8_t *ib = out + (tb.ib + pe.ib);
            uint8_t *vb = out + (tb.vb + pe.eb * W);
            const uint8_t *sv = reinterpret_cast<const uint8_t *>(slot_val + (size_t)t * slot_cap);
            const uint32_t iw = pe.count_internal >> 16;  // the index width (set by K2 for FIXED)
            const uint16_t *so = reinterpret_cast<const uint16_t *>(slot_bytes + (size_t)t * 2 * slot_cap);
            unsigned long long *buf = s_fix + 256 * (threadIdx.x >> 5);
            uint8_t *dst = ib, *pdst = pout ? pout + (ib - out) : nullptr;
            for (uint32_t b = 0; b < count; b += 256) {
                const uint32_t n = min(256u, count - b);
                for (uint32_t i = lane; i < n; i += 32) {
                    const unsigned long long x = pe.g0 + so[b + i];
                    if (iw == 4) reinterpret_cast<uint32_t *>(buf)[i] = (uint32_t)x;
                    else buf[i] = x;
                }
                __syncwarp();
                warp_copy4<false>(dst, reinterpret_cast<const uint8_t *>(buf), n * iw, lane);
                if (pdst) {  // fused assembly: the same bytes at their global offset
                    warp_copy4<false>(pdst, reinterpret_cast<const uint8_t *>(buf), n * iw, lane);
                    pdst += (size_t)n * iw;
                }
                __syncwarp();
                dst += (size_t)n * iw;
            }
            warp_copy(vb, sv, count * W, lane);
            if (pout) warp_copy(pout + (vb - out), sv, count * W, lane);
        }
        return;
    }
}

// LEB128 K4 with a shared-memory ring: each warp keeps S steps of slot bytes in flight through
// cp.async (LDGSTS, no registers held), plans 2S steps ahead, so a tile's DRAM latency overlaps
// the stores of the tiles before it (a register prefetch held one tile and ran 0.21 ms vs
// 0.15 ms at M3; 1-D TMA bulk copies per tile, 0.24 ms, were slower still).  Per tile and
// stage: 512 + 512 bytes of data (in-tile LEB128 bytes, values) and the tensor's emit bases;
// plans 2S steps ahead.  Tiles with a segment > kPref bytes take the synchronous copies.
constexpr uint32_t kRingData = 1024;

__device__ __forceinline__ void cp_async16(void *smem, const void *g) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}
// zero-fill form: src_bytes = 0 reads nothing and writes 16 zero bytes (no branch around it)
__device__ __forceinline__ void cp_async16_zfill(void *smem, const void *g, bool on) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(g), "r"(on ? 16u : 0u) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// n <= kPref bytes staged at s (16-byte aligned shared memory, vectors 0 .. n / 16 valid) to
// any destination: head bytes (lanes 0-15), 16-byte vectors funnel-shifted from two staged
// vectors, tail bytes (lanes 16-31) — the same split as warp_copy16.
template <int QV>
__device__ __forceinline__ void ring_vec(const uint8_t *s, uint8_t *dst, uint32_t head, uint32_t sh, int lane) {
    const uint4 *s16 = reinterpret_cast<const uint4 *>(s);
    const uint4 a = s16[lane], b = s16[lane + 1];
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    reinterpret_cast<uint4 *>(dst + head)[lane] =
        make_uint4(__funnelshift_r(w[QV], w[QV + 1], sh), __funnelshift_r(w[QV + 1], w[QV + 2], sh),
                   __funnelshift_r(w[QV + 2], w[QV + 3], sh), __funnelshift_r(w[QV + 3], w[QV + 4], sh));
}
// K4 proper: each lane group of L = 16 lanes (a half-warp) takes one tile, a warp two at a
// time, so the per-tile bookkeeping (plans, bases, addresses, first-gap bytes, copy issue)
// runs once per two tiles in each instruction; a ~330-byte values segment then takes two
// 16-lane passes instead of one 32-lane (0.154 -> 0.120 ms at M3).
template <int S, int P>
__host__ __device__ constexpr uint32_t pair_warp_bytes() { return S * P * (kRingData + 16) + 2 * S * P * 32; }

// n <= kPref bytes staged at s to any destination, by the L lanes hl = 0..L-1 of a lane group
template <int L>
__device__ __forceinline__ void ring_store_h(const uint8_t *s, uint8_t *dst, uint32_t n, int hl) {
    const uint32_t head = min(n, (uint32_t)((16u - ((uintptr_t)dst & 15u)) & 15u));
    const uint32_t rest = n - head, nv = rest >> 4, tail = rest & 15u;
    for (uint32_t b = hl; b < head; b += L) dst[b] = s[b];
    for (uint32_t b = hl; b < tail; b += L) dst[head + 16u * nv + b] = s[head + 16u * nv + b];
    const uint32_t sh = 8u * (head & 3u);
    for (uint32_t j = hl; j < nv; j += L) {
        switch (head >> 2) {
        case 0: ring_vec<0>(s, dst, head, sh, (int)j); break;
        case 1: ring_vec<1>(s, dst, head, sh, (int)j); break;
        case 2: ring_vec<2>(s, dst, head, sh, (int)j); break;
        default: ring_vec<3>(s, dst, head, sh, (int)j); break;
        }
    }
}
// the same from a 16-byte aligned global source of any length (dense tiles), U vectors per
// lane per round
template <int L, int U>
__device__ __forceinline__ void half_copy16(uint8_t *dst, const uint8_t *src, uint32_t n, int hl) {
    const uint32_t head = min(n, (uint32_t)((16u - ((uintptr_t)dst & 15u)) & 15u));
    const uint32_t rest = n - head, nv = rest >> 4, tail = rest & 15u;
    for (uint32_t b = hl; b < head; b += L) dst[b] = src[b];
    for (uint32_t b = hl; b < tail; b += L) dst[head + 16u * nv + b] = src[head + 16u * nv + b];
    uint4 *d16 = reinterpret_cast<uint4 *>(dst + head);
    const uint4 *s16 = reinterpret_cast<const uint4 *>(src);
    const uint32_t qv = head >> 2, sh = 8u * (head & 3u);
    // all U loads of a round issued before its stores (a dense tile's segment is up to 32 KiB:
    // with U = 1 every 16 lanes x 16 bytes cost a load-store round trip)
    for (uint32_t j0 = hl; j0 < nv; j0 += U * L) {
        uint4 a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t j = j0 + u * L;
            if (j < nv) {
                a[u] = __ldg(s16 + j);
                b[u] = __ldg(s16 + j + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t j = j0 + u * L;
            if (j >= nv) break;
            uint32_t w0, w1, w2, w3, w4;
            if (qv == 0) { w0 = a[u].x; w1 = a[u].y; w2 = a[u].z; w3 = a[u].w; w4 = b[u].x; }
            else if (qv == 1) { w0 = a[u].y; w1 = a[u].z; w2 = a[u].w; w3 = b[u].x; w4 = b[u].y; }
            else if (qv == 2) { w0 = a[u].z; w1 = a[u].w; w2 = b[u].x; w3 = b[u].y; w4 = b[u].z; }
            else { w0 = a[u].w; w1 = b[u].x; w2 = b[u].y; w3 = b[u].z; w4 = b[u].w; }
            d16[j] = make_uint4(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh), __funnelshift_r(w2, w3, sh),
                                __funnelshift_r(w3, w4, sh));
        }
    }
}

template <int W, int S, int L, int U>
__global__ void __launch_bounds__(256)
k_emit_pair(const TileEmit *__restrict__ plan, const TensorBase *__restrict__ bases, uint32_t ntiles, uint32_t slot_cap,
            const uint8_t *__restrict__ slot_bytes, const typename LaneOf<W>::T *__restrict__ slot_val,
            uint8_t *__restrict__ out, const ExtractSummary *summary, unsigned long long cap, PeerDst peer) {
    const EmitGate gate = emit_gate(summary, cap, peer);
    if (!gate.local) return;  // emit gate (async extract)
    uint8_t *const pout = gate.peer ? peer.base + gate.off : nullptr;  // fused assembly: the same bytes there too
    extern __shared__ __align__(16) uint8_t s_ring[];
    constexpr int P = 32 / L;  // tiles per warp step
    const int lane = threadIdx.x & 31, h = lane / L, hl = lane % L;
    uint8_t *const sdata = s_ring + (threadIdx.x >> 5) * pair_warp_bytes<S, P>();
    TensorBase *const sbase = reinterpret_cast<TensorBase *>(sdata + S * P * kRingData);
    TileEmit *const splan = reinterpret_cast<TileEmit *>(sdata + S * P * (kRingData + 16));
    const uint32_t wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    const uint32_t mine = wg < ntiles ? (ntiles - wg + nw - 1) / nw : 0;  // tiles of this warp: wg + m nw
    const uint32_t pairs = (mine + P - 1) / P;                            // step q: tiles m = Pq + h
    auto slot_i = [&](uint32_t t) { return slot_bytes + (size_t)t * 2 * slot_cap; };
    auto slot_v = [&](uint32_t t) { return reinterpret_cast<const uint8_t *>(slot_val + (size_t)t * slot_cap); };
    auto fast = [&](const TileEmit &p) {
        return (p.count_internal >> 16) <= kPref && (p.count_internal & 0xFFFFu) * W <= kPref;
    };
    auto issue_plan = [&](uint32_t q) {  // plan of this half's tile of pair q -> plan slot (q % 2S, h)
        const uint32_t m = P * q + h;
        if (m < mine && hl < 2)
            cp_async16(reinterpret_cast<uint8_t *>(splan + (q % (2 * S)) * P + h) + 16 * hl,
                       reinterpret_cast<const uint8_t *>(plan + (wg + m * nw)) + 16 * hl);
    };
    auto issue_data = [&](uint32_t q) {  // its slot bytes and emit bases -> stage (q % S, h)
        const uint32_t m = P * q + h;
        if (m >= mine) return;
        const TileEmit p = splan[(q % (2 * S)) * P + h];
        const uint32_t count = p.count_internal & 0xFFFFu, ni = p.count_internal >> 16, nv = count * W;
        if (count == 0 || !fast(p)) return;
        const uint32_t t = wg + m * nw;
        uint8_t *d = sdata + ((q % S) * P + h) * kRingData;
#pragma unroll
        for (int r = 0; r < 32 / L; ++r) {
            const uint32_t v = hl + L * r;
            cp_async16_zfill(d + 16 * v, slot_i(t) + 16 * v, v <= (ni >> 4));
            cp_async16_zfill(d + 512 + 16 * v, slot_v(t) + 16 * v, v <= (nv >> 4));
        }
        if (hl == 0) cp_async16(sbase + (q % S) * P + h, bases + p.k);
    };
    for (uint32_t q = 0; q < 2 * S - 1; ++q) issue_plan(q);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    for (uint32_t q = 0; q < S - 1; ++q) {
        issue_data(q);
        cp_async_commit();
    }
    for (uint32_t q = 0; q < pairs; ++q) {
        issue_plan(q + 2 * S - 1);  // into the slots of pair q - 1 (stored last iteration)
        issue_data(q + S - 1);      // into the stage of pair q - 1
        cp_async_commit();
        cp_async_wait<S - 1>();     // pair q's group (and the plans of pair q + S) landed
        __syncwarp();
        const uint32_t m = P * q + h;
        const TileEmit pc = m < mine ? splan[(q % (2 * S)) * P + h] : TileEmit{0, 0, 0, 0, 0};
        const uint32_t count = pc.count_internal & 0xFFFFu;
        if (count) {
            const bool f = fast(pc);
            const TensorBase tb = f ? sbase[(q % S) * P + h] : bases[pc.k];
            uint8_t *ib = out + (tb.ib + pc.ib);
            uint8_t *vb = out + (tb.vb + pc.eb * W);
            // the first gap: byte n = 7-bit group n, continuation bit on all but the last
            const unsigned long long g = pc.g0;
            const uint32_t L0 = leb_len(g);
            const uint32_t ni = pc.count_internal >> 16, nv = count * W;
            const uint8_t *sd = sdata + ((q % S) * P + h) * kRingData;
            const uint32_t t = wg + m * nw;
            for (int d = 0; d < (pout ? 2 : 1); ++d) {  // d = 1: fused assembly (NVLink stores)
                uint8_t *di = d ? pout + (ib - out) : ib;
                uint8_t *dv = d ? pout + (vb - out) : vb;
                for (uint32_t b = hl; b < L0; b += L)
                    di[b] = (uint8_t)(((g >> (7 * b)) & 0x7Fu) | (b + 1 < L0 ? 0x80u : 0u));
                if (f) {
                    ring_store_h<L>(sd, di + L0, ni, hl);
                    ring_store_h<L>(sd + 512, dv, nv, hl);
                } else {  // a dense tile: synchronous copies
                    half_copy16<L, U>(di + L0, slot_i(t), ni, hl);
                    half_copy16<L, U>(dv, slot_v(t), nv, hl);
                }
            }
        }
        __syncwarp();  // stage q % S and plan slots q % 2S are refilled from the next iterations
    }
    cp_async_wait<0>();
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
          unsigned long long *size_out, ExtractSticky *sticky, PeerDst peer) {
    const EmitGate gate = emit_gate(summary, cap, peer);
    const bool open = gate.local;
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
        if (sticky != nullptr && gate.fail) sticky->peer_fail = max(sticky->peer_fail, gate.fail);
    }
    if (!open) return;
    for (int dst = 0; dst < (gate.peer ? 2 : 1); ++dst)
    for (uint32_t k = blockIdx.x; k < T; k += gridDim.x) {
        const RecordRow r = table[k];
        uint8_t *o = (dst ? peer.base + gate.off : out) + r.record_offset;
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
    // K1's emission switches to vector order at this many changes per tile (DELTA_K1_DENSE_TILE
    // overrides it for experiments; results never depend on it)
    static const uint32_t dense_tile = [] {
        const char *e = getenv("DELTA_K1_DENSE_TILE");
        return e != nullptr ? (uint32_t)atoi(e) : kDenseTile;
    }();
    if (ev) cudaEventRecord(ev[0], s);
    if (a.ntiles)
        (a.index_codec ? (a.advance ? k_scan_tiles<W, false, true, true>
                                    : a.mode == 1 ? k_scan_tiles<W, true, false, true> : k_scan_tiles<W, false, false, true>)
                       : (a.advance ? k_scan_tiles<W, false, true> : a.mode == 1 ? k_scan_tiles<W, true> : k_scan_tiles<W>))
            <<<a.ntiles, 256, 0, s>>>(a.tiles, a.ntiles, a.prefetch_dist, a.slot_cap, a.slot_bytes,
                                      static_cast<LT *>(a.slot_val), a.meta, a.summary, a.redo_cap, dense_tile);
    if (ev) cudaEventRecord(ev[1], s);
    const uint32_t nblk = (a.ntiles + kTileBlock - 1) / kTileBlock;
    if (nblk)
        k_tiles_scan<<<nblk, kTileThreads, 0, s>>>(a.tiles, a.meta, a.ntiles, nblk, a.lb, a.epoch, a.plan,
                                                   a.entry_begin, a.tensor_byte_begin, a.ntensors, a.name_len,
                                                   a.numel, a.table, a.bases, a.width, a.index_codec, a.summary,
                                                   a.scan_size_out);
    if (ev && !a.prof_k1_only) {
        cudaEventRecord(ev[2], s);
        cudaEventRecord(ev[3], s);
    }
    return cudaGetLastError();
}

// K4's ring depth: 2 stages (measured: 3, 4, 6, 8 no faster, more shared memory per CTA);
// 16 lanes per tile, two tiles per warp step (measured: 0.154 ms with 32 lanes per tile,
// 0.120 with 16, 0.160 with 8 — the 8-lane form fits 3 CTAs per SM)
constexpr int kEmitStages = 2, kEmitLanes = 16;

template <int W, int L, int U>
static void launch_pair(const ExtractArgs &a, uint8_t *out, cudaStream_t s) {
    constexpr uint32_t psmem = 8 * pair_warp_bytes<kEmitStages, 32 / L>();
    static const bool attr = [] {
        cudaFuncSetAttribute(k_emit_pair<W, kEmitStages, L, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
        return true;
    }();
    (void)attr;
    k_emit_pair<W, kEmitStages, L, U><<<a.persist_ctas, 256, psmem, s>>>(
        a.plan, a.bases, a.ntiles, a.slot_cap, a.slot_bytes, static_cast<const typename LaneOf<W>::T *>(a.slot_val), out,
        a.summary, a.out_cap, a.peer);
}

// Dense tiles (segments > kPref bytes) are copied from global memory; the 4-deep unrolled copy
// costs registers (53 -> 118: 2 instead of 4 CTAs per SM), so it is taken only once the slots
// have grown past their initial 2 KiB per tile (some tile held > 1024 bf16 / 512 fp32 entries).
template <int W>
static void launch_ring(const ExtractArgs &a, uint8_t *out, cudaStream_t s) {
    if ((size_t)a.slot_cap * W > 2048) launch_pair<W, kEmitLanes, 4>(a, out, s);
    else launch_pair<W, kEmitLanes, 1>(a, out, s);
}

template <int W>
static cudaError_t emit_impl(const ExtractArgs &a, uint8_t *out, cudaStream_t s, cudaEvent_t *ev) {
    using LT = typename LaneOf<W>::T;
    if (ev) cudaEventRecord(ev[0], s);
    if (a.index_codec)
        k_emit_fixed<W><<<a.persist_ctas, 256, 0, s>>>(a.plan, a.bases, a.ntiles, a.slot_cap, a.slot_bytes,
                                                       static_cast<const LT *>(a.slot_val), out, a.summary, a.out_cap,
                                                       a.peer);
    else
        launch_ring<W>(a, out, s);
    if (ev) cudaEventRecord(ev[1], s);
    const uint32_t hb = a.ntensors < 65535u ? (a.ntensors ? a.ntensors : 1u) : 65535u;
    k_headers<<<hb, 128, 0, s>>>(a.table, a.ntensors, a.name_len, a.name_off, a.names, out, a.mode, a.summary,
                                 a.out_cap, a.size_out, a.sticky, a.peer);
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
