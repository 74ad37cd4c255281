// sd_internal.cuh — structures shared by the C-ABI host code (api.cu) and the sm_100a
// kernels (extract.cu, apply.cu).  Product code; shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sd {

// ---------------------------------------------------------------- extract geometry
constexpr int kScanThreads = 256;  // K1 block
constexpr int kScanVecs = 8;       // 16-byte vectors per thread per operand per tile
constexpr int kTileBytes = kScanThreads * kScanVecs * 16;  // 32 KiB of old + 32 KiB of new
// lanes per tile: 16384 (16-bit lanes) or 8192 (32-bit lanes) -> a lane offset fits a u16
constexpr uint32_t kDenseTile = 4096;  // K1: tiles with this many changes (25 %) emit in vector order
constexpr int kTileThreads = 256;  // threads of the tile-level scan kernel (K2)
constexpr int kTileBlock = kTileThreads * 4;  // tiles per block of the tile-level scans (4 per thread)
constexpr int kByteChunk = 4096;   // index-stream bytes per A2/A4 chunk (256 threads x 16)
constexpr int kHalo = 16;          // bytes before a chunk kept for varints that straddle it
constexpr uint32_t kStageGapBytes = 2048;

constexpr uint32_t kTileFirstOfTensor = 1u << 31;
constexpr uint32_t kTileAligned = 1u << 30;
constexpr uint32_t kTileTensorMask = (1u << 30) - 1;

// One tile = a run of lanes of one span of one tensor (never straddles a span).
struct TileDesc {
    const uint8_t *old_p;   // first lane of the tile
    const uint8_t *new_p;
    uint64_t lane_base;     // index of the tile's first lane within the fused tensor
    uint32_t nlanes;        // <= lanes per tile; 0 for the placeholder tile of an empty tensor
    uint32_t flags_tensor;  // tensor id | kTileFirstOfTensor | kTileAligned
};
static_assert(sizeof(TileDesc) == 32, "TileDesc is 32 bytes");

// K1 output per tile: changed-lane count, lane offsets (within the tile) of the first and
// last changed lane, and the LEB128 bytes of the gaps between consecutive changes inside
// the tile (the first change's gap depends on earlier tiles and is added by K2).
struct TileMeta {
    uint32_t count;
    uint16_t first_off, last_off;
    uint32_t internal_bytes;
    uint32_t pad;
};
static_assert(sizeof(TileMeta) == 16, "TileMeta is 16 bytes");

// K2 output per tile: everything K4 needs besides its tensor's bases, in one 32-byte load.
struct TileEmit {
    unsigned long long ib;   // LEB128 bytes of all tiles before this one (all tensors)
    unsigned long long eb;   // entries of all tiles before this one (all tensors)
    unsigned long long g0;   // gap of the tile's first change (to the previous change, or absolute)
    uint32_t count_internal; // changes in the tile | in-tile gap bytes (FIXED: index width) << 16
    uint32_t k;              // tensor
};
// K2's cross-block fold: per block of tiles its aggregate, published with a status word.
struct LbAgg {
    unsigned long long cnt;    // entries
    unsigned long long bytes;  // LEB128 bytes, except the first gap of the first non-empty tile
    unsigned long long fabs, labs;  // first / last change: lane index within its tensor
    uint32_t fk, lk;           // ... and its tensor
    uint32_t any, pad;         // any change at all
};
struct LbSlot {
    LbAgg agg, inc;            // the block's aggregate; its inclusive prefix (all blocks up to it)
    uint32_t status;           // (launch epoch << 2) | 1 once agg is written, | 2 once inc is
    uint32_t pad[3];
};

// Per tensor (written with the offset table): body offset of a tile's first index byte =
// ib + TileEmit::ib, of its first value = vb + TileEmit::eb * w.
struct TensorBase {
    unsigned long long ib, vb;
};
static_assert(sizeof(TileEmit) == 32, "TileEmit is 32 bytes");

// Device-written summary of one extract, read back by the host after the single sync.
struct ExtractSummary {
    unsigned long long M;           // total changed lanes (entries) over all tensors
    unsigned long long overflow;    // != 0: some tile had more entries than its slot holds
    unsigned long long max_count;   // largest per-tile count seen (sizes the slots on retry)
    unsigned long long idx_bytes;   // total LEB128 bytes over all tensors
    unsigned long long body_bytes;  // packed body size
    unsigned long long blocks_done; // K2 tickets (the last CTA writes the offset table)
    unsigned long long lb_ticket;   // K2 logical block ids (look-back order)
};

// Sticky outcome of the delta_extract_async calls since the last delta_extract_wait (folded
// in by K5 of every async extract; the per-call summary is reset by each call).
struct ExtractSticky {
    unsigned long long overflow;    // some call's tiles overflowed their slots
    unsigned long long max_count;   // largest per-tile count over those calls
    unsigned long long over_cap;    // some call's body exceeded its capacity
    unsigned long long need;        // largest such body
    unsigned long long peer_fail;   // fused assembly skipped: 1 a rank's size was ~0, 2 no room
};

// Fused emit + assembly (delta_extract_emit_async): a second destination for the body, e.g.
// the root's assembled-body buffer mapped with CUDA IPC, at the offset sum(sizes[q < rank]).
struct PeerDst {
    uint8_t *base = nullptr;               // nullptr: no second destination
    unsigned long long cap = 0;
    const unsigned long long *sizes = nullptr;  // n_ranks body sizes (device)
    uint32_t n_ranks = 0, rank = 0;
};

// Per-tensor row of the device offset table (same field order as delta_record_info).
struct RecordRow {
    unsigned long long record_offset, element_count, nnz, index_offset, index_bytes,
        values_offset, record_bytes;
};
static_assert(sizeof(RecordRow) == 56, "RecordRow matches delta_record_info");

// ---------------------------------------------------------------- apply
struct TargetDesc {
    uint8_t *w;
    unsigned long long numel;
    unsigned long long name_off;  // into the names blob (delta_merge: into the second body)
    unsigned long long name_len;
};

// Fixed-width index codec (reading R18): 4-byte indices iff N - 1 fits int32.
__host__ __device__ __forceinline__ uint32_t fixed_index_width(unsigned long long n) {
    return n <= 0x80000000ull ? 4u : 8u;
}

struct ApplyRec {  // located + verified record
    unsigned long long idx_off, idx_len, val_off, nnz, numel;
    uint8_t *w;
    unsigned long long mode;  // 0 replace (scatter-store), 1 additive (scatter-add)
};

// Status word codes written by the apply kernels (DELTA_D_* of sparsedelta.h).
enum : uint32_t {
    kOk = 0, kTruncated = 1, kOverlong = 2, kOverflow = 3, kNonIncreasing = 4, kRange = 5,
    kCount = 6, kName = 7, kNumel = 8, kMode = 9, kLayout = 10
};

struct ApplyState {
    uint32_t status;       // first error code of the current call (0 = ok): the gate
    uint32_t first_error;  // first error since the last delta_apply_wait (sticky)
    unsigned long long n_chunks;
};

// ---------------------------------------------------------------- launchers (extract.cu / apply.cu)
struct ExtractArgs {
    const TileDesc *tiles;
    uint32_t ntiles;
    uint32_t ntensors;
    uint32_t slot_cap;                // C: entries per tile slot (even)
    uint8_t *slot_bytes;              // ntiles x 2C LEB128 bytes of the gaps inside the tile
    void *slot_val;                   // ntiles x C lanes
    TileMeta *meta;                   // ntiles
    TileEmit *plan;                   // ntiles: K4's per-tile plan
    LbSlot *lb = nullptr;             // per tile block: K2's published aggregates
    uint32_t epoch = 0;               // K2 launch epoch (status words of older launches are stale)
    TensorBase *bases;                // ntensors: K4's per-tensor body bases
    const uint32_t *tensor_first_tile;  // ntensors
    unsigned long long *entry_begin;  // ntensors + 1 (E_k)
    unsigned long long *tensor_byte_begin;  // ntensors + 1 (B_k)
    RecordRow *table;                 // ntensors
    const uint32_t *name_len;         // ntensors
    const uint32_t *name_off;         // ntensors
    const uint8_t *names;             // blob
    const unsigned long long *numel;  // ntensors (N_k)
    ExtractSummary *summary;
    int width;                        // 2 or 4
    int persist_ctas;                 // grid for grid-stride kernels
    int sm_count;
    uint32_t prefetch_dist;           // K1 (0): L2 bulk prefetch distance in tiles (0 = off)
    int mode;                         // record mode: 0 replace, 1 additive
    int index_codec;                  // 0 LEB128 gaps, 1 fixed-width absolute (R18)
    bool advance = false;             // K1 also stores every changed new lane into old (extract-and-advance)
    bool prof_k1_only = false;        // profiling mode 3: events around K1 only (ev[0], ev[1])
    uint32_t redo_cap = 0;            // advance retry: only tiles with count > redo_cap run K1 again
    // emit gate (K4/K5 write nothing unless the scan fitted its slots and body <= out_cap);
    // size_out (device, may be NULL) receives the body size, or ~0 when the gate is closed
    unsigned long long out_cap = ~0ull;
    unsigned long long *size_out = nullptr;
    ExtractSticky *sticky = nullptr;  // async extracts: outcome folded in by K5
    unsigned long long *scan_size_out = nullptr;  // K2: the body size, or ~0 if a tile overflowed
    PeerDst peer;                     // K4/K5: fused assembly destination
};

// ev: nullptr, or events recorded around the kernels (scan: 4 = before K1, after K1,
// after the tile scans K2, after K3; emit: 3 = before K4, after K4, after K5).
cudaError_t launch_extract_scan(const ExtractArgs &a, cudaStream_t s, cudaEvent_t *ev);    // K1-K3
cudaError_t launch_extract_emit(const ExtractArgs &a, uint8_t *out, cudaStream_t s, cudaEvent_t *ev);  // K4-K5
cudaError_t launch_slots_regrow(const TileMeta *meta, uint32_t ntiles, int width, uint32_t old_cap,
                                const void *ob, const void *ov, uint32_t new_cap, void *nb, void *nv, int ctas,
                                cudaStream_t s);

struct ApplyArgs {
    const uint8_t *body;
    unsigned long long body_bytes;                 // bytes, or the capacity when body_bytes_dev is set
    const unsigned long long *body_bytes_dev = nullptr;  // device-resident size (chained apply)
    const TargetDesc *targets;
    uint32_t n;
    const uint8_t *names;
    const RecordRow *hint;            // device copy of the host hint, or nullptr
    ApplyRec *recs;                   // n
    unsigned long long *rec_chunk_begin;  // n + 1
    uint32_t *chunk_rec;              // chunk -> record
    unsigned int *chunk_count;
    unsigned long long *chunk_sum;
    unsigned long long *chunk_ord_base;
    unsigned long long *chunk_idx_base;
    unsigned long long chunk_cap;
    ApplyState *state;
    int width;
    int persist_ctas;
    int scatter_ctas;
    bool entry_major;                 // scatter store order (see k_scatter)
    bool dense_hint = false;          // body > w / 8 bytes per target lane (~5 % density): A4 at 6 CTAs/SM
    int index_codec;                  // 0 LEB128 gaps, 1 fixed-width absolute indices (R18)
};

cudaError_t launch_spdc_header(uint8_t *out, const uint32_t *digest, uint32_t format_version,
                               unsigned long long version, unsigned long long base_version, uint32_t elem_code,
                               uint32_t n_tensors, unsigned long long body_bytes, cudaStream_t s);
cudaError_t launch_blake3(const uint8_t *in, unsigned long long n, uint32_t *ws, uint32_t *out32, cudaStream_t s);

cudaError_t launch_record_sizes(const RecordRow *table, uint32_t n_local, const uint32_t *gidx,
                                unsigned long long *sizes, uint32_t n_global, cudaStream_t s);
cudaError_t launch_assemble_records(const uint8_t *src, uint8_t *dst, unsigned long long capacity,
                                    const unsigned long long *sizes, const uint32_t *gidx, uint32_t n_local,
                                    uint32_t n_global, unsigned long long *goff, unsigned long long *loff,
                                    uint32_t *status, int ctas, cudaStream_t s);
cudaError_t launch_assemble(const uint8_t *src, uint8_t *dst, unsigned long long capacity,
                            const unsigned long long *sizes, uint32_t rank, uint32_t *status, int ctas,
                            cudaStream_t s);

// ev: nullptr, or 5 events: before A1, after A1, A2, A3, A4.
cudaError_t launch_apply(const ApplyArgs &a, cudaStream_t s, cudaEvent_t *ev);  // A1-A4
// A1-A3, then (gated) every entry's absolute index and value written to idx_out / val_out at
// entry_base[record] + ordinal (delta_merge's decode of a body; targets carry no w).
cudaError_t launch_decode_only(const ApplyArgs &a, unsigned long long *idx_out, void *val_out,
                               const unsigned long long *entry_base, cudaStream_t s);
// delta_merge (merge.cu): see api.cu.  Entries are keyed (record << kKeyShift) | index, so
// element counts must stay below 2^40 (checked by the walk).
constexpr int kKeyShift = 40;
constexpr uint32_t kMergeTooLarge = 11;  // walk status: an element count >= 2^40
struct MergeArgs {
    const uint8_t *a, *b;                 // the two bodies
    unsigned long long a_bytes, b_bytes;
    uint32_t n;                           // records expected in each
    int width;
    TargetDesc *targets;                  // n: B's names / element counts, for A1 of both decodes
    RecordRow *ha, *hb;                   // n: table rows of a and b (the decodes' hints)
    uint32_t *name_len;                   // n
    unsigned long long *name_off;         // n (into body b)
    unsigned long long *numel;            // n
    unsigned long long *ea, *eb, *eu;     // n + 1 entry prefixes of a, b and the union
    uint32_t *status;                     // walk status (kOk / k* code)
    unsigned long long *ia, *ib;          // decoded keys (record << kKeyShift | index), ascending
    void *va, *vb;                        // decoded values
    uint32_t *tile_cnt;                   // merge-path tiles: kept entries per tile (scan input)
    unsigned long long *tile_off;         // tiles + 1: exclusive scan of tile_cnt
    unsigned long long ntiles;
    unsigned long long *split;            // ntiles + 1: a-entries before each tile boundary
    unsigned long long *bstat;            // ntiles + 1: look-back status of the tiles' LEB128 bytes
    unsigned long long *u;                // mu merged keys
    void *uv;                             // mu merged values
    uint32_t *len;                        // mu LEB128 lengths
    unsigned long long *lo;               // mu + 1 byte offsets (exclusive scan of len)
    unsigned long long *blk;              // scan scratch
    RecordRow *table;                     // n
    unsigned long long *body_size;        // 1
    unsigned long long ma, mb, mu;
};
cudaError_t launch_merge_walk(const MergeArgs &m, cudaStream_t s);
cudaError_t launch_merge_count(const MergeArgs &m, cudaStream_t s);    // tile_cnt, tile_off
cudaError_t launch_merge_place(const MergeArgs &m, cudaStream_t s);    // u, uv, eu, len, lo, table, body_size
cudaError_t launch_merge_emit(const MergeArgs &m, uint8_t *out, cudaStream_t s);

}  // namespace sd
