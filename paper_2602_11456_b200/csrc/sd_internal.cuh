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
constexpr int kEntryChunk = 4096;  // entries per K2/K4 chunk (256 threads x 16)
constexpr int kEntryPerThread = kEntryChunk / 256;
constexpr int kByteChunk = 4096;   // index-stream bytes per A2/A4 chunk (256 threads x 16)
constexpr int kHalo = 16;          // bytes before a chunk kept for varints that straddle it

// Tile-state words for the decoupled look-back (K1): top two bits are the flag.
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagIncl = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

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

// Device-written summary of one extract, read back by the host after the single sync.
struct ExtractSummary {
    unsigned long long M;           // total changed lanes (entries) over all tensors
    unsigned long long overflow;    // != 0: the entry workspace was too small
    unsigned long long idx_bytes;   // total LEB128 bytes over all tensors
    unsigned long long body_bytes;  // packed body size
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
    uint32_t name_off;  // into the names blob
    uint32_t name_len;
};

struct ApplyRec {  // located + verified record
    unsigned long long idx_off, idx_len, val_off, nnz, numel;
    uint8_t *w;
};

// Status word codes written by the apply kernels (DELTA_D_* of sparsedelta.h).
enum : uint32_t {
    kOk = 0, kTruncated = 1, kOverlong = 2, kOverflow = 3, kNonIncreasing = 4, kRange = 5,
    kCount = 6, kName = 7, kNumel = 8, kMode = 9, kLayout = 10
};

struct ApplyState {
    uint32_t status;     // first error code (0 = ok)
    uint32_t pad;
    unsigned long long n_chunks;
};

// ---------------------------------------------------------------- launchers (extract.cu / apply.cu)
struct ExtractArgs {
    const TileDesc *tiles;
    uint32_t ntiles;
    uint32_t ntensors;
    unsigned long long *tile_state;   // ntiles, zeroed
    unsigned int *ticket;             // zeroed
    void *ws_idx;                     // u32 or u64 entries
    void *ws_val;                     // lanes
    unsigned long long ws_cap;        // entries
    unsigned long long *entry_begin;  // ntensors + 1 (E_k)
    unsigned long long *tstart_partial;  // ntensors + 1
    unsigned int *chunk_bytes;        // per entry chunk
    unsigned long long *chunk_prefix; // per entry chunk
    unsigned long long chunk_cap;     // capacity of the chunk arrays
    unsigned long long *tensor_byte_begin;  // ntensors + 1 (B_k)
    RecordRow *table;                 // ntensors
    const uint32_t *name_len;         // ntensors
    const uint32_t *name_off;         // ntensors
    const uint8_t *names;             // blob
    const unsigned long long *numel;  // ntensors (N_k)
    ExtractSummary *summary;
    int width;                        // 2 or 4
    bool idx64;
    int persist_ctas;                 // grid for grid-stride kernels
};

// ev: nullptr, or events recorded around the kernels (scan: 4 = before K1, after K1, K2,
// K3; emit: 3 = before K4, after K4, after K5).
cudaError_t launch_extract_scan(const ExtractArgs &a, cudaStream_t s, cudaEvent_t *ev);    // K1-K3
cudaError_t launch_extract_emit(const ExtractArgs &a, uint8_t *out, cudaStream_t s, cudaEvent_t *ev);  // K4-K5

struct ApplyArgs {
    const uint8_t *body;
    unsigned long long body_bytes;
    const TargetDesc *targets;
    uint32_t n;
    const uint8_t *names;
    const RecordRow *hint;            // device copy of the host hint, or nullptr
    ApplyRec *recs;                   // n
    unsigned long long *rec_chunk_begin;  // n + 1
    unsigned int *chunk_count;
    unsigned long long *chunk_sum;
    unsigned long long *chunk_ord_base;
    unsigned long long *chunk_idx_base;
    unsigned long long chunk_cap;
    ApplyState *state;
    int width;
    int persist_ctas;
};

// ev: nullptr, or 5 events: before A1, after A1, A2, A3, A4.
cudaError_t launch_apply(const ApplyArgs &a, cudaStream_t s, cudaEvent_t *ev);  // A1-A4

}  // namespace sd
