// Internal structures shared by the host runtime (runtime.cpp) and the
// sm_100a kernels (kernels.cu).  Not part of the public C ABI (include/niyama.h).
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

#include "niyama.h"

namespace niyama {

// Sets niyama_last_error() for this thread and returns s (host translation units).
niyama_status set_error(niyama_status s, const char* msg);

// KV pool physical layout:
//   bf16: pool[layer][block][kv_head][K | V^T chunk]   (K and V^T of a block adjacent)
//   f32:  pool[layer][K=0|V=1][block][kv_head][chunk]
// A chunk is block_size * head_dim * elt bytes, contiguous; chunk_stride is the
// distance between consecutive (block, kv head) chunks of K (or of V).
// K (bf16): 8 x 16-byte core matrices — the 16-byte piece j of row s at
// (s / 8) * 8 * row_bytes + 128 j + 16 (s % 8).  A block is one bulk copy and lands
// as a canonical no-swizzle K-major UMMA operand (LBO 128 B, SBO 8 * row_bytes).
// V (bf16): stored TRANSPOSED in 16-key sub-blocks: sub-block u of a chunk is
// V^T [head_dim rows][16 keys] (32 B per row), 16-byte half c of row e at
// c ^ ((e >> 2) & 1) — the SWIZZLE_32B pattern.  One 4 KB sub-block is a
// canonical K-major UMMA SW32 operand (N = head_dim, K = 16 keys) for O += P V.
// K and V (f32 path): each token row is cut into 128-byte panels; inside a panel
// the 16-byte piece c of the row at slot s is at position c ^ (s & 7).

// Compact work list (a2 -> a4/a5).  The kernel expands item indices itself, so
// the per-iteration H2D stays small (tables + one record per slice / decode).
//
// Prefill slice: its work items are [tbase, tbase + nqt*Hkv); item t is q tile
// qt = nqt-1 - (t-tbase)/Hkv (largest key ranges first) of kv head (t-tbase)%Hkv,
// rows [qt*R, min(qt*R+R, c)) with R = 128/g chunk rows (128 MMA rows = g query
// heads x R rows).  (a4)
struct PrefillSlice {
  int32_t tbl;    // offset of the sequence's block table in the tables array
  int32_t o;      // slice offset (positions of rows are o + i)
  int32_t c;      // slice length
  int32_t row0;   // batch row of slice row 0
  int32_t nqt;    // q tiles = ceil(c / R)
  int32_t tbase;  // first tile index
  int32_t pad0, pad1;
};

// Decode row (sorted by ctx, longest first): unit (row, split s, kv head h) covers
// keys [s*L, min(ctx, (s+1)*L)) with L = split_len; its partial (when nsplit > 1)
// lives at the canonical index ubase + s*Hkv + h.  (a5, a6)
struct DecodeRow {
  int32_t tbl;
  int32_t ctx;
  int32_t row;     // batch row
  int32_t nsplit;
  int32_t ubase;
  int32_t pad0, pad1, pad2;
};

// Decode queue entry (a5): one per (row, split), in LPT order; unit id u of the
// queue is entry u / Hkv, kv head u % Hkv.  Everything a warp needs to start the
// unit is in this one 48-byte record, including the physical blocks of its first
// three 16-token stages, so claiming a unit costs one dependent load.
struct UnitRec {
  int32_t tbl;     // offset of the sequence's block table
  int32_t row;     // batch row
  int32_t k0, k1;  // key range [k0, k1)
  int32_t nsplit;  // splits of the row (1: write O/LSE directly)
  int32_t pbase;   // partial index of kv head 0: ubase + s * Hkv
  int32_t phys0;   // physical block of key k0 (stage 0)
  int32_t crow;    // sorted row index: completion counter crow * Hkv + kv head
  int32_t phys1;   // physical blocks of stages 1 and 2 (keys min(k0 + 16 s, k1 - 1)), so a
  int32_t phys2;   //   warp fills its 3-stage ring without a block-table round trip
  int32_t pad0, pad1;
};

// Merge row (a6), in readiness order (by the queue position of the row's last
// split): its items are (kv head, q head of the group).
struct MergeRec {
  int32_t row;     // batch row
  int32_t ubase;   // partial index of split 0, kv head 0
  int32_t nsplit;  // > 1
  int32_t crow;    // completion counter row
};

// Per-row info for the generic (f32) path.
struct RowInfo {
  int32_t tbl;
  int32_t n;  // visible keys
};

struct AppendParams {
  uint8_t* pool_k;
  uint8_t* pool_v;
  const uint8_t* k_new;
  const uint8_t* v_new;
  const int32_t* slot_map;  // [T] block * B + slot
  int64_t chunk_bytes;
  int64_t chunk_stride;  // bytes between consecutive (block, kv head) chunks
  int32_t T, Hkv, row_bytes, B;
  int32_t v_t;  // 1: V stored transposed in 16-key SW32 sub-blocks (bf16 path)
  // v_t only: V^T writes are grouped — vgrp[k] = first batch row of 8 consecutive rows
  // whose positions form one 8-aligned half of a 16-key sub-block (written as one 16-byte
  // V^T row segment per dim); velem[k] = every other row (element-wise 2-byte writes).
  const int32_t* vgrp;
  const int32_t* velem;
  int32_t n_grp, n_elem;
};

struct AttnParams {
  const uint8_t* pool_k;  // layer base of K
  const uint8_t* pool_v;  // layer base of V
  const void* q;
  void* o;
  float* lse;
  const int32_t* tables;
  const PrefillSlice* slices;
  const DecodeRow* drows;
  const UnitRec* uq;     // [n_units / Hkv] decode queue (LPT order)
  const MergeRec* mq;    // [n_merge_rows] merge queue (readiness order)
  int32_t* counters;     // [n_drows * Hkv] split-completion counters, cumulative over launches
  int32_t epoch;         // launches of this plan before this one (counter target (epoch+1)*nsplit)
  const RowInfo* rows;
  float* part_o;    // [n_units][g][d]
  float* part_ml;   // [n_units][g][2]
  int32_t* work;      // [0] tile queue, [1] unit queue, [2] CTA done counter, [3] merge queue (self-resetting)
  int64_t chunk_bytes;   // bytes of one (block, kv head) chunk
  int64_t chunk_stride;  // bytes between consecutive (block, kv head) chunks of pool_k / pool_v
  int32_t kv_adjacent;   // 1: pool_v = pool_k + chunk_bytes (K and V^T chunks of a block adjacent)
  int32_t dec_warps;     // bf16 decode warps per CTA: 12 (2-stage rings) or 8 (3-stage rings)
  int32_t T, Hq, Hkv, d, B, g, R;
  int32_t b_shift;    // log2(B) (block sizes are powers of two)
  int32_t hkv_shift;  // log2(Hkv) when Hkv is a power of two, else -1 (divide)
  int32_t n_tiles, n_units, n_slices, n_drows, split_len;
  int32_t n_merge_rows;  // rows with nsplit > 1
  int32_t prefill_ctas;  // CTAs [0, prefill_ctas) serve prefill items first; the rest decode at once
  int64_t* trace;  // optional per-CTA timeline [grid][4] (globaltimer ns), nullptr = off
  float scale_log2;     // softmax scale * log2(e)
  // niyama_append_attention: the KV append of this batch runs inside the launch
  // (append_total > 0 pieces, claimed through work[4], completion counted in work[5])
  AppendParams ap;
  int32_t append_total;
};


// Launchers (kernels.cu).  Return cudaSuccess or the launch error.
cudaError_t launch_append(const AppendParams& p, cudaStream_t s);
cudaError_t launch_gather(const uint8_t* pool_k, const uint8_t* pool_v, const int32_t* table, int32_t len,
                          int32_t Hkv, int32_t row_bytes, int32_t B, int64_t chunk_bytes, int32_t v_t, uint8_t* k_out,
                          uint8_t* v_out, cudaStream_t s);
cudaError_t configure_attention_bf16();  // per-device smem opt-in (current device)
cudaError_t launch_attention_bf16(const AttnParams& p, int grid, cudaStream_t s);
cudaError_t launch_attention_generic_f32(const AttnParams& p, cudaStream_t s);
int attention_bf16_smem_bytes();

}  // namespace niyama
