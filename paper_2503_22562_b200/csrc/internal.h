// Internal structures shared by the host runtime (runtime.cpp) and the
// sm_100a kernels (kernels.cu).  Not part of the public C ABI (include/niyama.h).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>

#include <cuda_runtime.h>

#include "niyama.h"

struct ncclWindow_vidmem;  // nccl.h: typedef ncclWindow_vidmem* ncclWindow_t

namespace niyama {

// Sets niyama_last_error() for this thread and returns s (host translation units).
niyama_status set_error(niyama_status s, const char* msg);

constexpr int kMaxGatherRanks = 8;  // §8(f)2: the ranks of one NVLink node

// ---- shared by the planner (runtime.cpp) and the predictor (predictor.cpp, a8), which
// models the same launch: one definition of every launch-shaping rule.
inline int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline niyama_tuning default_tuning() {
  niyama_tuning t{};
  t.prefill_ctas = 0;
  t.split_len = 0;
  t.decode_path = 0;
  t.prefill_split = 0;
  t.tail_div = NIYAMA_TAIL_DIV;
  t.tail_min = NIYAMA_TAIL_MIN;
  t.grid_cap = 0;
  t.plan_copy_stream = 1;
  t.prefill_pairs = 0;
  return t;
}

// Decode split length (a5), from batch totals only (split boundaries never depend
// on scheduling, so results stay bitwise deterministic): the power of two nearest
// (in log scale) to raw = sum ctx * Hkv / (4 units per resident warp), at least 128
// (measured: 64-key splits lose to 128 on small batches; rounding 131 up to 256 lost
// to 128), with at most 4095 splits per row.
inline int32_t choose_split_len(int64_t sum_ctx, int32_t max_ctx, int hkv, int num_sms) {
  const int64_t target = 4LL * num_sms * 8;
  const int64_t raw = ceil_div64(std::max<int64_t>(1, sum_ctx * hkv), target);
  int32_t s = 128;
  while ((2LL * s * s < raw * raw || ceil_div64(max_ctx, s) > 4095) && s < (1 << 20)) s *= 2;
  return s;
}

// CTA split of the bf16 launch.  Prefill tiles are
// tensor/MUFU-bound and decode streaming is HBM-bound, so the launch runs them side
// by side: CTAs [0, prefill_ctas) take prefill tiles first (longest first) and then
// join the decode queue; the others stream decode KV from the start.  The prefill
// share of the CTAs is its share of the estimated CTA-time: one 128-key prefill
// step costs a CTA about as long as streaming NIYAMA_STEP_BYTES of decode KV under
// load (measured: ~3.6 us per step vs ~44 GB/s per CTA on B200, tools/cap_sweep.py).
// A tile also pays a fixed setup (Q load, pipeline fill, epilogue) of about
// NIYAMA_TILE_SETUP_STEPS steps, which dominates short tiles (chunk at offset 0).
// `tile_cost` = sum over tiles of (steps + setup).  Shared by the planner and the
// predictor (a8), which simulates the same launch.
struct CtaSplit {
  int32_t grid, prefill_ctas;
};
inline CtaSplit cta_split(int64_t n_tiles, int64_t n_units, int64_t tile_cost, int64_t sum_ctx, int hkv, int d, int elt,
                   int g, int num_sms, int decode_path = 0) {
  CtaSplit r{};
  // a decode CTA runs one unit at a time (tensor-core pipeline) or one per warp (8+ warps)
  const int64_t units_per_cta = decode_path == 1 ? 1 : 8;
  r.grid = static_cast<int32_t>(
      std::max<int64_t>(1, std::min<int64_t>(num_sms, n_tiles + ceil_div64(n_units, units_per_cta))));
  if (n_tiles == 0) return r;
  if (n_units == 0) {
    r.prefill_ctas = r.grid;
    return r;
  }
  const double wp = static_cast<double>(tile_cost) * NIYAMA_STEP_BYTES;
  const double wd = static_cast<double>(sum_ctx) * hkv * d * 2.0 * elt *
                    (g > 4 && decode_path != 1 ? NIYAMA_WIDE_GROUP_DECODE_WEIGHT : 1.0);
  int64_t np = static_cast<int64_t>(std::ceil(r.grid * wp / (wp + wd)));
  // a tile-count floor keeps short-tile prefill off the tail (at most 4 tiles per prefill
  // CTA), itself capped at half the grid: with many long tiles (config 4: 1,024) it would
  // put every CTA on prefill first (measured 1,073 us vs 926 us at 80 prefill CTAs)
  np = std::max<int64_t>(np, std::min<int64_t>(ceil_div64(n_tiles, 4), ceil_div64(r.grid, 2)));
  np = std::min<int64_t>({np, n_tiles, static_cast<int64_t>(r.grid)});
  r.prefill_ctas = static_cast<int32_t>(std::max<int64_t>(1, np));
  return r;
}


// Prefill split-K (a4): when there are fewer q tiles than the CTAs the work split would
// give to prefill, each q tile's key range is cut into P contiguous parts run by different
// CTAs; the last part to finish merges the tile (log-sum-exp, part order: deterministic).
// P = floor(target prefill CTAs / q tiles), at most 16; per slice at most (its shortest
// tile's steps) / 4, so a part has >= 4 key steps.  `tile_cost` = sum of (steps + setup).
inline int32_t prefill_parts_target(int64_t q_tiles, int64_t n_units, int64_t tile_cost, int64_t sum_ctx, int hkv,
                                    int d, int elt, int g, int num_sms, int decode_path = 0, int prefill_split = 0) {
  if (q_tiles <= 0 || prefill_split == 0) return 1;
  double target = num_sms;
  if (n_units > 0) {
    const double wp = static_cast<double>(tile_cost) * NIYAMA_STEP_BYTES;
    const double wd = static_cast<double>(sum_ctx) * hkv * d * 2.0 * elt *
                      (g > 4 && decode_path != 1 ? NIYAMA_WIDE_GROUP_DECODE_WEIGHT : 1.0);
    target = std::ceil(num_sms * wp / (wp + wd));
  }
  return static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(16, static_cast<int64_t>(target) / q_tiles)));
}
inline int32_t prefill_parts_of_slice(int32_t target, int64_t min_steps) {
  return static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(target, min_steps / 4)));
}

// Prefill work items: with GQA packing a 128-row tile holds R = 128 / g chunk rows of
// the g query heads of one kv head (a4).
inline int32_t rows_per_tile(int g) { return 128 / (g > 0 ? g : 1); }
// Decode warps per CTA of the bf16 launch (12 when g <= 4, else 8)
inline int decode_warps(int g) { return g <= 4 ? 12 : 8; }
// Decode streams per CTA as the predictor models them: one pipeline (tensor-core path) or
// one per decode warp (mma.sync path).
// (decode_path 0 = auto resolves to 2 at g = 8, which also runs 8 compute warps)
inline int decode_streams(int g, int decode_path) {
  return decode_path == 1 ? 1 : decode_path == 2 ? 8 : decode_warps(g);
}

struct KvModel {
  int hq, hkv, d, elt, num_sms;
  niyama_tuning tune;
};
void kv_model(const niyama_kv* kv, KvModel* m);

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
  int32_t tbase;  // first work item: q tile (nqt-1 - (t-tbase)/(Hkv*parts)), kv head, key part
  int32_t parts;  // split-K: each q tile's key steps cut into `parts` contiguous ranges (1 = none)
  int32_t pbase;  // split tiles only: index of this slice's first q tile among all split tiles
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
  const uint8_t* pf_base;  // plan metadata to prefetch into L2 (pf_bytes, multiple of 16; 0 = none)
  uint32_t pf_bytes;
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
  float* ppart_o;   // prefill split-K partials [split tile][part][128 rows][d] (o / l)
  float* ppart_ml;  // [split tile][part][128 rows][2] (m in log2 units, l)
  int32_t* pcounters;  // [split tiles] parts finished, cumulative over launches (epoch)
  int32_t* work;      // [0] tile queue, [1] unit queue, [2] CTA done counter, [3] merge queue (self-resetting)
  int64_t chunk_bytes;   // bytes of one (block, kv head) chunk
  int64_t chunk_stride;  // bytes between consecutive (block, kv head) chunks of pool_k / pool_v
  int32_t kv_adjacent;   // 1: pool_v = pool_k + chunk_bytes (K and V^T chunks of a block adjacent)
  int32_t dec_warps;     // bf16 decode warps per CTA: 12 (2-stage rings) or 8 (3-stage rings)
  int32_t dec_mode;      // bf16 decode path: 0 = warp mma.sync streams, 1 = tensor-core CTA pipeline (128-token steps)
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
  // §8(f)2 fused all-gather: n > 0 stores every O / LSE value at (address + delta[r]) for
  // each rank r (delta = rank r's window mapping - this rank's window base), then the
  // last CTA publishes `epoch` into flags[rank] of every rank and waits for all n flags.
  struct Gather {
    int32_t n;          // ranks (0 = plain stores to o / lse)
    int32_t rank;
    uint32_t epoch;     // launches of this gather object, this one included (monotonic)
    uint32_t* flags;    // this rank's flag array [n] (window mapping)
    int64_t delta[kMaxGatherRanks];
  } gx;
  // Prefill CTA pairs (niyama_tuning.prefill_pairs): clusters of 2 CTAs take the two q tiles
  // (qt, qt - 1) of one kv head together; each CTA issues half of every K/V step's copies,
  // multicast into both CTAs' shared memory.  n_pair_items = sum over slices of
  // ceil(nqt / 2) * Hkv.  0 = one q tile per CTA.
  int32_t pairs;
  int32_t n_pair_items;
};


// Launchers (kernels.cu).  Return cudaSuccess or the launch error.
cudaError_t launch_append(const AppendParams& p, cudaStream_t s);
cudaError_t launch_gather(const uint8_t* pool_k, const uint8_t* pool_v, const int32_t* table, int32_t len,
                          int32_t Hkv, int32_t row_bytes, int32_t B, int64_t chunk_bytes, int32_t v_t, uint8_t* k_out,
                          uint8_t* v_out, cudaStream_t s);
cudaError_t configure_attention_bf16();  // per-device smem opt-in (current device)
cudaError_t launch_attention_bf16(const AttnParams& p, int grid, cudaStream_t s);
cudaError_t launch_attention_generic_f32(const AttnParams& p, cudaStream_t s);
// §8(f)2 (gather.cu, the one unit built against nccl_device.h): this process's address of
// every rank's copy of a symmetric window (offset 0), via the window's LSA mapping; blocking.
cudaError_t gather_resolve_peers(ncclWindow_vidmem* win, int world, uint64_t* host_out);
int attention_bf16_smem_bytes();

}  // namespace niyama
