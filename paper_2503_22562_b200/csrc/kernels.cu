// sm_100a kernels of the Niyama hybrid-batch paged-attention path.
//
//   kv_append_kernel        a3  scatter new K/V rows into the paged pool (core-matrix K, V^T)
//   kv_gather_kernel            read-back of a sequence (tests)
//   hybrid_attn_bf16_kernel a4-a6  ONE persistent launch:
//        prefill tiles  — TMA-engine bulk copies of paged K/V (one per block) into
//                         shared memory, S = Q K^T (SS) and O += P V (TS, P in TMEM)
//                         on tcgen05, two softmax warp sets on alternate key steps
//                         (online softmax, lazy rescale of O in TMEM);
//        decode units   — warp-level split-KV streaming (one 8 KB bulk copy per
//                         16-token stage into per-warp rings: 12 warps x 2 stages at
//                         g <= 4, 8 x 3 at g = 8; mma.sync m16n8k16 swap-AB with the
//                         GQA group on N), partials merged by log-sum-exp in-launch.
//   (niyama_append_attention: the append pieces run inside this launch first.)
//   hybrid_attn_generic_kernel  f32 path (config 1): SIMT warp per (row, kv head).
//
// Math (PAPER P:319 PagedAttention semantics, R1/R7/R10/R11): for row r
// with n_r visible keys and head h (kv head h/g): O = softmax(scale q K^T) V,
// LSE = ln sum exp(scale q K^T).  Scores are kept in the log2 domain
// (x = s * scale * log2 e) and exponentiated with ex2.approx.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace niyama {

using namespace ptx;

// ============================================================= append (a3)
// Byte offset, inside a (block, kv head) chunk, of V element (slot, dim e) in the
// transposed SW32 sub-block layout (internal.h): sub-block slot/16, row e, key slot%16.
__device__ __forceinline__ int vt_offset(int slot, int e, int head_dim) {
  const int k = slot & 15;
  return (slot >> 4) * (head_dim * 32) + e * 32 + ((((k >> 3) ^ (e >> 2)) & 1) << 4) + ((k & 7) << 1);
}

// Byte offset, inside a (block, kv head) chunk, of the 16-byte piece j (dims 8j..8j+7)
// of K row `slot` in the bf16 core-matrix layout: [slot/8][piece j][slot%8][16 B].  A
// block of B rows is B*row_bytes contiguous bytes, so one bulk copy per block lands a
// canonical no-swizzle K-major UMMA operand (LBO 128 B between pieces, SBO 8*row_bytes
// between 8-row groups) and ldmatrix reads 8 contiguous rows of a piece.
__device__ __forceinline__ int k_core_offset(int slot, int j, int row_bytes) {
  return (slot >> 3) * (row_bytes * 8) + j * 128 + ((slot & 7) << 4);
}

// One thread per 16-byte piece of a (row, kv head) vector, 32-bit index math (the
// launcher guarantees T*Hkv*pieces < 2^31).  Source rows are dense [T][Hkv][row_bytes];
// piece j of the K row at (block, slot) lands in panel j/8 at chunk position
// (j%8) ^ (slot%8).  V pieces go to the same place (f32) or are scattered element by
// element into the transposed sub-block (bf16, v_t).  Piece order: K pieces, then V^T
// 8-token segments, then element-wise V^T pieces.
__device__ __forceinline__ int append_total(const AppendParams& p) {
  const int pieces = p.row_bytes >> 4;
  const int d = p.row_bytes >> 1;
  return p.T * p.Hkv * pieces + (p.v_t ? p.n_grp * p.Hkv * d + p.n_elem * p.Hkv * pieces : 0);
}

__device__ __forceinline__ void append_piece(const AppendParams& p, const int idx) {
  const int pieces = p.row_bytes >> 4;  // 16 at d = 128 bf16
  const int nk = p.T * p.Hkv * pieces;  // K pieces (and V pieces when !v_t)
  const int d = p.row_bytes >> 1;       // head_dim (bf16)
  const int ng = p.v_t ? p.n_grp * p.Hkv * d : 0;
  {
    if (idx < nk) {  // K row pieces (and V when stored row-major)
      const int j = idx % pieces;
      const int rh = idx / pieces;
      const int h = rh % p.Hkv;
      const int r = rh / p.Hkv;
      const uint4 kv = __ldg(reinterpret_cast<const uint4*>(p.k_new) + idx);
      const int32_t sm = __ldg(p.slot_map + r);
      const int blk = sm / p.B;
      const int slot = sm - blk * p.B;
      const int64_t chunk = (static_cast<int64_t>(blk) * p.Hkv + h) * p.chunk_stride;
      if (p.v_t) {  // bf16: K in 8x16-byte core matrices (k_core_offset)
        *reinterpret_cast<uint4*>(p.pool_k + chunk + k_core_offset(slot, j, p.row_bytes)) = kv;
      } else {      // f32: K and V in swizzled 128-byte panels
        const int64_t dst_off = chunk + (j >> 3) * p.B * 128 + slot * 128 + (((j & 7) ^ (slot & 7)) << 4);
        *reinterpret_cast<uint4*>(p.pool_k + dst_off) = kv;
        *reinterpret_cast<uint4*>(p.pool_v + dst_off) = __ldg(reinterpret_cast<const uint4*>(p.v_new) + idx);
      }
    } else if (idx < nk + ng) {  // V^T: 8 tokens x one dim -> one 16-byte segment of row e
      const int k = idx - nk;
      const int e = k % d;
      const int gh = k / d;
      const int h = gh % p.Hkv;
      const int r0 = __ldg(p.vgrp + gh / p.Hkv);
      const uint16_t* src = reinterpret_cast<const uint16_t*>(p.v_new) + (static_cast<int64_t>(r0) * p.Hkv + h) * d + e;
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        w[q] = static_cast<uint32_t>(__ldg(src + static_cast<int64_t>(2 * q) * p.Hkv * d)) |
               (static_cast<uint32_t>(__ldg(src + static_cast<int64_t>(2 * q + 1) * p.Hkv * d)) << 16);
      const int32_t sm = __ldg(p.slot_map + r0);
      const int blk = sm / p.B;
      const int slot = sm - blk * p.B;  // 8-aligned
      const int64_t off = (static_cast<int64_t>(blk) * p.Hkv + h) * p.chunk_stride + vt_offset(slot, e, d);
      *reinterpret_cast<uint4*>(p.pool_v + off) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {  // V^T element-wise: row r, dims 8j..8j+7
      const int k = idx - nk - ng;
      const int j = k % pieces;
      const int rh = k / pieces;
      const int h = rh % p.Hkv;
      const int r = __ldg(p.velem + rh / p.Hkv);
      const uint4 vv = __ldg(reinterpret_cast<const uint4*>(p.v_new) + (static_cast<int64_t>(r) * p.Hkv + h) * pieces + j);
      const int32_t sm = __ldg(p.slot_map + r);
      const int blk = sm / p.B;
      const int slot = sm - blk * p.B;
      const int64_t chunk = (static_cast<int64_t>(blk) * p.Hkv + h) * p.chunk_stride;
      const uint32_t w[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<uint16_t*>(p.pool_v + chunk + vt_offset(slot, j * 8 + q, d)) =
            static_cast<uint16_t>(w[q >> 1] >> ((q & 1) * 16));
    }
  }
}

// Diagnostic A/B: the append kernel prefetches the plan's metadata into L2 (default off).
#ifndef NIYAMA_PLAN_PREFETCH
#define NIYAMA_PLAN_PREFETCH 0
#endif
__global__ void __launch_bounds__(256) kv_append_kernel(const AppendParams p) {
  grid_dep_launch();  // the attention launch that follows may start its prologue
#if NIYAMA_PLAN_PREFETCH
  if (blockIdx.x == 0 && p.pf_bytes > 0) {  // plan metadata into L2 for the attention launch
    const uint32_t chunk = 16384;
    for (uint32_t o = threadIdx.x * chunk; o < p.pf_bytes; o += blockDim.x * chunk)
      bulk_prefetch_l2(p.pf_base + o, min(chunk, p.pf_bytes - o));
  }
#endif
  const int total = append_total(p);
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x)
    append_piece(p, idx);
}

cudaError_t launch_append(const AppendParams& p, cudaStream_t s) {
  const int64_t pieces = p.row_bytes >> 4;
  const int64_t total = static_cast<int64_t>(p.T) * p.Hkv * pieces +
                        (p.v_t ? static_cast<int64_t>(p.n_grp) * p.Hkv * (p.row_bytes >> 1) +
                                     static_cast<int64_t>(p.n_elem) * p.Hkv * pieces
                               : 0);
  if (total == 0) return cudaSuccess;
  if (total >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  kv_append_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(p);
  return cudaGetLastError();
}

// ================================================================= gather
__global__ void kv_gather_kernel(const uint8_t* __restrict__ pool_k, const uint8_t* __restrict__ pool_v,
                                 const int32_t* __restrict__ table, int32_t len, int32_t Hkv, int32_t row_bytes,
                                 int32_t B, int64_t chunk_bytes, int32_t v_t, uint8_t* __restrict__ k_out,
                                 uint8_t* __restrict__ v_out) {
  const int pieces = row_bytes >> 4;
  const int64_t total = static_cast<int64_t>(len) * Hkv * pieces;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(idx % pieces);
    const int64_t th = idx / pieces;
    const int h = static_cast<int>(th % Hkv);
    const int t = static_cast<int>(th / Hkv);
    const int64_t blk = table[t / B];
    const int slot = t % B;
    const int64_t chunk = (blk * Hkv + h) * chunk_bytes;
    const int64_t src = chunk + static_cast<int64_t>(j >> 3) * B * 128 + slot * 128 + (((j & 7) ^ (slot & 7)) << 4);
    const int64_t dst = th * row_bytes + (static_cast<int64_t>(j) << 4);
    *reinterpret_cast<uint4*>(k_out + dst) =
        *reinterpret_cast<const uint4*>(pool_k + (v_t ? chunk + k_core_offset(slot, j, row_bytes) : src));
    if (v_t) {
      const int d = row_bytes >> 1;
      uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
      for (int q = 0; q < 8; ++q)
        w[q >> 1] |= static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(pool_v + chunk + vt_offset(slot, j * 8 + q, d)))
                     << ((q & 1) * 16);
      *reinterpret_cast<uint4*>(v_out + dst) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      *reinterpret_cast<uint4*>(v_out + dst) = *reinterpret_cast<const uint4*>(pool_v + src);
    }
  }
}

cudaError_t launch_gather(const uint8_t* pool_k, const uint8_t* pool_v, const int32_t* table, int32_t len,
                          int32_t Hkv, int32_t row_bytes, int32_t B, int64_t chunk_bytes, int32_t v_t, uint8_t* k_out,
                          uint8_t* v_out, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(len) * Hkv * (row_bytes >> 4);
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  kv_gather_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(pool_k, pool_v, table, len, Hkv, row_bytes, B,
                                                           chunk_bytes, v_t, k_out, v_out);
  return cudaGetLastError();
}

// ===================================================== fused bf16 attention
// CTA = 256 threads (8 warps), 1 CTA/SM, 512 TMEM columns.
// Shared memory map (from the 1024-aligned base), default (Q in shared memory):
//   [0,32K) Q tile (SW128; also the end-of-tile exchange) | [32K,128K) K stages x3 |
//   [128K,192K) V^T stages x2
// (NIYAMA_Q_TMEM=1: Q in TMEM, no Q tile; two S buffers instead of three — measured
// slower, the S-buffer reuse then sits in every other step's dependency cycle.)
// K stage: 128 rows in 8x16-byte core matrices (no swizzle, K-major: LBO 128 B, SBO
// 2 KB), one bulk copy per paged block.  V^T stage: 8 sub-blocks of [128 d][16 keys]
// (SW32, K-major).  TMEM: S/P buffers of 128 columns (P, bf16 pairs, overwrites its
// S), O (128 columns) [, Q (64 columns)].
// The decode role reuses [0, 192K) as per-warp rings of 8 KB stages.
namespace fa {
constexpr int kD = 128;             // head dim (bf16 path)
constexpr int kBN = 128;            // keys per prefill key tile
constexpr int kPanel = 128 * 128;   // one 64-column panel of a 128-row tile
constexpr int kTile = 2 * kPanel;   // 128 rows x 256 B = 32 KB (one region)
#ifndef NIYAMA_K_STAGES
#define NIYAMA_K_STAGES 3
#endif
#ifndef NIYAMA_V_STAGES
#define NIYAMA_V_STAGES 2
#endif
// Per-step event stamps (prefill roles, decode stages; tools/trace.py, tools/dec_trace.py):
// diagnostic builds only (tools/build_variant.py TAG -DNIYAMA_DIAG_STEPS=1).  The per-CTA
// phase timeline of niyama_debug_trace stays in every build.
#ifndef NIYAMA_DIAG_STEPS
#define NIYAMA_DIAG_STEPS 0
#endif
#ifndef NIYAMA_DIAG_HANG
#define NIYAMA_DIAG_HANG 0
#endif
// The K/V producers start an item's copies while the other warps load its Q tile
// (measured: config 2 99.4-99.9 -> 96.3 us, L70B prefill-only 426 -> 420 us,
// profiles/r02s3/ab_earlykv.txt); 0 restores the CTA-wide Q barrier.
#ifndef NIYAMA_EARLY_KV
#define NIYAMA_EARLY_KV 1
#endif
#ifndef NIYAMA_ONE_SLOAD
#define NIYAMA_ONE_SLOAD 0
#endif
#ifndef NIYAMA_DIAG_TILES
#define NIYAMA_DIAG_TILES 0
#endif
#ifndef NIYAMA_DIAG_HALF_KV
#define NIYAMA_DIAG_HALF_KV 0
#endif
constexpr int kKStages = NIYAMA_K_STAGES;  // K tile ring depth
constexpr int kVStages = NIYAMA_V_STAGES;  // V^T tile ring depth
#ifndef NIYAMA_Q_TMEM
#define NIYAMA_Q_TMEM 0
#endif
// Q in TMEM (QK^T as a TS MMA: only K is read from shared memory) leaves room for two S
// buffers; Q in shared memory (SS) for three.  Three win: with two, QK(j+2) waits for
// PV(j) to complete, putting two MMA-burst latencies (~0.7 K cycles each) and a softmax
// into every two steps (L70B prefill-only 556 -> 440 us with three).
constexpr bool kQTmem = NIYAMA_Q_TMEM != 0;
// P in TMEM columns of its own (default): S [2][128 cols] | P [2][64 cols of bf16 pairs] | O.
// An S buffer is free for QK_{j+2} as soon as the softmax of step j has LOADED it, not when
// PV_j has consumed P (the S-buffer cycle QK -> softmax -> PV -> QK was the prefill step's
// critical loop: ~5 K cycles per 3 steps, tools/trace.py).  0 = P over the consumed S
// columns with three S buffers (QK_{j+3} waits for PV_j).
#ifndef NIYAMA_P_SEPARATE
#define NIYAMA_P_SEPARATE 1
#endif
constexpr bool kPSep = NIYAMA_P_SEPARATE != 0;
static_assert(!(kPSep && kQTmem), "Q in TMEM needs the P-over-S layout");
constexpr int kSBufs = (kQTmem || kPSep) ? 2 : 3;  // S TMEM buffers: columns [128 b, 128 b + 128)
// Q staging tile (SS only) | K stages | V^T stages | end-of-tile exchange (2 KB; the Q
// tile's space when Q is staged in shared memory)
constexpr int kQOff = 0;
constexpr int kKOff = kQTmem ? 0 : kTile;          // K stage s at kKOff + s * kTile
constexpr int kVOff = kKOff + kKStages * kTile;    // V^T stage s at kVOff + s * kTile
constexpr int kXOff = kVOff + kVStages * kTile;  // 2 KB of its own (the Q tile stays intact)
constexpr int kPrefillBytes = kXOff + 2048;
constexpr int kThreads = 384;  // 12 warps: producers/MMA (0-3), softmax sets (4-7, 8-11)
// Decode: warps [0, p.dec_warps) stream units through per-warp rings of kDecSlots /
// dec_warps stages: 8 warps x 3 stages (g = 8: more work per byte, deeper rings) or 12 x 2
// (g <= 4: more warps in flight per SM).
constexpr int kDecSlots = 24;    // 8 KB stage slots shared by the rings (192 KB)
constexpr int kDecWarps = 12;    // the most decode warps per CTA
constexpr int kDecStage = 8192;  // 16 tokens of K (4 KB) + V^T (4 KB)
// Decode math: the 16 tokens of a stage on the MMA M dimension and the g <= 8 heads
// of the group on N (mma.sync m16n8k16, "swap-AB"): 8 MMAs for S^T = K Q^T and 8 for
// O^T += V^T P^T per stage (heads on M would pad g to 16 rows and need 16 + 16).

// Decode, tensor-core CTA pipeline (p.dec_mode == 1, DESIGN.md 6.1 "decode unit"): one
// pipeline per CTA over 128-token steps of one (row, kv head) unit at a time.  Swap-AB on
// tcgen05: S^T [128 tokens x 16] = K [128 x 128 d] . Q^T (the g <= 8 heads of the group,
// zero-padded to N = 16), softmax over the tokens per head (thread = TMEM lane = token),
// O^T [128 d x 16] += V^T [128 d x 128 tokens] . P^T (P^T bf16 in shared memory).
// Shared memory: 3 stages of 64 KB (K 128 rows core-matrix | V^T 8 SW32 sub-blocks) |
// 4 Q^T tiles (4 KB) | 2 P^T tiles (4 KB).  TMEM: S^T [2][16 cols] at 0, O^T [2][16] at 32.
constexpr int kD2Stages = 3;
constexpr int kD2Stage = 65536;
constexpr int kD2QOff = kD2Stages * kD2Stage;
constexpr int kD2QBufs = 4;
constexpr int kD2POff = kD2QOff + kD2QBufs * 4096;
constexpr int kD2Bytes = kD2POff + 2 * 4096;
constexpr uint32_t kIdescD2 = idesc_bf16_f32(128, 16, 0, 0);
constexpr int kDataBytes0 = kPrefillBytes > kDecSlots * kDecStage ? kPrefillBytes : kDecSlots * kDecStage;
constexpr int kDataBytes = kDataBytes0 > kD2Bytes ? kDataBytes0 : kD2Bytes;
static_assert(kDecWarps <= kThreads / 32, "decode warps");
// barrier indices
constexpr int kBarKFull = 0;                       // [kKStages]
constexpr int kBarKEmpty = kBarKFull + kKStages;   // [kKStages]
constexpr int kBarVFull = kBarKEmpty + kKStages;   // [kVStages]
constexpr int kBarVEmpty = kBarVFull + kVStages;   // [kVStages]
constexpr int kBarSFull = kBarVEmpty + kVStages;   // [kSBufs] QK^T committed into S[b]
constexpr int kBarPFull = kBarSFull + kSBufs;      // [kSBufs] softmax wrote P over S[b] (128 arrivals)
constexpr int kBarODone = kBarPFull + kSBufs;      // [kSBufs] PV from P[b] committed (P[b] free, O includes it)
constexpr int kBarSFree = kBarODone + kSBufs;      // [kSBufs] kPSep: softmax loaded S[b] (128 arrivals)
constexpr int kBarDec = kBarSFree + kSBufs;        // [kDecSlots] decode ring stages
constexpr int kBarDecEmpty = kBarDec + kDecSlots;  // [kDecSlots] decode_path 2: consumer done with the stage
constexpr int kB2Full = kBarDecEmpty + kDecSlots;  // [kD2Stages] K/V step landed (tx)
constexpr int kB2Empty = kB2Full + kD2Stages;  // [kD2Stages] PV of the step done (commit)
constexpr int kB2SFull = kB2Empty + kD2Stages;  // [2] QK^T committed into S^T[b]
constexpr int kB2SFree = kB2SFull + 2;          // [2] softmax loaded S^T[b] (128)
constexpr int kB2PFull = kB2SFree + 2;          // [2] P^T[b] written (128)
constexpr int kB2PFree = kB2PFull + 2;          // [2] PV from P^T[b] done (commit)
constexpr int kB2OFull = kB2PFree + 2;          // [2] unit's last PV into O^T[u%2] done (commit)
constexpr int kB2OFree = kB2OFull + 2;          // [2] epilogue loaded O^T[u%2] (128)
constexpr int kB2MLFull = kB2OFree + 2;         // [2] (m, l) of unit u written (128)
constexpr int kB2MLFree = kB2MLFull + 2;        // [2] epilogue read them (128)
constexpr int kB2QFull = kB2MLFree + 2;         // [kD2QBufs] Q^T tile written (1, after the producer warp)
constexpr int kB2QFree = kB2QFull + kD2QBufs;   // [kD2QBufs] unit's last QK^T done (commit)
constexpr int kB2DFull = kB2QFree + kD2QBufs;   // [4] unit descriptor published (1)
constexpr int kB2DFree = kB2DFull + 4;          // [4] producer, MMA, softmax, epilogue done with it (4)
constexpr int kNumBars = kB2DFree + 4;
constexpr int kBarBytes = (kNumBars * 8 + 63) & ~63;  // keeps the misc area 64-byte aligned (v4 accesses)
constexpr int kMiscBytes = 64 + kDecWarps * 16;      // tmem slot, item slot, per-warp desc counters
constexpr int kDescBytes = kDecWarps * 4 * 32;       // per-warp 4-entry UnitDesc rings (decode);
                                                     // the prefill softmax chain [2][128] floats (prefill)
static_assert(kDescBytes >= 2 * 128 * 4, "softmax chain must fit");
// decode-v2 scratch in the desc area: 4 descriptors (128 B) | first-step blocks [4][8] (128 B) | max [2][4][16] f32 (512 B) |
// l [2][4][16] f32 (512 B) | (m, l) [2][16] f32x2 (256 B)
constexpr int kD2Desc = 0, kD2Red = 256, kD2LRed = kD2Red + 512, kD2ML = kD2LRed + 512;
static_assert(kD2ML + 256 <= kDescBytes, "decode-v2 scratch must fit");
constexpr int kSmemBytes = 1024 /*align slack*/ + kDataBytes + kBarBytes + kMiscBytes + kDescBytes;
static_assert(kSmemBytes <= 232448, "exceeds 227 KB of dynamic shared memory");
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemP = 128 * kSBufs;  // kPSep: P[b] at kTmemP + 64 b
constexpr uint32_t kTmemO = kPSep ? kTmemP + 128 : 128 * kSBufs;  // O accumulator: 128 columns
static_assert(kTmemO + 128 <= kTmemCols, "TMEM columns");
constexpr uint32_t kTmemQ = kTmemO + 128;   // Q (kQTmem): 64 columns of bf16 pairs
constexpr uint32_t kIdescQK = idesc_bf16_f32(128, kBN, 0, 0);
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, kD, 0, 0);  // both operands K-major
}  // namespace fa

// ------------------------------------------------------- output stores (§8(f)2)
// Every O / LSE value of the launch goes through put_out.  Plain launch (gx.n == 0): one
// store.  Fused all-gather: the same value at the same window offset on every rank (peer
// mappings through NVLink; the own rank through its window mapping too), so the kernel's
// epilogues ARE the all-gather.
template <typename V>
__device__ __forceinline__ void put_out(const AttnParams& p, void* dst, const V& v) {
  if (p.gx.n == 0) {
    *reinterpret_cast<V*>(dst) = v;
    return;
  }
#pragma unroll 1
  for (int r = 0; r < p.gx.n; ++r) *reinterpret_cast<V*>(static_cast<uint8_t*>(dst) + p.gx.delta[r]) = v;
}

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* ptr) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys_u32(uint32_t* ptr, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(ptr), "r"(v) : "memory");
}

// The launch's last CTA: publish this launch's epoch to every rank's flag slot `rank`, then
// wait until every rank published it here.  Ordering (PTX memory model, causality is
// transitive): each CTA's output stores -> its fence.acq_rel.gpu + done count (observed by
// this CTA at gpu scope) -> this fence.acq_rel.sys + st.release.sys flag -> the peer's
// ld.acquire.sys.  A system-scope fence in every CTA instead measured +4 us per launch
// (config 2 at world 1: 100.4 vs 96.3 us).  Monotonic epochs, no reset.
// ~30 s without a peer = trap (a rank that never launches), never a silent hang.
__device__ __forceinline__ void gather_barrier(const AttnParams& p) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  for (int r = 0; r < p.gx.n; ++r)
    st_release_sys_u32(reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(p.gx.flags + p.gx.rank) + p.gx.delta[r]),
                       p.gx.epoch);
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int r = 0; r < p.gx.n; ++r) {
    while (static_cast<int32_t>(ld_acquire_sys_u32(p.gx.flags + r) - p.gx.epoch) < 0) {
      __nanosleep(64);
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 30ull * 1000000000ull) __trap();
    }
  }
}

// -------------------------------------------------------------- prefill tile
// Debug event log (niyama_debug_trace): CTA 0's first item, key tiles < 64, clock64 per role.
__device__ __forceinline__ void ev_stamp(int64_t* ev, int role, int j) {
  if (NIYAMA_DIAG_STEPS && ev != nullptr && j < 64) {
    int64_t c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    ev[role * 64 + j] = c;
  }
}

// 2^x on the FMA/ALU pipes (FA4-style): x = n + f with n = rint(x) (magic-number add),
// f in [-0.5, 0.5]; 2^f by a degree-3 polynomial (relative error < 1e-3, below bf16's
// 2^-8 rounding of P); n added to the exponent bits.  x < -125 (incl. masked -inf) -> 0.
#ifndef NIYAMA_POLY_EXP
#define NIYAMA_POLY_EXP 0
#endif
__device__ __forceinline__ float ex2_poly(float x) {
  const float xc = fmaxf(x, -125.f);
  const float t = xc + 12582912.f;       // 1.5 * 2^23: rint(xc) in the low mantissa bits
  const float n = t - 12582912.f;
  const float f = xc - n;
  float pl = fmaf(0.0555041087f, f, 0.2402265070f);
  pl = fmaf(pl, f, 0.6931471806f);
  pl = fmaf(pl, f, 1.0f);
  const float r = __int_as_float(__float_as_int(pl) + (__float_as_int(t) << 23));
  return x < -125.f ? 0.f : r;
}

// Causal mask of one 64-column slice of a score row: columns e > last become -inf.
__device__ __forceinline__ void mask_tail(uint32_t (&sr)[64], int last) {
#pragma unroll
  for (int e = 0; e < 64; ++e)
    if (e > last) sr[e] = 0xff800000u;  // -inf
}

struct TileDesc {
  int tbl, o, c, t0, row0, kvh, nkeys, nblk;
  int j0, j1;         // key steps [j0, j1) of this work item (split-K part; [0, nk) unsplit)
  int parts, part;    // split-K parts of the q tile and this item's part
  int stile;          // index of the q tile among split tiles (parts > 1)
};

// Expand work item t (PrefillSlice records; see internal.h): one key part of a 128-row q tile.
__device__ __forceinline__ TileDesc tile_desc(const AttnParams& p, int t) {
  int i = 0;
  while (i + 1 < p.n_slices && __ldg(&p.slices[i + 1].tbase) <= t) ++i;
  const PrefillSlice sl = p.slices[i];
  const int local = t - sl.tbase;
  const int tl = local / sl.parts;            // q tile of the slice (parts of a tile are consecutive)
  const int qt = sl.nqt - 1 - tl / p.Hkv;     // largest key ranges first
  TileDesc d;
  d.tbl = sl.tbl;
  d.o = sl.o;
  d.c = sl.c;
  d.t0 = qt * p.R;
  d.row0 = sl.row0;
  d.kvh = tl % p.Hkv;
  d.nkeys = sl.o + min(d.t0 + p.R, sl.c);
  d.nblk = (d.nkeys + p.B - 1) / p.B;
  const int nk = (d.nkeys + 127) >> 7;
  d.parts = sl.parts;
  d.part = local - tl * sl.parts;
  d.j0 = d.part * nk / sl.parts;
  d.j1 = (d.part + 1) * nk / sl.parts;
  d.stile = sl.pbase + tl;
  return d;
}

// Prefill CTA pairs (p.pairs): item t = (slice, q-tile pair, kv head); CTA `rank` of the
// cluster takes q tile nqt-1 - 2*pair - rank.  Both run the pair's key steps (those of the
// longer tile, rank 0's); a missing partner tile (odd nqt) is a tile with no valid rows.
__device__ __forceinline__ TileDesc tile_desc_pair(const AttnParams& p, int t, int rank) {
  int i = 0, base = 0;
  for (;; ++i) {
    const int npi = (p.slices[i].nqt + 1) / 2 * p.Hkv;
    if (i + 1 >= p.n_slices || t < base + npi) break;
    base += npi;
  }
  const PrefillSlice sl = p.slices[i];
  const int local = t - base;
  const int qp = local / p.Hkv;
  const int qt_a = sl.nqt - 1 - 2 * qp;  // rank 0's (longer) tile
  const int qt = qt_a - rank;
  TileDesc d;
  d.tbl = sl.tbl;
  d.o = sl.o;
  d.row0 = sl.row0;
  d.kvh = local - qp * p.Hkv;
  d.t0 = (qt >= 0 ? qt : qt_a) * p.R;
  d.c = qt >= 0 ? sl.c : d.t0;  // no partner tile: no valid rows (c - t0 = 0)
  d.nkeys = sl.o + min(qt_a * p.R + p.R, sl.c);
  d.nblk = (d.nkeys + p.B - 1) / p.B;
  d.parts = 1;
  d.part = 0;
  d.j0 = 0;
  d.j1 = (d.nkeys + 127) >> 7;
  d.stile = 0;
  return d;
}

// Split-K merge of one q tile (run by the CTA of its last part): for each of the 128 rows
// (g heads x R chunk rows) m = max_s m_s, w_s = 2^(m_s - m) l_s, o = sum_s w_s o~_s / sum_s w_s
// in part order (deterministic), LSE = (m + log2 sum w) ln 2.  Threads take (row, 4 dims).
__device__ __forceinline__ void prefill_merge(const AttnParams& p, const TileDesc& t) {
  using namespace fa;
  const int g = p.g, R = p.R;
  const int vrows = min(R, t.c - t.t0);
  const int64_t base = static_cast<int64_t>(t.stile) * t.parts * 128;
  for (int idx = threadIdx.x; idx < 128 * (kD / 4); idx += kThreads) {
    const int r = idx / (kD / 4), c4 = idx - r * (kD / 4);
    const int hh = r / R, i = r - hh * R;
    if (i >= vrows) continue;
    float M = -INFINITY;
    for (int s = 0; s < t.parts; ++s) M = fmaxf(M, __ldcg(p.ppart_ml + (base + s * 128 + r) * 2));
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < t.parts; ++s) {
      const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.ppart_ml + (base + s * 128 + r) * 2));
      const float w = ex2(ml.x - M) * ml.y;
      const float4 v = __ldcg(reinterpret_cast<const float4*>(p.ppart_o + (base + s * 128 + r) * kD) + c4);
      L += w;
      acc.x += w * v.x;
      acc.y += w * v.y;
      acc.z += w * v.z;
      acc.w += w * v.w;
    }
    const float inv = 1.f / L;
    const int h = t.kvh * g + hh;
    const int64_t trow = t.row0 + t.t0 + i;
    uint2 w2;
    w2.x = pack_bf16(acc.x * inv, acc.y * inv);
    w2.y = pack_bf16(acc.z * inv, acc.w * inv);
    put_out(p, static_cast<uint8_t*>(p.o) + ((static_cast<int64_t>(h) * p.T + trow) * kD + c4 * 4) * 2, w2);
    if (c4 == 0 && p.lse != nullptr) put_out(p, p.lse + static_cast<int64_t>(h) * p.T + trow, (M + __log2f(L)) * 0.69314718055994530942f);
  }
}

// Roles inside the 384-thread CTA: warp 0 lanes < 8 stream K tiles, warp 2 lanes < 8
// V^T tiles (bulk copies of the pre-laid-out paged blocks), warp 1 lane 0 issues the
// tcgen05 MMAs, warps 4-7 and 8-11 run the softmax of even / odd key steps (thread =
// TMEM lane = tile row r = hh*R + i, GQA packing).
// Pipeline per key tile j (global iteration g = it + j; S buffer g % 3):
//   MMA:     QK_{j+1} -> S[(g+1)%3] (once PV_{j-2} has read P from it),  PV_j (P from S[g%3])
//   softmax: S_g -> row max -> m chain from step j-1 -> [rare: wait PV_{j-1}, rescale O
//            in TMEM] -> exps -> P over S_g in TMEM -> arrive
__device__ __forceinline__ void prefill_tile(const AttnParams& p, const TileDesc& t, uint32_t sbase, uint32_t bars,
                                             uint32_t tmem, float* xch, uint8_t* xch_base, uint32_t& kv_it, uint32_t& it) {
  using namespace fa;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int g = p.g, R = p.R;
  const uint32_t rank = p.pairs ? cluster_ctarank() : 0u;
  const int vrows = min(R, t.c - t.t0);
  const int nk = (t.nkeys + kBN - 1) / kBN;   // key steps of the whole q tile
  const int j0 = t.j0, j1 = t.j1, n = j1 - j0;  // this item's steps (split-K part)
#if NIYAMA_DIAG_TILES  // per-tile stamps instead (main loop): [claim | Q ready | tile end][tile]
  int64_t* ev = nullptr;
#else
  int64_t* ev = (p.trace != nullptr && blockIdx.x == 0 && it == 0) ? p.trace + 8 * 160 : nullptr;  // [10][64]
#endif

  // ---- Q tile: rows r = hh*R + i  <-  q[row0 + t0 + i][kvh*g + hh][:]
  if (kQTmem) {  // TMEM lane r, columns [kTmemQ, +64): dims (2c, 2c+1) in column c
    if (warp >= 4 && warp < 8) {
      const int r = (warp & 3) * 32 + lane;
      const int hh = r / R, i = r - hh * R;
      uint32_t w[64];
      if (i < vrows) {
        const uint4* src = reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(p.q) +
                                                          (((t.row0 + t.t0 + i) * static_cast<int64_t>(p.Hq) + t.kvh * g + hh) * kD) * 2);
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const uint4 v = __ldg(src + c);
          w[4 * c] = v.x, w[4 * c + 1] = v.y, w[4 * c + 2] = v.z, w[4 * c + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 64; ++c) w[c] = 0u;
      }
      const uint32_t qa = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + kTmemQ;
      tmem_st32(qa, *reinterpret_cast<uint32_t(*)[32]>(w));
      tmem_st32(qa + 32, *reinterpret_cast<uint32_t(*)[32]>(w + 32));
      tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  } else {
    // All of a thread's pieces are loaded before any is stored, so the ~6 loads per
    // thread are in flight together (one memory latency per tile instead of six: the
    // serial version took ~10 K cycles per tile, tools/tile_trace.py).
    // NIYAMA_EARLY_KV: the K/V producer warps (0, 2) skip the Q load and start the item's
    // bulk copies at once, so the ring fill overlaps the Q load; the other 10 warps load Q
    // and meet at a named barrier (the QK issuer is one of them).
    const uint8_t* q = static_cast<const uint8_t*>(p.q);
    constexpr int kLoaders = NIYAMA_EARLY_KV ? kThreads - 64 : kThreads;
    const bool loader = !NIYAMA_EARLY_KV || (warp != 0 && warp != 2);
    const int lidx = NIYAMA_EARLY_KV ? (warp == 1 ? lane : (warp - 2) * 32 + lane) : tid;
    if (loader) {
      constexpr int kQPer = (128 * 16 + kLoaders - 1) / kLoaders;
      uint4 qv[kQPer];
#pragma unroll
      for (int k = 0; k < kQPer; ++k) {
        const int idx = lidx + k * kLoaders;
        const int r = idx >> 4, j = idx & 15;
        const int hh = r / R, i = r - hh * R;
        qv[k] = make_uint4(0, 0, 0, 0);
        if (idx < 128 * 16 && i < vrows) {
          const int64_t row = t.row0 + t.t0 + i;
          qv[k] = __ldg(reinterpret_cast<const uint4*>(q + ((row * p.Hq + t.kvh * g + hh) * kD) * 2 + j * 16));
        }
      }
#pragma unroll
      for (int k = 0; k < kQPer; ++k) {
        const int idx = lidx + k * kLoaders;
        if (idx >= 128 * 16) break;
        const int r = idx >> 4, j = idx & 15;
        st_shared_v4(sbase + kQOff + (j >> 3) * kPanel + r * 128 + (((j & 7) ^ (r & 7)) << 4), qv[k].x, qv[k].y,
                     qv[k].z, qv[k].w);
      }
      fence_proxy_async_smem();
      if (NIYAMA_EARLY_KV)
        named_bar_sync(13, kLoaders);
      else
        __syncthreads();
    }
  }
#if NIYAMA_DIAG_TILES
  if (p.trace != nullptr && blockIdx.x == 0 && tid == 0 && p.trace[8 * 160 + 3 * 64] < 64) {
    int64_t c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    p.trace[8 * 160 + 64 + p.trace[8 * 160 + 3 * 64]] = c;
  }
#endif

  if (warp == 0 || warp == 2) {
    // ---------------- producers: 128-key K tiles (warp 0), V^T tiles (warp 2).
    // Lane u < 8 owns piece u of every step: K = block u of the step (two 128-byte
    // panels of B rows, at B = 16), V^T = the 16-key sub-block u.  Its block-table
    // lookup for step j+1 is issued before step j's copies, so the lookups of a
    // step run in parallel and off the critical path (a deeper lookahead measured no
    // change); lane 0 arms the barrier.
    const bool isK = warp == 0;
    const uint8_t* pool = isK ? p.pool_k : p.pool_v;
    const uint32_t ring = sbase + (isK ? kKOff : kVOff);
    const int bar_full = isK ? kBarKFull : kBarVFull, bar_empty = isK ? kBarKEmpty : kBarVEmpty;
    const uint32_t nstg = isK ? kKStages : kVStages;
    const int bpt = kBN / p.B;                  // K: blocks per key step
    const int npc = isK ? bpt : kBN / 16;       // pieces per step
    auto piece_off = [&](int j) -> int64_t {    // byte offset of this lane's piece of step j
      if (lane >= npc || j >= nk) return 0;
      if (isK) {
        const int lb = min(j * bpt + lane, t.nblk - 1);  // past the end: finite data, masked (P = 0)
        return (static_cast<int64_t>(__ldg(p.tables + t.tbl + lb)) * p.Hkv + t.kvh) * p.chunk_stride;
      }
      const int key = j * kBN + 16 * lane;
      const int lb = min(key >> p.b_shift, t.nblk - 1);
      return (static_cast<int64_t>(__ldg(p.tables + t.tbl + lb)) * p.Hkv + t.kvh) * p.chunk_stride +
             static_cast<int64_t>((key & (p.B - 1)) >> 4) * 4096;
    };
    int64_t next = piece_off(j0);
    for (int j = j0; j < j1; ++j) {
      const int64_t cur = next;
      next = piece_off(j + 1);
      const uint32_t k_it = kv_it + (j - j0);
      const int st = k_it % nstg;
      const uint32_t full = bars + 8 * (bar_full + st);
      if (lane == 0) {
        mbar_wait(bars + 8 * (bar_empty + st), ((k_it / nstg) & 1) ^ 1);
        ev_stamp(ev, isK ? 0 : 1, j);
        mbar_expect_tx(full, NIYAMA_DIAG_HALF_KV ? kTile / 2 : kTile);
      }
      __syncwarp();
      const uint32_t dst0 = ring + st * kTile;
      // CTA pairs: this CTA issues the pieces it owns (odd/even lanes; a single K piece: rank 0)
      // multicast into both CTAs of the cluster, whose full barriers each expect the whole step
      const bool own = !p.pairs || (npc >= 2 ? (lane & 1) == static_cast<int>(rank) : rank == 0);
      if (lane < (NIYAMA_DIAG_HALF_KV ? npc / 2 : npc) && own) {  // (diagnostic: half the bytes, wrong results)
        const uint32_t bytes = isK ? static_cast<uint32_t>(p.chunk_bytes) : 4096u;
        const uint32_t dst = dst0 + lane * bytes;  // K: one copy per block (B rows x 256 B); V^T: sub-block
        if (p.pairs)
          bulk_g2s_mc(dst, pool + cur, bytes, full, 0x3);
        else
          bulk_g2s(dst, pool + cur, bytes, full);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- QK^T issuer.  Issuing blocks while earlier MMAs execute (the
      // tensor pipe's queue is a few MMAs deep; a burst of 8 takes ~0.7 K cycles,
      // tools/umma_issue_test.cu), so QK^T and PV have an issuing thread each: neither
      // stream's readiness waits behind the other's issue.
      for (int j = j0; j < j1; ++j) {
        const uint32_t k_it = kv_it + (j - j0), gj = it + (j - j0);
        const int st = k_it % kKStages, sb = gj % kSBufs;
        if (gj >= kSBufs)  // S[sb] free: loaded by softmax_{j-2} (kPSep) / PV_{j-3} read its P
          mbar_wait(bars + 8 * ((kPSep ? kBarSFree : kBarODone) + sb), ((gj - kSBufs) / kSBufs) & 1);
        mbar_wait(bars + 8 * (kBarKFull + st), (k_it / kKStages) & 1);
        tc_fence_after();
        ev_stamp(ev, 2, j);
        const uint32_t qa = sbase + kQOff, ka = sbase + kKOff + st * kTile;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t koff = (kk >> 2) * kPanel + (kk & 3) * 32;
          if (kQTmem)
            umma_ts(tmem + sb * 128, tmem + kTmemQ + kk * 8, noswz_desc(ka + kk * 256, 128, 2048), kIdescQK, kk > 0);
          else
            umma_f16(tmem + sb * 128, sw128_desc(qa + koff, 16, 1024), noswz_desc(ka + kk * 256, 128, 2048),
                     kIdescQK, kk > 0);
        }
        umma_commit(bars + 8 * (kBarSFull + sb));
        if (p.pairs)  // the stage is free only when both CTAs' QK^T have read it
          umma_commit_mc(bars + 8 * (kBarKEmpty + st), 0x3);
        else
          umma_commit(bars + 8 * (kBarKEmpty + st));
        ev_stamp(ev, 9, j);
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {
      // ---------------- PV issuer
      for (int j = j0; j < j1; ++j) {
        const uint32_t k_it = kv_it + (j - j0), gj = it + (j - j0);
        const int st = k_it % kVStages, sb = gj % kSBufs;
        mbar_wait(bars + 8 * (kBarPFull + sb), (gj / kSBufs) & 1);
        mbar_wait(bars + 8 * (kBarVFull + st), (k_it / kVStages) & 1);
        tc_fence_after();
        ev_stamp(ev, 3, j);
        const uint32_t va = sbase + kVOff + st * kTile;
        // O += P V: A = P (bf16, 128 rows x 16 keys per MMA) from TMEM columns
        // [S[sb] + 8 kk, +8) (TS form), B = the V^T sub-block kk (SW32 K-major)
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          umma_ts(tmem + kTmemO, tmem + (kPSep ? kTmemP + sb * 64 : sb * 128) + kk * 8, sw32_desc(va + kk * 4096, 16, 256), kIdescPV,
                  (j > j0 || kk > 0) ? 1u : 0u);
        umma_commit(bars + 8 * (kBarODone + sb));
        if (p.pairs)
          umma_commit_mc(bars + 8 * (kBarVEmpty + st), 0x3);
        else
          umma_commit(bars + 8 * (kBarVEmpty + st));
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax: two warp sets take alternate key steps (set = parity
    // of the global step gj), so one set's exponentials (MUFU-bound) overlap the
    // other's TMEM loads, row max, P stores and barrier waits.  Thread = tile row r
    // (TMEM lane r) in both sets.  The running max is a chain: the set on step j
    // receives m_{j-1} from the other set (shared memory + named barrier) after its
    // own row max, decides m_j (lazy: raised only when it grows by > 8 in log2
    // units) and passes it on.  Each set keeps its partial row sum l at the max it
    // last used; the two are combined in the epilogue.  S is read from TMEM twice
    // (row max, then exponentials) in 64-column halves to bound registers.
    const int quarter = warp & 3;
    const int set = (warp - 4) >> 2;
    const int r = quarter * 32 + lane;
    const int hh = r / R, i = r - hh * R;
    const bool valid = i < vrows;
    const int pos = t.o + t.t0 + (valid ? i : 0);  // last visible key of this row
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    uint8_t* smem_gen = xch_base;
    volatile float* chain = reinterpret_cast<volatile float*>(xch);  // [set][128]: m passed by that set
    const int bar_in = 1 + 4 * set + quarter, bar_out = 1 + 4 * (set ^ 1) + quarter;
    float m_set = -INFINITY, l = 0.f;  // this set's partial sum, expressed at max m_set
    float m_ref = -INFINITY;           // max of the latest step this set handled
    const float sl2 = p.scale_log2;
    const bool tracer = quarter == 0 && lane == 0;
    for (int j = j0; j < j1; ++j) {
      const uint32_t gj = it + (j - j0);
      if (static_cast<int>(gj & 1) != set) continue;
      const int sb = gj % kSBufs;
      mbar_wait(bars + 8 * (kBarSFull + sb), (gj / kSBufs) & 1);
      tc_fence_after();
      if (tracer) ev_stamp(ev, 4, j);
#if NIYAMA_DIAG_SKIP_SOFTMAX  // timing diagnostic only: P = S bits, no softmax work (wrong results)
      tc_fence_before();
      if (kPSep) mbar_arrive(bars + 8 * (kBarSFree + sb));
      mbar_arrive(bars + 8 * (kBarPFull + sb));
      continue;
#endif
      const int kbase = j * kBN;
      const bool diag = kbase + kBN - 1 > pos;
#if NIYAMA_ONE_SLOAD
      // S is loaded from TMEM once (128 registers) and P packed in place over the consumed
      // values; S[sb] is released to QK_{j+2} right after the load
      uint32_t sr[128];
      tmem_ld128(lane_addr + sb * 128, sr);
      if (kPSep) {
        tc_fence_before();
        mbar_arrive(bars + 8 * (kBarSFree + sb));
      }
      if (diag) {
        mask_tail(*reinterpret_cast<uint32_t(*)[64]>(sr), pos - kbase);
        mask_tail(*reinterpret_cast<uint32_t(*)[64]>(sr + 64), pos - (kbase + 64));
      }
      float mx;
      {
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = __uint_as_float(sr[k]);
#pragma unroll
        for (int e = 8; e < 128; ++e) m8[e & 7] = fmaxf(m8[e & 7], __uint_as_float(sr[e]));
        mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      }
#else
      float mx = -INFINITY;
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t sr[64];
        tmem_ld64(lane_addr + sb * 128 + hf * 64, sr);
        if (diag) mask_tail(sr, pos - (kbase + hf * 64));
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = __uint_as_float(sr[k]);
#pragma unroll
        for (int e = 8; e < 64; ++e) m8[e & 7] = fmaxf(m8[e & 7], __uint_as_float(sr[e]));
        mx = fmaxf(mx, fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                             fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))));
      }
#endif
      float m_prev = -INFINITY;
      if (j > j0) {  // m_{j-1} from the other set
        named_bar_sync(bar_in, 64);
        m_prev = chain[(set ^ 1) * 128 + r];
      }
      const float m_new = fmaxf(m_prev, mx * sl2);
      const bool need = m_new > m_prev + 8.0f;  // lazy rescale: p <= 2^8 otherwise
      const float m_use = need ? m_new : m_prev;
      if (j + 1 < j1) {  // pass m_j on
        chain[set * 128 + r] = m_use;
        named_bar_arrive(bar_out, 64);
      }
      if (m_use != m_set) {
        l *= ex2(m_set - m_use);  // 0 while this set has no sum yet (m_set = -inf)
        m_set = m_use;
      }
      m_ref = m_use;
      if (tracer) ev_stamp(ev, 5, j);
      if (j > j0 && __any_sync(0xffffffffu, need)) {
        // rare: rescale O after PV_{j-1} (PV_j waits for our P).  A parity wait is only
        // unambiguous while the barrier is at most one phase behind the awaited one: this
        // set knows PV_{j-4} is done (its P-free wait at step j-2) but not PV_{j-3}, which
        // shares PV_{j-1}'s barrier when there are 2 S buffers.  So first wait for PV_{j-2}
        // (its barrier's previous phase, PV_{j-4}, is known complete; completion of PV_{j-2}
        // implies PV_{j-3}), then for PV_{j-1}.  (Waiting for PV_{j-1} alone returned early
        // whenever PV_{j-3} was still running: O rescaled under a running PV, an
        // intermittent wrong row found by tools/gather_stress.py.)
        const float alpha = ex2(m_prev - m_use);
        if (gj >= 2) mbar_wait(bars + 8 * (kBarODone + (gj - 2) % kSBufs), ((gj - 2) / kSBufs) & 1);
        mbar_wait(bars + 8 * (kBarODone + (gj - 1) % kSBufs), ((gj - 1) / kSBufs) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < kD / 32; ++c) {
          uint32_t ov[32];
          tmem_ld32(lane_addr + kTmemO + c * 32, ov);
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
          tmem_st32(lane_addr + kTmemO + c * 32, ov);
        }
        tmem_wait_st();
      }
      if (tracer) ev_stamp(ev, 7, j);
      const float nm = -m_use;
      float sum0 = 0.f, sum1 = 0.f;
#if NIYAMA_ONE_SLOAD
#pragma unroll
      for (int c = 0; c < 64; ++c) {  // P pair c overwrites sr[c] (its S values were sr[2c], sr[2c+1], c <= 2c)
        const float e0 = ex2(fmaf(__uint_as_float(sr[2 * c]), sl2, nm));
        const float e1 = ex2(fmaf(__uint_as_float(sr[2 * c + 1]), sl2, nm));
        if (c & 1) sum1 += e0 + e1; else sum0 += e0 + e1;
        sr[c] = pack_bf16(e0, e1);
      }
      if (kPSep && gj >= kSBufs) {  // P[sb] free: PV_{j-2} done
        mbar_wait(bars + 8 * (kBarODone + sb), ((gj - kSBufs) / kSBufs) & 1);
        tc_fence_after();
      }
      tmem_st32(lane_addr + (kPSep ? kTmemP + sb * 64 : sb * 128), *reinterpret_cast<uint32_t(*)[32]>(sr));
      tmem_st32(lane_addr + (kPSep ? kTmemP + sb * 64 : sb * 128) + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
#else
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t sr[64];
        tmem_ld64(lane_addr + sb * 128 + hf * 64, sr);
        if (kPSep && hf == 1) {  // S[sb] fully loaded: QK_{j+2} may overwrite it
          tc_fence_before();
          mbar_arrive(bars + 8 * (kBarSFree + sb));
        }
        if (diag) mask_tail(sr, pos - (kbase + hf * 64));
        // p = 2^(s*scale*log2e - m): one FFMA + one MUFU.EX2 each; P (bf16 pairs, even key
        // in the low half) overwrites the consumed columns [32 hf, 32 hf + 32) of S[sb]
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          float e0, e1;
          if (NIYAMA_POLY_EXP > 0 && c % (NIYAMA_POLY_EXP > 0 ? NIYAMA_POLY_EXP : 1) == 0) {
            // every NIYAMA_POLY_EXP-th pair on the FMA pipe instead of MUFU (FA4's trick)
            e0 = ex2_poly(fmaf(__uint_as_float(sr[2 * c]), sl2, nm));
            e1 = ex2_poly(fmaf(__uint_as_float(sr[2 * c + 1]), sl2, nm));
          } else {
            e0 = ex2(fmaf(__uint_as_float(sr[2 * c]), sl2, nm));
            e1 = ex2(fmaf(__uint_as_float(sr[2 * c + 1]), sl2, nm));
          }
          if (c & 1) sum1 += e0 + e1; else sum0 += e0 + e1;
          pk[c] = pack_bf16(e0, e1);
        }
        if (kPSep && hf == 0 && gj >= kSBufs) {  // P[sb] free: PV_{j-2} done
          mbar_wait(bars + 8 * (kBarODone + sb), ((gj - kSBufs) / kSBufs) & 1);
          tc_fence_after();
        }
        tmem_st32(lane_addr + (kPSep ? kTmemP + sb * 64 : sb * 128) + hf * 32, pk);
      }
#endif
      l += sum0 + sum1;
      if (tracer) ev_stamp(ev, 8, j);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bars + 8 * (kBarPFull + sb));
      if (tracer) ev_stamp(ev, 6, j);
    }
    // ---------------- epilogue: combine the sets' (l, m); O / l -> bf16 (set s writes
    // dims [64 s, 64 s + 64)), LSE
    mbar_wait(bars + 8 * (kBarODone + (it + n - 1) % kSBufs), ((it + n - 1) / kSBufs) & 1);
    tc_fence_after();
    {
      // every MMA of the tile has completed, so the Q tile's shared memory is free:
      // exchange (l, m_set) of the two sets through it
      float2* xq = reinterpret_cast<float2*>(smem_gen + kXOff);
      xq[set * 128 + r] = make_float2(l, m_set);
      named_bar_sync(9 + quarter, 64);
      // the set that handled step j1-2 may have passed its ODone wait early (same
      // two-phases-behind ambiguity as above); the set of the last step waited for PV_{j1-1}
      // unambiguously, and O is read only after this barrier with it
      tc_fence_after();
      const float2 other = xq[(set ^ 1) * 128 + r];
      m_ref = fmaxf(m_set, other.y);  // the max of the last step (the chain never decreases)
      l = l * ex2(m_set - m_ref) + other.x * ex2(other.y - m_ref);
    }
    const float inv_l = 1.f / l;
    const int h = t.kvh * g + hh;
    const int64_t trow = t.row0 + t.t0 + i;
    const uint32_t col0 = static_cast<uint32_t>(set * 64);
    uint8_t* orow = static_cast<uint8_t*>(p.o) + ((static_cast<int64_t>(h) * p.T + trow) * kD + col0) * 2;
    if (t.parts > 1) {
      // split-K part: the normalised partial o / l (fp32) and (m, l) of this row; the part
      // that completes the tile merges (prefill_merge)
      const int64_t slot = (static_cast<int64_t>(t.stile) * t.parts + t.part) * 128 + r;
      float* po = p.ppart_o + slot * kD + col0;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t ov[32];
        tmem_ld32(lane_addr + kTmemO + col0 + c * 32, ov);
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          __stcg(reinterpret_cast<float4*>(po + c * 32 + e),
                 make_float4(__uint_as_float(ov[e]) * inv_l, __uint_as_float(ov[e + 1]) * inv_l,
                             __uint_as_float(ov[e + 2]) * inv_l, __uint_as_float(ov[e + 3]) * inv_l));
      }
      if (set == 0) __stcg(reinterpret_cast<float2*>(p.ppart_ml + slot * 2), make_float2(m_ref, l));
      __threadfence();
    } else {
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t ov[32];
      tmem_ld32(lane_addr + kTmemO + col0 + c * 32, ov);
      if (valid) {
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(ov[e + 0]) * inv_l, __uint_as_float(ov[e + 1]) * inv_l);
          w.y = pack_bf16(__uint_as_float(ov[e + 2]) * inv_l, __uint_as_float(ov[e + 3]) * inv_l);
          w.z = pack_bf16(__uint_as_float(ov[e + 4]) * inv_l, __uint_as_float(ov[e + 5]) * inv_l);
          w.w = pack_bf16(__uint_as_float(ov[e + 6]) * inv_l, __uint_as_float(ov[e + 7]) * inv_l);
          put_out(p, orow + (c * 32 + e) * 2, w);
        }
      }
    }
    if (set == 0 && valid && p.lse != nullptr)
      put_out(p, p.lse + static_cast<int64_t>(h) * p.T + trow, (m_ref + __log2f(l)) * 0.69314718055994530942f);
    }
  }
  kv_it += n;
  it += n;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t.parts > 1) {
    // split-K completion: the part that brings the tile's count to (epoch + 1) * parts merges
    volatile int* flag = reinterpret_cast<volatile int*>(xch_base + kXOff + 2040);
    if (tid == 0) {
      const int old = atomicAdd(p.pcounters + t.stile, 1);
      *flag = old + 1 == (p.epoch + 1) * t.parts;
    }
    __syncthreads();
    const bool last = *flag != 0;
    __syncthreads();
    if (last) {
      __threadfence();
      prefill_merge(p, t);
      __syncthreads();
    }
  }
}

// --------------------------------------------------------------- decode unit
struct UnitDesc {
  int id, tbl, row, kvh, k0, k1, nsplit, crow;
};

// Per-warp unit-descriptor ring (4 entries) and its published count live in shared
// memory; lane 0 writes, the warp reads after __syncwarp (which orders shared
// memory among the warp's lanes), so plain st/ld.shared suffice.
__device__ __forceinline__ void desc_store(uint32_t ring, int k, const UnitDesc& d) {
  const uint32_t a = ring + (k & 3) * 32;
  asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(d.id), "r"(d.tbl), "r"(d.row), "r"(d.kvh)
               : "memory");
  asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(a + 16), "r"(d.k0), "r"(d.k1), "r"(d.nsplit),
               "r"(d.crow)
               : "memory");
}
__device__ __forceinline__ UnitDesc desc_load(uint32_t ring, int k) {
  const uint32_t a = ring + (k & 3) * 32;
  UnitDesc d;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(d.id), "=r"(d.tbl), "=r"(d.row), "=r"(d.kvh) : "r"(a)
               : "memory");
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(d.k0), "=r"(d.k1), "=r"(d.nsplit), "=r"(d.crow)
               : "r"(a + 16)
               : "memory");
  return d;
}
__device__ __forceinline__ void count_store(uint32_t a, int v) {
  asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int count_load(uint32_t a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

// x / Hkv and x % Hkv without a runtime integer division (a ~100-cycle dependent
// sequence) whenever Hkv is a power of two.
__device__ __forceinline__ int div_hkv(const AttnParams& p, int x) {
  return p.hkv_shift >= 0 ? x >> p.hkv_shift : x / p.Hkv;
}

// Unit = (row, split s, kv head h); d.id = its canonical partial index ubase + s*Hkv + h.
__device__ __forceinline__ UnitDesc make_unit(const UnitRec& r, int h) {
  UnitDesc d;
  d.id = r.pbase + h;
  d.tbl = r.tbl;
  d.row = r.row;
  d.kvh = h;
  d.k0 = r.k0;
  d.k1 = r.k1;
  d.nsplit = r.nsplit;
  d.crow = r.crow;
  return d;
}

// Stage s of a unit = 16 tokens of one kv head: K then V (4 KB each at d = 128 bf16).
// `phys` is the physical block holding the stage (looked up one stage ahead).
__device__ __forceinline__ void decode_issue(const AttnParams& p, const UnitDesc& u, int s, int phys,
                                             uint32_t stage, uint32_t bar) {
  const int tok = u.k0 + 16 * s;
  const int sub = (tok & (p.B - 1)) >> 4;  // 16-token sub-block of the block
  const int64_t chunk = (static_cast<int64_t>(phys) * p.Hkv + u.kvh) * p.chunk_stride;
  // Streamed once: evict-first keeps the KV stream from displacing reused lines in L2
  // (measured: config 2 108.6 -> 102.6 us, decode-only 95.7 -> 91.3 us per launch).
  const uint64_t pol = policy_evict_first();
  mbar_expect_tx(bar, fa::kDecStage);
  if (p.kv_adjacent && p.B == 16) {  // the block's K chunk and V^T chunk are one 8 KB run
    bulk_g2s_hint(stage, p.pool_k + chunk, 8192, bar, pol);
  } else {
    bulk_g2s_hint(stage, p.pool_k + chunk + sub * 4096, 4096, bar, pol);  // K: 16 rows = two 8-row core groups
    bulk_g2s_hint(stage + 4096, p.pool_v + chunk + sub * 4096, 4096, bar, pol);  // V^T sub-block [128 d][16 keys]
  }
}



// Load side of a decode warp (lane 0 only).  It walks a continuous stream of
// 16-token stages across unit boundaries, keeping kDecStages in flight.  Every
// dependent global load is issued one step before its value is needed: the
// block-table entry of the NEXT stage is fetched while the current one is issued,
// and the next unit is prepared one step per issued stage (queue atomic -> its
// row index -> row record -> descriptor + first block), so lane 0 never waits on
// memory in the issue path.  Each new unit's descriptor is published to the
// compute lanes through a 4-entry per-warp ring in shared memory (+ a counter).
template <int kDecStages>
struct DecodeLoader {
  UnitDesc cur;
  int s, nst;
  int phys;  // block of stage s of cur (32-bit: loaded one stage before it is consumed)
  int nxt_id, nxt_step;  // 0 nothing, 1 id claimed, 2 record requested
  int reserved;          // this warp's pre-assigned first unit (decode-first CTAs), -1 if none
  int id_base;           // ids [0, id_base) are pre-assigned; the queue counter hands out the rest
  int4 nxt_a, nxt_b, nxt_c;  // raw UnitRec of the next unit, unpacked only when it starts
  int nd;                // descriptors published so far (lane 0's copy of the shared count)
  int ph1, ph2;          // blocks of stages 1 and 2 of cur (from its record)
  bool warm;             // initial ring fill done: the next-unit claim may proceed
  bool done;
  uint32_t issued;

  __device__ __forceinline__ void advance(const AttnParams& p) {
    if (nxt_step == 0) {
      if (reserved >= 0) {
        nxt_id = reserved;
        reserved = -1;
      } else {
        nxt_id = id_base + atomicAdd(p.work + 1, 1);
      }
    } else if (nxt_step == 1) {
      if (nxt_id < p.n_units) {
        const int4* rp = reinterpret_cast<const int4*>(p.uq + div_hkv(p, nxt_id));
        nxt_a = __ldg(rp);
        nxt_b = __ldg(rp + 1);
        nxt_c = __ldg(rp + 2);
      }
    } else {
      return;
    }
    ++nxt_step;
  }
  __device__ __forceinline__ void issue_next(const AttnParams& p, uint32_t ring, uint32_t bar0, uint32_t descs,
                                             uint32_t n_desc) {
    using namespace fa;
    if (done) return;
    if (s == nst) {
      while (nxt_step < 2) advance(p);
      const int k = nd;
      if (nxt_id >= p.n_units) {
        done = true;
        UnitDesc end{};
        end.id = -1;  // end of stream
        desc_store(descs, k, end);
        __threadfence_block();  // descriptor before count (decode_path 2: read by another warp)
        count_store(n_desc, ++nd);
        return;
      }
      const UnitRec rec{nxt_a.x, nxt_a.y, nxt_a.z, nxt_a.w, nxt_b.x, nxt_b.y, nxt_b.z, nxt_b.w, nxt_c.x, nxt_c.y, 0, 0};
      cur = make_unit(rec, nxt_id - div_hkv(p, nxt_id) * p.Hkv);
      phys = rec.phys0;
      ph1 = rec.phys1;
      ph2 = rec.phys2;
      s = 0;
      nst = (cur.k1 - cur.k0 + 15) >> 4;
      nxt_step = 0;
      desc_store(descs, k, cur);
      __threadfence_block();
      count_store(n_desc, ++nd);
    }
    const uint32_t slot = issued % kDecStages;
    decode_issue(p, cur, s, phys, ring + slot * kDecStage, bar0 + 8 * slot);
    ++s;
    ++issued;
    if (s < nst) {
      if (s <= 2) {
        phys = s == 1 ? ph1 : ph2;  // from the unit record
      } else {
        const int lb_prev = (cur.k0 + 16 * (s - 1)) >> p.b_shift, lb = (cur.k0 + 16 * s) >> p.b_shift;
        if (lb != lb_prev) phys = __ldg(p.tables + cur.tbl + lb);  // consumed by the next call
      }
    }
    // During the initial ring fill only the claim itself (step 0) is issued: its
    // result is first needed after the fill, so the fill never waits on it.
    if (warm || nxt_step == 0) advance(p);
  }
};

// Raw Q fragments of unit u (A operand rows = the g heads of its group; lanes with
// gid >= g load a valid row and are zeroed by q_mask at use, so no instruction
// depends on the loads until the fragments are consumed).
__device__ __forceinline__ void load_q_frags(const AttnParams& p, const UnitDesc& u, int gid, int tig,
                                             uint32_t (&qa0)[8], uint32_t (&qa2)[8]) {
  const int g = p.g;
  const __nv_bfloat16* qrow = static_cast<const __nv_bfloat16*>(p.q) +
                              (static_cast<int64_t>(u.row) * p.Hq + u.kvh * g + (gid < g ? gid : 0)) * fa::kD;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    qa0[kk] = __ldg(reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * tig));
    qa2[kk] = __ldg(reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 8 + 2 * tig));
  }
}

// Make split unit `c`'s partial (stored by every lane) visible, then count it
// (a6 completion counter; c = crow * Hkv + kv head, -1 = nothing pending).
__device__ __forceinline__ void publish_split(const AttnParams& p, int c, int lane) {
  if (c < 0) return;
  __threadfence();
  __syncwarp();
  if (lane == 0) atomicAdd(p.counters + c, 1);
}

__device__ __forceinline__ int ld_acquire_gpu(const int* ptr) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}

// Compute side: every lane of the warp.  Split rows write an fp32 partial
// (m, l, o~) at index `unit id` (fire and forget); unsplit rows write O / LSE.
// Descriptor k of a consumer warp's ring is published by its producer warp: wait for the
// count, then order the descriptor loads after it.
__device__ __forceinline__ void wait_desc(uint32_t n_desc, int k) {
#ifndef NIYAMA_NO_WATCHDOG
  uint32_t polls = 0;
#endif
  while (count_load(n_desc) <= k) {
    __nanosleep(32);  // a tight shared-memory spin starves the producer warp on this SMSP
#ifndef NIYAMA_NO_WATCHDOG
    if (++polls == (NIYAMA_DIAG_HANG ? (1u << 20) : (1u << 28))) {
      if (NIYAMA_DIAG_HANG && (threadIdx.x & 31) == 0)
        printf("consumer cta %d warp %d: waits for desc %d, count %d\n", blockIdx.x, threadIdx.x >> 5, k,
               count_load(n_desc));
      __trap();
    }
#endif
  }
  __threadfence_block();
}

// decode_path 2: producer warp (lane 0) of consumer warps c0 and c0 + 1.  It runs both
// consumers' DecodeLoader streams (claims, records, table prefetch, descriptor publishing,
// one 8 KB bulk copy per stage) and refills a consumer's slot as soon as its empty barrier
// shows the consumer is done with it — taking the loader's ~30 % of the per-stage cycle off
// the compute warps (ncu round 2: the lane-0 loader was the largest block of decode stall
// samples at g = 8, where warps 8-11 had no decode work at all).
template <int kDecWarpsT, int kDecStages>
__device__ __forceinline__ void decode_producer(const AttnParams& p, uint32_t sbase, uint32_t bars, uint32_t descs_base,
                                                uint32_t n_desc_base, int c0) {
  using namespace fa;
  DecodeLoader<kDecStages> ld[2];
  const int dec_first = p.n_tiles > 0 ? p.prefill_ctas : 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int c = c0 + i;
    ld[i].s = ld[i].nst = 0;
    ld[i].nxt_step = 0;
    ld[i].nxt_id = 0;
    ld[i].id_base = (static_cast<int>(gridDim.x) - dec_first) * kDecWarpsT;
    ld[i].reserved = static_cast<int>(blockIdx.x) >= dec_first
                         ? (static_cast<int>(blockIdx.x) - dec_first) * kDecWarpsT + c
                         : -1;
    ld[i].done = false;
    ld[i].issued = 0;
    ld[i].phys = 0;
    ld[i].warm = false;
    ld[i].ph1 = ld[i].ph2 = 0;
    ld[i].nd = 0;
  }
  auto ring = [&](int i) { return sbase + (c0 + i) * kDecStages * kDecStage; };
  auto fbar = [&](int i) { return bars + 8 * (kBarDec + (c0 + i) * kDecStages); };
  auto ebar = [&](int i) { return bars + 8 * (kBarDecEmpty + (c0 + i) * kDecStages); };
  auto descs = [&](int i) { return descs_base + (c0 + i) * 4 * 32; };
  auto ndesc = [&](int i) { return n_desc_base + (c0 + i) * 16; };
  for (int k = 0; k < kDecStages; ++k)
#pragma unroll
    for (int i = 0; i < 2; ++i) ld[i].issue_next(p, ring(i), fbar(i), descs(i), ndesc(i));
  ld[0].warm = ld[1].warm = true;
#ifndef NIYAMA_NO_WATCHDOG
  uint32_t idle = 0;
#endif
  while (!(ld[0].done && ld[1].done)) {
    bool any = false;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (ld[i].done) continue;
      const uint32_t slot = ld[i].issued % kDecStages;
      const uint32_t use = ld[i].issued / kDecStages;  // >= 1 here: the initial fill covered use 0
      if (mbar_test(ebar(i) + 8 * slot, (use - 1) & 1)) {
        ld[i].issue_next(p, ring(i), fbar(i), descs(i), ndesc(i));
        any = true;
      }
    }
    if (!any) __nanosleep(20);  // yield the SMSP to the consumer warps while their slots are busy
#ifndef NIYAMA_NO_WATCHDOG
    if (any) {
      idle = 0;
    } else if (++idle == (NIYAMA_DIAG_HANG ? (1u << 20) : (1u << 28))) {
#if NIYAMA_DIAG_HANG
      for (int i = 0; i < 2; ++i) {
        uint64_t st;
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(st) : "r"(ebar(i) + 8 * (ld[i].issued % kDecStages)));
        printf("producer cta %d c %d: issued %u done %d s %d nst %d nxt_id %d nd %d ebar %llx\n", blockIdx.x, c0 + i,
               ld[i].issued, ld[i].done, ld[i].s, ld[i].nst, ld[i].nxt_id, ld[i].nd, (unsigned long long)st);
      }
#endif
      __trap();
    }
#endif
  }
}

// kProd (decode_path 2): this warp only computes; a producer warp (decode_producer) claims its
// units, publishes their descriptors and issues its stage copies, and the warp hands each
// consumed stage back through the slot's empty barrier.  Otherwise lane 0 is the warp's own
// loader (DecodeLoader), interleaved with the compute.
template <int kDecWarpsT, int kDecStages, bool kProd = false>
__device__ __forceinline__ void decode_warp_loop(const AttnParams& p, uint32_t sbase, uint32_t bars,
                                                 uint32_t descs, uint32_t n_desc) {
  using namespace fa;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int g = p.g;
  const uint32_t ring = sbase + warp * kDecStages * kDecStage;
  const uint32_t bar0 = bars + 8 * (kBarDec + warp * kDecStages);
  uint32_t dec_iter = 0;
  const float sl2 = p.scale_log2;
  const int mi = lane >> 3, rr = lane & 7;

  DecodeLoader<kDecStages> ld;
  ld.s = ld.nst = 0;
  ld.nxt_step = 0;
  ld.nxt_id = 0;
  {
    // CTAs that start with decode get one pre-assigned unit per warp (LPT order), so
    // the first claim is a plain load instead of an atomic; prefill-first CTAs and
    // every later claim use the queue counter.
    const int dec_first = p.n_tiles > 0 ? p.prefill_ctas : 0;
    ld.id_base = (static_cast<int>(gridDim.x) - dec_first) * kDecWarpsT;
    ld.reserved = static_cast<int>(blockIdx.x) >= dec_first
                      ? (static_cast<int>(blockIdx.x) - dec_first) * kDecWarpsT + warp
                      : -1;
  }
  ld.done = false;
  ld.issued = 0;
  ld.phys = 0;
  ld.warm = false;
  ld.ph1 = ld.ph2 = 0;
  ld.nd = 0;
  if (!kProd && lane == 0) {
    count_store(n_desc, 0);
    for (int k = 0; k < kDecStages; ++k) ld.issue_next(p, ring, bar0, descs, n_desc);
  }
  ld.warm = true;
  __syncwarp();
  const uint32_t ebar0 = bars + 8 * (kBarDecEmpty + warp * kDecStages);  // kProd: slot empty barriers

  uint32_t qn0[8], qn2[8];
  bool qn_valid = false;
  int pending = -1;  // completion counter of the last split unit, not yet published
  for (int ck = 0;; ++ck) {
    __syncwarp();
    if (kProd) wait_desc(n_desc, ck);
    const UnitDesc u = desc_load(descs, ck);
    if (u.id < 0) break;
    const int nst = (u.k1 - u.k0 + 15) >> 4;
    uint32_t qa0[8], qa2[8];
    if (qn_valid) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) qa0[kk] = qn0[kk], qa2[kk] = qn2[kk];
    } else {
      load_q_frags(p, u, gid, tig, qa0, qa2);
    }
    qn_valid = false;
    if (gid >= g) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) qa0[kk] = qa2[kk] = 0u;
    }
    float o[8][4];  // O^T m-tiles: (dim 16md + gid (+8), heads 2tig, 2tig+1)
#pragma unroll
    for (int n = 0; n < 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m = -INFINITY, l = 0.f;      // head 2*tig
    float mB = -INFINITY, lB = 0.f;    // head 2*tig + 1
    for (int s = 0; s < nst; ++s) {
      const uint32_t slot = dec_iter % kDecStages;
      const uint32_t ph = (dec_iter / kDecStages) & 1;
      const uint32_t stg = ring + slot * kDecStage;
      // diagnostics (p.trace, decode-only launches): warp 0 of CTA 0, first 64 stages
      // (compiled in only with NIYAMA_DIAG_STEPS: the per-stage checks and stores cost ~5 % of
      // the decode loop's stall samples, ncu round 2)
      int64_t* dev = (NIYAMA_DIAG_STEPS && p.trace != nullptr && p.n_tiles == 0 && blockIdx.x == 0 && warp == 0 &&
                      lane == 0 && dec_iter < 64) ? p.trace + 8 * 160 : nullptr;
      auto dstamp = [&](int role) {
        if (dev != nullptr) dev[role * 64 + dec_iter] = static_cast<int64_t>(clock64());
      };
      dstamp(0);
      mbar_wait(bar0 + 8 * slot, ph);
      dstamp(1);
      // S^T [16 tok x 8 heads] = K [16 tok x 128 d] . Q^T: A = K via ldmatrix (matrices
      // (tok 0-7, c), (tok 8-15, c), (tok 0-7, c+1), (tok 8-15, c+1)), B = Q fragments.
      float st[4] = {0.f, 0.f, 0.f, 0.f};
      const int ttok = (mi & 1) * 8 + rr;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t addr = stg + (ttok >> 3) * 2048 + (kk * 2 + (mi >> 1)) * 128 + ((ttok & 7) << 4);
        uint32_t a0, a1, a2, a3;
        ldsm_x4(addr, a0, a1, a2, a3);
        mma_bf16_16816(st, a0, a1, a2, a3, qa0[kk], qa2[kk]);
      }
      dstamp(2);
      // st: (tok gid, head 2tig), (tok gid, head 2tig+1), (tok gid+8, 2tig), (tok gid+8, 2tig+1)
      const int tb = u.k0 + 16 * s;
      float x0 = st[0] * sl2, x1 = st[1] * sl2, x2 = st[2] * sl2, x3 = st[3] * sl2;
      if (tb + 16 > u.k1) {
        if (tb + gid >= u.k1) x0 = x1 = -INFINITY;
        if (tb + gid + 8 >= u.k1) x2 = x3 = -INFINITY;
      }
      float mxA = fmaxf(x0, x2), mxB = fmaxf(x1, x3);  // column (head) max over the 16 tokens
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, off));
        mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, off));
      }
      const float mnA = fmaxf(m, mxA), mnB = fmaxf(mB, mxB);
      if (mnA > m) {
        const float alpha = ex2(m - mnA);
        l *= alpha;
#pragma unroll
        for (int md = 0; md < 8; ++md) {
          o[md][0] *= alpha;
          o[md][2] *= alpha;
        }
        m = mnA;
      }
      if (mnB > mB) {
        const float alpha = ex2(mB - mnB);
        lB *= alpha;
#pragma unroll
        for (int md = 0; md < 8; ++md) {
          o[md][1] *= alpha;
          o[md][3] *= alpha;
        }
        mB = mnB;
      }
      const float p0 = ex2(x0 - m), p1 = ex2(x1 - mB), p2 = ex2(x2 - m), p3 = ex2(x3 - mB);
      l += p0 + p2;
      lB += p1 + p3;
      dstamp(3);
      // P^T as the B operand: transpose the two 8x8 (tok x head) halves in registers
      const uint32_t pb0 = movmatrix_trans(pack_bf16(p0, p1)), pb1 = movmatrix_trans(pack_bf16(p2, p3));
      // O^T [128 d x 8 heads] += V^T [128 d x 16 tok] . P^T: A = V^T m-tile via ldmatrix
#pragma unroll
      for (int md = 0; md < 8; ++md) {
        const int dr = 16 * md + (mi & 1) * 8 + rr;
        const uint32_t addr = stg + 4096 + dr * 32 + ((((mi >> 1) ^ (dr >> 2)) & 1) << 4);
        uint32_t a0, a1, a2, a3;
        ldsm_x4(addr, a0, a1, a2, a3);
        mma_bf16_16816(o[md], a0, a1, a2, a3, pb0, pb1);
      }
      // Publish the previous split unit once two stages of this one have gone by: its
      // partial stores have landed by then, so the fence costs nothing.
      if (s == 1 || s == nst - 1) {
        publish_split(p, pending, lane);
        pending = -1;
      }
      if (NIYAMA_DIAG_STEPS && p.trace != nullptr && dec_iter == 0 && warp == 0 && lane == 0) {  // diagnostics: first stage done
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[8 * blockIdx.x + 7] = static_cast<int64_t>(t);
      }
      __syncwarp();
      dstamp(4);
      if (lane == 0) {
        if (kProd)
          mbar_arrive(ebar0 + 8 * slot);  // hand the slot back to the producer
        else
          ld.issue_next(p, ring, bar0, descs, n_desc);  // refill this slot
      }
      dstamp(5);
      ++dec_iter;
      // prefetch the next unit's Q fragments once its descriptor is published
      if (!qn_valid && s + 2 >= nst) {
        __syncwarp();
        if (count_load(n_desc) > ck + 1) {
          if (kProd) __threadfence_block();  // the descriptor was written before the count
          const UnitDesc nu = desc_load(descs, ck + 1);
          if (nu.id >= 0) {
            load_q_frags(p, nu, gid, tig, qn0, qn2);
            qn_valid = true;
          }
        }
      }
    }
    if (u.nsplit > 1) pending = u.crow * p.Hkv + u.kvh;  // published two stages into the next unit
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, off);
      lB += __shfl_xor_sync(0xffffffffu, lB, off);
    }
    const int hA = 2 * tig, hB = 2 * tig + 1;  // this lane's heads (columns of O^T)
    const float invA = 1.f / l, invB = 1.f / lB;
    if (u.nsplit == 1) {
      // transpose (d, head) 8x8 blocks back to (head, d): lane (head gid) gets dims 2tig, 2tig+1
      __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(p.o) +
                            (static_cast<int64_t>(u.kvh * g + gid) * p.T + u.row) * kD;
#pragma unroll
      for (int md = 0; md < 8; ++md) {
        const uint32_t lo = movmatrix_trans(pack_bf16(o[md][0] * invA, o[md][1] * invB));
        const uint32_t hi = movmatrix_trans(pack_bf16(o[md][2] * invA, o[md][3] * invB));
        if (gid < g) {
          put_out(p, orow + 16 * md + 2 * tig, lo);
          put_out(p, orow + 16 * md + 8 + 2 * tig, hi);
        }
      }
      if (gid == 0 && p.lse != nullptr) {
        if (hA < g) put_out(p, p.lse + static_cast<int64_t>(u.kvh * g + hA) * p.T + u.row, (m + __log2f(l)) * 0.69314718055994530942f);
        if (hB < g) put_out(p, p.lse + static_cast<int64_t>(u.kvh * g + hB) * p.T + u.row, (mB + __log2f(lB)) * 0.69314718055994530942f);
      }
    } else {
      float* poA = p.part_o + (static_cast<int64_t>(u.id) * g + hA) * kD;
      float* poB = p.part_o + (static_cast<int64_t>(u.id) * g + hB) * kD;
#pragma unroll
      for (int md = 0; md < 8; ++md) {
        if (hA < g) {
          __stcg(poA + 16 * md + gid, o[md][0] * invA);
          __stcg(poA + 16 * md + 8 + gid, o[md][2] * invA);
        }
        if (hB < g) {
          __stcg(poB + 16 * md + gid, o[md][1] * invB);
          __stcg(poB + 16 * md + 8 + gid, o[md][3] * invB);
        }
      }
      if (gid == 0) {
        if (hA < g) __stcg(reinterpret_cast<float2*>(p.part_ml + (static_cast<int64_t>(u.id) * g + hA) * 2), make_float2(m, l));
        if (hB < g) __stcg(reinterpret_cast<float2*>(p.part_ml + (static_cast<int64_t>(u.id) * g + hB) * 2), make_float2(mB, lB));
      }
    }
  }
  publish_split(p, pending, lane);  // the last split unit of this warp
  if (p.trace != nullptr && warp == 0 && lane == 0) {  // diagnostics: warp 0 ran out of units
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[8 * blockIdx.x + 5] = static_cast<int64_t>(t);
  }

}

// a6 — merge the partials of every split (row, kv head, q head) item (SURVEY §8 a6:
// m = max_s m_s, w_s = e^(m_s - m) l_s, o = sum_s w_s o~_s / sum_s w_s, lse = m + ln
// sum_s w_s).  Run by warps whose decode queue is exhausted, so it overlaps the
// decode tail: items are claimed in readiness order (merge queue) and each waits
// for its (row, kv head) completion counter.  No deadlock: every unit is claimed
// before any warp merges, and unit processing never waits on a merge.  Lane s
// reads split s's (m, l); o slices are accumulated in split order, so the result
// is deterministic.
__device__ __forceinline__ void merge_tail(const AttnParams& p) {
  const int lane = threadIdx.x & 31;
  const int g = p.g;
  const int per_row = p.Hkv * g;
  const int items = p.n_merge_rows * per_row;
  for (;;) {
    int it = 0;
    if (lane == 0) it = atomicAdd(p.work + 3, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= items) break;
    const MergeRec rec = p.mq[it / per_row];
    const int kvh = (it / g) % p.Hkv, hh = it % g;
    {
      const int target = (p.epoch + 1) * rec.nsplit;
      const int* cnt = p.counters + rec.crow * p.Hkv + kvh;
      uint32_t polls = 0;
      while (ld_acquire_gpu(cnt) < target) {
        __nanosleep(64);
#ifndef NIYAMA_NO_WATCHDOG
        if (++polls == (1u << 26)) __trap();  // a lost completion: fail loudly, never hang
#endif
      }
    }
    const int ns = rec.nsplit;
    auto pidx = [&](int sp) -> int64_t {
      return static_cast<int64_t>(rec.ubase + sp * p.Hkv + kvh) * g + hh;
    };
    const int h = kvh * g + hh;
    __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(p.o) + (static_cast<int64_t>(h) * p.T + rec.row) * fa::kD;
    if (ns <= 32) {
      // one round trip: (m, l) of split `lane` and up to 32 o~ slices are loaded together
      float2 ml = make_float2(-INFINITY, 0.f);
      if (lane < ns) ml = __ldcg(reinterpret_cast<const float2*>(p.part_ml + pidx(lane) * 2));
      float4 v[32];
#pragma unroll
      for (int k = 0; k < 32; ++k)
        v[k] = k < ns ? __ldcg(reinterpret_cast<const float4*>(p.part_o + pidx(k) * fa::kD + lane * 4))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
      float M = ml.x;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
      const float w = lane < ns ? ex2(ml.x - M) * ml.y : 0.f;
      float L = w;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k >= ns) break;
        const float wk = __shfl_sync(0xffffffffu, w, k);
        acc.x += wk * v[k].x;
        acc.y += wk * v[k].y;
        acc.z += wk * v[k].z;
        acc.w += wk * v[k].w;
      }
      const float inv = 1.f / L;
      uint2 w2;
      w2.x = pack_bf16(acc.x * inv, acc.y * inv);
      w2.y = pack_bf16(acc.z * inv, acc.w * inv);
      put_out(p, orow + lane * 4, w2);
      if (lane == 0 && p.lse != nullptr)
        put_out(p, p.lse + static_cast<int64_t>(h) * p.T + rec.row, (M + __log2f(L)) * 0.69314718055994530942f);
      continue;
    }
    float M = -INFINITY;
    for (int base = 0; base < ns; base += 32)
      if (base + lane < ns) M = fmaxf(M, __ldcg(p.part_ml + pidx(base + lane) * 2));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int base = 0; base < ns; base += 32) {
      float w = 0.f;
      if (base + lane < ns) {
        const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.part_ml + pidx(base + lane) * 2));
        w = ex2(ml.x - M) * ml.y;
      }
      float ws = w;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, off);
      L += ws;
      const int cnt = min(32, ns - base);
      for (int k0 = 0; k0 < cnt; k0 += 16) {
        float4 v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k)
          v[k] = (k0 + k < cnt) ? __ldcg(reinterpret_cast<const float4*>(p.part_o + pidx(base + k0 + k) * fa::kD +
                                                                         lane * 4))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float wk = __shfl_sync(0xffffffffu, w, k0 + k);
          acc.x += wk * v[k].x;
          acc.y += wk * v[k].y;
          acc.z += wk * v[k].z;
          acc.w += wk * v[k].w;
        }
      }
    }
    const float inv = 1.f / L;
    uint2 w2;
    w2.x = pack_bf16(acc.x * inv, acc.y * inv);
    w2.y = pack_bf16(acc.z * inv, acc.w * inv);
    put_out(p, orow + lane * 4, w2);
    if (lane == 0 && p.lse != nullptr)
      put_out(p, p.lse + static_cast<int64_t>(h) * p.T + rec.row, (M + __log2f(L)) * 0.69314718055994530942f);
  }
}

// ------------------------------------------------- decode, tensor-core CTA pipeline
// (p.dec_mode == 1; constants and barriers in fa::kD2* / kB2*).  Roles:
//   warp 0        producer: claims units (pre-assigned first unit per decode-first CTA,
//                 then the queue counter), publishes their descriptors, writes each
//                 unit's Q^T tile, and streams its 128-token steps: per paged block one
//                 bulk copy of its K rows and one of its V^T sub-blocks (evict-first).
//   warp 1 lane 0 MMA issuer: QK^T of step j+1 is issued before PV of step j, so the
//                 softmax of j overlaps the tensor core.
//   warps 4-7     softmax: thread = TMEM lane = token of the step; per-head max over the
//                 step's 128 tokens (shuffles + 4-warp exchange), lazy O rescale (max
//                 grows by > 8 in log2 units), P^T (bf16) into shared memory; per-thread
//                 partial sums l, reduced once per unit.
//   warps 8-11    epilogue: thread = TMEM lane = head dim; O^T / l -> O (bf16, unsplit
//                 rows) or the fp32 partial (split rows) + the completion count (a6).
__device__ __forceinline__ uint32_t d2_pt_off(int h, int t) {  // P^T [K = 128 tokens][N = 16 heads], K-major
  return (h >> 3) * 2048 + (t >> 3) * 128 + (h & 7) * 16 + (t & 7) * 2;
}

__device__ __forceinline__ void decode_cta_v2(const AttnParams& p, uint32_t sbase, uint32_t bars, uint32_t tmem,
                                              uint32_t scratch) {
  using namespace fa;
  // diagnostics (p.trace): CTA 0, steps < 64: clock64 per role (0 copies issued, 1 QK issued,
  // 2 S ready (softmax), 3 P written, 4 PV issued, 5 stage full seen by the MMA, 6 stage empty
  // seen by the producer)
  int64_t* tr2 = (NIYAMA_DIAG_STEPS && p.trace != nullptr && blockIdx.x == 0) ? p.trace + 8 * 160 : nullptr;
  auto stamp = [&](int role, uint32_t j) {
    if (tr2 != nullptr && j < 64) tr2[role * 64 + j] = static_cast<int64_t>(clock64());
  };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = p.g;
  const uint32_t descs = scratch + kD2Desc;
  auto bar = [&](int b) { return bars + 8 * b; };
  const int tb = p.B < 128 ? p.B : 128;  // tokens of one block inside a step
  if (warp == 2) {
    // ---------------------------------------------------------- unit warp
    // Claims units up to 4 ahead of the pipeline (ring of 4 descriptors + 4 Q^T tiles), so
    // the claim -> record -> Q round trips never stall the K/V stream.  Each descriptor
    // also carries the physical blocks of the unit's first step.
    const int dec_first = p.n_tiles > 0 ? p.prefill_ctas : 0;
    const int id_base = static_cast<int>(gridDim.x) - dec_first;
    int reserved = static_cast<int>(blockIdx.x) >= dec_first ? static_cast<int>(blockIdx.x) - dec_first : -1;
    int next = 0;
    if (lane == 0) next = reserved >= 0 ? reserved : id_base + atomicAdd(p.work + 1, 1);
    for (uint32_t u = 0;; ++u) {
      const int id = __shfl_sync(0xffffffffu, next, 0);
      // claim the unit after this one now: its round trip overlaps this one's preparation
      if (lane == 0 && id < p.n_units) next = id_base + atomicAdd(p.work + 1, 1);
      UnitDesc d{};
      d.id = -1;
      int phys0 = 0;
      if (id < p.n_units) {
        const int hkv_id = div_hkv(p, id);
        const int4* rp = reinterpret_cast<const int4*>(p.uq + hkv_id);
        const int4 a = __ldg(rp), b = __ldg(rp + 1);
        d.kvh = id - hkv_id * p.Hkv;
        d.id = b.y + d.kvh;  // pbase + kv head
        d.tbl = a.x;
        d.row = a.y;
        d.k0 = a.z;
        d.k1 = a.w;
        d.nsplit = b.x;
        d.crow = b.w;
        const int nblk_tbl = (d.k1 + p.B - 1) >> p.b_shift;
        if (lane * tb < 128) phys0 = __ldg(p.tables + d.tbl + min((d.k0 + lane * tb) >> p.b_shift, nblk_tbl - 1));
      }
      const int ds = u & 3;
      mbar_wait(bar(kB2DFree + ds), ((u >> 2) & 1) ^ 1);
      if (d.id >= 0) {
        const int qb = u % kD2QBufs;  // == ds: the Q^T tile is freed with the descriptor (last QK^T)
        const uint32_t qt = sbase + kD2QOff + qb * 4096;
        const uint8_t* qsrc = static_cast<const uint8_t*>(p.q) +
                              (static_cast<int64_t>(d.row) * p.Hq + d.kvh * g) * (kD * 2);
        for (int pc = lane; pc < g * 16; pc += 32) {
          const int h = pc >> 4, j = pc & 15;
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(qsrc + pc * 16));
          st_shared_v4(qt + (h >> 3) * 2048 + j * 128 + (h & 7) * 16, v.x, v.y, v.z, v.w);
        }
        fence_proxy_async_smem();
        if (lane < 8) asm volatile("st.shared.s32 [%0], %1;" ::"r"(descs + 128 + ds * 32 + lane * 4), "r"(phys0) : "memory");
      }
      __syncwarp();
      if (lane == 0) {
        desc_store(descs, ds, d);
        mbar_arrive(bar(kB2DFull + ds));
      }
      if (d.id < 0) break;
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------- producer
    const uint64_t pol = policy_evict_first();
    const uint32_t bytes_blk = static_cast<uint32_t>(tb) * 512u;  // K rows + V^T sub-blocks
    uint32_t st = 0;
    for (uint32_t u = 0;; ++u) {
      const int ds = u & 3;
      mbar_wait(bar(kB2DFull + ds), (u >> 2) & 1);
      const UnitDesc d = desc_load(descs, ds);
      if (d.id < 0) break;
      const int nsteps = (d.k1 - d.k0 + 127) >> 7;
      const int nblk_tbl = (d.k1 + p.B - 1) >> p.b_shift;
      int phys_next = 0;
      if (lane < 8) asm volatile("ld.shared.s32 %0, [%1];" : "=r"(phys_next) : "r"(descs + 128 + ds * 32 + lane * 4) : "memory");
      auto lookup = [&](int s) {
        const int k = d.k0 + 128 * s + lane * tb;
        return (lane * tb < 128 && s < nsteps) ? __ldg(p.tables + d.tbl + min(k >> p.b_shift, nblk_tbl - 1)) : 0;
      };
      for (int s = 0; s < nsteps; ++s, ++st) {
        const int phys = phys_next;
        phys_next = lookup(s + 1);
        const int k = d.k0 + 128 * s;
        const int valid = min(128, d.k1 - k);
        const int nb = (valid + tb - 1) / tb;
        const int slot = st % kD2Stages;
        const uint32_t stg = sbase + slot * kD2Stage;
        if (lane == 0) {
          mbar_wait(bar(kB2Empty + slot), ((st / kD2Stages) & 1) ^ 1);
          stamp(6, st);
          mbar_expect_tx(bar(kB2Full + slot), nb * bytes_blk);
        }
        __syncwarp();
        if (lane < nb) {
          const int64_t chunk = (static_cast<int64_t>(phys) * p.Hkv + d.kvh) * p.chunk_stride;
          bulk_g2s_hint(stg + lane * tb * 256, p.pool_k + chunk, tb * 256, bar(kB2Full + slot), pol);
          bulk_g2s_hint(stg + 32768 + lane * tb * 256, p.pool_v + chunk, tb * 256, bar(kB2Full + slot), pol);
        }
        if (lane == 0) stamp(0, st);
      }
      if (lane == 0) mbar_arrive(bar(kB2DFree + ds));
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      struct Pend {
        int slot, b, u, first, last;
      } pd{0, 0, 0, 0, 0};
      bool pending = false;
      uint32_t st = 0;
      auto issue_pv = [&](const Pend& q, uint32_t qst) {
        mbar_wait(bar(kB2PFull + q.b), (qst >> 1) & 1);
        if (q.first) mbar_wait(bar(kB2OFree + (q.u & 1)), ((q.u >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t va = sbase + q.slot * kD2Stage + 32768, pa = sbase + kD2POff + q.b * 4096;
        // descriptors built once; the start-address field (bits 0-13, 16-byte units) advances per k-step
        const uint64_t vd = sw32_desc(va, 16, 256), pdsc = noswz_desc(pa, 128, 2048);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_f16(tmem + 32 + 16 * (q.u & 1), vd + static_cast<uint64_t>(kk * (4096 >> 4)),
                   pdsc + static_cast<uint64_t>(kk * (256 >> 4)), kIdescD2, (q.first && kk == 0) ? 0u : 1u);
        stamp(4, qst);
        umma_commit(bar(kB2Empty + q.slot));
        umma_commit(bar(kB2PFree + q.b));
        if (q.last) umma_commit(bar(kB2OFull + (q.u & 1)));
      };
      for (uint32_t u = 0;; ++u) {
        mbar_wait(bar(kB2DFull + (u & 3)), (u >> 2) & 1);
        const UnitDesc d = desc_load(descs, u & 3);
        if (d.id < 0) break;
        const int qb = u % kD2QBufs;
        const int nsteps = (d.k1 - d.k0 + 127) >> 7;
        const uint32_t qa = sbase + kD2QOff + qb * 4096;
        for (int s = 0; s < nsteps; ++s, ++st) {
          const int slot = st % kD2Stages, b = st & 1;
          mbar_wait(bar(kB2Full + slot), (st / kD2Stages) & 1);
          stamp(5, st);
          mbar_wait(bar(kB2SFree + b), ((st >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t ka = sbase + slot * kD2Stage;
          const uint64_t kd = noswz_desc(ka, 128, 2048), qd = noswz_desc(qa, 128, 2048);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_f16(tmem + 16 * b, kd + static_cast<uint64_t>(kk * (256 >> 4)), qd + static_cast<uint64_t>(kk * (256 >> 4)),
                     kIdescD2, kk > 0 ? 1u : 0u);
          umma_commit(bar(kB2SFull + b));
          stamp(1, st);
          if (s == nsteps - 1) umma_commit(bar(kB2DFree + (u & 3)));  // Q^T tile read: the slot may be refilled
          if (pending) issue_pv(pd, st - 1);
          pd = Pend{slot, static_cast<int>(b), static_cast<int>(u), s == 0, s == nsteps - 1};
          pending = true;
        }
      }
      if (pending) issue_pv(pd, st - 1);
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------- softmax
    const int r = tid - 128;  // token of the step (TMEM lane)
    const int w4 = warp - 4;
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(w4 * 32) << 16);
    const float sl2 = p.scale_log2;
    uint32_t st = 0;
    for (uint32_t u = 0;; ++u) {
      mbar_wait(bar(kB2DFull + (u & 3)), (u >> 2) & 1);
      const UnitDesc d = desc_load(descs, u & 3);
      if (d.id < 0) break;
      const int nsteps = (d.k1 - d.k0 + 127) >> 7;
      float m[8], lt[8];
#pragma unroll
      for (int h = 0; h < 8; ++h) m[h] = -INFINITY, lt[h] = 0.f;
      for (int s = 0; s < nsteps; ++s, ++st) {
        const int b = st & 1;
        mbar_wait(bar(kB2SFull + b), (st >> 1) & 1);
        tc_fence_after();
        if (r == 0) stamp(2, st);
        uint32_t sr[16];
        tmem_ld16(lane_addr + 16 * b, sr);
        tc_fence_before();
        mbar_arrive(bar(kB2SFree + b));
        if (r == 0) stamp(7, st);
        const bool valid = d.k0 + 128 * s + r < d.k1;
        float x[8], mx[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          x[h] = (valid && h < g) ? __uint_as_float(sr[h]) * sl2 : -INFINITY;
          mx[h] = x[h];
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
          for (int h = 0; h < 8; ++h)
            if (h < g) mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], off));
        const uint32_t red = scratch + kD2Red + b * 256;
        if (lane < g) {  // mx[lane] without a dynamic register index
          float v = mx[0];
#pragma unroll
          for (int h = 1; h < 8; ++h)
            if (lane == h) v = mx[h];
          st_shared_f32(red + w4 * 64 + lane * 4, v);
        }
        named_bar_sync(1, 128);
        if (r == 0) stamp(8, st);
        bool rescale = false;
        float alpha[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          alpha[h] = 1.f;
          if (h < g) {
            float v = ld_shared_f32(red + h * 4);
#pragma unroll
            for (int w = 1; w < 4; ++w) v = fmaxf(v, ld_shared_f32(red + w * 64 + h * 4));
            if (s == 0) {
              m[h] = v;
            } else if (v > m[h] + 8.0f) {  // lazy rescale (P <= 2^8 otherwise)
              alpha[h] = ex2(m[h] - v);
              m[h] = v;
              rescale = true;
            }
          }
        }
        if (rescale) {  // uniform across the 128 threads: O^T *= alpha per head column, after PV(st-1)
          mbar_wait(bar(kB2PFree + ((st - 1) & 1)), ((st - 1) >> 1) & 1);
          tc_fence_after();
          uint32_t ov[16];
          tmem_ld16(lane_addr + 32 + 16 * (u & 1), ov);
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            ov[h] = __float_as_uint(__uint_as_float(ov[h]) * alpha[h]);
            lt[h] *= alpha[h];
          }
          tmem_st16(lane_addr + 32 + 16 * (u & 1), ov);
          tmem_wait_st();
          tc_fence_before();
        }
        mbar_wait(bar(kB2PFree + b), ((st >> 1) & 1) ^ 1);  // PV(st-2) has read P^T[b]
        const uint32_t pt = sbase + kD2POff + b * 4096;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          if (h < g) {
            const float pv = ex2(x[h] - m[h]);
            lt[h] += pv;
            st_shared_u16(pt + d2_pt_off(h, r), __bfloat16_as_ushort(__float2bfloat16_rn(pv)));
          }
        }
        if (r == 0) stamp(9, st);
        fence_proxy_async_smem();
        mbar_arrive(bar(kB2PFull + b));
        if (r == 0) stamp(3, st);
      }
      // per-head l over the 128 threads, then (m, l) to the epilogue
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int h = 0; h < 8; ++h)
          if (h < g) lt[h] += __shfl_xor_sync(0xffffffffu, lt[h], off);
      const uint32_t lred = scratch + kD2LRed + (u & 1) * 256;
      if (lane < g) {
        float v = lt[0];
#pragma unroll
        for (int h = 1; h < 8; ++h)
          if (lane == h) v = lt[h];
        st_shared_f32(lred + w4 * 64 + lane * 4, v);
      }
      named_bar_sync(1, 128);
      mbar_wait(bar(kB2MLFree + (u & 1)), ((u >> 1) & 1) ^ 1);
      if (r < g) {
        float l = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) l += ld_shared_f32(lred + w * 64 + r * 4);
        float mm = m[0];
#pragma unroll
        for (int h = 1; h < 8; ++h)
          if (r == h) mm = m[h];
        st_shared_v2f(scratch + kD2ML + (u & 1) * 128 + r * 8, mm, l);
      }
      mbar_arrive(bar(kB2MLFull + (u & 1)));
      if (r == 0) mbar_arrive(bar(kB2DFree + (u & 3)));
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ epilogue
    const int r = tid - 256;  // head dim (TMEM lane)
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>((warp - 8) * 32) << 16);
    for (uint32_t u = 0;; ++u) {
      mbar_wait(bar(kB2DFull + (u & 3)), (u >> 2) & 1);
      const UnitDesc d = desc_load(descs, u & 3);
      if (d.id < 0) break;
      mbar_wait(bar(kB2OFull + (u & 1)), (u >> 1) & 1);
      mbar_wait(bar(kB2MLFull + (u & 1)), (u >> 1) & 1);
      tc_fence_after();
      uint32_t ov[16];
      tmem_ld16(lane_addr + 32 + 16 * (u & 1), ov);
      tc_fence_before();
      mbar_arrive(bar(kB2OFree + (u & 1)));
      float mh[8], lh[8];
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        if (h < g) {
          const float2 ml = ld_shared_v2f(scratch + kD2ML + (u & 1) * 128 + h * 8);
          mh[h] = ml.x;
          lh[h] = ml.y;
        } else {
          mh[h] = 0.f;
          lh[h] = 1.f;
        }
      }
      mbar_arrive(bar(kB2MLFree + (u & 1)));
      if (d.nsplit == 1) {
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          if (h < g) {
            __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(p.o) +
                                  (static_cast<int64_t>(d.kvh * g + h) * p.T + d.row) * kD;
            put_out(p, orow + r, __float2bfloat16_rn(__uint_as_float(ov[h]) / lh[h]));
            if (r == 0 && p.lse != nullptr)
              put_out(p, p.lse + static_cast<int64_t>(d.kvh * g + h) * p.T + d.row, (mh[h] + __log2f(lh[h])) * 0.69314718055994530942f);
          }
        }
      } else {
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          if (h < g) {
            __stcg(p.part_o + (static_cast<int64_t>(d.id) * g + h) * kD + r, __uint_as_float(ov[h]) / lh[h]);
            if (r == 0) __stcg(reinterpret_cast<float2*>(p.part_ml + (static_cast<int64_t>(d.id) * g + h) * 2),
                               make_float2(mh[h], lh[h]));
          }
        }
        __threadfence();
        named_bar_sync(2, 128);
        if (r == 0) atomicAdd(p.counters + d.crow * p.Hkv + d.kvh, 1);
      }
      if (r == 0) mbar_arrive(bar(kB2DFree + (u & 3)));
    }
  }
}

__global__ void __launch_bounds__(fa::kThreads, 1) hybrid_attn_bf16_kernel(const AttnParams p) {
  using namespace fa;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bars = sbase + kDataBytes;
  uint8_t* misc = smem + kDataBytes + kBarBytes;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(misc);
  volatile int* item_slot = reinterpret_cast<volatile int*>(misc + 16);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  uint64_t t_entry = 0;
  if (p.trace != nullptr && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_entry));

  // one barrier per thread (a serial loop of ~90 inits by one thread sat in every launch's
  // prologue); the fence by each initialising thread, then the CTA barrier below
  static_assert(kNumBars <= kThreads, "one mbarrier per initialising thread");
  if (tid < kNumBars) {
    {
      const int b = tid;
      uint32_t cnt = 1;
      if (b >= kBarPFull && b < kBarPFull + kSBufs) cnt = 128;
      if (b >= kBarSFree && b < kBarSFree + kSBufs) cnt = 128;
      if ((b >= kB2SFree && b < kB2PFull + 2) || (b >= kB2OFree && b < kB2MLFree + 2)) cnt = 128;
      if (b >= kB2DFree && b < kB2DFree + 4) cnt = 4;  // producer, MMA (after the last QK^T), softmax, epilogue
      // CTA pairs: a K/V stage is free once both CTAs' MMAs have read it (multicast commits)
      if (p.pairs && ((b >= kBarKEmpty && b < kBarKEmpty + kKStages) || (b >= kBarVEmpty && b < kBarVEmpty + kVStages)))
        cnt = 2;
      mbar_init(bars + 8 * b, cnt);
    }
    fence_mbar_init();
  }
  const bool any_items = p.n_tiles > 0 && static_cast<int>(blockIdx.x) < p.prefill_ctas;
  const bool dec_v2 = p.dec_mode == 1 && p.n_units > 0;
  const bool need_tmem = any_items || dec_v2;
  if (need_tmem && warp == 1) {
    tmem_alloc(smem_u32(tmem_slot), kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (p.pairs) cluster_sync_all();  // both CTAs' barriers exist before any multicast copy or commit
  const uint32_t tmem = need_tmem ? *tmem_slot : 0u;
  // Launched with programmatic stream serialization: everything above touched only
  // on-chip state; every global access below comes after the preceding grid (the
  // KV append) has completed and its writes are visible.
  grid_dep_wait();

  if (p.append_total > 0) {
    // niyama_append_attention: this batch's KV append (a3) inside the launch.  CTAs claim
    // kThreads pieces at a time until the queue is empty and count the pieces they
    // finished; only then does any CTA wait for the count to reach the total.  Every
    // piece is therefore claimed by a CTA that is already running, so the wait needs no
    // co-residency of the grid.  The pool writes (generic proxy) are fenced for the
    // bulk-copy (async proxy) reads that follow, on both sides of the release/acquire.
    for (;;) {
      if (tid == 0) *item_slot = atomicAdd(p.work + 4, kThreads);
      __syncthreads();
      const int base = *item_slot;
      __syncthreads();
      if (base >= p.append_total) break;
      const int n = min(kThreads, p.append_total - base);
      if (tid < n) append_piece(p.ap, base + tid);
      fence_proxy_async_global();
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(p.work + 5, n);
      }
    }
    if (tid == 0) {
      uint32_t polls = 0;
      while (ld_acquire_gpu(p.work + 5) < p.append_total) {
        __nanosleep(32);
#ifndef NIYAMA_NO_WATCHDOG
        if (++polls == (1u << 26)) __trap();
#endif
      }
      fence_proxy_async_global();
    }
    __syncthreads();
  }

  uint64_t t_start = 0;
  if (p.trace != nullptr && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  int n_done_items = 0;
  uint32_t kv_it = 0, it = 0;
  while (any_items) {
#if NIYAMA_DIAG_TILES  // CTA 0: clock64 at the claim, after the Q load and at the tile end; count at [3][0]
    int64_t* tev = (p.trace != nullptr && blockIdx.x == 0 && tid == 0 && n_done_items < 64) ? p.trace + 8 * 160 : nullptr;
    if (tev) {
      int64_t c;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
      tev[n_done_items] = c;
      tev[3 * 64] = n_done_items;
    }
#endif
    if (p.pairs) {
      // the cluster's rank-0 CTA claims a q-tile pair; its partner reads the claim through DSMEM
      const uint32_t rank = cluster_ctarank();
      if (rank == 0 && tid == 0) *item_slot = atomicAdd(p.work + 0, 1);
      cluster_sync_all();
      const int item = rank == 0 ? *item_slot : ld_shared_cluster_s32(mapa_shared(smem_u32(const_cast<int*>(item_slot)), 0));
      __syncthreads();
      if (item >= p.n_pair_items) break;
      prefill_tile(p, tile_desc_pair(p, item, static_cast<int>(rank)), sbase, bars, tmem,
                   reinterpret_cast<float*>(misc + kMiscBytes), smem, kv_it, it);
      ++n_done_items;
      continue;
    }
    if (tid == 0) *item_slot = atomicAdd(p.work + 0, 1);
    __syncthreads();
    const int item = *item_slot;
    __syncthreads();
    if (item >= p.n_tiles) break;
    prefill_tile(p, tile_desc(p, item), sbase, bars, tmem, reinterpret_cast<float*>(misc + kMiscBytes), smem, kv_it, it);
#if NIYAMA_DIAG_TILES
    if (tev) {
      int64_t c;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
      tev[2 * 64 + n_done_items] = c;
      tev[4 * 64 + n_done_items] = item;
    }
#endif
    ++n_done_items;
  }
  uint64_t t_prefill = 0;
  if (p.trace != nullptr && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_prefill));
  // Switch roles: the decode rings overwrite prefill buffers through the async proxy.  All
  // bulk copies of the prefill were consumed before the last item barrier.
  fence_proxy_async_smem();
  __syncthreads();
  if (p.pairs) cluster_sync_all();  // no partner copy or commit targets this CTA from here on
  if (dec_v2) {
    // tensor-core decode pipeline; its shared memory starts zeroed (padding rows of the
    // Q^T / P^T tiles, and V^T columns of partial steps must be finite: they meet P = 0)
    for (int i = tid * 16; i < kD2Bytes; i += kThreads * 16) st_shared_v4(sbase + i, 0u, 0u, 0u, 0u);
    fence_proxy_async_smem();
    __syncthreads();
    decode_cta_v2(p, sbase, bars, tmem, smem_u32(misc + kMiscBytes));
    tc_fence_before();
    __syncthreads();
    if (p.n_merge_rows > 0) merge_tail(p);
  } else if (p.n_units > 0 && p.dec_mode == 2) {
    // producer/consumer decode: warps 0-7 compute (3-stage rings), warps 8-11 load for two each
    const uint32_t descs0 = smem_u32(misc + kMiscBytes), n_desc0 = smem_u32(misc + 64);
    if (warp < 8) {
      if ((tid & 31) == 0) count_store(n_desc0 + 16 * warp, 0);
      __syncthreads();
      decode_warp_loop<8, 3, true>(p, sbase, bars, descs0 + warp * 4 * 32, n_desc0 + 16 * warp);
    } else {
      __syncthreads();  // the consumers' descriptor counts are zeroed
      if ((tid & 31) == 0) decode_producer<8, 3>(p, sbase, bars, descs0, n_desc0, 2 * (warp - 8));
      __syncwarp();
    }
    if (p.n_merge_rows > 0) merge_tail(p);
  } else if (p.n_units > 0 && warp < p.dec_warps) {  // the other warps only serve the prefill softmax
    UnitDesc* descs = reinterpret_cast<UnitDesc*>(misc + kMiscBytes) + 4 * warp;
    const uint32_t n_desc = smem_u32(misc + 64 + 16 * warp);
    if (p.dec_warps == 12)
      decode_warp_loop<12, 2>(p, sbase, bars, smem_u32(descs), n_desc);
    else
      decode_warp_loop<8, 3>(p, sbase, bars, smem_u32(descs), n_desc);
    if (p.n_merge_rows > 0) merge_tail(p);
  }
  uint64_t t_decode = 0;
  if (p.trace != nullptr && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_decode));
  tc_fence_before();
  __syncthreads();
  if (p.trace != nullptr && tid == 0) {
    uint64_t t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    int64_t* tr = p.trace + 8 * blockIdx.x;
    tr[0] = static_cast<int64_t>(t_start);
    tr[1] = static_cast<int64_t>(t_prefill);
    tr[2] = static_cast<int64_t>(t_end);
    tr[3] = n_done_items;
    tr[4] = static_cast<int64_t>(t_decode);
    tr[6] = static_cast<int64_t>(t_entry);
  }
  if (need_tmem && warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
  if (tid == 0) {  // (the __syncthreads above ordered every thread's output stores before this fence)
    __threadfence();
    const int done = atomicAdd(p.work + 2, 1);
    if (done == static_cast<int>(gridDim.x) - 1) {  // last CTA: reset the queues for the next launch
      p.work[0] = 0;
      p.work[1] = 0;
      p.work[2] = 0;
      p.work[3] = 0;
      p.work[4] = 0;
      p.work[5] = 0;
      __threadfence();
      if (p.gx.n > 0) gather_barrier(p);
    }
  }
}

int attention_bf16_smem_bytes() { return fa::kSmemBytes; }

// The dynamic shared-memory opt-in is a per-device attribute: niyama_kv_create sets it
// on the pool's device (current at that point), so every device that owns a bf16 pool has it.
cudaError_t configure_attention_bf16() {
  return cudaFuncSetAttribute(hybrid_attn_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fa::kSmemBytes);
}

cudaError_t launch_attention_bf16(const AttnParams& p, int grid, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(fa::kThreads);
  cfg.dynamicSmemBytes = fa::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (p.pairs) {  // prefill CTA pairs: clusters of 2 consecutive CTAs
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.numAttrs = 2;
  }
  return cudaLaunchKernelEx(&cfg, hybrid_attn_bf16_kernel, p);
}

// ==================================================== generic f32 (config 1)
// One warp per (batch row, kv head); the g query heads of the group share each
// K/V load.  Element e of a token row lives at panel (e*4)/128, chunk
// ((e*4)%128)/16 swizzled by slot%8 (same pool layout as the bf16 path).
template <int kMaxDPerLane, int kMaxG>
__global__ void __launch_bounds__(128) hybrid_attn_generic_f32_kernel(const AttnParams p) {
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wg >= p.T * p.Hkv) return;
  const int r = wg / p.Hkv, kvh = wg - r * p.Hkv;
  const RowInfo ri = p.rows[r];
  const int d = p.d, g = p.g;
  const int dpl = d / 32;
  const float* q = static_cast<const float*>(p.q);
  float qv[kMaxG][kMaxDPerLane], acc[kMaxG][kMaxDPerLane], m[kMaxG], l[kMaxG];
#pragma unroll
  for (int hh = 0; hh < kMaxG; ++hh) {
    m[hh] = -INFINITY;
    l[hh] = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxDPerLane; ++k) {
      acc[hh][k] = 0.f;
      qv[hh][k] = (hh < g && k < dpl) ? q[(static_cast<int64_t>(r) * p.Hq + kvh * g + hh) * d + lane + 32 * k] : 0.f;
    }
  }
  for (int t = 0; t < ri.n; ++t) {
    const int64_t blk = p.tables[ri.tbl + t / p.B];
    const int slot = t % p.B;
    const int64_t base = (blk * p.Hkv + kvh) * p.chunk_stride + slot * 128;
    float kv[kMaxDPerLane], vv[kMaxDPerLane];
#pragma unroll
    for (int k = 0; k < kMaxDPerLane; ++k) {
      if (k < dpl) {
        const int byte = (lane + 32 * k) * 4;
        const int panel = byte >> 7, within = byte & 127;
        const int64_t off = base + static_cast<int64_t>(panel) * p.B * 128 + ((((within >> 4) ^ (slot & 7))) << 4) +
                            (within & 15);
        kv[k] = *reinterpret_cast<const float*>(p.pool_k + off);
        vv[k] = *reinterpret_cast<const float*>(p.pool_v + off);
      } else {
        kv[k] = vv[k] = 0.f;
      }
    }
#pragma unroll
    for (int hh = 0; hh < kMaxG; ++hh) {
      if (hh >= g) break;
      float dot = 0.f;
#pragma unroll
      for (int k = 0; k < kMaxDPerLane; ++k) dot = fmaf(qv[hh][k], kv[k], dot);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
      const float x = dot * p.scale_log2;
      const float mn = fmaxf(m[hh], x);
      const float a = exp2f(m[hh] - mn), w = exp2f(x - mn);
      l[hh] = l[hh] * a + w;
#pragma unroll
      for (int k = 0; k < kMaxDPerLane; ++k) acc[hh][k] = acc[hh][k] * a + w * vv[k];
      m[hh] = mn;
    }
  }
  float* o = static_cast<float*>(p.o);
#pragma unroll
  for (int hh = 0; hh < kMaxG; ++hh) {
    if (hh >= g) break;
    const int h = kvh * g + hh;
#pragma unroll
    for (int k = 0; k < kMaxDPerLane; ++k)
      if (k < dpl) o[(static_cast<int64_t>(h) * p.T + r) * d + lane + 32 * k] = acc[hh][k] / l[hh];
    if (lane == 0 && p.lse != nullptr)
      p.lse[static_cast<int64_t>(h) * p.T + r] = (m[hh] + log2f(l[hh])) * 0.69314718055994530942f;
  }
}

cudaError_t launch_attention_generic_f32(const AttnParams& p, cudaStream_t s) {
  const int warps = p.T * p.Hkv;
  if (warps == 0) return cudaSuccess;
  const int blocks = (warps + 3) / 4;
  if (p.d > 128 || p.g > 8) return cudaErrorInvalidValue;
  hybrid_attn_generic_f32_kernel<4, 8><<<blocks, 128, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace niyama
