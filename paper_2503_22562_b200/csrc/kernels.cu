// sm_100a kernels of the Niyama hybrid-batch paged-attention path.
//
//   kv_append_kernel        a3  scatter new K/V rows into the swizzled paged pool
//   kv_gather_kernel            read-back of a sequence (tests)
//   hybrid_attn_bf16_kernel a4-a6  ONE persistent launch:
//        prefill tiles  — TMA-engine bulk copies of paged K/V into SW128 smem,
//                         S = Q K^T and O += P V on tcgen05 (accumulators in TMEM),
//                         one softmax thread per TMEM lane (online softmax, lazy
//                         rescale of O in TMEM);
//        decode units   — warp-level split-KV streaming (bulk copies into a per-warp
//                         3-stage ring, mma.sync m16n8k16 with the GQA group on M),
//                         partials merged by log-sum-exp by the last split of a row.
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
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace niyama {

using namespace ptx;

// ============================================================= append (a3)
// One thread per 16-byte piece of a (row, kv head) vector, 32-bit index math (the
// launcher guarantees T*Hkv*pieces < 2^31).  Source rows are dense [T][Hkv][row_bytes];
// piece j of the row at (block, slot) lands in panel j/8 at chunk position
// (j%8) ^ (slot%8).  K and V move together; all loads are issued before the stores.
__global__ void __launch_bounds__(256) kv_append_kernel(const AppendParams p) {
  const int pieces = p.row_bytes >> 4;  // 16 at d = 128 bf16
  const int total = p.T * p.Hkv * pieces;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int j = idx % pieces;
    const int rh = idx / pieces;
    const int h = rh % p.Hkv;
    const int r = rh / p.Hkv;
    const uint4 kv = __ldg(reinterpret_cast<const uint4*>(p.k_new) + idx);
    const uint4 vv = __ldg(reinterpret_cast<const uint4*>(p.v_new) + idx);
    const int32_t sm = __ldg(p.slot_map + r);
    const int blk = sm / p.B;
    const int slot = sm - blk * p.B;
    const int64_t dst_off = (static_cast<int64_t>(blk) * p.Hkv + h) * p.chunk_bytes + (j >> 3) * p.B * 128 +
                            slot * 128 + (((j & 7) ^ (slot & 7)) << 4);
    *reinterpret_cast<uint4*>(p.pool_k + dst_off) = kv;
    *reinterpret_cast<uint4*>(p.pool_v + dst_off) = vv;
  }
}

cudaError_t launch_append(const AppendParams& p, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(p.T) * p.Hkv * (p.row_bytes >> 4);
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
                                 int32_t B, int64_t chunk_bytes, uint8_t* __restrict__ k_out,
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
    const int64_t src = (blk * Hkv + h) * chunk_bytes + static_cast<int64_t>(j >> 3) * B * 128 + slot * 128 +
                        (((j & 7) ^ (slot & 7)) << 4);
    const int64_t dst = th * row_bytes + (static_cast<int64_t>(j) << 4);
    *reinterpret_cast<uint4*>(k_out + dst) = *reinterpret_cast<const uint4*>(pool_k + src);
    *reinterpret_cast<uint4*>(v_out + dst) = *reinterpret_cast<const uint4*>(pool_v + src);
  }
}

cudaError_t launch_gather(const uint8_t* pool_k, const uint8_t* pool_v, const int32_t* table, int32_t len,
                          int32_t Hkv, int32_t row_bytes, int32_t B, int64_t chunk_bytes, uint8_t* k_out,
                          uint8_t* v_out, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(len) * Hkv * (row_bytes >> 4);
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  kv_gather_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(pool_k, pool_v, table, len, Hkv, row_bytes, B,
                                                           chunk_bytes, k_out, v_out);
  return cudaGetLastError();
}

// ===================================================== fused bf16 attention
// CTA = 384 threads (3 warpgroups), 1 CTA/SM, 512 TMEM columns.  Warpgroups 0-1 (softmax,
// decode, merge) run with 224 registers, warpgroup 2 (bulk-copy producers, MMA issuer) with 56.
// Shared memory map (bytes from the 1024-aligned base):
//   [0, 64K)            Q_A, Q_B tiles (2 panels x 128 rows x 128 B each, SW128)
//   [64K, +3*32K)       K stages (128 keys x 256 B each)
//   [.., +2*32K)        V stages
// TMEM: S_A/P_A cols [0,128), S_B/P_B [128,256), O_A [256,384), O_B [384,512).
// The decode role reuses [0, 192K) as 8 warps x 3 stages x 8 KB.
namespace fa {
constexpr int kD = 128;            // head dim (bf16 path)
constexpr int kBN = 128;           // keys per prefill key tile
constexpr int kNSK = 3;            // K stages (released after both QK^T of a key tile)
constexpr int kNSV = 2;            // V stages (released after both PV of a key tile)
constexpr int kPanel = 128 * 128;  // one 64-column panel of a 128-row tile
constexpr int kTile = 2 * kPanel;  // 128 rows x 256 B
constexpr int kQOff = 0;           // Q_X at kQOff + X * kTile
constexpr int kKOff = 2 * kTile;
constexpr int kVOff = kKOff + kNSK * kTile;
constexpr int kDataBytes = kVOff + kNSV * kTile;  // 224 KB
constexpr int kThreads = 384;
constexpr int kWarpLoad = 8, kWarpMMA = 9;  // warp 8: lane 0 streams K, lane 1 streams V; warp 9 lane 0: MMA
constexpr int kRegsMath = 216, kRegsCtl = 72;  // setmaxnreg budgets: warpgroups 0-1 / warpgroup 2
static_assert(2 * kRegsMath + kRegsCtl <= 65536 / kThreads / 8 * 8 * 3, "setmaxnreg budgets exceed the launch allocation");
constexpr int kDecWarps = 8;
constexpr int kDecStages = 3;
constexpr int kDecStage = 8192;  // 16 tokens of K (4 KB) + V (4 KB)
static_assert(kDecWarps * kDecStages * kDecStage <= kDataBytes, "decode ring must fit");
// barrier indices
constexpr int kBarKFull = 0;
constexpr int kBarKEmpty = kBarKFull + kNSK;
constexpr int kBarVFull = kBarKEmpty + kNSK;
constexpr int kBarVEmpty = kBarVFull + kNSV;
constexpr int kBarSFull = kBarVEmpty + kNSV;  // [2] per Q tile: QK^T committed
constexpr int kBarPFull = kBarSFull + 2;      // [2] per Q tile: P written to TMEM (128 arrivals)
constexpr int kBarODone = kBarPFull + 2;      // [2] per Q tile: PV committed
constexpr int kBarDec = kBarODone + 2;        // kDecWarps x kDecStages
constexpr int kNumBars = kBarDec + kDecWarps * kDecStages;
constexpr int kMiscBytes = 64 + kDecWarps * 16;      // tmem slot, item slot, per-warp desc counters
constexpr int kDescBytes = kDecWarps * 4 * 40;       // per-warp 4-entry UnitDesc rings
constexpr int kSmemBytes = 1024 /*align slack*/ + kDataBytes + kNumBars * 8 + kMiscBytes + kDescBytes;
static_assert(kSmemBytes <= 232448, "exceeds 227 KB of dynamic shared memory");
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemS = 0;    // S_X / P_X at kTmemS + 128 X
constexpr uint32_t kTmemO = 256;  // O_X at kTmemO + 128 X
constexpr uint32_t kIdescQK = idesc_bf16_f32(128, kBN, 0, 0);
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, kD, 0, 1);
}  // namespace fa

// -------------------------------------------------------------- prefill pair
// Debug event log (niyama_debug_trace): CTA 0's first item, key tiles < 64, clock64 per role.
__device__ __forceinline__ void ev_stamp(int64_t* ev, int role, int j) {
  if (ev != nullptr && j < 64) {
    int64_t c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    ev[role * 64 + j] = c;
  }
}

// A prefill work item = a PAIR of 128-row Q tiles (X = 0: q-tile 2qp, X = 1: q-tile
// 2qp+1) of one kv head; both stream the same K/V tiles.  Tile X's rows r = hh*R + i
// hold chunk row t0[X] + i of query head kvh*g + hh (GQA packing, R = 128/g).
struct PairDesc {
  int tbl, o, c, row0, kvh, nblk;
  int t0[2], vrows[2], nk[2];
};

__device__ __forceinline__ PairDesc pair_desc(const AttnParams& p, int item) {
  int i = 0;
  while (i + 1 < p.n_slices && __ldg(&p.slices[i + 1].tbase) <= item) ++i;
  const PrefillSlice sl = p.slices[i];
  const int local = item - sl.tbase;
  const int npair = (sl.nqt + 1) >> 1;
  const int qp = npair - 1 - local / p.Hkv;  // largest key ranges first
  PairDesc d;
  d.tbl = sl.tbl;
  d.o = sl.o;
  d.c = sl.c;
  d.row0 = sl.row0;
  d.kvh = local % p.Hkv;
  int nkeys_max = 0;
#pragma unroll
  for (int X = 0; X < 2; ++X) {
    d.t0[X] = (2 * qp + X) * p.R;
    d.vrows[X] = max(0, min(p.R, sl.c - d.t0[X]));
    const int nkeys = d.vrows[X] > 0 ? sl.o + d.t0[X] + d.vrows[X] : 0;
    d.nk[X] = (nkeys + fa::kBN - 1) / fa::kBN;
    nkeys_max = max(nkeys_max, nkeys);
  }
  d.nblk = (nkeys_max + p.B - 1) / p.B;
  return d;
}

__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Roles: warp 8 lane 0 streams K tiles and lane 1 V tiles (bulk copies of pre-swizzled
// paged blocks), warp 9 lane 0 issues tcgen05 MMAs, warps 0-3 run the
// softmax of tile A and warps 4-7 that of tile B (thread = TMEM lane = tile row).
// MMA order per key tile j:  PV_A(j), QK_A(j+1), PV_B(j), QK_B(j+1) — the tensor pipe
// executes in issue order, so "S_X(j+1) ready" implies "PV_X(j) done": the softmax of
// tile X may rescale O_X right after S_X(j+1) lands, and P_X(j) (bf16, written into
// the first 64 columns of S_X) is consumed by PV_X(j) from TMEM before QK_X(j+1)
// overwrites S_X.
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// kMath = true: warpgroups 0-1 (Q load, softmax of tiles A/B); false: warpgroup 2
// (bulk-copy producers, MMA issuer).  Both instantiations run the same named-barrier
// sequence, so the two register budgets never share a code path.
template <bool kMath>
__device__ __forceinline__ void prefill_pair(const AttnParams& p, const PairDesc& t, uint32_t sbase, uint32_t bars,
                                             uint32_t tmem, uint32_t& kv_it, uint32_t (&it)[2]) {
  using namespace fa;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int g = p.g, R = p.R;
  const int nk = max(t.nk[0], t.nk[1]);
  int64_t* ev = (p.trace != nullptr && blockIdx.x == 0 && kv_it == 0) ? p.trace + 8 * 160 : nullptr;  // [10 roles][64]

  // ---- Q tiles: tile X row r = hh*R + i  <-  q[row0 + t0[X] + i][kvh*g + hh][:]
  if constexpr (kMath) {
    const uint8_t* q = static_cast<const uint8_t*>(p.q);
    for (int idx = tid; idx < 2 * 128 * 16; idx += 256) {
      const int X = idx >> 11, r = (idx >> 4) & 127, j = idx & 15;
      const int hh = r / R, i = r - hh * R;
      const int vrowsX = X ? t.vrows[1] : t.vrows[0], t0X = X ? t.t0[1] : t.t0[0];
      uint4 v = make_uint4(0, 0, 0, 0);
      if (i < vrowsX) {
        const int64_t row = t.row0 + t0X + i;
        v = __ldg(reinterpret_cast<const uint4*>(q + ((row * p.Hq + t.kvh * g + hh) * kD) * 2 + j * 16));
      }
      st_shared_v4(sbase + kQOff + X * kTile + (j >> 3) * kPanel + r * 128 + (((j & 7) ^ (r & 7)) << 4), v.x, v.y,
                   v.z, v.w);
    }
    fence_proxy_async_smem();
  }
  named_bar_sync(1, kThreads);  // Q tiles in smem

  if (!kMath && warp == kWarpLoad) {
    if (lane < 2) {
      // ---------------- producers (two lanes, independent thread scheduling): 128-key K / V tiles
      const bool isK = lane == 0;
      const int ns = isK ? kNSK : kNSV;
      const uint8_t* pool = isK ? p.pool_k : p.pool_v;
      const uint32_t ring = sbase + (isK ? kKOff : kVOff);
      const int bar_full = isK ? kBarKFull : kBarVFull, bar_empty = isK ? kBarKEmpty : kBarVEmpty;
      const int bpt = kBN / p.B;  // blocks per key tile
      const uint32_t seg = static_cast<uint32_t>(p.B) * 128;
      for (int j = 0; j < nk; ++j) {
        const uint32_t k_it = kv_it + j;
        const int st = k_it % ns;
        const uint32_t ph = (k_it / ns) & 1;
        mbar_wait(bars + 8 * (bar_empty + st), ph ^ 1);
        ev_stamp(ev, isK ? 0 : 1, j);
        const uint32_t full = bars + 8 * (bar_full + st);
        mbar_expect_tx(full, kTile);
        for (int b = 0; b < bpt; ++b) {
          int lb = j * bpt + b;
          if (lb >= t.nblk) lb = t.nblk - 1;  // finite data; masked out (P = 0)
          const int64_t phys = __ldg(p.tables + t.tbl + lb);
          const int64_t off = (phys * p.Hkv + t.kvh) * p.chunk_bytes;
          for (int pn = 0; pn < 2; ++pn)
            bulk_g2s(ring + st * kTile + pn * kPanel + b * seg, pool + off + pn * seg, seg, full);
        }
      }
    }
  } else if (!kMath && warp == kWarpMMA) {
    if (lane == 0) {
      // ---------------- tcgen05 issuer
      auto qk = [&](int X, int j) {
        const uint32_t k_it = kv_it + j;
        const int st = k_it % kNSK;
        mbar_wait(bars + 8 * (kBarKFull + st), (k_it / kNSK) & 1);
        tc_fence_after();
        if (X == 0) ev_stamp(ev, 2, j);
        const uint32_t qa = sbase + kQOff + X * kTile, ka = sbase + kKOff + st * kTile;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t koff = (kk >> 2) * kPanel + (kk & 3) * 32;
          umma_f16(tmem + kTmemS + 128 * X, sw128_desc(qa + koff, 16, 1024), sw128_desc(ka + koff, 16, 1024),
                   kIdescQK, kk > 0);
        }
        umma_commit(bars + 8 * (kBarSFull + X));
      };
      auto pv = [&](int X, int j) {
        const uint32_t k_it = kv_it + j;
        const int st = k_it % kNSV;
        mbar_wait(bars + 8 * (kBarPFull + X), (it[X] + j) & 1);
        mbar_wait(bars + 8 * (kBarVFull + st), (k_it / kNSV) & 1);
        tc_fence_after();
        if (X == 0) ev_stamp(ev, 3, j);
        const uint32_t va = sbase + kVOff + st * kTile;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          umma_ts(tmem + kTmemO + 128 * X, tmem + kTmemS + 128 * X + kk * 8, sw128_desc(va + kk * 2048, kPanel, 1024),
                  kIdescPV, (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(bars + 8 * (kBarODone + X));
      };
      if (t.nk[0] > 0) qk(0, 0);
      if (t.nk[1] > 0) qk(1, 0);
      umma_commit(bars + 8 * (kBarKEmpty + kv_it % kNSK));
      for (int j = 0; j < nk; ++j) {
        if (j < t.nk[0]) pv(0, j);
        if (j + 1 < t.nk[0]) qk(0, j + 1);
        if (j < t.nk[1]) pv(1, j);
        umma_commit(bars + 8 * (kBarVEmpty + (kv_it + j) % kNSV));
        if (j + 1 < t.nk[1]) qk(1, j + 1);
        if (j + 1 < nk) umma_commit(bars + 8 * (kBarKEmpty + (kv_it + j + 1) % kNSK));
      }
    }
  } else if (kMath) {
    // ---------------- softmax of tile X: this thread owns tile row r (TMEM lane r)
    const int X = warp >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int hh = r / R, i = r - hh * R;
    const int vrowsX = X ? t.vrows[1] : t.vrows[0], t0X = X ? t.t0[1] : t.t0[0];
    const int nkX = X ? t.nk[1] : t.nk[0];
    const uint32_t itX = X ? it[1] : it[0];
    const bool valid = i < vrowsX;
    const int pos = t.o + t0X + (valid ? i : 0);  // last visible key of this row
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t s_addr = lane_addr + kTmemS + 128 * X, o_addr = lane_addr + kTmemO + 128 * X;
    float m_ref = -INFINITY, l = 0.f;
    const float sl2 = p.scale_log2;
    for (int j = 0; j < nkX; ++j) {
      mbar_wait(bars + 8 * (kBarSFull + X), (itX + j) & 1);
      tc_fence_after();
      if (X == 0 && r == 0) ev_stamp(ev, 4, j);
      const int kbase = j * kBN;
      const bool diag = kbase + kBN - 1 > pos;  // diagonal / tail tile: causal mask on raw scores
      // exp pass: p = 2^(s*scale*log2e - m_ref) (one FFMA + one MUFU.EX2 each), row max of the
      // raw scores tracked on the side (scale > 0 commutes with max).  P stays in registers
      // (bf16x2) until the reference is verified.
      uint32_t pk[64];
      float sum0 = 0.f, sum1 = 0.f;
      auto exp_pass = [&](float ref, float& mxraw) {
        const float nm = -ref;
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = -INFINITY;
        sum0 = sum1 = 0.f;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {  // 32 columns per TMEM load keeps register pressure low
          uint32_t sr[32];
          tmem_ld32(s_addr + q4 * 32, sr);
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int e = q4 * 32 + 2 * c;
            const float s0 = (diag && kbase + e > pos) ? -INFINITY : __uint_as_float(sr[2 * c]);
            const float s1 = (diag && kbase + e + 1 > pos) ? -INFINITY : __uint_as_float(sr[2 * c + 1]);
            m8[(2 * c) & 7] = fmaxf(m8[(2 * c) & 7], s0);
            m8[(2 * c + 1) & 7] = fmaxf(m8[(2 * c + 1) & 7], s1);
            const float e0 = ex2(fmaf(s0, sl2, nm)), e1 = ex2(fmaf(s1, sl2, nm));
            if (c & 1) sum1 += e0 + e1; else sum0 += e0 + e1;
            pk[q4 * 16 + c] = pack_bf16(e0, e1);
          }
        }
        mxraw = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      };
      if (j == 0) {
        // first key tile: the reference is the tile's own row max (max pass, then exps)
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = -INFINITY;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          uint32_t sr[32];
          tmem_ld32(s_addr + q4 * 32, sr);
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float v = (diag && kbase + q4 * 32 + e > pos) ? -INFINITY : __uint_as_float(sr[e]);
            m8[e & 7] = fmaxf(m8[e & 7], v);
          }
        }
        m_ref = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))) *
                sl2;
      }
      float mxraw;
      exp_pass(m_ref, mxraw);
      if (X == 0 && r == 0) ev_stamp(ev, 5, j);
      const float m_new = fmaxf(m_ref, mxraw * sl2);
      const bool need = m_new > m_ref + 8.0f;  // lazy rescale: p <= 2^8 otherwise
      if (__any_sync(0xffffffffu, need)) {
        // rare: rescale O_X (PV_X(j-1) completed before QK_X(j) ran; PV_X(j) waits for our P),
        // then redo the exps against the new reference (S is intact: P is not written yet)
        const float alpha = need ? ex2(m_ref - m_new) : 1.f;
#pragma unroll 1
        for (int c = 0; c < kD / 32; ++c) {
          uint32_t ov[32];
          tmem_ld32(o_addr + c * 32, ov);
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
          tmem_st32(o_addr + c * 32, ov);
        }
        if (need) {
          l *= alpha;
          m_ref = m_new;
        }
        float unused;
        exp_pass(m_ref, unused);
      }
      if (X == 0 && r == 0) ev_stamp(ev, 7, j);
      {
        uint32_t (&p0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&pk[0]);
        uint32_t (&p1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&pk[32]);
        tmem_st32(s_addr, p0);  // P_X(j) as bf16x2 over S_X's first 64 columns
        tmem_st32(s_addr + 32, p1);
      }
      l += sum0 + sum1;
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bars + 8 * (kBarPFull + X));
      if (X == 0 && r == 0) ev_stamp(ev, 6, j);
    }
    if (nkX > 0) {
      // ---------------- epilogue: O / l -> bf16, LSE
      mbar_wait(bars + 8 * (kBarODone + X), (itX + nkX - 1) & 1);
      tc_fence_after();
      const float inv_l = 1.f / l;
      const int h = t.kvh * g + hh;
      const int64_t trow = t.row0 + t0X + i;
      uint8_t* orow = static_cast<uint8_t*>(p.o) + ((static_cast<int64_t>(h) * p.T + trow) * kD) * 2;
#pragma unroll 1
      for (int c = 0; c < kD / 32; ++c) {
        uint32_t ov[32];
        tmem_ld32(o_addr + c * 32, ov);
        if (valid) {
#pragma unroll
          for (int e = 0; e < 32; e += 8) {
            uint4 w;
            w.x = pack_bf16(__uint_as_float(ov[e + 0]) * inv_l, __uint_as_float(ov[e + 1]) * inv_l);
            w.y = pack_bf16(__uint_as_float(ov[e + 2]) * inv_l, __uint_as_float(ov[e + 3]) * inv_l);
            w.z = pack_bf16(__uint_as_float(ov[e + 4]) * inv_l, __uint_as_float(ov[e + 5]) * inv_l);
            w.w = pack_bf16(__uint_as_float(ov[e + 6]) * inv_l, __uint_as_float(ov[e + 7]) * inv_l);
            *reinterpret_cast<uint4*>(orow + (c * 32 + e) * 2) = w;
          }
        }
      }
      if (valid && p.lse != nullptr)
        p.lse[static_cast<int64_t>(h) * p.T + trow] = (m_ref + __log2f(l)) * 0.69314718055994530942f;
    }
  }
  kv_it += nk;
  it[0] += t.nk[0];
  it[1] += t.nk[1];
  tc_fence_before();
  named_bar_sync(2, kThreads);  // item done: Q/K/V smem and TMEM free for the next item
  tc_fence_after();
}

// --------------------------------------------------------------- decode unit
struct UnitDesc {
  int id, tbl, ctx, row, kvh, k0, k1, nsplit, ubase, pad;
};

// Unit = (row, split s, kv head h); d.id = its canonical partial index ubase + s*Hkv + h.
__device__ __forceinline__ UnitDesc make_unit(const AttnParams& p, const DecodeRow& r, int s, int h) {
  UnitDesc d;
  d.id = r.ubase + s * p.Hkv + h;
  d.tbl = r.tbl;
  d.ctx = r.ctx;
  d.row = r.row;
  d.kvh = h;
  d.k0 = s * p.split_len;
  d.k1 = min(r.ctx, d.k0 + p.split_len);
  d.nsplit = r.nsplit;
  d.ubase = r.ubase;
  d.pad = 0;
  return d;
}

// Stage s of a unit = 16 tokens of one kv head: K then V (4 KB each at d = 128 bf16).
// `phys` is the physical block holding the stage (looked up one stage ahead).
__device__ __forceinline__ void decode_issue(const AttnParams& p, const UnitDesc& u, int s, int64_t phys,
                                             uint32_t stage, uint32_t bar) {
  const int tok = u.k0 + 16 * s;
  const int sub = (tok % p.B) >> 4;
  const int64_t off = (phys * p.Hkv + u.kvh) * p.chunk_bytes + sub * 2048;
  const uint32_t seg = static_cast<uint32_t>(p.B) * 128;
  mbar_expect_tx(bar, fa::kDecStage);
  if (seg == 2048) {  // B = 16: the (block, head) chunk is one contiguous 4 KB run per K / V
    bulk_g2s(stage, p.pool_k + off, 4096, bar);
    bulk_g2s(stage + 4096, p.pool_v + off, 4096, bar);
  } else {
    bulk_g2s(stage, p.pool_k + off, 2048, bar);
    bulk_g2s(stage + 2048, p.pool_k + off + seg, 2048, bar);
    bulk_g2s(stage + 4096, p.pool_v + off, 2048, bar);
    bulk_g2s(stage + 6144, p.pool_v + off + seg, 2048, bar);
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
struct DecodeLoader {
  UnitDesc cur;
  int s, nst;
  int64_t phys;  // block of stage s of cur
  int nxt_id, nxt_row, nxt_step;  // 0 nothing, 1 id requested, 2 row index, 3 row record, 4 ready
  DecodeRow nxt_r;
  UnitDesc nxt;
  int64_t nxt_phys0;
  bool done;
  uint32_t issued;

  __device__ __forceinline__ void advance(const AttnParams& p) {
    if (nxt_step == 0) {
      nxt_id = atomicAdd(p.work + 1, 1);
    } else if (nxt_step == 1) {
      if (nxt_id < p.n_units) nxt_row = __ldg(p.urow + nxt_id / p.Hkv);  // row << 12 | split
    } else if (nxt_step == 2) {
      if (nxt_id < p.n_units) nxt_r = p.drows[nxt_row >> 12];
    } else if (nxt_step == 3) {
      if (nxt_id < p.n_units) {
        nxt = make_unit(p, nxt_r, nxt_row & 4095, nxt_id % p.Hkv);
        nxt_phys0 = __ldg(p.tables + nxt.tbl + nxt.k0 / p.B);
      }
    } else {
      return;
    }
    ++nxt_step;
  }
  __device__ __forceinline__ void issue_next(const AttnParams& p, uint32_t ring, uint32_t bar0, UnitDesc* descs,
                                             volatile int* n_desc) {
    using namespace fa;
    if (done) return;
    if (s == nst) {
      while (nxt_step < 4) advance(p);
      const int k = *n_desc;
      if (nxt_id >= p.n_units) {
        done = true;
        descs[k & 3].id = -1;  // end of stream
        *n_desc = k + 1;
        return;
      }
      cur = nxt;
      phys = nxt_phys0;
      s = 0;
      nst = (cur.k1 - cur.k0 + 15) >> 4;
      nxt_step = 0;
      descs[k & 3] = cur;
      *n_desc = k + 1;
    }
    const uint32_t slot = issued % kDecStages;
    decode_issue(p, cur, s, phys, ring + slot * kDecStage, bar0 + 8 * slot);
    ++s;
    ++issued;
    if (s < nst) {
      const int lb_prev = (cur.k0 + 16 * (s - 1)) / p.B, lb = (cur.k0 + 16 * s) / p.B;
      if (lb != lb_prev) phys = __ldg(p.tables + cur.tbl + lb);  // consumed by the next call
    }
    advance(p);
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

// Compute side: every lane of the warp.  Split rows write an fp32 partial
// (m, l, o~) at index `unit id` (fire and forget); unsplit rows write O / LSE.
__device__ __forceinline__ void decode_warp_loop(const AttnParams& p, uint32_t sbase, uint32_t bars,
                                                 UnitDesc* descs, volatile int* n_desc) {
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
  const int ktok = (mi >> 1) * 8 + rr;  // K (non-trans): matrices (tok 0-7,c),(0-7,c+1),(8-15,c),(8-15,c+1)
  const int vtok = (mi & 1) * 8 + rr;   // V (trans):     matrices (tok 0-7,d),(8-15,d),(0-7,d+8),(8-15,d+8)

  DecodeLoader ld;
  ld.s = ld.nst = 0;
  ld.nxt_step = 0;
  ld.nxt_id = ld.nxt_row = 0;
  ld.done = false;
  ld.issued = 0;
  ld.phys = ld.nxt_phys0 = 0;
  if (lane == 0) {
    *n_desc = 0;
    for (int k = 0; k < kDecStages; ++k) ld.issue_next(p, ring, bar0, descs, n_desc);
  }
  __syncwarp();

  uint32_t qn0[8], qn2[8];
  bool qn_valid = false;
  for (int ck = 0;; ++ck) {
    __syncwarp();
    const UnitDesc u = descs[ck & 3];
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
    float o[16][4];
#pragma unroll
    for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int s = 0; s < nst; ++s) {
      const uint32_t slot = dec_iter % kDecStages;
      const uint32_t ph = (dec_iter / kDecStages) & 1;
      const uint32_t stg = ring + slot * kDecStage;
      mbar_wait(bar0 + 8 * slot, ph);
      // S = Q K^T over 16 tokens (2 n-tiles of 8)
      float sc0[4] = {0.f, 0.f, 0.f, 0.f}, sc1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int chunk = (kk & 3) * 2 + (mi & 1);
        const uint32_t addr = stg + (kk >> 2) * 2048 + ktok * 128 + ((chunk ^ (ktok & 7)) << 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(addr, b0, b1, b2, b3);
        mma_bf16_16816(sc0, qa0[kk], 0u, qa2[kk], 0u, b0, b1);
        mma_bf16_16816(sc1, qa0[kk], 0u, qa2[kk], 0u, b2, b3);
      }
      const int tb = u.k0 + 16 * s;
      float x0 = sc0[0] * sl2, x1 = sc0[1] * sl2, x2 = sc1[0] * sl2, x3 = sc1[1] * sl2;
      if (tb + 16 > u.k1) {
        const int t0 = tb + 2 * tig;
        if (t0 >= u.k1) x0 = -INFINITY;
        if (t0 + 1 >= u.k1) x1 = -INFINITY;
        if (t0 + 8 >= u.k1) x2 = -INFINITY;
        if (t0 + 9 >= u.k1) x3 = -INFINITY;
      }
      float mx = fmaxf(fmaxf(x0, x1), fmaxf(x2, x3));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m, mx);
      if (m_new > m) {
        const float alpha = ex2(m - m_new);
        l *= alpha;
#pragma unroll
        for (int n = 0; n < 16; ++n) {
          o[n][0] *= alpha;
          o[n][1] *= alpha;
        }
        m = m_new;
      }
      const float p0 = ex2(x0 - m), p1 = ex2(x1 - m), p2 = ex2(x2 - m), p3 = ex2(x3 - m);
      l += (p0 + p1) + (p2 + p3);
      const uint32_t pa0 = pack_bf16(p0, p1), pa2 = pack_bf16(p2, p3);
      // O += P V  (16 tokens x 128 dims = 16 n-tiles)
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) {
        const int dchunk = 2 * n2 + (mi >> 1);
        const uint32_t addr = stg + 4096 + (dchunk >> 3) * 2048 + vtok * 128 + (((dchunk & 7) ^ (vtok & 7)) << 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(addr, b0, b1, b2, b3);
        mma_bf16_16816(o[2 * n2], pa0, 0u, pa2, 0u, b0, b1);
        mma_bf16_16816(o[2 * n2 + 1], pa0, 0u, pa2, 0u, b2, b3);
      }
      __syncwarp();
      if (lane == 0) ld.issue_next(p, ring, bar0, descs, n_desc);  // refill this slot
      ++dec_iter;
      // prefetch the next unit's Q fragments once its descriptor is published
      if (!qn_valid && s + 2 >= nst) {
        __syncwarp();
        if (*n_desc > ck + 1) {
          const UnitDesc nu = descs[(ck + 1) & 3];
          if (nu.id >= 0) {
            load_q_frags(p, nu, gid, tig, qn0, qn2);
            qn_valid = true;
          }
        }
      }
    }
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    if (gid < g) {
      const float inv = 1.f / l;
      if (u.nsplit == 1) {
        const int h = u.kvh * g + gid;
        __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(p.o) + (static_cast<int64_t>(h) * p.T + u.row) * kD;
#pragma unroll
        for (int n = 0; n < 16; ++n)
          *reinterpret_cast<uint32_t*>(orow + n * 8 + 2 * tig) = pack_bf16(o[n][0] * inv, o[n][1] * inv);
        if (tig == 0 && p.lse != nullptr)
          p.lse[static_cast<int64_t>(h) * p.T + u.row] = (m + __log2f(l)) * 0.69314718055994530942f;
      } else {
        float* po = p.part_o + (static_cast<int64_t>(u.id) * g + gid) * kD;
#pragma unroll
        for (int n = 0; n < 16; ++n)
          __stcg(reinterpret_cast<float2*>(po + n * 8 + 2 * tig), make_float2(o[n][0] * inv, o[n][1] * inv));
        if (tig == 0)
          __stcg(reinterpret_cast<float2*>(p.part_ml + (static_cast<int64_t>(u.id) * g + gid) * 2), make_float2(m, l));
      }
    }
  }
}

// a6 — after the grid barrier: merge the partials of every split (row, kv head, q head)
// item, one warp per item (m = max_s m_s, w_s = e^(m_s - m) l_s,
// o = sum_s w_s o~_s / sum_s w_s, lse = m + ln sum_s w_s).  Lane s reads split s's
// (m, l); the o slices are read 16 splits at a time (16 loads in flight per lane) and
// accumulated in split order, so the result is deterministic.  Rows with nsplit > 1
// form the prefix [0, n_merge_rows) of the sorted DecodeRow records.
__device__ __forceinline__ void merge_phase(const AttnParams& p) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * fa::kDecWarps + (threadIdx.x >> 5);  // warps 0..kDecWarps-1 of each CTA
  const int nw = gridDim.x * fa::kDecWarps;
  const int g = p.g;
  const int items = p.n_merge_rows * p.Hkv * g;
  for (int it = gw; it < items; it += nw) {
    const int hh = it % g;
    const int pair = it / g;
    const int r = pair / p.Hkv, kvh = pair - r * p.Hkv;
    const DecodeRow dr = p.drows[r];
    const int ns = dr.nsplit;
    auto pidx = [&](int sp) -> int64_t {
      return static_cast<int64_t>(dr.ubase + sp * p.Hkv + kvh) * g + hh;
    };
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
    const int h = kvh * g + hh;
    __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(p.o) + (static_cast<int64_t>(h) * p.T + dr.row) * fa::kD;
    uint2 w2;
    w2.x = pack_bf16(acc.x * inv, acc.y * inv);
    w2.y = pack_bf16(acc.z * inv, acc.w * inv);
    *reinterpret_cast<uint2*>(orow + lane * 4) = w2;
    if (lane == 0 && p.lse != nullptr)
      p.lse[static_cast<int64_t>(h) * p.T + dr.row] = (M + __log2f(L)) * 0.69314718055994530942f;
  }
}

__global__ void __launch_bounds__(fa::kThreads, 1) hybrid_attn_bf16_kernel(const AttnParams p) {
  using namespace fa;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bars = sbase + kDataBytes;
  uint8_t* misc = smem + kDataBytes + kNumBars * 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(misc);
  volatile int* item_slot = reinterpret_cast<volatile int*>(misc + 16);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  if (tid == 0) {
    for (int b = kBarKFull; b < kBarVEmpty + kNSV; ++b) mbar_init(bars + 8 * b, 1);
    for (int X = 0; X < 2; ++X) {
      mbar_init(bars + 8 * (kBarSFull + X), 1);
      mbar_init(bars + 8 * (kBarPFull + X), 128);
      mbar_init(bars + 8 * (kBarODone + X), 1);
    }
    for (int b = kBarDec; b < kNumBars; ++b) mbar_init(bars + 8 * b, 1);
    fence_mbar_init();
  }
  const bool any_items = p.n_tiles > 0;
  if (any_items && warp == kWarpMMA) {
    tmem_alloc(smem_u32(tmem_slot), kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = any_items ? *tmem_slot : 0u;
  uint32_t kv_it = 0, it[2] = {0, 0};

  if (warp >= 8) {
    // ===== warpgroup 2: producers + MMA issuer (few registers); never rejoins the math path
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtl));
    while (any_items) {
      named_bar_sync(3, kThreads);  // item id published by thread 0
      const int item = *item_slot;
      named_bar_sync(4, kThreads);  // everyone has read it
      if (item >= p.n_tiles) break;
      prefill_pair<false>(p, pair_desc(p, item), sbase, bars, tmem, kv_it, it);
    }
    if (any_items && warp == kWarpMMA) {  // all TMEM reads ended before the last item barrier
      tc_fence_after();
      tmem_dealloc(tmem, kTmemCols);
    }
    return;
  }

  // ===== warpgroups 0-1: Q load + softmax, then decode and merge (many registers)
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsMath));
  uint64_t t_start = 0;
  if (p.trace != nullptr && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  int n_done_items = 0;
  while (any_items) {
    if (tid == 0) *item_slot = atomicAdd(p.work + 0, 1);
    named_bar_sync(3, kThreads);
    const int item = *item_slot;
    named_bar_sync(4, kThreads);
    if (item >= p.n_tiles) break;
    prefill_pair<true>(p, pair_desc(p, item), sbase, bars, tmem, kv_it, it);
    ++n_done_items;
  }
  uint64_t t_prefill = 0;
  if (p.trace != nullptr && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_prefill));
  // Switch roles: the decode rings overwrite prefill buffers through the async proxy.  All
  // bulk copies of the prefill were consumed before the last item barrier.
  fence_proxy_async_smem();
  named_bar_sync(5, 256);
  if (p.n_units > 0) {
    UnitDesc* descs = reinterpret_cast<UnitDesc*>(misc + kMiscBytes) + 4 * warp;
    volatile int* n_desc = reinterpret_cast<volatile int*>(misc + 64 + 16 * warp);
    decode_warp_loop(p, sbase, bars, descs, n_desc);
  }
  uint64_t t_decode = 0, t_barrier = 0;
  if (p.n_merge_rows > 0) {
    // grid barrier (cooperative launch: every CTA is resident), then the a6 merge phase
    named_bar_sync(6, 256);
    if (tid == 0) {
      if (p.trace != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_decode));
      __threadfence();
      atomicAdd(p.work + 3, 1);
      while (atomicAdd(p.work + 3, 0) < static_cast<int>(gridDim.x)) __nanosleep(100);
      __threadfence();
      if (p.trace != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_barrier));
    }
    named_bar_sync(7, 256);
    merge_phase(p);
  }
  named_bar_sync(8, 256);
  if (p.trace != nullptr && tid == 0) {
    uint64_t t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    int64_t* tr = p.trace + 8 * blockIdx.x;
    tr[0] = static_cast<int64_t>(t_start);
    tr[1] = static_cast<int64_t>(t_prefill);
    tr[2] = static_cast<int64_t>(t_end);
    tr[3] = n_done_items;
    tr[4] = static_cast<int64_t>(t_decode);
    tr[5] = static_cast<int64_t>(t_barrier);
  }
  if (tid == 0) {
    __threadfence();
    const int done = atomicAdd(p.work + 2, 1);
    if (done == static_cast<int>(gridDim.x) - 1) {  // last CTA: reset the queues for the next launch
      p.work[0] = 0;
      p.work[1] = 0;
      p.work[2] = 0;
      p.work[3] = 0;
      __threadfence();
    }
  }
}

int attention_bf16_smem_bytes() { return fa::kSmemBytes; }

cudaError_t launch_attention_bf16(const AttnParams& p, int grid, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(hybrid_attn_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         fa::kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  // Cooperative launch: the decode merge phase follows a grid-wide barrier, which
  // needs every CTA resident (1 CTA/SM, grid <= #SMs).
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(fa::kThreads);
  cfg.dynamicSmemBytes = fa::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  // NIYAMA_NO_COOP=1: diagnostic switch to measure the cooperative-launch overhead (the
  // grid is <= #SMs at 1 CTA/SM, so all CTAs are resident on an otherwise idle GPU).
  static const bool no_coop = std::getenv("NIYAMA_NO_COOP") != nullptr;
  attr[0].val.cooperative = (p.n_merge_rows > 0 && !no_coop) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
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
    const int64_t base = (blk * p.Hkv + kvh) * p.chunk_bytes + slot * 128;
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
