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

#include "internal.h"
#include "ptx.cuh"

namespace niyama {

using namespace ptx;

// ============================================================= append (a3)
// One thread per 16-byte piece of a (row, kv head) vector.  Source rows are
// dense [T][Hkv][row_bytes]; the destination piece j of the row at (block,
// slot) lands in panel j/8 at chunk position (j%8) ^ (slot%8).
__global__ void kv_append_kernel(const AppendParams p) {
  const int pieces = p.row_bytes >> 4;
  const int64_t total = static_cast<int64_t>(p.T) * p.Hkv * pieces;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(idx % pieces);
    const int64_t rh = idx / pieces;
    const int h = static_cast<int>(rh % p.Hkv);
    const int r = static_cast<int>(rh / p.Hkv);
    const int32_t sm = p.slot_map[r];
    const int64_t blk = sm / p.B;
    const int slot = sm - static_cast<int>(blk) * p.B;
    const int64_t src_off = rh * p.row_bytes + (static_cast<int64_t>(j) << 4);
    const int64_t dst_off = (blk * p.Hkv + h) * p.chunk_bytes + static_cast<int64_t>(j >> 3) * p.B * 128 +
                            slot * 128 + (((j & 7) ^ (slot & 7)) << 4);
    const uint4 kv = __ldg(reinterpret_cast<const uint4*>(p.k_new + src_off));
    const uint4 vv = __ldg(reinterpret_cast<const uint4*>(p.v_new + src_off));
    *reinterpret_cast<uint4*>(p.pool_k + dst_off) = kv;
    *reinterpret_cast<uint4*>(p.pool_v + dst_off) = vv;
  }
}

cudaError_t launch_append(const AppendParams& p, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(p.T) * p.Hkv * (p.row_bytes >> 4);
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
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
// Shared memory map (bytes from the 1024-aligned base):
//   [0, 32K)            Q tile   (2 panels x 128 rows x 128 B, SW128)
//   [32K, 32K+NS*32K)   K stages (128 keys x 256 B each)
//   [.., +NS*32K)       V stages
//   [.., +32K)          P tile   (2 panels x 128 rows x 128 B, SW128, bf16)
// The decode role reuses [0, 192K) as 8 warps x 3 stages x 8 KB.
namespace fa {
constexpr int kD = 128;            // head dim (bf16 path)
constexpr int kBN = 128;           // keys per prefill tile
constexpr int kNS = 2;             // K/V stages
constexpr int kPanel = 128 * 128;  // one 64-column panel of a 128-row tile
constexpr int kTile = 2 * kPanel;  // 128 rows x 256 B
constexpr int kQOff = 0;
constexpr int kKOff = kTile;
constexpr int kVOff = kKOff + kNS * kTile;
constexpr int kPOff = kVOff + kNS * kTile;
constexpr int kDataBytes = kPOff + kTile;  // 192 KB
constexpr int kDecStages = 3;
constexpr int kDecStage = 8192;  // 16 tokens of K (4 KB) + V (4 KB)
static_assert(8 * kDecStages * kDecStage <= kDataBytes, "decode ring must fit");
// barrier indices
constexpr int kBarKFull = 0;
constexpr int kBarVFull = kBarKFull + kNS;
constexpr int kBarKVEmpty = kBarVFull + kNS;
constexpr int kBarSFull = kBarKVEmpty + kNS;
constexpr int kBarSFree = kBarSFull + 2;
constexpr int kBarPFull = kBarSFree + 2;
constexpr int kBarODone = kBarPFull + 1;
constexpr int kBarDec = kBarODone + 1;  // 8 warps x 3 stages
constexpr int kNumBars = kBarDec + 8 * kDecStages;
constexpr int kSmemBytes = 1024 /*align slack*/ + kDataBytes + kNumBars * 8 + 64;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemO = 256;  // O accumulator columns [256, 384); S buffers at 0 and 128
constexpr uint32_t kIdescQK = idesc_bf16_f32(128, kBN, 0, 0);
constexpr uint32_t kIdescPV = idesc_bf16_f32(128, kD, 0, 1);
}  // namespace fa

// -------------------------------------------------------------- prefill tile
// Roles inside the 256-thread CTA: warp 0 lane 0 = bulk-copy producer, warp 1
// lane 0 = tcgen05 issuer, warps 4-7 = softmax (thread = TMEM lane = tile row).
__device__ __forceinline__ void prefill_tile(const AttnParams& p, const PrefillTile& t, uint8_t* smem,
                                             uint32_t sbase, uint32_t bars, uint32_t tmem, uint32_t& kv_iter,
                                             uint32_t& s_iter, uint32_t& pv_iter) {
  using namespace fa;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int g = p.g, R = p.R;
  const int vrows = min(R, t.c - t.t0);
  const int nk = (t.nkeys + kBN - 1) / kBN;

  // ---- Q tile: rows r = hh*R + i  <-  q[row0 + t0 + i][kvh*g + hh][:]
  {
    const uint8_t* q = static_cast<const uint8_t*>(p.q);
    for (int idx = tid; idx < 128 * 16; idx += 256) {
      const int r = idx >> 4, j = idx & 15;
      const int hh = r / R, i = r - hh * R;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (i < vrows) {
        const int64_t row = t.row0 + t.t0 + i;
        v = __ldg(reinterpret_cast<const uint4*>(q + ((row * p.Hq + t.kvh * g + hh) * kD) * 2 + j * 16));
      }
      st_shared_v4(sbase + kQOff + (j >> 3) * kPanel + r * 128 + (((j & 7) ^ (r & 7)) << 4), v.x, v.y, v.z, v.w);
    }
    fence_proxy_async_smem();
    __syncthreads();
  }

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer: K and V tiles of 128 keys, block by block
      const int bpt = kBN / p.B;  // blocks per tile
      const uint32_t seg = static_cast<uint32_t>(p.B) * 128;
      for (int j = 0; j < nk; ++j) {
        const uint32_t it = kv_iter + j;
        const int st = it % kNS;
        const uint32_t ph = (it / kNS) & 1;
        mbar_wait(bars + 8 * (kBarKVEmpty + st), ph ^ 1);
        const uint32_t kfull = bars + 8 * (kBarKFull + st), vfull = bars + 8 * (kBarVFull + st);
        mbar_expect_tx(kfull, kTile);
        mbar_expect_tx(vfull, kTile);
        for (int b = 0; b < bpt; ++b) {
          int lb = j * bpt + b;
          if (lb >= t.nblk) lb = t.nblk - 1;  // finite data; masked out (P = 0)
          const int64_t phys = p.tables[t.tbl + lb];
          const int64_t off = (phys * p.Hkv + t.kvh) * p.chunk_bytes;
          for (int pn = 0; pn < 2; ++pn) {
            const uint32_t dst = pn * kPanel + b * seg;
            bulk_g2s(sbase + kKOff + st * kTile + dst, p.pool_k + off + pn * seg, seg, kfull);
            bulk_g2s(sbase + kVOff + st * kTile + dst, p.pool_v + off + pn * seg, seg, vfull);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- tcgen05 issuer
      for (int j = 0; j <= nk; ++j) {
        if (j < nk) {
          const uint32_t si = s_iter + j;
          const uint32_t sb = si & 1, sph = (si >> 1) & 1;
          const uint32_t it = kv_iter + j;
          const int st = it % kNS;
          const uint32_t ph = (it / kNS) & 1;
          mbar_wait(bars + 8 * (kBarSFree + sb), sph ^ 1);
          mbar_wait(bars + 8 * (kBarKFull + st), ph);
          tc_fence_after();
          const uint32_t qa = sbase + kQOff, ka = sbase + kKOff + st * kTile;
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk) {
            const uint32_t koff = (kk >> 2) * kPanel + (kk & 3) * 32;
            umma_f16(tmem + sb * 128, sw128_desc(qa + koff, 16, 1024), sw128_desc(ka + koff, 16, 1024), kIdescQK,
                     kk > 0);
          }
          umma_commit(bars + 8 * (kBarSFull + sb));
        }
        if (j >= 1) {
          const int jj = j - 1;
          const uint32_t it = kv_iter + jj;
          const int st = it % kNS;
          const uint32_t ph = (it / kNS) & 1;
          mbar_wait(bars + 8 * kBarPFull, (pv_iter + jj) & 1);
          mbar_wait(bars + 8 * (kBarVFull + st), ph);
          tc_fence_after();
          const uint32_t pa = sbase + kPOff, va = sbase + kVOff + st * kTile;
#pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk) {
            const uint32_t poff = (kk >> 2) * kPanel + (kk & 3) * 32;
            umma_f16(tmem + kTmemO, sw128_desc(pa + poff, 16, 1024), sw128_desc(va + kk * 2048, kPanel, 1024),
                     kIdescPV, (jj > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(bars + 8 * (kBarKVEmpty + st));
          umma_commit(bars + 8 * kBarODone);
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax: this thread owns tile row r (TMEM lane r)
    const int quarter = warp - 4;
    const int r = quarter * 32 + lane;
    const int hh = r / R, i = r - hh * R;
    const bool valid = i < vrows;
    const int pos = t.o + t.t0 + (valid ? i : 0);  // last visible key of this row
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    float m_ref = -INFINITY, l = 0.f;
    const float sl2 = p.scale_log2;
    for (int j = 0; j < nk; ++j) {
      const uint32_t si = s_iter + j;
      const uint32_t sb = si & 1, sph = (si >> 1) & 1;
      mbar_wait(bars + 8 * (kBarSFull + sb), sph);
      tc_fence_after();
      float s[kBN];
#pragma unroll
      for (int c = 0; c < kBN / 32; ++c) {
        uint32_t raw[32];
        tmem_ld32(lane_addr + sb * 128 + c * 32, raw);
#pragma unroll
        for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(raw[e]);
      }
      tc_fence_before();
      mbar_arrive(bars + 8 * (kBarSFree + sb));
      const int kbase = j * kBN;
      float mx = -INFINITY;
      if (kbase + kBN - 1 <= pos) {
#pragma unroll
        for (int e = 0; e < kBN; ++e) {
          s[e] *= sl2;
          mx = fmaxf(mx, s[e]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < kBN; ++e) {
          s[e] = (kbase + e <= pos) ? s[e] * sl2 : -INFINITY;
          mx = fmaxf(mx, s[e]);
        }
      }
      const float m_new = fmaxf(m_ref, mx);
      const bool need = m_new > m_ref + 8.0f;  // lazy rescale (p <= 2^8 otherwise)
      if (j > 0) {
        mbar_wait(bars + 8 * kBarODone, (pv_iter + j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, need)) {
          const float alpha = need ? ex2(m_ref - m_new) : 1.f;
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
      }
      if (need) {
        l *= ex2(m_ref - m_new);  // 0 on the first tile (m_ref = -inf)
        m_ref = m_new;
      }
      float sum = 0.f;
      const uint32_t prow = sbase + kPOff + r * 128;
#pragma unroll
      for (int c = 0; c < kBN / 8; ++c) {
        float e0 = ex2(s[c * 8 + 0] - m_ref), e1 = ex2(s[c * 8 + 1] - m_ref);
        float e2 = ex2(s[c * 8 + 2] - m_ref), e3 = ex2(s[c * 8 + 3] - m_ref);
        float e4 = ex2(s[c * 8 + 4] - m_ref), e5 = ex2(s[c * 8 + 5] - m_ref);
        float e6 = ex2(s[c * 8 + 6] - m_ref), e7 = ex2(s[c * 8 + 7] - m_ref);
        sum += ((e0 + e1) + (e2 + e3)) + ((e4 + e5) + (e6 + e7));
        st_shared_v4(prow + (c >> 3) * kPanel + (((c & 7) ^ (r & 7)) << 4), pack_bf16(e0, e1), pack_bf16(e2, e3),
                     pack_bf16(e4, e5), pack_bf16(e6, e7));
      }
      l += sum;
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(bars + 8 * kBarPFull);
    }
    // ---------------- epilogue: O / l -> bf16, LSE
    mbar_wait(bars + 8 * kBarODone, (pv_iter + nk - 1) & 1);
    tc_fence_after();
    const float inv_l = 1.f / l;
    const int h = t.kvh * g + hh;
    const int64_t trow = t.row0 + t.t0 + i;
    uint8_t* orow = static_cast<uint8_t*>(p.o) + ((static_cast<int64_t>(h) * p.T + trow) * kD) * 2;
#pragma unroll 1
    for (int c = 0; c < kD / 32; ++c) {
      uint32_t ov[32];
      tmem_ld32(lane_addr + kTmemO + c * 32, ov);
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
    if (valid && p.lse != nullptr) p.lse[static_cast<int64_t>(h) * p.T + trow] = (m_ref + __log2f(l)) * 0.69314718055994530942f;
  }
  kv_iter += nk;
  s_iter += nk;
  pv_iter += nk;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
}

// --------------------------------------------------------------- decode unit
__device__ __forceinline__ void decode_issue(const AttnParams& p, const DecodeUnit& u, int s, uint32_t stage,
                                             uint32_t bar) {
  const int tok = u.k0 + 16 * s;
  const int lb = tok / p.B;
  const int sub = (tok - lb * p.B) >> 4;
  const int64_t phys = p.tables[u.tbl + lb];
  const int64_t off = (phys * p.Hkv + u.kvh) * p.chunk_bytes + sub * 2048;
  const uint32_t seg = static_cast<uint32_t>(p.B) * 128;
  mbar_expect_tx(bar, fa::kDecStage);
  bulk_g2s(stage, p.pool_k + off, 2048, bar);
  bulk_g2s(stage + 2048, p.pool_k + off + seg, 2048, bar);
  bulk_g2s(stage + 4096, p.pool_v + off, 2048, bar);
  bulk_g2s(stage + 6144, p.pool_v + off + seg, 2048, bar);
}

__device__ __forceinline__ void decode_warp_loop(const AttnParams& p, uint32_t sbase, uint32_t bars) {
  using namespace fa;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int g = p.g;
  const uint32_t ring = sbase + warp * kDecStages * kDecStage;
  const uint32_t bar0 = bars + 8 * (kBarDec + warp * kDecStages);
  uint32_t dec_iter = 0;
  const float sl2 = p.scale_log2;
  // ldmatrix lane geometry
  const int mi = lane >> 3, rr = lane & 7;
  const int ktok = (mi >> 1) * 8 + rr;  // K (non-trans): matrices (tok 0-7,c),(0-7,c+1),(8-15,c),(8-15,c+1)
  const int vtok = (mi & 1) * 8 + rr;   // V (trans):     matrices (tok 0-7,d),(8-15,d),(0-7,d+8),(8-15,d+8)
  while (true) {
    int ui = 0;
    if (lane == 0) ui = atomicAdd(p.work + 1, 1);
    ui = __shfl_sync(0xffffffffu, ui, 0);
    if (ui >= p.n_units) break;
    const DecodeUnit u = p.units[ui];
    const int nst = (u.k1 - u.k0 + 15) >> 4;
    if (lane == 0) {
      const int pre = nst < kDecStages ? nst : kDecStages;
      for (int s = 0; s < pre; ++s) {
        const uint32_t slot = (dec_iter + s) % kDecStages;
        decode_issue(p, u, s, ring + slot * kDecStage, bar0 + 8 * slot);
      }
    }
    // Q fragments (A operand, rows = heads of the group, rows >= g are zero)
    uint32_t qa0[8], qa2[8];
    {
      const __nv_bfloat16* qrow = static_cast<const __nv_bfloat16*>(p.q) +
                                  (static_cast<int64_t>(u.row) * p.Hq + u.kvh * g + (gid < g ? gid : 0)) * kD;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t a = __ldg(reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * tig));
        uint32_t b = __ldg(reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 8 + 2 * tig));
        qa0[kk] = gid < g ? a : 0u;
        qa2[kk] = gid < g ? b : 0u;
      }
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
      if (lane == 0 && s + kDecStages < nst) decode_issue(p, u, s + kDecStages, stg, bar0 + 8 * slot);
      ++dec_iter;
    }
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    const int D = kD;
    if (u.nsplit == 1) {
      if (gid < g) {
        const int h = u.kvh * g + gid;
        const float inv = 1.f / l;
        __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(p.o) + (static_cast<int64_t>(h) * p.T + u.row) * D;
#pragma unroll
        for (int n = 0; n < 16; ++n)
          *reinterpret_cast<uint32_t*>(orow + n * 8 + 2 * tig) = pack_bf16(o[n][0] * inv, o[n][1] * inv);
        if (tig == 0 && p.lse != nullptr)
          p.lse[static_cast<int64_t>(h) * p.T + u.row] = (m + __log2f(l)) * 0.69314718055994530942f;
      }
    } else {
      const int pidx = u.pbase + u.split;
      if (gid < g) {
        const float inv = 1.f / l;
        float* po = p.part_o + (static_cast<int64_t>(pidx) * g + gid) * D;
#pragma unroll
        for (int n = 0; n < 16; ++n)
          __stcg(reinterpret_cast<float2*>(po + n * 8 + 2 * tig), make_float2(o[n][0] * inv, o[n][1] * inv));
        if (tig == 0) __stcg(reinterpret_cast<float2*>(p.part_ml + (static_cast<int64_t>(pidx) * g + gid) * 2),
                             make_float2(m, l));
      }
      __threadfence();
      __syncwarp();
      int prev = 0;
      if (lane == 0) prev = atomicAdd(p.counters + u.pair, 1);
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev == u.nsplit - 1) {
        // a6: last split merges all partials of this (row, kv head), in split order.
        __threadfence();
        for (int hh = 0; hh < g; ++hh) {
          float M = -INFINITY;
          for (int sp = 0; sp < u.nsplit; ++sp)
            M = fmaxf(M, __ldcg(p.part_ml + (static_cast<int64_t>(u.pbase + sp) * g + hh) * 2));
          float L = 0.f;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int sp = 0; sp < u.nsplit; ++sp) {
            const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.part_ml + (static_cast<int64_t>(u.pbase + sp) * g + hh) * 2));
            const float w = ex2(ml.x - M) * ml.y;
            L += w;
            const float4 v = __ldcg(reinterpret_cast<const float4*>(p.part_o + (static_cast<int64_t>(u.pbase + sp) * g + hh) * D + lane * 4));
            acc.x += w * v.x;
            acc.y += w * v.y;
            acc.z += w * v.z;
            acc.w += w * v.w;
          }
          const float inv = 1.f / L;
          const int h = u.kvh * g + hh;
          __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(p.o) + (static_cast<int64_t>(h) * p.T + u.row) * D;
          uint2 w2;
          w2.x = pack_bf16(acc.x * inv, acc.y * inv);
          w2.y = pack_bf16(acc.z * inv, acc.w * inv);
          *reinterpret_cast<uint2*>(orow + lane * 4) = w2;
          if (lane == 0 && p.lse != nullptr)
            p.lse[static_cast<int64_t>(h) * p.T + u.row] = (M + __log2f(L)) * 0.69314718055994530942f;
        }
        if (lane == 0) p.counters[u.pair] = 0;  // ready for the next launch
      }
    }
  }
}

__global__ void __launch_bounds__(256, 1) hybrid_attn_bf16_kernel(const AttnParams p) {
  using namespace fa;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bars = sbase + kDataBytes;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kDataBytes + kNumBars * 8);
  int* item_slot = reinterpret_cast<int*>(smem + kDataBytes + kNumBars * 8 + 16);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  if (tid == 0) {
    for (int b = kBarKFull; b < kBarKVEmpty + kNS; ++b) mbar_init(bars + 8 * b, 1);
    mbar_init(bars + 8 * (kBarSFull + 0), 1);
    mbar_init(bars + 8 * (kBarSFull + 1), 1);
    mbar_init(bars + 8 * (kBarSFree + 0), 128);
    mbar_init(bars + 8 * (kBarSFree + 1), 128);
    mbar_init(bars + 8 * kBarPFull, 128);
    mbar_init(bars + 8 * kBarODone, 1);
    for (int b = kBarDec; b < kNumBars; ++b) mbar_init(bars + 8 * b, 1);
    fence_mbar_init();
  }
  const bool any_tiles = p.n_tiles > 0;
  if (any_tiles && warp == 1) {
    tmem_alloc(smem_u32(tmem_slot), kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = any_tiles ? *tmem_slot : 0u;

  uint32_t kv_iter = 0, s_iter = 0, pv_iter = 0;
  while (any_tiles) {
    if (tid == 0) *item_slot = atomicAdd(p.work + 0, 1);
    __syncthreads();
    const int item = *item_slot;
    __syncthreads();
    if (item >= p.n_tiles) break;
    prefill_tile(p, p.tiles[item], smem, sbase, bars, tmem, kv_iter, s_iter, pv_iter);
  }
  // Switch roles: the ring overwrites prefill buffers through the async proxy.
  fence_proxy_async_smem();
  __syncthreads();
  if (p.n_units > 0) decode_warp_loop(p, sbase, bars);

  tc_fence_before();
  __syncthreads();
  if (any_tiles && warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
  if (tid == 0) {
    __threadfence();
    const int done = atomicAdd(p.work + 2, 1);
    if (done == static_cast<int>(gridDim.x) - 1) {  // last CTA: reset the queues for the next launch
      p.work[0] = 0;
      p.work[1] = 0;
      p.work[2] = 0;
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
  hybrid_attn_bf16_kernel<<<grid, 256, fa::kSmemBytes, s>>>(p);
  return cudaGetLastError();
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
