// tcgen05 SS MMA rate vs shared-memory placement of the operands (1 CTA, 1 thread
// issuing M=128 N=128 K=16 bf16 MMAs back to back into one TMEM accumulator).
//   A: SW128 K-major at smem offset a_off;  B: SW128 K-major (128 rows) or SW32 K-major
//   (V^T sub-block: [128 rows][32 B]) at b_off.  Prints ns per MMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2503_22562_b200/csrc -o tools/umma_layout_test tools/umma_layout_test.cu
#include <cstdio>
#include <cstdint>

#include "ptx.cuh"

using namespace niyama::ptx;

__global__ void rate_kernel(int n, uint32_t a_off, uint32_t b_off, int b_sw32, int n256) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(smem_u32(&tslot), 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t a = smem_u32(sm) + a_off, b = smem_u32(sm) + b_off;
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, n256 == 1 ? 256 : 128, 0, 0);
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      ad[i] = sw128_desc(a + (i & 3) * 32, 16, 1024);
      bd[i] = b_sw32 == 1   ? sw32_desc(b + (i & 7) * 4096, 16, 256)
              : b_sw32 == 2 ? noswz_desc(b + (i & 7) * 256, 128, 2048)   // K tile, per-block 4 KB runs
              : b_sw32 == 3 ? noswz_desc(b + (i & 7) * 4096, 128, 256)   // V^T 16-key sub-block
                            : sw128_desc(b + (i & 3) * 32, 16, 1024);
    }
    if (n256 >= 3) {  // 8 SS + commit (+ 8 TS + commit) per group, mbarrier per group
      __shared__ __align__(8) uint64_t gb[2];
      mbar_init(smem_u32(&gb[0]), 1);
      mbar_init(smem_u32(&gb[1]), 1);
      fence_mbar_init();
      for (int i = 0; i < n; i += 16) {
#pragma unroll
        for (int k = 0; k < 8; ++k) umma_f16(tmem + 256, ad[k], bd[k], idesc, 1u);
        umma_commit(smem_u32(&gb[0]));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (n256 == 3) umma_f16(tmem + 128, ad[k], bd[k], idesc, 1u);
          else umma_ts(tmem + 128, tmem + k * 8, bd[k], idesc, 1u);
        }
        umma_commit(smem_u32(&gb[1]));
      }
    } else if (n256 == 2) {  // TS: A (128 x 16 bf16) from TMEM columns [8k, 8k+8)
      for (int i = 0; i < n; i += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) umma_ts(tmem + 256, tmem + k * 8, bd[k], idesc, 1u);
      }
    } else {
      for (int i = 0; i < n; i += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) umma_f16(tmem + 256, ad[k], bd[k], idesc, 1u);
      }
    }
    umma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const int n = 1 << 15;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 20; ++w) rate_kernel<<<1, 128, 220 * 1024>>>(n, 0, 32768, 0, 0);
  struct C { uint32_t a, b; int sw32, n256; } cs[] = {
      {0, 16384, 0, 0},  {0, 32768, 0, 0},  {0, 49152, 0, 0},  {0, 65536, 0, 0},  {0, 98304, 0, 0},
      {0, 131072, 0, 0}, {0, 163840, 0, 0}, {32768, 65536, 0, 0}, {32768, 98304, 0, 0}, {65536, 98304, 0, 0},
      {0, 4096, 0, 0},   {0, 8192, 0, 0},   {0, 1024 * 36, 0, 0}, {0, 1024 * 40, 0, 0}, {0, 1024 * 48, 0, 0},
      {0, 32768, 1, 0},  {0, 65536, 1, 0},  {0, 98304, 1, 0},  {0, 16384, 1, 0},  {0, 8192, 1, 0},
      {0, 32768, 0, 1},  {0, 65536, 0, 1},  {0, 98304, 0, 1},
      {0, 32768, 2, 0},  {0, 65536, 2, 0},  {0, 32768, 3, 0},  {0, 65536, 3, 0},
      {0, 32768, 1, 2},  {0, 32768, 0, 2},  {0, 32768, 2, 2},
      {0, 32768, 2, 3},  {0, 32768, 1, 4}};
  for (auto c : cs) {
    float best = 1e9f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      rate_kernel<<<1, 128, 220 * 1024>>>(n, c.a, c.b, c.sw32, c.n256);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("%s A@%6u B@%6u B=%s N=%d : %7.2f ns/mma  (%s)\n", c.n256 == 2 ? "TS" : c.n256 == 3 ? "SS8+commit x2" : c.n256 == 4 ? "SS8+c,TS8+c" : "SS", c.a, c.b, c.sw32 == 1 ? "SW32 " : c.sw32 == 2 ? "NOSWK" : c.sw32 == 3 ? "NOSWV" : "SW128", c.n256 == 1 ? 256 : 128,
           best * 1e6 / n, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
