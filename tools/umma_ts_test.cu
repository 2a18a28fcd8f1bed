// Micro-test of tcgen05.mma with the A operand in TMEM ("TS"): O = P V with
// P [128 x 128] bf16 written by tcgen05.st as packed bf16x2 columns (row = lane),
// V [128 keys x 128 d] bf16 in SW128 MN-major smem (the hybrid kernel's V tile layout).
// Variants: A tmem column advance per K=16 step of 8 (hypothesis) or 16 columns.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2503_22562_b200/csrc -o tools/umma_ts_test tools/umma_ts_test.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "ptx.cuh"

using namespace niyama::ptx;

__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) ts_kernel(const __nv_bfloat16* P, const __nv_bfloat16* V, float* O,
                                                    int col_step) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(sm);
  // V -> smem, SW128 MN-major: panel (d/64), key row at 128 B, 16 B chunk c at c ^ (key & 7)
  for (int idx = tid; idx < 128 * 16; idx += 128) {
    const int k = idx >> 4, j = idx & 15;
    const uint4 v = *reinterpret_cast<const uint4*>(V + k * 128 + j * 8);
    st_shared_v4(sbase + (j >> 3) * 16384 + k * 128 + (((j & 7) ^ (k & 7)) << 4), v.x, v.y, v.z, v.w);
  }
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(smem_u32(&tslot), 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t lane_addr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  // P row `tid` -> TMEM columns 0..63 as packed bf16x2 (low half = even key)
  {
    uint32_t r[32];
    for (int half = 0; half < 2; ++half) {
      for (int c = 0; c < 32; ++c) {
        const int key = 2 * (half * 32 + c);
        const __nv_bfloat16 lo = P[tid * 128 + key], hi = P[tid * 128 + key + 1];
        r[c] = static_cast<uint32_t>(__bfloat16_as_ushort(lo)) | (static_cast<uint32_t>(__bfloat16_as_ushort(hi)) << 16);
      }
      tmem_st32(lane_addr + half * 32, r);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, 128, 0, 1);
    for (int kk = 0; kk < 8; ++kk)
      umma_ts(tmem + 128, tmem + kk * col_step, sw128_desc(sbase + kk * 2048, 16384, 1024), idesc, kk > 0);
    umma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  uint32_t o[32];
  for (int c = 0; c < 4; ++c) {
    tmem_ld32(lane_addr + 128 + c * 32, o);
    for (int e = 0; e < 32; ++e) O[tid * 128 + c * 32 + e] = __uint_as_float(o[e]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

int main() {
  std::vector<__nv_bfloat16> P(128 * 128), V(128 * 128);
  std::vector<float> Pf(128 * 128), Vf(128 * 128);
  srand(1);
  for (int i = 0; i < 128 * 128; ++i) {
    P[i] = __float2bfloat16((rand() % 2001 - 1000) / 1000.f);
    V[i] = __float2bfloat16((rand() % 2001 - 1000) / 1000.f);
    Pf[i] = __bfloat162float(P[i]);
    Vf[i] = __bfloat162float(V[i]);
  }
  std::vector<float> ref(128 * 128, 0.f);
  for (int m = 0; m < 128; ++m)
    for (int k = 0; k < 128; ++k)
      for (int n = 0; n < 128; ++n) ref[m * 128 + n] += Pf[m * 128 + k] * Vf[k * 128 + n];
  __nv_bfloat16 *dP, *dV;
  float* dO;
  cudaMalloc(&dP, 128 * 128 * 2);
  cudaMalloc(&dV, 128 * 128 * 2);
  cudaMalloc(&dO, 128 * 128 * 4);
  cudaMemcpy(dP, P.data(), 128 * 128 * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), 128 * 128 * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int step : {8, 16, 4}) {
    cudaMemset(dO, 0, 128 * 128 * 4);
    ts_kernel<<<1, 128, 40 * 1024>>>(dP, dV, dO, step);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> out(128 * 128);
    cudaMemcpy(out.data(), dO, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int i = 0; i < 128 * 128; ++i) maxerr = fmax(maxerr, fabs(out[i] - ref[i]));
    printf("col_step=%2d err=%s max_abs_err=%.3e  out[0]=%f ref[0]=%f\n", step, cudaGetErrorString(e), maxerr,
           out[0], ref[0]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
