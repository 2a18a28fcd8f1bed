// Does tcgen05.mma issue block while earlier MMAs execute?  One thread issues N MMAs
// (M=128 N=128 K=16, SS) back to back; clock64 after the issue loop and after the
// commit's mbarrier completes.  If issue time ~ completion time, the issuing thread is
// throttled to the tensor pipe's execution rate (shallow MMA queue).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2503_22562_b200/csrc -o tools/umma_issue_test tools/umma_issue_test.cu
#include <cstdio>
#include <cstdint>

#include "ptx.cuh"

using namespace niyama::ptx;

__global__ void k(int n, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
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
  const uint32_t a = smem_u32(sm), b = a + 32768;
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
    uint64_t ad[4], bd[4];
    for (int i = 0; i < 4; ++i) ad[i] = sw128_desc(a + i * 32, 16, 1024), bd[i] = sw128_desc(b + i * 32, 16, 1024);
    uint32_t ph = 0;
    for (int rep = 0; rep < 3; ++rep) {
      long long t0 = clock64();
      for (int i = 0; i < n; i += 4) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_f16(tmem + 256, ad[kk], bd[kk], idesc, 1u);
      }
      long long t1 = clock64();
      umma_commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), ph);
      ph ^= 1;
      long long t2 = clock64();
      out[rep * 2] = t1 - t0;
      out[rep * 2 + 1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  long long* d;
  cudaMalloc(&d, 64);
  long long h[6];
  for (int n : {4, 8, 16, 32, 64, 256}) {
    k<<<1, 128, 80 * 1024>>>(n, d);
    cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
    printf("n=%4d  issue %6lld cycles (%5.1f/mma)  complete %6lld cycles (%5.1f/mma)  [%s]\n", n, h[4], (double)h[4] / n,
           h[5], (double)h[5] / n, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
