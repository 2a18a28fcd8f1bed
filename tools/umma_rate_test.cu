// tcgen05 MMA issue/execute rate micro-benchmark (1 CTA): cycles per MMA for
//   SS  M=128 N=64  K=16 (QK^T at 64-key tiles)
//   SS  M=128 N=128 K=16 (QK^T at 128-key tiles)
//   TS  M=128 N=128 K=16 (PV with P in TMEM)
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2503_22562_b200/csrc -o tools/umma_rate_test tools/umma_rate_test.cu
#include <cstdio>
#include <cstdint>

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

__global__ void rate_kernel(long long* out, int n, int only) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 150 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
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
    uint32_t phase = 0;
    for (int variant = only; variant < only + 1; ++variant) {
      const int N = (variant == 0) ? 64 : (variant == 6 ? 256 : 128);
      const int bmn = (variant == 2 || variant == 4 || variant == 7) ? 1 : 0;
      const uint32_t idesc = idesc_bf16_f32(128, N, 0, bmn);
      long long t0 = clock64();
      for (int i = 0; i < n; ++i) {
        if (variant < 2 || variant == 6)
          umma_f16(tmem + 256, sw128_desc(a + (i & 3) * 32, 16, 1024), sw128_desc(b + (i & 3) * 32, 16, 1024), idesc,
                   i > 0);
        else if (variant == 2)  // TS, B MN-major (V tile)
          umma_ts(tmem + 256, tmem + (i & 7) * 8, sw128_desc(b + (i & 7) * 2048, 8192, 1024), idesc, i > 0);
        else if (variant == 3)  // SS with A and B both 128 rows: K-major
          umma_f16(tmem + 256, sw128_desc(a + (i & 3) * 32, 16, 1024), sw128_desc(a + 16384 + (i & 3) * 32, 16, 1024),
                   idesc, i > 0);
        else if (variant == 4)  // SS, A K-major (P in smem), B MN-major (V tile)
          umma_f16(tmem + 256, sw128_desc(a + (i & 3) * 32, 16, 1024), sw128_desc(b + (i & 7) * 2048, 8192, 1024),
                   idesc, i > 0);
        else if (variant == 5)  // TS, B K-major
          umma_ts(tmem + 256, tmem + (i & 7) * 8, sw128_desc(b + (i & 3) * 32, 16, 1024), idesc, i > 0);
        else if (variant == 8)  // SS, A SW128 K-major (P), B SW32 K-major (V^T sub-block, the kernel's PV)
          umma_f16(tmem + 256, sw128_desc(a + (i & 3) * 32, 16, 1024), sw32_desc(b + (i & 7) * 4096, 16, 256), idesc,
                   i > 0);
        else if (variant == 9)  // SS, A SW128 (Q), B SW128 (K), operands 64 KB apart (the kernel's QK)
          umma_f16(tmem + 256, sw128_desc(a + (i & 3) * 32, 16, 1024), sw128_desc(a + 65536 + (i & 3) * 32, 16, 1024),
                   idesc, i > 0);
        else  // 7: SS, A K-major, B MN-major with 16 KB panels (128-key V tile)
          umma_f16(tmem + 256, sw128_desc(a + (i & 3) * 32, 16, 1024), sw128_desc(b + (i & 7) * 2048, 16384, 1024),
                   idesc, i > 0);
      }
      long long t1 = clock64();
      umma_commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), phase);
      phase ^= 1;
      long long t2 = clock64();
      out[variant * 2] = t1 - t0;
      out[variant * 2 + 1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 128);
  cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int n = 1 << 16;
  const char* names[10] = {"SS N64 B K-major", "SS N128 B K-major", "TS N128 B MN-major", "SS N128 A,B 128 rows",
                          "SS N128 B MN-major (8K panel)", "TS N128 B K-major", "SS N256 B K-major",
                          "SS N128 B MN-major (16K panel)", "SS N128 B SW32 K-major (PV)", "SS N128 QK 64K apart"};
  const double F = 2.0 * 128 * 16;
  const double flop[10] = {F * 64, F * 128, F * 128, F * 128, F * 128, F * 128, F * 256, F * 128, F * 128, F * 128};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 20; ++w) rate_kernel<<<1, 128, 160 * 1024>>>(d, n, 1);  // clock warm-up
  for (int rep = 0; rep < 2; ++rep)
    for (int v = 0; v < 10; ++v) {
      cudaEventRecord(a);
      rate_kernel<<<1, 128, 160 * 1024>>>(d, n, v);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("%-34s %8.2f ns/mma  %7.2f TFLOP/s per SM (x148 = %6.0f)  %s\n", names[v], ms * 1e6 / n,
             flop[v] * n / (ms * 1e-3) / 1e12, 148 * flop[v] * n / (ms * 1e-3) / 1e12,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
