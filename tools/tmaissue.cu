// Per-SM throughput of the prefill tile's copy pattern (diagnostic).
// One CTA per SM (G CTAs).  "K" producer: 32 KB stages made of `nk` copies issued by
// lanes 0..kl-1 of warp 0; "V" producer: 32 KB stages of `nv` copies by lanes of warp 2;
// ring depth dk / dv; a consumer warp (warp 1 lane 0) waits full and frees immediately.
// Source chunks are 4 KB pieces at random (permuted) addresses inside `wrap` bytes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmaissue tools/tmaissue.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint32_t bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory"); }
__device__ __forceinline__ void arrive(uint32_t bar) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory"); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t n, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(n), "r"(bar) : "memory");
}

__global__ void __launch_bounds__(128, 1) kern(const uint8_t* src, const int* perm, int nperm, int steps, int nk, int nv,
                                               int dk, int dv, int kl, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = smem_u32(sm);
  const uint32_t kfull = smem_u32(&bars[0]), kempty = smem_u32(&bars[4]), vfull = smem_u32(&bars[8]), vempty = smem_u32(&bars[12]);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) { mbar_init(kfull + 8 * i, 1); mbar_init(kempty + 8 * i, 1); mbar_init(vfull + 8 * i, 1); mbar_init(vempty + 8 * i, 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 0 || warp == 2) {
    const bool isK = warp == 0;
    const int n = isK ? nk : nv, d = isK ? dk : dv;
    const uint32_t ring = base + (isK ? 0 : 3 * 32768);
    const uint32_t full = isK ? kfull : vfull, empty = isK ? kempty : vempty;
    const int per = 32768 / n;
    const int lanes = isK ? kl : 8;
    for (int j = 0; j < steps; ++j) {
      const int st = j % d;
      if (lane == 0) {
        wait(empty + 8 * st, ((j / d) & 1) ^ 1);
        expect_tx(full + 8 * st, 32768);
      }
      __syncwarp();
      for (int c = lane; c < n; c += lanes) {
        if (lane < lanes) {
          const int chunk = perm[(blockIdx.x * 977 + j * 8 + (c * per) / 4096 + (isK ? 0 : 5000)) % nperm];
          bulk(ring + st * 32768 + c * per, src + (size_t)chunk * 4096 + (c * per) % 4096, per, full + 8 * st);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (int j = 0; j < steps; ++j) {
      wait(kfull + 8 * (j % dk), (j / dk) & 1);
      arrive(kempty + 8 * (j % dk));
      wait(vfull + 8 * (j % dv), (j / dv) & 1);
      arrive(vempty + 8 * (j % dv));
    }
    sink[blockIdx.x] = 1;
  }
}

int main() {
  const size_t wrap = (size_t)64 << 20;  // 64 MB of 4 KB chunks (L2-resident-ish)
  const int nperm = (int)(wrap / 4096);
  uint8_t* buf; int *perm, *sink;
  cudaMalloc(&buf, wrap); cudaMalloc(&perm, nperm * 4); cudaMalloc(&sink, 4096);
  cudaMemset(buf, 1, wrap);
  int* h = new int[nperm];
  for (int i = 0; i < nperm; ++i) h[i] = i;
  uint64_t x = 88172645463325252ull;
  for (int i = nperm - 1; i > 0; --i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; int j = (int)(x % (uint64_t)(i + 1)); int t = h[i]; h[i] = h[j]; h[j] = t; }
  cudaMemcpy(perm, h, nperm * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct C { int nk, nv, dk, dv, kl; const char* what; } cs[] = {
    {16, 8, 2, 2, 8, "prefill today: K 16x2KB by 8 lanes, V 8x4KB, rings 2/2"},
    {16, 8, 3, 3, 8, "rings 3/3"},
    {16, 8, 2, 2, 1, "K by ONE lane"},
    {8, 8, 2, 2, 8, "K 8x4KB"},
    {4, 4, 2, 2, 8, "K 4x8KB, V 4x8KB"},
    {1, 1, 2, 2, 8, "K 1x32KB, V 1x32KB"},
    {16, 8, 2, 2, 16, "K by 16 lanes"},
  };
  const int steps = 2000;
  for (int G : {16, 128}) for (auto c : cs) {
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      kern<<<G, 128, 6 * 32768>>>(buf, perm, nperm, steps, c.nk, c.nv, c.dk, c.dv, c.kl, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    const double per_sm = 65536.0 * steps / (ms * 1e-3) / 1e9;
    printf("G=%3d %-55s per SM %6.1f GB/s  step %.2f us  (%s)\n", G, c.what, per_sm, ms * 1e3 / steps, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
