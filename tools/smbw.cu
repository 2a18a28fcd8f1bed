// Per-SM load throughput (does one SM cap below its share of HBM/L2?):
// grid G CTAs x 8 warps, each warp streams its range through a 3-stage ring of 8 KB
// bulk copies (cp.async.bulk, the decode path's pattern) or 16-byte cp.async, or
// ld.global.v4; source either distinct (HBM) or wrapped inside `wrap` bytes (L2).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/smbw tools/smbw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint32_t bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory"); }
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t n, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(n), "r"(bar) : "memory");
}

// mode 0: bulk (ops per 8 KB stage = sub); mode 1: cp.async 16 B by all lanes
__global__ void __launch_bounds__(256, 1) ring(const uint8_t* src, size_t per_warp, size_t wrap, int mode, int sub, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int chunk = 8192, depth = 3;
  __shared__ __align__(8) uint64_t bars[8 * 4];
  const size_t gw = (size_t)blockIdx.x * 8 + w;
  uint32_t rbase = smem_u32(sm) + w * depth * chunk;
  uint32_t bar0 = smem_u32(&bars[w * 4]);
  if (lane == 0) for (int s = 0; s < depth; ++s) mbar_init(bar0 + 8 * s, mode == 0 ? 1 : 32);
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const int n = (int)(per_warp / chunk);
  auto addr = [&](int i) { return src + ((gw * per_warp + (size_t)i * chunk) % wrap); };
  auto issue = [&](int i) {
    int s = i % depth;
    if (mode == 0) {
      if (lane == 0) {
        expect_tx(bar0 + 8 * s, chunk);
        for (int k = 0; k < sub; ++k) bulk(rbase + s * chunk + k * (chunk / sub), addr(i) + k * (chunk / sub), chunk / sub, bar0 + 8 * s);
      }
    } else {
      const uint8_t* a = addr(i);
      for (int k = 0; k < chunk / 512; ++k)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(rbase + s * chunk + k * 512 + lane * 16), "l"(a + k * 512 + lane * 16) : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar0 + 8 * s) : "memory");
    }
  };
  for (int i = 0; i < depth && i < n; ++i) issue(i);
  int acc = 0;
  for (int i = 0; i < n; ++i) {
    int s = i % depth;
    while (!try_wait(bar0 + 8 * s, (i / depth) & 1)) {}
    acc += *(volatile int*)(sm + w * depth * chunk + s * chunk + lane * 4);
    __syncwarp();
    if (i + depth < n) issue(i + depth);
  }
  if (acc == 0x12345) sink[0] = acc;
}

__global__ void __launch_bounds__(256, 1) ldg(const uint8_t* src, size_t per_warp, size_t wrap, int* sink) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t gw = (size_t)blockIdx.x * 8 + w;
  int acc = 0;
  for (size_t off = 0; off < per_warp; off += 8 * 512) {
    int4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int4* a = (const int4*)(src + ((gw * per_warp + off + k * 512) % wrap) + lane * 16);
      asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(a));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].w;
  }
  if (acc == 0x12345) sink[0] = acc;
}

int main() {
  const size_t bytes = (size_t)2 << 30;
  uint8_t* buf; int* sink;
  cudaMalloc(&buf, bytes); cudaMalloc(&sink, 4); cudaMemset(buf, 1, bytes);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const size_t per_warp = (size_t)4 << 20;  // 4 MB per warp
  for (int l2 = 0; l2 < 2; ++l2)
    for (int G : {4, 16, 37, 74, 148}) {
      const size_t wrap = l2 ? ((size_t)16 << 20) : bytes;
      const size_t pw = l2 ? per_warp : (bytes / ((size_t)G * 8)) / 8192 * 8192;
      for (int m = 0; m < 4; ++m) {  // 0: bulk 1 op, 1: bulk 4 ops, 2: cp.async, 3: ldg
        float ms = 0;
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(a);
          if (m < 2) ring<<<G, 256, 3 * 8192 * 8>>>(buf, pw, wrap, 0, m == 0 ? 1 : 4, sink);
          else if (m == 2) ring<<<G, 256, 3 * 8192 * 8>>>(buf, pw, wrap, 1, 1, sink);
          else ldg<<<G, 256>>>(buf, pw, wrap, sink);
          cudaEventRecord(b); cudaEventSynchronize(b);
          cudaEventElapsedTime(&ms, a, b);
        }
        const double gbs = (double)pw * G * 8 / 1e9 / (ms * 1e-3);
        const char* nm[4] = {"bulk8K", "bulk4x2K", "cp.async", "ldg.v4"};
        printf("%s G=%3d %-9s total %7.0f GB/s  per SM %6.1f GB/s  (%s)\n", l2 ? "L2 " : "HBM", G, nm[m], gbs, gbs / G,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  return 0;
}
