// HBM streaming micro-benchmark for sm_100a: which load pattern saturates HBM?
//   mode 0: per-warp ring of cp.async.bulk copies (chunk bytes, depth) — each warp streams its own range
//   mode 1: per-CTA ring, one producer lane, chunk bytes, depth — all warps wait on the stage
//   mode 2: ld.global.nc.v4 by every thread, unroll 8
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bwtest tools/bwtest.cu
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

// mode 0: every warp streams [start, start+per_warp) in chunks of `chunk` with `depth` stages
__global__ void __launch_bounds__(256, 1) warp_ring(const uint8_t* src, size_t per_warp, int chunk, int depth, int sub, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __shared__ __align__(8) uint64_t bars[8 * 16];
  const size_t gw = (size_t)blockIdx.x * nw + w;
  const uint8_t* base = src + gw * per_warp;
  uint32_t ring = smem_u32(sm) + w * depth * chunk;
  uint32_t bar0 = smem_u32(&bars[w * 16]);
  if (lane == 0) for (int s = 0; s < depth; ++s) mbar_init(bar0 + 8 * s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const int n = (int)(per_warp / chunk);
  auto issue = [&](int i) {
    int s = i % depth;
    expect_tx(bar0 + 8 * s, chunk);
    for (int k = 0; k < sub; ++k) bulk(ring + s * chunk + k * (chunk / sub), base + (size_t)i * chunk + k * (chunk / sub), chunk / sub, bar0 + 8 * s);
  };
  if (lane == 0) for (int i = 0; i < depth && i < n; ++i) issue(i);
  int acc = 0;
  for (int i = 0; i < n; ++i) {
    int s = i % depth;
    while (!try_wait(bar0 + 8 * s, (i / depth) & 1)) {}
    acc += *(volatile int*)(sm + w * depth * chunk + s * chunk + lane * 4);
    __syncwarp();
    if (lane == 0 && i + depth < n) issue(i + depth);
  }
  if (acc == 0x12345) sink[0] = acc;
}

// mode 2: plain vector loads
__global__ void __launch_bounds__(512) ldg_stream(const int4* src, size_t n16, int* sink) {
  int acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    int4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(src + i + k * stride));
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].w;
  }
  if (acc == 0x12345) sink[0] = acc;
}

int main() {
  const size_t bytes = (size_t)2 << 30;
  uint8_t* buf; int* sink;
  cudaMalloc(&buf, bytes); cudaMalloc(&sink, 4); cudaMemset(buf, 1, bytes);
  cudaFuncSetAttribute(warp_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct Cfg { int warps, chunk, depth, sub; } cfgs[] = {
    {8, 8192, 3, 4}, {8, 8192, 3, 2}, {8, 8192, 3, 1}, {8, 4096, 6, 1}, {8, 4096, 4, 1}, {8, 8192, 2, 1},
    {4, 16384, 3, 1}, {4, 16384, 3, 8}, {8, 2048, 8, 1}, {8, 16384, 1, 1}, {2, 32768, 3, 1}, {1, 65536, 3, 1},
    {8, 4096, 3, 1}, {8, 8192, 3, 4}};
  for (auto c : cfgs) {
    size_t smem = (size_t)c.warps * c.depth * c.chunk;
    if (smem > 200 * 1024) continue;
    size_t per_warp = (bytes / ((size_t)sms * c.warps)) / c.chunk * c.chunk;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      warp_ring<<<sms, c.warps * 32, smem>>>(buf, per_warp, c.chunk, c.depth, c.sub, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    double gb = (double)per_warp * sms * c.warps / 1e9;
    printf("bulk warps=%d chunk=%6d depth=%d ops/chunk=%d inflight/SM=%6zu KB : %7.0f GB/s  (err=%s)\n", c.warps, c.chunk, c.depth, c.sub, smem / 1024, gb / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
  }
  for (int threads : {256, 512}) for (int mult : {1, 2, 4, 8}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      ldg_stream<<<sms * mult, threads>>>((const int4*)buf, bytes / 16, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("ldg threads=%d blocks=%d*SM : %7.0f GB/s\n", threads, mult, bytes / 1e9 / (ms * 1e-3));
  }
  return 0;
}
