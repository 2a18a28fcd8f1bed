// Standalone check of the prefill Q-tile TMA load (kernels.cu prefill_stream): a 3-D tensor
// map over Q [T][Hq][128] bf16, box {64, g, R}, 128-byte swizzle, passed inside a
// __grid_constant__ parameter struct, loaded by one thread with mbarrier completion; every
// thread then checks the landed tile against the SW128 K-major layout (tile row i*g + hh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../include -I../paper_2503_22562_b200/csrc tools/tma_q_test.cu -o /tmp/tma_q_test
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#include "ptx.cuh"
using namespace niyama::ptx;

struct Params {
  int T, Hq, g, R, row0, kvh;
  uint16_t* out;  // [128 rows][128] the tile as the kernel sees it (unswizzled by address math)
  int* status;
  alignas(64) CUtensorMap map;
};

__global__ void k_test(const __grid_constant__ Params p) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  const uint32_t sbase = smem_u32(sm), b = smem_u32(&bar);
  if (threadIdx.x == 0) {
    mbar_init(b, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(b, 32768);
    tma_load_3d(sbase, &p.map, 0, p.kvh * p.g, p.row0, b);
    tma_load_3d(sbase + 16384, &p.map, 64, p.kvh * p.g, p.row0, b);
    uint32_t polls = 0;
    while (!mbar_try_wait(b, 0)) {
      if (++polls == (1u << 22)) {
        printf("TMA never completed\n");
        *p.status = 1;
        return;
      }
    }
  }
  __syncthreads();
  // thread r reads tile row r: 16-byte chunk j of panel (j>>3) at r*128 + ((j&7) ^ (r&7))*16
  const int r = threadIdx.x;
  if (r < 128) {
    for (int j = 0; j < 16; ++j) {
      const uint4 v = *reinterpret_cast<const uint4*>(sm + (j >> 3) * 16384 + r * 128 + (((j & 7) ^ (r & 7)) << 4));
      reinterpret_cast<uint4*>(p.out + r * 128)[j] = v;
    }
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  for (int g : {4, 8}) {
    const int T = 100, Hq = 8 * g, R = 128 / g;
    std::vector<uint16_t> hq(static_cast<size_t>(T) * Hq * 128);
    for (size_t i = 0; i < hq.size(); ++i) hq[i] = static_cast<uint16_t>(i * 2654435761u >> 16);
    uint16_t* dq;
    cudaMalloc(&dq, hq.size() * 2);
    cudaMemcpy(dq, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice);
    Params p{};
    p.T = T, p.Hq = Hq, p.g = g, p.R = R, p.row0 = 90, p.kvh = 3;  // rows 90..90+R-1: past T for R > 10
    cudaMalloc(&p.out, 128 * 128 * 2);
    cudaMalloc(&p.status, 4);
    cudaMemset(p.status, 0, 4);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    EncodeTiledFn enc = reinterpret_cast<EncodeTiledFn>(f);
    const cuuint64_t dims[3] = {128, static_cast<cuuint64_t>(Hq), static_cast<cuuint64_t>(T)};
    const cuuint64_t strides[2] = {256, static_cast<cuuint64_t>(Hq) * 256};
    const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(g), static_cast<cuuint32_t>(R)};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&p.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dq, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("g=%d encode: %d (query %d)\n", g, static_cast<int>(r), static_cast<int>(q));
    cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    k_test<<<1, 128, 40000>>>(p);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<uint16_t> out(128 * 128);
    int st = 0;
    cudaMemcpy(out.data(), p.out, out.size() * 2, cudaMemcpyDeviceToHost);
    cudaMemcpy(&st, p.status, 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int row = 0; row < 128; ++row) {
      const int i = row / g, hh = row % g;
      const int trow = p.row0 + i, h = p.kvh * g + hh;
      for (int e2 = 0; e2 < 128; ++e2) {
        const uint16_t want = trow < T ? hq[(static_cast<size_t>(trow) * Hq + h) * 128 + e2] : 0;
        if (out[row * 128 + e2] != want) ++bad;
      }
    }
    printf("g=%d status %d mismatches %d of %d\n", g, st, bad, 128 * 128);
  }
  return 0;
}
