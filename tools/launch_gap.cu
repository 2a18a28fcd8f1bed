// Back-to-back launch cost of an empty 148 x 256 kernel vs its dynamic smem size
// (diagnostic: how much of a persistent kernel's event time is launch overhead).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/launch_gap tools/launch_gap.cu
#include <cstdio>
__global__ void empty_kernel(int* p) {
  extern __shared__ int sm[];
  if (p && threadIdx.x == 0 && blockIdx.x == 100000) p[0] = sm[0];
}
__global__ void spin_kernel(int* p, long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t;
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < ns);
  if (p && threadIdx.x == 0 && blockIdx.x == 100000) p[0] = 1;
}
int main() {
  cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(spin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int smems[] = {0, 48 * 1024, 100 * 1024, 200 * 1024, 227 * 1024};
  for (int rep = 0; rep < 2; ++rep)
    for (int sm : smems) {
      for (int i = 0; i < 10; ++i) empty_kernel<<<148, 256, sm>>>(nullptr);
      cudaEventRecord(a);
      for (int i = 0; i < 200; ++i) empty_kernel<<<148, 256, sm>>>(nullptr);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("empty 148x256 smem %6d B: %.2f us per launch\n", sm, ms * 1e3 / 200);
      cudaEventRecord(a);
      for (int i = 0; i < 100; ++i) spin_kernel<<<148, 256, sm>>>(nullptr, 50000);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("spin 50us 148x256 smem %6d B: %.2f us per launch (%s)\n", sm, ms * 1e3 / 100,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
