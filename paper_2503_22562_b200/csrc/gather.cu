// §8(f)2 fused all-gather: peer addresses of an NCCL symmetric window.  The only
// translation unit that includes the NCCL device API; the attention kernel itself takes
// plain per-rank address offsets (AttnParams::Gather) and needs no NCCL types.
#include <nccl.h>
#include <nccl_device.h>

#include "internal.h"

namespace niyama {

__global__ void resolve_peers_kernel(ncclWindow_t win, int world, uint64_t* out) {
  const int r = threadIdx.x;
  // world rank r -> its window copy as mapped into this process (ncclGetPeerPointer
  // translates world ranks to the window's LSA team, one NVLink node)
  if (r < world) out[r] = reinterpret_cast<uint64_t>(ncclGetPeerPointer(win, 0, r));
}

cudaError_t gather_resolve_peers(ncclWindow_vidmem* win, int world, uint64_t* host_out) {
  uint64_t* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(uint64_t) * kMaxGatherRanks);
  if (e != cudaSuccess) return e;
  resolve_peers_kernel<<<1, 32>>>(win, world, d);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(host_out, d, sizeof(uint64_t) * world, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}

}  // namespace niyama
