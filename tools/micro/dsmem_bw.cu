// DSMEM bandwidth microbenchmark (B200): clusters of C CTAs (one per SM); each
// CTA pushes `bytes` from its shared memory into the next CTA's shared memory
// with cp.async.bulk.shared::cluster.shared::cta, completion counted on the
// receiver's mbarrier, `iters` times. Prints aggregate GB/s per SM.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int C>
__global__ void __cluster_dims__(C, 1, 1) push_kernel(int bytes, int iters, unsigned long long* cycles) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  unsigned char* src = sm;
  unsigned char* dst = sm + bytes;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cl.sync();
  const unsigned next = (rank + 1) % C;
  // remote addresses of the next CTA's dst buffer and mbarrier
  uint32_t rdst, rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(su32(dst)), "r"(next));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(su32(&bar)), "r"(next));
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes));
    }
    cl.sync();  // every receiver armed before anyone sends
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(rdst), "r"(su32(src)), "r"(bytes), "r"(rbar) : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(su32(&bar)), "r"(it & 1));
    }
    __syncthreads();
  }
  cl.sync();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

int main() {
  const int bytes = 64 * 1024, iters = 200;
  unsigned long long* d;
  cudaMalloc(&d, 1024 * sizeof(unsigned long long));
  auto run = [&](auto kern, int C) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * bytes);
    const int grid = (148 / C) * C;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<grid, 128, 2 * bytes>>>(bytes, 10, d);
    cudaEventRecord(a);
    kern<<<grid, 128, 2 * bytes>>>(bytes, iters, d);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double per_sm = (double)bytes * iters / (ms / 1e3) / 1e9;
    printf("cluster %d grid %d: %s, %.3f ms, %.1f GB/s per SM received, %.2f TB/s aggregate\n", C, grid,
           cudaGetErrorString(e), ms, per_sm, per_sm * grid / 1e3);
  };
  run(push_kernel<2>, 2);
  run(push_kernel<4>, 4);
  run(push_kernel<8>, 8);
  return 0;
}
