// Microbenchmark for the (f)1 design question: can window sums be accumulated
// with L2 reductions at HBM speed? 1 GiB of FP32 complex signals (N = 2^16,
// B = 2048) read once; variant 0: plain read + register sum (HBM floor);
// variant 1: red.global.add.v2.f32 of every element into its window's sum
// (W = 16 signals per window, coalesced, p-major like K7's ring).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bw red_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const float2* __restrict__ x, long long n, float* out) {
  float a = 0.f, b = 0.f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float2 v = __ldcs(x + i);
    a += v.x;
    b += v.y;
  }
  if (a + b == 1234.5f) out[0] = a;
}

__global__ void red(const float2* __restrict__ x, long long n, int N, int W, float2* s) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float2 v = __ldcs(x + i);
    const long long sig = i / N, k = i % N;
    float2* d = s + (sig / W) * N + k;
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(d), "f"(v.x), "f"(v.y) : "memory");
  }
}

int main() {
  const int N = 1 << 16, B = 2048, W = 16;
  const long long n = (long long)N * B;
  float2 *x, *s;
  float* o;
  cudaMalloc(&x, n * sizeof(float2));
  cudaMalloc(&s, (long long)(B / W) * N * sizeof(float2));
  cudaMalloc(&o, 4);
  cudaMemset(x, 0, n * sizeof(float2));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int nsm = 148;
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemset(s, 0, (long long)(B / W) * N * sizeof(float2));
      cudaEventRecord(a);
      if (v == 0) rd<<<nsm * 8, 256>>>(x, n, o);
      else red<<<nsm * 8, 256>>>(x, n, N, W, s);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 3) printf("%s: %.3f ms, %.1f GB/s of input\n", v ? "red.v2.f32 window sums" : "plain read", ms,
                           n * 8 / ms / 1e6);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
