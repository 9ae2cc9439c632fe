// Thread-level + threadblock-level Stockham FFT engine for one signal held by
// TPS = N/E threads (E elements each, radix-E register butterflies, swizzled
// shared-memory exchanges between passes). Used by the single-pass kernel (K1)
// and by both halves of the two-pass four-step kernel (K3).
//
// Pass sequence: radix E repeated, then one remainder pass (radix N / E^k).
// The index contract is the reference's Stockham DIT sweep
// (_kernels_py.py:16-17): leg t of butterfly (p, q) at q + s(p + m t), output
// c at q + s(r p + c), so after any pass with cumulative radix product S the
// buffer holds the canonical stage-boundary intermediate Z_S.
#pragma once

#include "tfft_common.cuh"

namespace tfft {

__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }

template <typename T, int N_, int E_, bool INV>
struct Fft {
  static constexpr int N = N_;
  static constexpr int E = (E_ < N_) ? E_ : N_;
  static constexpr int TPS = N / E;
  static constexpr int LOGN = ilog2(N);
  static constexpr int LOGE = ilog2(E);
  static constexpr int NFULL = LOGN / LOGE;
  static constexpr int REM = N >> (NFULL * LOGE);
  static constexpr int NPASS = NFULL + (REM > 1 ? 1 : 0);
  static constexpr int RLAST = (REM > 1) ? REM : E;

  template <int P> __host__ __device__ static constexpr int radix() { return (P < NFULL) ? E : REM; }
  template <int P> __host__ __device__ static constexpr int stride() { return 1 << (P * LOGE); }

  // position index (element = tau + TPS * pos) of last-pass output register k
  static __device__ __forceinline__ constexpr int out_pos(int k) {
    return k / RLAST + (E / RLAST) * (k % RLAST);
  }

  // twiddle multiply + radix-R butterflies of pass P on the register set v
  template <int P>
  static __device__ __forceinline__ void compute(C<T> (&v)[E], int tau, const C<T>* __restrict__ tw) {
    constexpr int R = radix<P>();
    constexpr int S = stride<P>();
    constexpr int M = N / (S * R);
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
      if constexpr (S > 1) {
        const int j = tau + TPS * u;
        const int q = j & (S - 1);
#pragma unroll
        for (int t = 1; t < R; ++t) v[u * R + t] = cmul<T>(v[u * R + t], __ldg(tw + q * t * M));
      }
      dft<T, R, INV>(&v[u * R]);
    }
  }

  template <int P>
  static __device__ __forceinline__ void read(const C<T>* buf, C<T> (&v)[E], int tau, int key) {
    constexpr int R = radix<P>();
#pragma unroll
    for (int u = 0; u < E / R; ++u)
#pragma unroll
      for (int t = 0; t < R; ++t) v[u * R + t] = buf[swz<T>(tau + TPS * u + (N / R) * t) ^ key];
  }

  template <int P>
  static __device__ __forceinline__ void write(C<T>* buf, const C<T> (&v)[E], int tau, int key) {
    constexpr int R = radix<P>();
    constexpr int S = stride<P>();
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
      const int j = tau + TPS * u;
      const int q = j & (S - 1);
      const int p = j >> ilog2(S);
#pragma unroll
      for (int c = 0; c < R; ++c) buf[swz<T>(q + S * (R * p + c)) ^ key] = v[u * R + c];
    }
  }

  template <int P>
  static __device__ __forceinline__ void rest(C<T>* buf, C<T> (&v)[E], int tau, const C<T>* tw, int key) {
    if constexpr (P < NPASS) {
      __syncthreads();
      write<P - 1>(buf, v, tau, key);
      __syncthreads();
      read<P>(buf, v, tau, key);
      compute<P>(v, tau, tw);
      rest<P + 1>(buf, v, tau, tw, key);
    }
  }

  // v: legs of pass 0 (= input elements tau + TPS*k, already loaded by the
  // caller from buf's linear layout). On return v holds the outputs at
  // positions tau + TPS*out_pos(k); the last smem read is complete for this
  // thread but the caller must barrier before overwriting buf.
  // Contains NPASS-1 pairs of CTA-wide barriers: every thread must call it.
  // `key` XORs the low swizzle bits per slot (K3 packs many columns per CTA).
  static __device__ __forceinline__ void run(C<T>* buf, C<T> (&v)[E], int tau, const C<T>* tw, int key = 0) {
    compute<0>(v, tau, tw);
    rest<1>(buf, v, tau, tw, key);
  }

  // smem address of position a of a slot buffer (the swizzled layout)
  static __device__ __forceinline__ int phys(int a, int key) { return swz<T>(a) ^ key; }
};

}  // namespace tfft
