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

// TWG tables hold only the rows load_tw reads (1 = compact; 0 = every power)
#ifndef TFFT_TW_COMPACT
#define TFFT_TW_COMPACT 1
#endif

namespace tfft {

__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }

// CTA-wide barrier (BAR_THREADS == 0) or a named barrier (id 1) over the
// first BAR_THREADS threads, for warp-specialised kernels whose producer warp
// does not take part in the exchanges.
template <int BAR_THREADS>
__device__ __forceinline__ void fft_sync() {
  if constexpr (BAR_THREADS == 0) __syncthreads();
  else asm volatile("bar.sync 1, %0;" ::"n"(BAR_THREADS) : "memory");
}

// Exchange synchronisation of one signal's TPS threads. BAR_THREADS >= 0: as
// fft_sync. BAR_THREADS == -1 ("group" mode, tau-fastest thread maps): a
// signal whose threads fit in one warp syncs with __syncwarp; a wider one
// uses named barrier `bar_id` over its own TPS threads only, so signals (and
// warps) of one CTA never wait for each other.
template <int BAR_THREADS, int TPS>
__device__ __forceinline__ void fft_sync_grp(int bar_id) {
  if constexpr (BAR_THREADS >= 0) fft_sync<BAR_THREADS>();
  else if constexpr (TPS <= 32) __syncwarp();
  else asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(TPS) : "memory");
}

// PF: issue the next pass's twiddle loads before the exchange barriers so their
// L1/L2 latency hides behind the shared-memory round trip (costs E registers).
// TWS: where the twiddles come from.
//   false: the global w_N table (tw[m] = w_N^m), read through the read-only path;
//   true : per-pass tables in shared memory built by build_pass_tables():
//          pass P's block holds w_{S R}^{q t} at (t - 1) * S + q, q fastest, so
//          the lanes of a warp (consecutive q) read consecutive words: no bank
//          conflicts, unlike strided reads of a w_N copy (up to 8-way).
// TWG (with TWS): per leg group, load only w^1 (and w^4, w^8, w^12 at radix
//          8/16) of a pass's table and form the other powers by one or two
//          complex products: 4 instead of 15 shared-memory twiddle reads per
//          radix-16 group, for kernels whose shared-memory pipe is the limiter.
template <typename T, int N_, int E_, bool INV, bool PF = false, int BAR_THREADS = 0, bool TWS = false,
          bool TWG = false>
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

  // Padded shared-memory layout: one spare slot after every 16 elements, so
  // Stockham scatter writes (consecutive threads 16 + 1 elements apart after a
  // radix-16 pass) and strided reads hit distinct banks for both 8-byte and
  // 16-byte elements; offsets that are multiples of 16 fold into compile-time
  // constants (the XOR swizzle cost ~20% integer ops).
  static constexpr int LOGP = 4;
  static constexpr int NPAD = N + (N >> LOGP);  // elements a slot buffer occupies
  static __device__ __forceinline__ int phys(int a) { return a + (a >> LOGP); }

  // rows of pass P's block: every power t = 1..R-1, or with TWG only the
  // powers load_tw reads (t = 1, 4, 8, 12 for radix 16; 1, 4 for 8; 1 below)
  static constexpr bool CMP = TWG && TWS && TFFT_TW_COMPACT;
  template <int R>
  __host__ __device__ static constexpr int nrows() {
    return !CMP ? R - 1 : (R >= 16 ? 4 : (R >= 8 ? 2 : 1));
  }
  // table row ri holds the power t = row_pow(ri)
  __host__ __device__ static constexpr int row_pow(int ri) { return CMP ? (ri == 0 ? 1 : 4 * ri) : ri + 1; }

  // offset of pass P's block in the per-pass table: sum over earlier passes
  // P' >= 1 of rows(R') S' (= S_P - E for P >= 1 without TWG); PASS_TABLE
  // entries in all
  template <int P>
  __host__ __device__ static constexpr int pass_off() {
    if constexpr (P <= 1) return 0;
    else return pass_off<P - 1>() + nrows<radix<P - 1>()>() * stride<P - 1>();
  }
  static constexpr int PASS_TABLE = NPASS > 1 ? pass_off<NPASS>() : 0;

  // per-pass twiddle tables from the global w_N table (direction included),
  // cooperatively by threads [tid0, tid0 + nthr)
  static __device__ __forceinline__ void build_pass_tables(C<T>* dst, const C<T>* __restrict__ wn, int tid,
                                                           int nthr) {
    build_from<1>(dst, wn, tid, nthr);
  }
  template <int P>
  static __device__ __forceinline__ void build_from(C<T>* dst, const C<T>* __restrict__ wn, int tid, int nthr) {
    if constexpr (P < NPASS) {
      constexpr int R = radix<P>();
      constexpr int S = stride<P>();
      constexpr int M = N / (S * R);
      for (int i = tid; i < nrows<R>() * S; i += nthr) {
        const int t = row_pow(i / S), q = i % S;
        dst[pass_off<P>() + i] = wn[q * t * M];
      }
      build_from<P + 1>(dst, wn, tid, nthr);
    }
  }

  template <int P>
  static __device__ __forceinline__ void load_tw(C<T> (&w)[E], int tau, const C<T>* __restrict__ tw) {
    constexpr int R = radix<P>();
    constexpr int S = stride<P>();
    constexpr int M = N / (S * R);
    if constexpr (S > 1) {
#pragma unroll
      for (int u = 0; u < E / R; ++u) {
        const int q = (tau + TPS * u) & (S - 1);
        if constexpr (TWG && TWS && R >= 4) {
          // w^1, w^4, w^8, w^12 at b[0], b[S], b[2S], b[3S] (compact) or b[(t - 1) S]
          const C<T>* b = tw + pass_off<P>() + q;
          constexpr int S4 = CMP ? S : 3 * S, S8 = CMP ? 2 * S : 7 * S, S12 = CMP ? 3 * S : 11 * S;
          w[u * R + 1] = b[0];
          w[u * R + 2] = cmul<T>(w[u * R + 1], w[u * R + 1]);
          w[u * R + 3] = cmul<T>(w[u * R + 2], w[u * R + 1]);
          if constexpr (R >= 8) {
            w[u * R + 4] = b[S4];
#pragma unroll
            for (int t = 1; t < 4; ++t) w[u * R + 4 + t] = cmul<T>(w[u * R + 4], w[u * R + t]);
          }
          if constexpr (R == 16) {
            w[u * R + 8] = b[S8];
            w[u * R + 12] = b[S12];
#pragma unroll
            for (int t = 1; t < 4; ++t) {
              w[u * R + 8 + t] = cmul<T>(w[u * R + 8], w[u * R + t]);
              w[u * R + 12 + t] = cmul<T>(w[u * R + 12], w[u * R + t]);
            }
          }
          continue;
        }
#pragma unroll
        for (int t = 1; t < R; ++t) {
          if constexpr (TWS) w[u * R + t] = tw[pass_off<P>() + (t - 1) * S + q];
          else w[u * R + t] = __ldg(tw + q * t * M);
        }
      }
    }
  }

  // twiddle multiply (from w) + radix-R butterflies of pass P
  template <int P>
  static __device__ __forceinline__ void apply(C<T> (&v)[E], const C<T> (&w)[E]) {
    constexpr int R = radix<P>();
    constexpr int S = stride<P>();
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
      if constexpr (S > 1) {
#pragma unroll
        for (int t = 1; t < R; ++t) v[u * R + t] = cmul<T>(v[u * R + t], w[u * R + t]);
      }
      dft<T, R, INV>(&v[u * R]);
    }
  }

  template <int P>
  static __device__ __forceinline__ void compute(C<T> (&v)[E], int tau, const C<T>* __restrict__ tw) {
    C<T> w[E];
    load_tw<P>(w, tau, tw);
    apply<P>(v, w);
  }

  template <int P>
  static __device__ __forceinline__ void read(const C<T>* buf, C<T> (&v)[E], int tau) {
    constexpr int R = radix<P>();
#pragma unroll
    for (int u = 0; u < E / R; ++u)
#pragma unroll
      for (int t = 0; t < R; ++t) v[u * R + t] = buf[phys(tau + TPS * u + (N / R) * t)];
  }

  template <int P>
  static __device__ __forceinline__ void write(C<T>* buf, const C<T> (&v)[E], int tau) {
    constexpr int R = radix<P>();
    constexpr int S = stride<P>();
#pragma unroll
    for (int u = 0; u < E / R; ++u) {
      const int j = tau + TPS * u;
      const int q = j & (S - 1);
      const int p = j >> ilog2(S);
#pragma unroll
      for (int c = 0; c < R; ++c) buf[phys(q + S * (R * p + c))] = v[u * R + c];
    }
  }

  template <int P>
  static __device__ __forceinline__ void rest(C<T>* buf, C<T> (&v)[E], int tau, const C<T>* tw, int bar_id) {
    if constexpr (P < NPASS) {
      C<T> w[E];
      if constexpr (PF) load_tw<P>(w, tau, tw);
      fft_sync_grp<BAR_THREADS, TPS>(bar_id);
      write<P - 1>(buf, v, tau);
      fft_sync_grp<BAR_THREADS, TPS>(bar_id);
      read<P>(buf, v, tau);
      if constexpr (!PF) load_tw<P>(w, tau, tw);
      apply<P>(v, w);
      rest<P + 1>(buf, v, tau, tw, bar_id);
    }
  }

  // v: legs of pass 0 (= input elements tau + TPS*k, loaded by the caller).
  // On return v holds the outputs at positions tau + TPS*out_pos(k); the last
  // smem read is complete for this thread but the caller must barrier before
  // overwriting buf. Contains NPASS-1 pairs of CTA-wide barriers: every thread
  // must call it. buf spans NPAD elements (padded layout).
  // bar_id: the named barrier of this signal's thread group in group mode
  static __device__ __forceinline__ void run(C<T>* buf, C<T> (&v)[E], int tau, const C<T>* tw, int bar_id = 1) {
    compute<0>(v, tau, tw);
    rest<1>(buf, v, tau, tw, bar_id);
  }
};

}  // namespace tfft
