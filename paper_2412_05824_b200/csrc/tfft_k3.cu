// K3: two-pass (four-step) batched FFT for 2^13 < N <= 2^22 (FP32 from 2^14).
//
// N = N1 x N2 with N1 = the reference plan's first stage span (fft_core.py
// stage boundaries), so the pass-A output IS the canonical stage-1
// intermediate Z[p][q] = sum_v x[p + N2 v] w_N1^{qv}, stored
// at q + N1 p; stage-1 strikes flip it in registers before the w_N^{pq}
// twiddle, exactly where the reference's injector fires.
//
//   pass A: for each signal and each block of CB consecutive columns p, load
//           the N1 x CB tile (CB contiguous elements per row v: coalesced),
//           N1-point FFTs in shared memory (one padded column slot each, with a
//           per-column skew against bank conflicts), twiddle w_N^{pq}, store
//           rows of Z contiguously.
//   pass B: for each block of CB consecutive q, load the N2 x CB tile of Z,
//           N2-point FFTs, transpose through shared memory, store
//           y[q + N1 k] in CB-contiguous runs.
//
// Both passes are one persistent kernel launch each; the engine (tfft_fft.cuh)
// is the same one K1 uses.
#include <cmath>
#include <vector>

#include "tfft_fft.cuh"
#include "tfft_internal.h"
#include "tfft_k3.h"
#include "tfft_k4.h"
#include <cstdlib>
#include "tfft_aux.h"

namespace tfft {

template <typename T, int LOGL>
struct ColCfg {
  static constexpr int L = 1 << LOGL;
  static constexpr int EMAX = 16;
  static constexpr int E = EMAX < L ? EMAX : L;
  static constexpr int TPS = L / E;
  static constexpr int BPC = (int)sizeof(C<T>);
  static constexpr int CB0 = 65536 / (L * BPC);
  static constexpr int CB = CB0 < 2 ? 2 : (CB0 > 32 ? 32 : CB0);
  static constexpr int NT = CB * TPS;
  // bank-row slots (16 float2 / 8 double2 per 128 B); each column slot is the
  // engine's padded buffer plus room for a per-column skew that spreads the
  // rows one shared-memory phase of the transposing loader touches
  static constexpr int PB = sizeof(T) == 4 ? 16 : 8;
  static constexpr int NPAD = L + L / PB;
  static constexpr int SLOTP = NPAD + PB;
  static constexpr int RPP = PB / CB > 1 ? PB / CB : 1;
  static __device__ __forceinline__ int base(int c) { return c * SLOTP + ((c * RPP) & (PB - 1)); }
  static constexpr int TILE = CB * SLOTP;
  static constexpr int SMEM = TILE * BPC;
};

struct ColArgs {
  const void* src;
  void* dst;
  int64_t batch;
  int64_t n;        // full transform length N
  int64_t pitch;    // row pitch (elements) of the src matrix view
  int64_t ncols;    // columns of the view (N / L)
  int64_t n1;       // N1 (output stride of pass B, layout of Z)
  const void* tw;   // omega_L^m (conj for inverse), L entries
  const void* hi;   // omega_N^{h * 2^lo_bits}
  const void* lo;   // omega_N^{l}
  int lo_bits;
  const DevFault* faults;
  int nfaults;
  int strike_stage; // stage index whose boundary pass A's output is (1), or -1
  Counters* counters;
  // MODE 2 (one reference stage as one radix-L Stockham pass):
  int64_t s;        // S = product of the earlier stages' spans (1 for stage 0)
  int stage;        // stage index: strikes with this stage flip the loaded legs
  int last;         // last stage (inverse: x 1/N)
};

// stage passes: two CTAs per SM (TFFT_COL2_MINB=2) spill and measured 15-20% slower
#ifndef TFFT_COL2_MINB
#define TFFT_COL2_MINB 1
#endif
template <typename T, int LOGL, bool INV, int MODE>
__global__ void __launch_bounds__(ColCfg<T, LOGL>::NT, MODE == 2 ? TFFT_COL2_MINB : 1) col_kernel(ColArgs a) {
  using K = ColCfg<T, LOGL>;
  using F = Fft<T, K::L, K::EMAX, INV>;
  using CT = C<T>;
  constexpr int L = K::L, E = K::E, TPS = K::TPS, CB = K::CB, NT = K::NT;
  extern __shared__ __align__(128) unsigned char smem[];
  CT* tile = reinterpret_cast<CT*>(smem);

  const int tid = threadIdx.x;
  const int g = tid / TPS;
  const int tau = tid % TPS;
  CT* slot = tile + K::base(g);
  const CT* __restrict__ src = static_cast<const CT*>(a.src);
  CT* __restrict__ dst = static_cast<CT*>(a.dst);
  const CT* __restrict__ tw = static_cast<const CT*>(a.tw);
  const int64_t ncb = a.ncols / CB;
  const int64_t ntiles = a.batch * ncb;
  bool bad = false;

  // the L x CB tile (rows contiguous in global): element e = i*NT + tid is
  // row e / CB, column e % CB. Loads for tile t+grid are issued before tile
  // t's FFT so their HBM latency hides behind the shared-memory passes.
  CT ld[E];
  auto issue = [&](int64_t t) {
    const int64_t sg = t / ncb;
    const CT* s = src + sg * a.n + (t - sg * ncb) * CB;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int e = i * NT + tid;
      ld[i] = __ldcs(s + (int64_t)(e / CB) * a.pitch + e % CB);
    }
  };
  if (blockIdx.x < ntiles) issue(blockIdx.x);

#pragma unroll 1
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t sig = t / ncb;
    const int64_t c0 = (t - sig * ncb) * CB;
    if constexpr (MODE == 0 || MODE == 2) {
      if (MODE == 0 || a.stage == 0) {
#pragma unroll
        for (int i = 0; i < E; ++i) bad |= !finite2<T>(ld[i]);
      }
      if (a.nfaults > 0) {
        const int st = MODE == 0 ? 0 : a.stage;
        for (int f = fault_lo(a.faults, a.nfaults, sig); f < a.nfaults && a.faults[f].signal == sig; ++f) {
          const DevFault fl = a.faults[f];
          if (fl.signal != sig || fl.stage != st) continue;
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const int e = i * NT + tid;
            if (c0 + e % CB + (int64_t)(e / CB) * a.pitch == fl.element) {
              if (fl.part == 0) ld[i].x = flip_bits(ld[i].x, fl.bit);
              else ld[i].y = flip_bits(ld[i].y, fl.bit);
            }
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int e = i * NT + tid;
      tile[K::base(e % CB) + F::phys(e / CB)] = ld[i];
    }
    __syncthreads();
    if (t + gridDim.x < ntiles) issue(t + gridDim.x);
    // ---- column FFTs
    CT v[E];
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = slot[F::phys(tau + TPS * k)];
    if constexpr (MODE == 2) {
      // DIT Stockham stage: leg t of column j = q + S p' times w_{S L}^{q t}
      // (= w_N^{q t N / (S L)}, two-level table), then the L-point DFT
      if (a.s > 1) {
        // w_N^{m}, m = q t N / (S L), t = tau + TPS k: the base (t = tau) and
        // the step (TPS) from the two-level table, then E - 1 products (as
        // K4's pass A) instead of two table loads per leg
        const CT* __restrict__ hi = static_cast<const CT*>(a.hi);
        const CT* __restrict__ lo = static_cast<const CT*>(a.lo);
        const int64_t lomask = (int64_t(1) << a.lo_bits) - 1;
        const int64_t q = (c0 + g) & (a.s - 1);
        const int64_t scale = a.n / (a.s * L);
        const int64_t mb = (q * (int64_t)tau * scale) & (a.n - 1);
        const int64_t ms = (q * (int64_t)TPS * scale) & (a.n - 1);
        TwRun<T> w(cmul<T>(__ldg(hi + (mb >> a.lo_bits)), __ldg(lo + (mb & lomask))),
                   cmul<T>(__ldg(hi + (ms >> a.lo_bits)), __ldg(lo + (ms & lomask))));
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = cmul<T>(v[k], w.next(k));
      }
    }
    F::run(slot, v, tau, tw);
    if constexpr (MODE == 2) {
      const bool scl = INV && a.last;
      const T sc = (T)(1.0 / (double)a.n);
      if (a.s == 1) {
        // stage 0: column j's L outputs are contiguous at j L + c
        CT* d = dst + sig * a.n + (c0 + g) * L;
#pragma unroll
        for (int k = 0; k < E; ++k) __stcs(d + tau + TPS * F::out_pos(k), scl ? cscale<T>(v[k], sc) : v[k]);
        __syncthreads();  // tile reuse by the next load
      } else {
        // S >= CB: the tile is one p', q = q0 .. q0 + CB - 1; output c of
        // column q at q + S (L p' + c): L rows of CB contiguous, pitch S
        __syncthreads();
#pragma unroll
        for (int k = 0; k < E; ++k) slot[F::phys(tau + TPS * F::out_pos(k))] = v[k];
        __syncthreads();
        const int64_t q0 = c0 & (a.s - 1), p0 = c0 / a.s;
        CT* d = dst + sig * a.n + q0 + a.s * L * p0;
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int e = i * NT + tid;
          const int r = e / CB, c = e % CB;
          const CT val = tile[K::base(c) + F::phys(r)];
          __stcs(d + (int64_t)r * a.s + c, scl ? cscale<T>(val, sc) : val);
        }
        __syncthreads();
      }
    } else if constexpr (MODE == 0) {
      // twiddle w_N^{p q} (two-level table) and store Z[p][q] at q + N1 p
      const int64_t p = c0 + g;
      const CT* __restrict__ hi = static_cast<const CT*>(a.hi);
      const CT* __restrict__ lo = static_cast<const CT*>(a.lo);
      const int64_t lomask = (int64_t(1) << a.lo_bits) - 1;
      CT* d = dst + sig * a.n + p * L;
      const int f1 = (a.nfaults > 0 && a.strike_stage == 1) ? fault_lo(a.faults, a.nfaults, sig) : 0;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int q = tau + TPS * F::out_pos(k);
        if (a.nfaults > 0 && a.strike_stage == 1) {
          for (int f = f1; f < a.nfaults && a.faults[f].signal == sig; ++f) {
            const DevFault fl = a.faults[f];
            if (fl.signal == sig && fl.stage == 1 && fl.element == q + p * L) {
              if (fl.part == 0) v[k].x = flip_bits(v[k].x, fl.bit);
              else v[k].y = flip_bits(v[k].y, fl.bit);
            }
          }
        }
        const int64_t m = p * (int64_t)q;
        const CT w = cmul<T>(__ldg(hi + (m >> a.lo_bits)), __ldg(lo + (m & lomask)));
        d[q] = cmul<T>(v[k], w);
      }
      __syncthreads();  // tile reuse by the next load
    } else {
      // transpose through the tile, then y[q + N1 k] in CB-contiguous runs
      __syncthreads();
#pragma unroll
      for (int k = 0; k < E; ++k) slot[F::phys(tau + TPS * F::out_pos(k))] = v[k];
      __syncthreads();
      CT* d = dst + sig * a.n + c0;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int e = i * NT + tid;
        const int r = e / CB, c = e % CB;
        CT val = tile[K::base(c) + F::phys(r)];
        if constexpr (INV) val = cscale<T>(val, (T)(1.0 / (double)a.n));
        __stcs(d + (int64_t)r * a.n1 + c, val);
      }
      __syncthreads();
    }
  }
  if constexpr (MODE == 0 || MODE == 2) {
    if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0 && a.counters) atomicOr(&a.counters->nonfinite, 1ull);
  }
}

template <typename T, int LOGL, bool INV, int MODE>
static int launch_col(const ColArgs& a, int num_sms, cudaStream_t st) {
  using K = ColCfg<T, LOGL>;
  auto kern = col_kernel<T, LOGL, INV, MODE>;
  static LaunchCfg cfg;
  const int dev = current_device();
  if (!cfg.done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
    if (e != cudaSuccess) return (int)e;
    cfg.done[dev] = true;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K::NT, K::SMEM);
  if (e != cudaSuccess) return (int)e;
  if (per_sm < 1) per_sm = 1;
  const int64_t ntiles = a.batch * (a.ncols / K::CB);
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > ntiles) grid = ntiles;
  if (grid < 1) return 0;
  kern<<<(unsigned)grid, K::NT, K::SMEM, st>>>(a);
  return (int)cudaGetLastError();
}

template <typename T, bool INV, int MODE>
static int dispatch_col(int logl, const ColArgs& a, int num_sms, cudaStream_t st) {
  switch (logl) {
#define TFFT_COL(L) \
  case L: return launch_col<T, L, INV, MODE>(a, num_sms, st);
    TFFT_COL(6) TFFT_COL(7) TFFT_COL(8) TFFT_COL(9) TFFT_COL(10) TFFT_COL(11)
#undef TFFT_COL
    default:
      return (int)cudaErrorInvalidValue;
  }
}

static int col(int prec, bool inv, int mode, int logl, const ColArgs& a, int num_sms, cudaStream_t st) {
  if (mode == 2) {
    if (prec == 0)
      return inv ? dispatch_col<float, true, 2>(logl, a, num_sms, st) : dispatch_col<float, false, 2>(logl, a, num_sms, st);
    return inv ? dispatch_col<double, true, 2>(logl, a, num_sms, st) : dispatch_col<double, false, 2>(logl, a, num_sms, st);
  }
  if (prec == 0) {
    if (mode == 0) return inv ? dispatch_col<float, true, 0>(logl, a, num_sms, st) : dispatch_col<float, false, 0>(logl, a, num_sms, st);
    return inv ? dispatch_col<float, true, 1>(logl, a, num_sms, st) : dispatch_col<float, false, 1>(logl, a, num_sms, st);
  }
  if (mode == 0) return inv ? dispatch_col<double, true, 0>(logl, a, num_sms, st) : dispatch_col<double, false, 0>(logl, a, num_sms, st);
  return inv ? dispatch_col<double, true, 1>(logl, a, num_sms, st) : dispatch_col<double, false, 1>(logl, a, num_sms, st);
}

// ---------------------------------------------------------------------------
// plan: tables + intermediate workspace

struct K3Plan {
  int64_t n = 0;
  int prec = 0;
  int l1 = 0, l2 = 0;  // log2 N1, log2 N2
  int lo_bits = 0;
  bool stage1 = false;
  int num_sms = 148;
  void* tw1[2] = {nullptr, nullptr};
  void* tw2[2] = {nullptr, nullptr};
  void* hi[2] = {nullptr, nullptr};
  void* lo[2] = {nullptr, nullptr};
  void* enc[2] = {nullptr, nullptr};
  void* inter = nullptr;
  size_t inter_cap = 0;
  bool k4 = false;       // fused L2-ring kernel available for this split
  void* ring = nullptr;  // K4 intermediate ring (3 group slots)
  size_t ring_cap = 0;
  void* sync = nullptr;  // K4 ticket + per-group completion counters
  size_t sync_cap = 0;
};

namespace {

// omega_M^{k * step} for k < count, extended precision, rounded once
int upload_table(int prec, int64_t M, int64_t step, int64_t count, bool conj, void** out) {
  const long double two_pi = 6.283185307179586476925286766559005768L;
  const size_t cb = prec == 0 ? 8 : 16;
  std::vector<unsigned char> host(count * cb);
  for (int64_t k = 0; k < count; ++k) {
    const int64_t m = (k * step) % M;
    const long double ang = two_pi * (long double)m / (long double)M;
    long double re = cosl(ang), im = -sinl(ang);
    if (4 * m == M) { re = 0; im = -1; }
    if (2 * m == M) { re = -1; im = 0; }
    if (4 * m == 3 * M) { re = 0; im = 1; }
    if (m == 0) { re = 1; im = 0; }
    if (conj) im = -im;
    if (prec == 0) {
      float* f = (float*)host.data();
      f[2 * k] = (float)re;
      f[2 * k + 1] = (float)im;
    } else {
      double* d = (double*)host.data();
      d[2 * k] = (double)re;
      d[2 * k + 1] = (double)im;
    }
  }
  cudaError_t e = cudaMalloc(out, host.size());
  if (e != cudaSuccess) return (int)e;
  return (int)cudaMemcpy(*out, host.data(), host.size(), cudaMemcpyHostToDevice);
}

int ilog2i(int64_t v) {
  int r = 0;
  while ((int64_t(1) << r) < v) ++r;
  return r;
}

}  // namespace

// ---------------------------------------------------------------------------
// Fused two-sided ABFT over the stage passes (abft.py:648-665, :592-624).
// The first and the last stage walk items (window w, column block): the CB
// columns of every signal of the window in turn, then one pseudo-signal.
//  first stage (PH 0): c_in = row . x and ||x||^2 partials from the loaded
//    legs (the row slice is read once per item), s_in += w_j x_j in
//    registers; after the window's signals the pseudo-signal s_in gets the
//    same stage pass, written to its own buffer -- so the later stages carry
//    FFT(s_in) along at 1/W extra work instead of a separate window FFT;
//  last stage (PH 2): c_out partials and s_out += w_j y_j from the outputs;
//    the pseudo-signal's output IS FFT(s_in), compared in place with s_out
//    (group-divergence partials). x and y are read / written exactly once.
struct StageAbft {
  int64_t win;         // W = T * bs signals per window
  int64_t nwin;
  int64_t weight0;     // global index of row 0
  const void* row;     // left checksum row
  int enc;             // ENC_WANG / ENC_ONES
  void* pseudo_dst;    // [nwin][N] (PH 0 output of the pseudo-signals)
  const void* pseudo_src;  // [nwin][N] (PH 2 input)
  double* sig_part;    // [B][P][5]: PH 0 fills 0..2, PH 2 fills 3..4 (zeroed)
  int64_t parts;       // P
  double* gpart;       // [nwin][ncb * NW][2] (PH 2)
};

template <typename T, int LOGL, int PH>
__global__ void __launch_bounds__(ColCfg<T, LOGL>::NT) stage_abft_kernel(ColArgs a, StageAbft b) {
  using K = ColCfg<T, LOGL>;
  using F = Fft<T, K::L, K::EMAX, false>;
  using CT = C<T>;
  constexpr int L = K::L, E = K::E, TPS = K::TPS, CB = K::CB, NT = K::NT, NW = NT / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  CT* tile = reinterpret_cast<CT*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int g = tid / TPS;
  const int tau = tid % TPS;
  CT* slot = tile + K::base(g);
  const CT* __restrict__ src = static_cast<const CT*>(a.src);
  CT* __restrict__ dst = static_cast<CT*>(a.dst);
  const CT* __restrict__ tw = static_cast<const CT*>(a.tw);
  const int64_t ncb = a.ncols / CB;
  const int64_t nitems = b.nwin * ncb;
  bool bad = false;
  CT ld[E];
  // one sub-tile: signal sig (pseudo when sig >= batch) of column block c0
  auto issue = [&](const CT* base) {
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int e = i * NT + tid;
      ld[i] = __ldcs(base + (int64_t)(e / CB) * a.pitch + e % CB);
    }
  };
  auto land = [&]() {
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int e = i * NT + tid;
      tile[K::base(e % CB) + F::phys(e / CB)] = ld[i];
    }
    __syncthreads();
  };
  auto warp_sum = [&](T v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = radd(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
  };

  // the first load of item `it` (its window's first signal)
  auto item_base = [&](int64_t it) {
    const int64_t w = it / ncb, cb = it % ncb;
    return src + (w * b.win) * a.n + cb * CB;
  };
  if ((int64_t)blockIdx.x < nitems) issue(item_base(blockIdx.x));
#pragma unroll 1
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int64_t w = it / ncb, cb = it % ncb;
    const int64_t c0 = cb * CB;
    const int64_t w0 = w * b.win, w1 = min(w0 + b.win, a.batch);
    const int64_t col = c0 + g;
    const int64_t itn = it + gridDim.x;  // the next item: its first load is issued during this one's last sub-tile
    CT acc[E];
#pragma unroll
    for (int k = 0; k < E; ++k) acc[k] = mk<T>(0, 0);
    CT rw[E];
    if constexpr (PH == 0) {
      const CT* __restrict__ row = static_cast<const CT*>(b.row);
#pragma unroll
      for (int k = 0; k < E; ++k) rw[k] = __ldg(row + col + (int64_t)(tau + TPS * k) * a.pitch);
    }
    // twiddle base / step of this column (last stage, S > 1): w_N^{q t N / (S L)}
    CT tw0 = mk<T>(1, 0), tstep = mk<T>(1, 0);
    if constexpr (PH == 2) {
      const CT* __restrict__ hi = static_cast<const CT*>(a.hi);
      const CT* __restrict__ lo = static_cast<const CT*>(a.lo);
      const int64_t lomask = (int64_t(1) << a.lo_bits) - 1;
      const int64_t q = col & (a.s - 1);
      const int64_t scale = a.n / (a.s * L);
      const int64_t mb = (q * (int64_t)tau * scale) & (a.n - 1);
      const int64_t ms = (q * (int64_t)TPS * scale) & (a.n - 1);
      tw0 = cmul<T>(__ldg(hi + (mb >> a.lo_bits)), __ldg(lo + (mb & lomask)));
      tstep = cmul<T>(__ldg(hi + (ms >> a.lo_bits)), __ldg(lo + (ms & lomask)));
    }
#pragma unroll 1
    for (int64_t j = w0; j <= w1; ++j) {  // j == w1: the window's pseudo-signal
      const bool pseudo = j == w1;
      if (PH == 0 && pseudo) {
        __syncthreads();  // the slots' last readers are done
      } else {
        land();
      }
      // next sub-tile's loads in flight during this one's passes (across items)
      if (j + 1 < w1) issue(src + (j + 1) * a.n + c0);
      else if (PH == 2 && j + 1 == w1) issue(static_cast<const CT*>(b.pseudo_src) + w * a.n + c0);
      else if (((PH == 0 && j + 1 == w1) || (PH == 2 && pseudo)) && itn < nitems) issue(item_base(itn));
      CT v[E];
      if (PH == 0 && pseudo) {
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = acc[k];
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = slot[F::phys(tau + TPS * k)];
      }
      const T wj = (T)(b.weight0 + j + 1);
      if constexpr (PH == 0) {
        if (!pseudo) {
          // c_in, ||x||^2 and s_in from the clean legs, then the strikes
          T r5[3] = {0, 0, 0};
#pragma unroll
          for (int k = 0; k < E; ++k) {
            bad |= !finite2<T>(v[k]);
            r5[0] = rfma(rw[k].x, v[k].x, rfma(-rw[k].y, v[k].y, r5[0]));
            r5[1] = rfma(rw[k].x, v[k].y, rfma(rw[k].y, v[k].x, r5[1]));
            r5[2] = rfma(v[k].x, v[k].x, rfma(v[k].y, v[k].y, r5[2]));
            acc[k] = mk<T>(rfma(wj, v[k].x, acc[k].x), rfma(wj, v[k].y, acc[k].y));
          }
#pragma unroll
          for (int q = 0; q < 3; ++q) r5[q] = warp_sum(r5[q]);
          if (lane == 0) {
            double* dp = b.sig_part + (j * b.parts + cb * NW + wp) * 5;
#pragma unroll
            for (int q = 0; q < 3; ++q) dp[q] = (double)r5[q];
          }
        }
      }
      if (!pseudo && a.nfaults > 0) {  // this stage's strikes on the canonical intermediate
        for (int f = fault_lo(a.faults, a.nfaults, j); f < a.nfaults && a.faults[f].signal == j; ++f) {
          const DevFault fl = a.faults[f];
          if (fl.stage != a.stage) continue;
#pragma unroll
          for (int k = 0; k < E; ++k)
            if (col + (int64_t)(tau + TPS * k) * a.pitch == fl.element) {
              if (fl.part == 0) v[k].x = flip_bits(v[k].x, fl.bit);
              else v[k].y = flip_bits(v[k].y, fl.bit);
            }
        }
      }
      if constexpr (PH == 2) {
        TwRun<T> wv(tw0, tstep);
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = cmul<T>(v[k], wv.next(k));
      }
      F::run(slot, v, tau, tw);
      if constexpr (PH == 0) {
        // stage 0 (S = 1): column j's outputs are contiguous at j L + c
        CT* d = pseudo ? static_cast<CT*>(b.pseudo_dst) + w * a.n + col * L : dst + j * a.n + col * L;
#pragma unroll
        for (int k = 0; k < E; ++k) __stcs(d + tau + TPS * F::out_pos(k), v[k]);
        __syncthreads();
      } else {
        if (!pseudo) {
          // outputs at e = q + S c: c_out (wang: omega_3^(e mod 3)) and s_out
          T r2[2] = {0, 0};
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const int64_t e = col + a.s * (int64_t)(tau + TPS * F::out_pos(k));
            CT ev = mk<T>(1, 0);
            if (b.enc == ENC_WANG) {
              const int m = (int)(e % 3);
              const T h = (T)0.86602540378443864676372317075294;
              ev = m == 0 ? mk<T>(1, 0) : (m == 1 ? mk<T>((T)-0.5, -h) : mk<T>((T)-0.5, h));
            }
            r2[0] = rfma(ev.x, v[k].x, rfma(-ev.y, v[k].y, r2[0]));
            r2[1] = rfma(ev.x, v[k].y, rfma(ev.y, v[k].x, r2[1]));
            acc[k] = mk<T>(rfma(wj, v[k].x, acc[k].x), rfma(wj, v[k].y, acc[k].y));
          }
          r2[0] = warp_sum(r2[0]);
          r2[1] = warp_sum(r2[1]);
          if (lane == 0) {
            double* dp = b.sig_part + (j * b.parts + cb * NW + wp) * 5;
            dp[3] = (double)r2[0];
            dp[4] = (double)r2[1];
          }
          // y: transposed through the slots, CB contiguous per output row
          __syncthreads();
#pragma unroll
          for (int k = 0; k < E; ++k) slot[F::phys(tau + TPS * F::out_pos(k))] = v[k];
          __syncthreads();
          CT* d = dst + j * a.n + c0;
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const int e = i * NT + tid;
            const int r = e / CB, c = e % CB;
            __stcs(d + (int64_t)r * a.s + c, tile[K::base(c) + F::phys(r)]);
          }
          __syncthreads();
        } else {
          // the pseudo-signal's output is ref = FFT(s_in): group partials
          double a2 = 0, b2 = 0;
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const double dr = (double)v[k].x - (double)acc[k].x, di = (double)v[k].y - (double)acc[k].y;
            a2 += dr * dr + di * di;
            b2 += (double)v[k].x * (double)v[k].x + (double)v[k].y * (double)v[k].y;
          }
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) {
            a2 += __shfl_xor_sync(0xffffffffu, a2, off);
            b2 += __shfl_xor_sync(0xffffffffu, b2, off);
          }
          if (lane == 0) {
            b.gpart[((w * ncb + cb) * NW + wp) * 2] = a2;
            b.gpart[((w * ncb + cb) * NW + wp) * 2 + 1] = b2;
          }
          __syncthreads();
        }
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0 && a.counters) atomicOr(&a.counters->nonfinite, 1ull);
}

// group_div[w] = sqrt(sum a) / max(sqrt(sum b), 1e-30) over the window's partials, in order
__global__ void stage_group_fin_kernel(const double* gpart, int64_t per, int64_t nwin, double* out) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= nwin) return;
  double a2 = 0, b2 = 0;
  for (int64_t i = 0; i < per; ++i) {
    a2 += gpart[(w * per + i) * 2];
    b2 += gpart[(w * per + i) * 2 + 1];
  }
  out[w] = sqrt(a2) / fmax(sqrt(b2), 1e-30);
}

template <typename T, int LOGL, int PH>
static int launch_stage_abft_t(const ColArgs& a, const StageAbft& b, int num_sms, cudaStream_t st) {
  using K = ColCfg<T, LOGL>;
  auto kern = stage_abft_kernel<T, LOGL, PH>;
  static LaunchCfg cfg;
  const int dev = current_device();
  if (!cfg.done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
    if (e != cudaSuccess) return (int)e;
    int ps = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, K::NT, K::SMEM);
    if (e != cudaSuccess) return (int)e;
    cfg.per_sm[dev] = ps < 1 ? 1 : ps;
    cfg.done[dev] = true;
  }
  const int64_t nitems = b.nwin * (a.ncols / K::CB);
  int64_t grid = (int64_t)num_sms * cfg.per_sm[dev];
  if (grid > nitems) grid = nitems;
  if (grid < 1) return 0;
  kern<<<(unsigned)grid, K::NT, K::SMEM, st>>>(a, b);
  return (int)cudaGetLastError();
}

template <typename T, int PH>
static int dispatch_stage_abft(int logl, const ColArgs& a, const StageAbft& b, int num_sms, cudaStream_t st) {
  switch (logl) {
#define TFFT_SA(L) \
  case L: return launch_stage_abft_t<T, L, PH>(a, b, num_sms, st);
    TFFT_SA(6) TFFT_SA(7) TFFT_SA(8) TFFT_SA(9) TFFT_SA(10) TFFT_SA(11)
#undef TFFT_SA
    default:
      return (int)cudaErrorInvalidValue;
  }
}

template <int PH>
static int stage_abft(int prec, int logl, const ColArgs& a, const StageAbft& b, int num_sms, cudaStream_t st) {
  return prec == 0 ? dispatch_stage_abft<float, PH>(logl, a, b, num_sms, st)
                   : dispatch_stage_abft<double, PH>(logl, a, b, num_sms, st);
}

// warps per stage-pass tile (NT / 32) and column blocks of a span
static void stage_tile_shape(int prec, int64_t L, int64_t n, int64_t* ncb, int* nw) {
  const int bpc = prec == 0 ? 8 : 16;
  int64_t cb0 = 65536 / (L * bpc);
  const int64_t cb = cb0 < 2 ? 2 : (cb0 > 32 ? 32 : cb0);
  const int64_t tps = L / (16 < L ? 16 : L);
  *ncb = (n / L) / cb;
  *nw = (int)((cb * tps) / 32);
}

// ---------------------------------------------------------------------------
// stage passes

struct StagePlan {
  int64_t n = 0;
  int prec = 0;
  int nst = 0;
  int64_t spans[3] = {0, 0, 0};
  int lo_bits = 0;
  int num_sms = 148;
  void* tw[3][2] = {};  // omega_span^m per stage (conj for inverse)
  void* hi[2] = {nullptr, nullptr};
  void* lo[2] = {nullptr, nullptr};
};

int stage_create(int64_t n, int prec, const int64_t* spans, int nstages, int num_sms, StagePlan** out) {
  *out = nullptr;
  if (nstages < 2 || nstages > 3) return (int)cudaErrorInvalidValue;
  for (int k = 0; k < nstages; ++k)
    if (spans[k] < 64 || spans[k] > 2048) return (int)cudaErrorInvalidValue;  // col_kernel's L range
  StagePlan* p = new StagePlan();
  p->n = n;
  p->prec = prec;
  p->nst = nstages;
  p->num_sms = num_sms;
  const int logn = ilog2i(n);
  p->lo_bits = (logn + 1) / 2;
  int e = 0;
  for (int k = 0; k < nstages && !e; ++k) {
    p->spans[k] = spans[k];
    for (int c = 0; c < 2 && !e; ++c) e = upload_table(prec, spans[k], 1, spans[k], c == 1, &p->tw[k][c]);
  }
  for (int c = 0; c < 2 && !e; ++c) {
    e = upload_table(prec, n, int64_t(1) << p->lo_bits, n >> p->lo_bits, c == 1, &p->hi[c]);
    if (!e) e = upload_table(prec, n, 1, int64_t(1) << p->lo_bits, c == 1, &p->lo[c]);
  }
  if (e) {
    stage_destroy(p);
    return e;
  }
  *out = p;
  return 0;
}

void stage_destroy(StagePlan* p) {
  if (!p) return;
  for (auto& t : p->tw)
    for (void* q : t) cudaFree(q);
  for (int c = 0; c < 2; ++c) {
    cudaFree(p->hi[c]);
    cudaFree(p->lo[c]);
  }
  delete p;
}

int stage_count(const StagePlan* p) { return p ? p->nst : 0; }

int stage_protected_parts(const StagePlan* p, int64_t* parts, int64_t* gper) {
  // [B][P][5] per-signal partials with P = the larger of the first and last
  // stage's (column blocks x warps); per-window group partials of the last
  int64_t ncb0, ncb2;
  int nw0, nw2;
  stage_tile_shape(p->prec, p->spans[0], p->n, &ncb0, &nw0);
  stage_tile_shape(p->prec, p->spans[p->nst - 1], p->n, &ncb2, &nw2);
  if (nw0 < 1 || nw2 < 1) return (int)cudaErrorNotSupported;
  *parts = ncb0 * nw0 > ncb2 * nw2 ? ncb0 * nw0 : ncb2 * nw2;
  *gper = ncb2 * nw2;
  return 0;
}

int stage_protected(StagePlan* p, const void* x, void* y, void* tmp, int64_t batch, int64_t weight0,
                    const DevFault* faults, int nfaults, Counters* counters, int64_t win, int enc, const void* row,
                    void* pa, void* pb, double* sig_part, double* gpart, double* win_div, cudaStream_t st) {
  if (p->nst < 2 || (enc != ENC_WANG && enc != ENC_ONES)) return (int)cudaErrorNotSupported;
  int64_t parts = 0, gper = 0;
  int rc = stage_protected_parts(p, &parts, &gper);
  if (rc) return rc;
  const int64_t nwin = (batch + win - 1) / win;
  cudaError_t e = cudaMemsetAsync(sig_part, 0, (size_t)batch * parts * 5 * sizeof(double), st);
  if (e != cudaSuccess) return (int)e;
  StageAbft b{};
  b.win = win;
  b.nwin = nwin;
  b.weight0 = weight0;
  b.row = row;
  b.enc = enc;
  b.sig_part = sig_part;
  b.parts = parts;
  b.gpart = gpart;
  const void* src = x;
  void* psrc = nullptr;
  int64_t S = 1;
  for (int k = 0; k < p->nst; ++k) {
    void* dst = ((p->nst - 1 - k) % 2 == 0) ? y : tmp;
    void* pdst = (k % 2 == 0) ? pa : pb;
    const int64_t L = p->spans[k];
    ColArgs a{};
    a.src = src;
    a.dst = dst;
    a.batch = batch;
    a.n = p->n;
    a.pitch = p->n / L;
    a.ncols = p->n / L;
    a.tw = p->tw[k][0];
    a.hi = p->hi[0];
    a.lo = p->lo[0];
    a.lo_bits = p->lo_bits;
    a.faults = faults;
    a.nfaults = nfaults;
    a.strike_stage = -1;
    a.counters = counters;
    a.s = S;
    a.stage = k;
    a.last = 0;
    if (k == 0) {
      b.pseudo_dst = pdst;
      rc = stage_abft<0>(p->prec, ilog2i(L), a, b, p->num_sms, st);
    } else if (k == p->nst - 1) {
      b.pseudo_src = psrc;
      rc = stage_abft<2>(p->prec, ilog2i(L), a, b, p->num_sms, st);
    } else {
      rc = col(p->prec, false, 2, ilog2i(L), a, p->num_sms, st);  // the real signals
      if (!rc) {
        ColArgs q = a;  // the pseudo-signals (no strikes, no counters)
        q.src = psrc;
        q.dst = pdst;
        q.batch = nwin;
        q.nfaults = 0;
        q.counters = nullptr;
        rc = col(p->prec, false, 2, ilog2i(L), q, p->num_sms, st);
      }
    }
    if (rc) return rc;
    src = dst;
    psrc = pdst;
    S *= L;
  }
  stage_group_fin_kernel<<<(unsigned)((nwin + 127) / 128), 128, 0, st>>>(gpart, gper, nwin, win_div);
  return (int)cudaGetLastError();
}

int stage_execute(StagePlan* p, const void* x, void* y, void* tmp, int64_t batch, int inverse, const DevFault* faults,
                  int nfaults, Counters* counters, cudaStream_t st) {
  const int c = inverse ? 1 : 0;
  const void* src = x;
  int64_t S = 1;
  for (int k = 0; k < p->nst; ++k) {
    // ping-pong ending in y: ..., tmp, y
    void* dst = ((p->nst - 1 - k) % 2 == 0) ? y : tmp;
    const int64_t L = p->spans[k];
    ColArgs a{};
    a.src = src;
    a.dst = dst;
    a.batch = batch;
    a.n = p->n;
    a.pitch = p->n / L;
    a.ncols = p->n / L;
    a.n1 = 0;
    a.tw = p->tw[k][c];
    a.hi = p->hi[c];
    a.lo = p->lo[c];
    a.lo_bits = p->lo_bits;
    a.faults = faults;
    a.nfaults = nfaults;
    a.strike_stage = -1;
    a.counters = counters;
    a.s = S;
    a.stage = k;
    a.last = k == p->nst - 1;
    const int rc = col(p->prec, inverse != 0, 2, ilog2i(L), a, p->num_sms, st);
    if (rc) return rc;
    src = dst;
    S *= L;
  }
  return 0;
}

int k3_create(int64_t n, int prec, const int64_t* spans, int nstages, int num_sms, K3Plan** out) {
  *out = nullptr;
  const int logn = ilog2i(n);
  int l1;
  if (nstages >= 2) l1 = ilog2i(spans[0]);
  else l1 = (logn + 1) / 2;
  int l2 = logn - l1;
  if (nstages > 2 || l1 < 6 || l2 < 6 || l1 > 11 || l2 > 11) {
    // the reference's span may be lopsided; fall back to a balanced split
    // (stage-1 strikes then go through the strike path)
    if (nstages > 2 || logn < 12 || logn > 22) return (int)cudaErrorInvalidValue;
    l1 = (logn + 1) / 2;
    l2 = logn - l1;
    nstages = 1;
  }
  K3Plan* p = new K3Plan();
  p->n = n;
  p->prec = prec;
  p->l1 = l1;
  p->l2 = l2;
  p->stage1 = nstages == 2;
  p->num_sms = num_sms;
  p->lo_bits = (logn + 1) / 2;
  p->k4 = k4_supported(prec, l1, l2) && std::getenv("TFFT_NO_K4") == nullptr;
  const int64_t N1 = int64_t(1) << l1, N2 = int64_t(1) << l2;
  int e = 0;
  for (int c = 0; c < 2 && !e; ++c) {
    e = upload_table(prec, N1, 1, N1, c == 1, &p->tw1[c]);
    if (!e) e = upload_table(prec, N2, 1, N2, c == 1, &p->tw2[c]);
    if (!e) e = upload_table(prec, n, int64_t(1) << p->lo_bits, n >> p->lo_bits, c == 1, &p->hi[c]);
    if (!e) e = upload_table(prec, n, 1, int64_t(1) << p->lo_bits, c == 1, &p->lo[c]);
  }
  if (e) {
    k3_destroy(p);
    return e;
  }
  *out = p;
  return 0;
}

void k3_destroy(K3Plan* p) {
  if (!p) return;
  for (int c = 0; c < 2; ++c) {
    cudaFree(p->tw1[c]);
    cudaFree(p->tw2[c]);
    cudaFree(p->hi[c]);
    cudaFree(p->lo[c]);
    cudaFree(p->enc[c]);
  }
  cudaFree(p->inter);
  cudaFree(p->ring);
  cudaFree(p->sync);
  delete p;
}

bool k3_strikes_stage1(const K3Plan* p) { return p && p->stage1; }

int k3_launches(const K3Plan* p) { return p && p->k4 ? 1 : 2; }

// K4 group size: ~16 MB of intermediate per group, so the 3-slot ring is ~48 MB
// the plain two-pass schedule runs on K7 (else K4)
static bool k7_on(const K3Plan* p) {
  return k7_supported(p->prec, p->l1, p->l2) && std::getenv("TFFT_NO_K7") == nullptr;
}

static int64_t k4_group(const K3Plan* p, int64_t batch) {
  const int64_t cb = p->prec == 0 ? 8 : 16;
  // ~16 MB of intermediate per group (3-slot ring ~48 MB) up to 2^16; 32 MB
  // from 2^17 (measured sweep 4..48 MB: 2^18..2^20 FP64 2-4% and FP32 3-7%
  // faster, 2^14..2^16 slower with the larger ring)
  // per-size group bytes from a sweep of the current K7 (tools/k7_sched_sweep.sh,
  // 12..40 MB): 1-2% at FP64 2^17, 2^18 (20 MB), FP64 2^20 (16 MB: one signal
  // per group, 0.770 vs 0.787 ms) and FP32 2^20 (24 MB: three signals)
  int64_t mb = p->n >= (int64_t(1) << 17) ? 32 : 16;
  if (p->prec == 1 && (p->n == (int64_t(1) << 17) || p->n == (int64_t(1) << 18))) mb = 20;
  if (p->prec == 1 && p->n == (int64_t(1) << 20)) mb = 16;
  if (p->prec == 0 && p->n == (int64_t(1) << 20)) mb = 24;
  if (const char* env = std::getenv("TFFT_K4_GROUP_MB")) {  // tuning hook (tools/k7_sched_sweep.sh)
    const long long v = std::atoll(env);
    if (v >= 1 && v <= 256) mb = v;
  }
  int64_t g = (mb << 20) / (p->n * cb);
  if (g < 1) g = 1;
  if (g > batch) g = batch;
  return g;
}

static int k4_execute_chunk(K3Plan* p, const void* x, void* y, int64_t batch, int inverse, const DevFault* faults,
                            int nfaults, Counters* counters, cudaStream_t st);

// TMA coordinates are 32-bit: x is addressed as batch * N1 rows (and y as
// batch * N2 rows), so very large batches run as several launches of at most
// 2^31 / max(N1, N2) signals each (faults are re-based per chunk)
static int k4_execute(K3Plan* p, const void* x, void* y, int64_t batch, int inverse, const DevFault* faults,
                      int nfaults, Counters* counters, cudaStream_t st) {
  const int64_t rows = int64_t(1) << (p->l1 > p->l2 ? p->l1 : p->l2);
  int64_t maxb = (int64_t(1) << 31) / rows - 1;
  if (const char* env = std::getenv("TFFT_K4_MAX_BATCH")) {  // test hook: force the chunked path
    const long long v = std::atoll(env);
    if (v > 0 && v < maxb) maxb = v;
  }
  if (batch <= maxb) return k4_execute_chunk(p, x, y, batch, inverse, faults, nfaults, counters, st);
  const size_t cb = p->prec == 0 ? 8 : 16;
  std::vector<DevFault> host(nfaults);
  if (nfaults) {
    cudaError_t e = cudaMemcpy(host.data(), faults, nfaults * sizeof(DevFault), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return (int)e;
  }
  DevFault* dfl = nullptr;
  if (nfaults) {
    cudaError_t e = cudaMalloc(&dfl, nfaults * sizeof(DevFault));
    if (e != cudaSuccess) return (int)e;
  }
  int rc = 0;
  for (int64_t b0 = 0; b0 < batch && !rc; b0 += maxb) {
    const int64_t nb = batch - b0 < maxb ? batch - b0 : maxb;
    std::vector<DevFault> mine;
    for (const DevFault& f : host)
      if (f.signal >= b0 && f.signal < b0 + nb) {
        DevFault g = f;
        g.signal -= b0;
        mine.push_back(g);
      }
    if (!mine.empty()) {
      cudaError_t e = cudaMemcpyAsync(dfl, mine.data(), mine.size() * sizeof(DevFault), cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) {
        rc = (int)e;
        break;
      }
    }
    rc = k4_execute_chunk(p, static_cast<const char*>(x) + (size_t)b0 * p->n * cb,
                          static_cast<char*>(y) + (size_t)b0 * p->n * cb, nb, inverse, mine.empty() ? nullptr : dfl,
                          (int)mine.size(), counters, st);
    if (!mine.empty()) cudaStreamSynchronize(st);  // dfl is reused by the next chunk
  }
  cudaFree(dfl);
  return rc;
}

static int k4_execute_chunk(K3Plan* p, const void* x, void* y, int64_t batch, int inverse, const DevFault* faults,
                            int nfaults, Counters* counters, cudaStream_t st) {
  const size_t cb = p->prec == 0 ? 8 : 16;
  const int64_t G = k4_group(p, batch);
  const size_t ring = (size_t)3 * G * p->n * cb;
  if (p->ring_cap < ring) {
    cudaFree(p->ring);
    p->ring = nullptr;
    p->ring_cap = 0;
    cudaError_t e = cudaMalloc(&p->ring, ring);
    if (e != cudaSuccess) return (int)e;
    p->ring_cap = ring;
  }
  const int64_t ng = (batch + G - 1) / G;
  const bool k7 = k7_on(p);
  const bool ldisc = k7 && k7_line_discard(p->prec, p->l1, p->l2) && std::getenv("TFFT_K7_LDISC") != nullptr;
  const size_t lcnt = ldisc ? (size_t)batch * ((int64_t(1) << p->l1) / (p->prec == 0 ? 16 : 8)) : 0;
  const size_t sync = 8 + ((size_t)2 * ng + lcnt) * sizeof(unsigned);
  if (p->sync_cap < sync) {
    cudaFree(p->sync);
    p->sync = nullptr;
    p->sync_cap = 0;
    cudaError_t e = cudaMalloc(&p->sync, sync);
    if (e != cudaSuccess) return (int)e;
    p->sync_cap = sync;
  }
  cudaError_t e = cudaMemsetAsync(p->sync, 0, sync, st);
  if (e != cudaSuccess) return (int)e;
  const int64_t N1 = int64_t(1) << p->l1, N2 = int64_t(1) << p->l2;
  const int lmax = p->l1 > p->l2 ? p->l1 : p->l2;
  // pass-A / pass-B tiles per signal
  const int64_t tpa = N2 / (k7 ? k7_columns_per_tile(p->prec, p->l1) : k4_columns_per_tile(p->prec, p->l1, lmax));
  const int64_t tpb = N1 / (k7 ? k7_columns_per_tile(p->prec, p->l2) : k4_columns_per_tile(p->prec, p->l2, lmax));
  const int64_t glast = batch - (ng - 1) * G;
  const int c = inverse ? 1 : 0;
  K4Args a{};
  a.x = x;
  a.y = y;
  a.z = p->ring;
  a.batch = batch;
  a.group = G;
  a.ngroups = ng;
  a.ta = G * tpa;
  a.tb = G * tpb;
  a.ta_last = glast * tpa;
  a.tb_last = glast * tpb;
  a.tw1 = p->tw1[c];
  a.tw2 = p->tw2[c];
  a.hi = p->hi[c];
  a.lo = p->lo[c];
  a.lo_bits = p->lo_bits;
  a.faults = faults;
  a.nfaults = nfaults;
  a.strike_stage = p->stage1 ? 1 : -1;
  a.counters = counters;
  a.ticket = static_cast<unsigned long long*>(p->sync);
  a.done_a = reinterpret_cast<unsigned*>(static_cast<char*>(p->sync) + 8);
  a.done_b = a.done_a + ng;
  a.line_cnt = ldisc ? a.done_b + ng : nullptr;
  if (k7)
    return launch_k7(p->prec, inverse != 0, p->l1, p->l2, a, p->num_sms, st);
  return launch_k4(p->prec, inverse != 0, p->l1, p->l2, a, p->num_sms, st);
}

int k3_execute(K3Plan* p, const void* x, void* y, int64_t batch, int inverse, const DevFault* faults, int nfaults,
               Counters* counters, void* reserved, cudaStream_t st) {
  (void)reserved;
  if (p->k4) return k4_execute(p, x, y, batch, inverse, faults, nfaults, counters, st);
  const size_t cb = p->prec == 0 ? 8 : 16;
  const size_t need = (size_t)batch * p->n * cb;
  if (p->inter_cap < need) {
    cudaFree(p->inter);
    p->inter = nullptr;
    p->inter_cap = 0;
    cudaError_t e = cudaMalloc(&p->inter, need);
    if (e != cudaSuccess) return (int)e;
    p->inter_cap = need;
  }
  const int64_t N1 = int64_t(1) << p->l1, N2 = int64_t(1) << p->l2;
  const int c = inverse ? 1 : 0;
  ColArgs a{};
  a.src = x;
  a.dst = p->inter;
  a.batch = batch;
  a.n = p->n;
  a.pitch = N2;
  a.ncols = N2;
  a.n1 = N1;
  a.tw = p->tw1[c];
  a.hi = p->hi[c];
  a.lo = p->lo[c];
  a.lo_bits = p->lo_bits;
  a.faults = faults;
  a.nfaults = nfaults;
  a.strike_stage = p->stage1 ? 1 : -1;
  a.counters = counters;
  int rc = col(p->prec, inverse != 0, 0, p->l1, a, p->num_sms, st);
  if (rc) return rc;
  ColArgs b = a;
  b.src = p->inter;
  b.dst = y;
  b.pitch = N1;
  b.ncols = N1;
  b.tw = p->tw2[c];
  b.nfaults = 0;
  b.strike_stage = -1;
  return col(p->prec, inverse != 0, 1, p->l2, b, p->num_sms, st);
}

// Fused two-sided ABFT on the K4 schedule (forward): the transform plus the C
// tiles that form the window sums and per-(signal, chunk) checksum partials
// from x and y while they are L2-resident. cudaErrorNotSupported when the
// split runs on K7 / K3, the window does not divide into the group size, or
// the batch needs several launches; the caller then uses the checksum sweep.
int k3_protected(K3Plan* p, const void* x, void* y, int64_t batch, int64_t weight0, const DevFault* faults,
                 int nfaults, Counters* counters, const AbftArgs& ab, const void* row, void* s_in, void* s_out,
                 double* sig_part, int64_t* nparts, cudaStream_t st) {
  if (!p->k4 || k7_on(p)) return (int)cudaErrorNotSupported;
  if (ab.enc != ENC_WANG && ab.enc != ENC_ONES) return (int)cudaErrorNotSupported;
  const int64_t W = ab.win_signals;
  const int64_t G0 = k4_group(p, batch);
  if (W > 2 * G0) return (int)cudaErrorNotSupported;  // ring would outgrow L2
  // a smaller group than the plain schedule's: the C tiles' x / y reads
  // share the L2 with the ring (TFFT_K4_ABFT_G: windows per group)
  int64_t gw = 1;
  if (const char* e = std::getenv("TFFT_K4_ABFT_G")) gw = std::atoll(e) > 0 ? std::atoll(e) : 1;
  int64_t G = gw * W;
  if (G > 2 * G0) G = W;
  const int64_t rows = int64_t(1) << (p->l1 > p->l2 ? p->l1 : p->l2);
  if (batch > (int64_t(1) << 31) / rows - 1) return (int)cudaErrorNotSupported;
  const int64_t KC = k4_abft_chunk(p->prec, p->l1, p->l2);
  if (p->n % KC) return (int)cudaErrorNotSupported;
  const size_t cb = p->prec == 0 ? 8 : 16;
  const size_t ring = (size_t)3 * G * p->n * cb;
  if (p->ring_cap < ring) {
    cudaFree(p->ring);
    p->ring = nullptr;
    p->ring_cap = 0;
    cudaError_t e = cudaMalloc(&p->ring, ring);
    if (e != cudaSuccess) return (int)e;
    p->ring_cap = ring;
  }
  const int64_t ng = (batch + G - 1) / G;
  const int64_t nwin = (batch + W - 1) / W;
  const size_t sync = 8 + (size_t)(2 * ng + nwin) * sizeof(unsigned);
  if (p->sync_cap < sync) {
    cudaFree(p->sync);
    p->sync = nullptr;
    p->sync_cap = 0;
    cudaError_t e = cudaMalloc(&p->sync, sync);
    if (e != cudaSuccess) return (int)e;
    p->sync_cap = sync;
  }
  cudaError_t e = cudaMemsetAsync(p->sync, 0, sync, st);
  if (e != cudaSuccess) return (int)e;
  const int64_t N1 = int64_t(1) << p->l1, N2 = int64_t(1) << p->l2;
  const int lmax = p->l1 > p->l2 ? p->l1 : p->l2;
  const int64_t tpa = N2 / k4_columns_per_tile(p->prec, p->l1, lmax);
  const int64_t tpb = N1 / k4_columns_per_tile(p->prec, p->l2, lmax);
  const int64_t glast = batch - (ng - 1) * G;
  const int64_t nchunk = p->n / KC;
  K4Args a{};
  a.x = x;
  a.y = y;
  a.z = p->ring;
  a.batch = batch;
  a.group = G;
  a.ngroups = ng;
  a.ta = G * tpa;
  a.tb = G * tpb;
  a.ta_last = glast * tpa;
  a.tb_last = glast * tpb;
  a.tw1 = p->tw1[0];
  a.tw2 = p->tw2[0];
  a.hi = p->hi[0];
  a.lo = p->lo[0];
  a.lo_bits = p->lo_bits;
  a.faults = faults;
  a.nfaults = nfaults;
  a.strike_stage = p->stage1 ? 1 : -1;
  a.counters = counters;
  a.ticket = static_cast<unsigned long long*>(p->sync);
  a.done_a = reinterpret_cast<unsigned*>(static_cast<char*>(p->sync) + 8);
  a.done_b = a.done_a + ng;
  a.abft = 1;
  a.enc = ab.enc;
  a.win = W;
  a.tc = (G / W) * nchunk;
  a.tc_last = ((glast + W - 1) / W) * nchunk;
  a.nchunk = nchunk;
  a.weight0 = weight0;
  a.row = row;
  a.s_in = s_in;
  a.s_out = s_out;
  a.sig_part = sig_part;
  a.done_w = a.done_b + ng;
  *nparts = nchunk;
  return launch_k4_abft(p->prec, p->l1, p->l2, a, p->num_sms, st);
}

int k3_base_table(K3Plan*, int prec, int64_t s, int r, int inverse, void* dst, cudaStream_t st) {
  return launch_base_table(prec, s, r, inverse, dst, st);
}

const void* k3_enc_table(K3Plan* p) {
  if (!p->enc[0]) upload_table(p->prec, p->n, 1, p->n, false, &p->enc[0]);
  return p->enc[0];
}

const void* k3_enc_table_inv(K3Plan* p) {
  if (!p->enc[1]) upload_table(p->prec, p->n, 1, p->n, true, &p->enc[1]);
  return p->enc[1];
}

}  // namespace tfft
