// K1 / K2: single-pass batched FFT (N <= 2^13 FP32, 2^12 FP64), optionally with
// the fused two-sided ABFT epilogue (reference abft.py:592-665 done on-chip).
//
// Persistent CTAs; each CTA owns SPT "slots" of TPS threads, one signal per slot
// per pipeline step. Signal tiles arrive through 1-D bulk async copies
// (cp.async.bulk, the TMA engine) into an NSTAGE-deep shared-memory ring
// guarded by mbarriers, so HBM reads for step i+NSTAGE-1 overlap the radix work
// of step i. The FFT runs in place in the stage buffer; the last pass stores
// straight from registers to HBM (coalesced: thread tau writes tau + TPS*k).
//
// ABFT (template flag, zero cost when off): per signal, c_in = row . x and the
// floor ||x||^2 are formed from the registers the first pass loaded, c_out =
// enc . y from the registers the last pass stores; per verification window,
// s_in = sum w_j x_j and s_out = sum w_j y_j accumulate in registers across the
// window's signals and FFT(s_in) runs in-CTA at the window end. No extra HBM
// traffic beyond O(B) scalars and O(#windows) partial columns.
#include "tfft_fft.cuh"
#include "tfft_internal.h"

namespace tfft {

// Tunable shapes (swept on the B200 with tools/tune_k1.py; the production
// choice per (precision, N) is k1_variant()).
struct K1Var {
  int emax32, emax64;  // elements per thread (radix of the main passes)
  int nt;              // target threads per CTA
  int st_small, st_big;  // pipeline stages for tiles <= 32 KB / larger
  int minb;            // __launch_bounds__ min blocks per SM
  int pf;              // prefetch next-pass twiddles before the barriers
};
constexpr K1Var kK1Var[] = {
    {16, 16, 256, 3, 2, 1, 0},  // 0 production default: radix 16, 3-stage ring
    {16, 16, 256, 3, 2, 1, 1},  // 1 + twiddle prefetch
    {16, 16, 256, 2, 2, 2, 0},  // 2 2 stages, 2 blocks/SM
    {16, 16, 256, 2, 2, 2, 1},  // 3 2 stages, 2 blocks/SM, prefetch
    {16, 16, 128, 3, 2, 2, 0},  // 4 128-thread CTAs
    {16, 16, 512, 3, 2, 1, 0},  // 5 512-thread CTAs
    {16, 16, 256, 4, 2, 1, 0},  // 6 4-stage ring
    {8, 8, 256, 3, 2, 2, 0},    // 7 radix 8
};

template <typename T, int LOGN, bool INV, bool ABFT, int V = 0>
struct K1 {
  static constexpr K1Var VAR = kK1Var[V];
  static constexpr int N = 1 << LOGN;
  static constexpr int EMAX = sizeof(T) == 4 ? VAR.emax32 : VAR.emax64;
  using F = Fft<T, N, EMAX, INV, VAR.pf != 0>;
  static constexpr int E = F::E;
  static constexpr int TPS = F::TPS;
  static constexpr int NT_TARGET = VAR.nt;
  static constexpr int SPT = TPS >= NT_TARGET ? 1 : NT_TARGET / TPS;
  static constexpr int NT = SPT * TPS;
  static constexpr int MINB = (NT <= 1024 / VAR.minb) ? VAR.minb : 1;
  // slot g's signal lands at g * SLOT (linear, by the bulk copy) and the
  // passes re-lay it out padded inside the same NPAD elements; SLOT keeps the
  // bulk-copy destinations 16-byte aligned
  static constexpr int SLOT = (F::NPAD + (16 / (int)sizeof(C<T>)) - 1) / (16 / (int)sizeof(C<T>)) *
                              (16 / (int)sizeof(C<T>));
  static constexpr int TILE = SPT * SLOT;
  static constexpr int TILE_BYTES = TILE * (int)sizeof(C<T>);
  static constexpr int NSTAGE = TILE_BYTES <= 32768 ? VAR.st_small : VAR.st_big;
  static constexpr int NWARP_SLOT = TPS >= 32 ? TPS / 32 : 1;
  static constexpr int RED_BYTES = SPT * NWARP_SLOT * 5 * 8;
  static constexpr int SMEM = (NSTAGE + (ABFT ? 1 : 0)) * TILE_BYTES + RED_BYTES + 64 + NSTAGE * 8;
};

// deterministic reduction of NV doubles over the TPS threads of a slot;
// result valid in the slot's tau == 0 thread. Contains a CTA barrier when
// TPS > 32 (every thread must call).
template <int TPS, int NV>
__device__ __forceinline__ void slot_reduce(double (&r)[NV], double* red, int g, int tau) {
  if constexpr (TPS <= 32) {
#pragma unroll
    for (int off = TPS / 2; off >= 1; off >>= 1)
#pragma unroll
      for (int k = 0; k < NV; ++k) r[k] += __shfl_xor_sync(0xffffffffu, r[k], off);
  } else {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
      for (int k = 0; k < NV; ++k) r[k] += __shfl_xor_sync(0xffffffffu, r[k], off);
    constexpr int NW = TPS / 32;
    const int w = tau >> 5;
    if ((tau & 31) == 0)
#pragma unroll
      for (int k = 0; k < NV; ++k) red[(g * NW + w) * NV + k] = r[k];
    __syncthreads();
    if (tau == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        double acc = red[(g * NW) * NV + k];
        for (int i = 1; i < NW; ++i) acc += red[(g * NW + i) * NV + k];
        r[k] = acc;
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* addr, double v) {
  atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

template <typename T, int LOGN, bool INV, bool ABFT, int V>
__global__ void __launch_bounds__(K1<T, LOGN, INV, ABFT, V>::NT, K1<T, LOGN, INV, ABFT, V>::MINB)
    k1_kernel(K1Args a) {
  using K = K1<T, LOGN, INV, ABFT, V>;
  using F = typename K::F;
  using CT = C<T>;
  constexpr int N = K::N, E = K::E, TPS = K::TPS, SPT = K::SPT, NSTAGE = K::NSTAGE;

  extern __shared__ __align__(128) unsigned char smem[];
  CT* tiles = reinterpret_cast<CT*>(smem);
  CT* wbuf = tiles + NSTAGE * K::TILE;  // ABFT window buffer (one tile)
  double* red = reinterpret_cast<double*>(smem + (NSTAGE + (ABFT ? 1 : 0)) * K::TILE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(red) + K::RED_BYTES);
  int* flag = reinterpret_cast<int*>(full + NSTAGE);

  const int tid = threadIdx.x;
  const int g = tid / TPS;
  const int tau = tid % TPS;
  const CT* __restrict__ x = static_cast<const CT*>(a.x);
  CT* __restrict__ y = static_cast<CT*>(a.y);
  const CT* __restrict__ tw = static_cast<const CT*>(a.tw);
  const int64_t B = a.batch;

  // ---- work decomposition --------------------------------------------------
  // plain: item k = tile of SPT consecutive signals (one step)
  // ABFT mode 0: item k = SPT consecutive windows, slot g runs window k*SPT+g
  // ABFT mode 1: item k = piece (k % P) of window (k / P), split over the slots
  const int64_t W = ABFT ? a.abft.win_signals : 1;
  const int64_t P = ABFT ? a.abft.pieces : 1;
  const int mode = ABFT ? a.abft.mode : 0;
  int64_t nitems;
  if (!ABFT) nitems = (B + SPT - 1) / SPT;
  else if (mode == 0) nitems = (a.abft.nwin + SPT - 1) / SPT;
  else nitems = a.abft.nwin * P;

  auto slot_run = [&](int64_t item, int gg, int64_t& start, int64_t& len) {
    if (!ABFT) {
      start = item * SPT + gg;
      len = start < B ? 1 : 0;
    } else if (mode == 0) {
      const int64_t w = item * SPT + gg;
      start = w * W;
      len = (w < a.abft.nwin) ? min(W, B - start) : 0;
    } else {
      const int64_t wi = item / P, pi = item % P;
      const int64_t w0 = wi * W, w1 = min(w0 + W, B);
      const int64_t pl = (W + P - 1) / P;
      const int64_t ps = min(w0 + pi * pl, w1), pe = min(ps + pl, w1);
      const int64_t sl = (pe - ps + SPT - 1) / SPT;
      start = min(ps + gg * sl, pe);
      len = min(start + sl, pe) - start;
    }
    if (len < 0) len = 0;
  };
  auto item_len = [&](int64_t item) {
    int64_t s, l, mx = 0;
    for (int gg = 0; gg < SPT; ++gg) {
      slot_run(item, gg, s, l);
      mx = l > mx ? l : mx;
    }
    return mx;
  };

  // ---- producer (thread 0): issues the bulk copies of one pipeline step ------
  int64_t p_item = blockIdx.x, p_i = 0, p_len = 0;
  if (tid == 0) {
#pragma unroll 1
    for (int s = 0; s < NSTAGE; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    p_len = p_item < nitems ? item_len(p_item) : 0;
  }
  __syncthreads();
  auto produce = [&](int stage) {  // thread 0 only
    while (p_item < nitems && p_i >= p_len) {
      p_item += gridDim.x;
      p_i = 0;
      p_len = p_item < nitems ? item_len(p_item) : 0;
    }
    if (p_item >= nitems) return;
    CT* dst = tiles + stage * K::TILE;
    if (!ABFT && SPT == 1) {
      mbar_expect_tx(&full[stage], (uint32_t)(N * sizeof(CT)));
      bulk_g2s(dst, x + p_item * N, N * sizeof(CT), &full[stage]);
    } else {
      uint32_t bytes = 0;
      int64_t st[SPT];
      bool ok[SPT];
      for (int gg = 0; gg < SPT; ++gg) {
        int64_t s, l;
        slot_run(p_item, gg, s, l);
        ok[gg] = p_i < l;
        st[gg] = s + p_i;
        bytes += ok[gg] ? (uint32_t)(N * sizeof(CT)) : 0u;
      }
      mbar_expect_tx(&full[stage], bytes);
      for (int gg = 0; gg < SPT; ++gg)
        if (ok[gg]) bulk_g2s(dst + gg * K::SLOT, x + st[gg] * N, N * sizeof(CT), &full[stage]);
    }
    ++p_i;
  };
  if (tid == 0)
    for (int s = 0; s < NSTAGE; ++s) produce(s);

  // ---- ABFT per-thread state -------------------------------------------------
  CT s_in[ABFT ? E : 1], s_out[ABFT ? E : 1];
  int enc_mod3[ABFT ? E : 1];
  if constexpr (ABFT) {
#pragma unroll
    for (int k = 0; k < E; ++k) {
      s_in[k] = mk<T>(0, 0);
      s_out[k] = mk<T>(0, 0);
      enc_mod3[k] = (tau + TPS * F::out_pos(k)) % 3;
    }
  }
  const CT* __restrict__ row = static_cast<const CT*>(a.abft.row);
  bool bad_input = false;
  double dmax = 0.0;  // largest per-signal divergence this thread decided

  uint32_t it = 0;
#pragma unroll 1
  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
    int64_t my_start, my_len;
    slot_run(item, g, my_start, my_len);
    const int64_t len = item_len(item);
#pragma unroll 1
    for (int64_t i = 0; i < len; ++i, ++it) {
      const int stage = it % NSTAGE;
      mbar_wait(&full[stage], (it / NSTAGE) & 1);
      CT* buf = tiles + stage * K::TILE + g * K::SLOT;
      const bool valid = i < my_len;
      const int64_t sig = my_start + i;

      CT v[E];
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = buf[tau + TPS * k];
      if (valid) {
#pragma unroll
        for (int k = 0; k < E; ++k) bad_input |= !finite2<T>(v[k]);
      }

      double red5[5] = {0, 0, 0, 0, 0};
      if constexpr (ABFT) {
        if (valid) {
          // c_in = row . x and ||x||^2 from the clean input (abft.py:656-659)
          CT ci = mk<T>(0, 0);
          T fl = 0;
          const T w = (T)(a.weight0 + sig + 1);
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const CT r = __ldg(row + tau + TPS * k);
            ci = cadd<T>(ci, cmul<T>(r, v[k]));
            fl = rfma(v[k].x, v[k].x, rfma(v[k].y, v[k].y, fl));
            s_in[k] = mk<T>(rfma(w, v[k].x, s_in[k].x), rfma(w, v[k].y, s_in[k].y));
          }
          red5[0] = (double)ci.x;
          red5[1] = (double)ci.y;
          red5[2] = (double)fl;
        }
      }
      // stage-0 strikes: flip the freshly loaded element (fault.py:99-107)
      if (a.nfaults > 0 && valid) {
        for (int f = fault_lo(a.faults, a.nfaults, sig); f < a.nfaults && a.faults[f].signal == sig; ++f) {
          const DevFault fl = a.faults[f];
          if (fl.signal != sig || fl.stage != 0 || (int)(fl.element % TPS) != tau) continue;
          const int k0 = (int)(fl.element / TPS);
#pragma unroll
          for (int k = 0; k < E; ++k)
            if (k == k0) {
              if (fl.part == 0) v[k].x = flip_bits(v[k].x, fl.bit);
              else v[k].y = flip_bits(v[k].y, fl.bit);
            }
        }
      }

      F::run(buf, v, tau, tw);
      fence_proxy_async();
      __syncthreads();  // every read of this stage buffer is done: refill it
      if (tid == 0) produce(stage);

      if constexpr (INV) {
        const T sc = (T)(1.0 / (double)N);
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = cscale<T>(v[k], sc);
      }
      if (valid) {
        CT* yo = y + sig * N + tau;
#pragma unroll
        for (int k = 0; k < E; ++k) st_cs(yo + TPS * F::out_pos(k), v[k]);
      }
      if constexpr (ABFT) {
        if (valid) {
          const T w = (T)(a.weight0 + sig + 1);
          CT co = mk<T>(0, 0);
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const int pk = F::out_pos(k);
            CT e;
            if (a.abft.enc == ENC_WANG) {
              const T h = (T)0.86602540378443864676372317075294;  // sin(2 pi/3)
              const int m = enc_mod3[k];
              e = m == 0 ? mk<T>(1, 0) : (m == 1 ? mk<T>((T)-0.5, -h) : mk<T>((T)-0.5, h));
            } else if (a.abft.enc == ENC_ONES) {
              e = mk<T>(1, 0);
            } else {
              e = __ldg(tw + tau + TPS * pk);  // omega_N^k (forward table)
            }
            co = cadd<T>(co, cmul<T>(e, v[k]));
            s_out[pk] = mk<T>(rfma(w, v[k].x, s_out[pk].x), rfma(w, v[k].y, s_out[pk].y));
          }
          red5[3] = (double)co.x;
          red5[4] = (double)co.y;
        }
        slot_reduce<TPS, 5>(red5, red, g, tau);
        if (valid && tau == 0) {
          const double cin_r = red5[0], cin_i = red5[1];
          const double co_r = red5[3], co_i = red5[4];
          const double floor_v = sqrt(red5[2]) / sqrt((double)N);
          double dv;
          if (!isfinite(co_r) || !isfinite(co_i)) {
            dv = __longlong_as_double(0x7ff0000000000000ll);
          } else {
            const double den = fmax(fmax(hypot(cin_r, cin_i), floor_v), 1e-30);
            dv = hypot(cin_r - co_r, cin_i - co_i) / den;
          }
          a.abft.c_in[2 * sig] = cin_r;
          a.abft.c_in[2 * sig + 1] = cin_i;
          a.abft.c_out[2 * sig] = co_r;
          a.abft.c_out[2 * sig + 1] = co_i;
          a.abft.floors[sig] = floor_v;
          a.abft.div[sig] = dv;
          if (dv > a.abft.delta) atomicAdd(&a.counters->triggered, 1ull);
          dmax = fmax(dmax, dv);
        }
      }
    }

    // ---- end of item: verification-window work (abft.py:592-624, fused) -----
    if constexpr (ABFT) {
      const int64_t wi_mode1 = item / P;
      bool have_window = false;  // this slot (mode 0) / slot 0 (mode 1) finalizes a window
      int64_t wid = 0;
      if (mode == 0) {
        wid = item * SPT + g;
        have_window = wid < a.abft.nwin;
        if (have_window) {
#pragma unroll
          for (int k = 0; k < E; ++k) wbuf[g * K::SLOT + tau + TPS * k] = s_in[k];
        }
        __syncthreads();
      } else {
        // combine the slots' partials in slot order, then (if the window is split
        // into pieces) publish the piece partial; the last piece finalizes
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
          for (int k = 0; k < E; ++k) wbuf[g * K::SLOT + tau + TPS * k] = pass == 0 ? s_in[k] : s_out[k];
          __syncthreads();
          if (g == 0) {
#pragma unroll
            for (int k = 0; k < E; ++k) {
              CT acc = wbuf[tau + TPS * k];
              for (int gg = 1; gg < SPT; ++gg) acc = cadd<T>(acc, wbuf[gg * K::SLOT + tau + TPS * k]);
              if (pass == 0) s_in[k] = acc;
              else s_out[k] = acc;
            }
          }
          __syncthreads();
        }
        wid = wi_mode1;
        bool last = true;
        if (P > 1) {
          CT* ws = static_cast<CT*>(a.abft.ws) + item * 2 * N;
          if (g == 0) {
#pragma unroll
            for (int k = 0; k < E; ++k) {
              ws[tau + TPS * k] = s_in[k];
              ws[N + tau + TPS * k] = s_out[k];
            }
          }
          __threadfence();
          __syncthreads();
          if (tid == 0) {
            const unsigned prev = atomicAdd(&a.abft.win_count[wid], 1u);
            *flag = (prev == (unsigned)(P - 1));
          }
          __syncthreads();
          last = *flag != 0;
          if (last) {
            __threadfence();
            if (g == 0) {
              const CT* wsw = static_cast<const CT*>(a.abft.ws) + wid * P * 2 * N;
#pragma unroll
              for (int k = 0; k < E; ++k) {
                CT ai = __ldcg(wsw + tau + TPS * k);
                CT ao = __ldcg(wsw + N + tau + TPS * k);
                for (int64_t pi = 1; pi < P; ++pi) {
                  ai = cadd<T>(ai, __ldcg(wsw + pi * 2 * N + tau + TPS * k));
                  ao = cadd<T>(ao, __ldcg(wsw + pi * 2 * N + N + tau + TPS * k));
                }
                s_in[k] = ai;
                s_out[k] = ao;
              }
            }
            if (tid == 0) a.abft.win_count[wid] = 0;
          }
        }
        have_window = last && g == 0;
        if (last) {
          if (g == 0) {
#pragma unroll
            for (int k = 0; k < E; ++k) wbuf[tau + TPS * k] = s_in[k];
          }
          __syncthreads();
        }
        if (!last) {
#pragma unroll
          for (int k = 0; k < E; ++k) {
            s_in[k] = mk<T>(0, 0);
            s_out[k] = mk<T>(0, 0);
          }
          continue;
        }
      }
      // in-CTA FFT of s_in (working precision, as _fft_column) vs s_out
      CT v[E];
      CT* wb = wbuf + g * K::SLOT;
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = wb[tau + TPS * k];
      F::run(wb, v, tau, tw);
      double r2[2] = {0, 0};
      if (have_window) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int pk = F::out_pos(k);
          const double dr = (double)v[k].x - (double)s_out[pk].x;
          const double di = (double)v[k].y - (double)s_out[pk].y;
          r2[0] += dr * dr + di * di;
          r2[1] += (double)v[k].x * (double)v[k].x + (double)v[k].y * (double)v[k].y;
        }
      }
      slot_reduce<TPS, 2>(r2, red, g, tau);
      if (have_window && tau == 0) a.abft.win_div[wid] = sqrt(r2[0]) / fmax(sqrt(r2[1]), 1e-30);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < E; ++k) {
        s_in[k] = mk<T>(0, 0);
        s_out[k] = mk<T>(0, 0);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad_input) && (tid & 31) == 0) atomicOr(&a.counters->nonfinite, 1ull);
  if (ABFT && dmax > 0.0) atomic_max_nonneg(&a.counters->max_div_bits, dmax);  // once per thread, not per signal
}

// ---------------------------------------------------------------------------
// host-side dispatch

// production variant per (precision, log2 N) — chosen from the B200 sweep
// (tools/tune_k1.py, profiles/round1_k1_variants.txt)
template <typename T, int LOGN>
constexpr int prod_variant() {
  return 0;
}

template <typename T, int LOGN, bool INV, bool ABFT, int V>
static int launch_one(const K1Args& a, int num_sms, cudaStream_t st) {
  using K = K1<T, LOGN, INV, ABFT, V>;
  auto kern = k1_kernel<T, LOGN, INV, ABFT, V>;
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
  int64_t nitems;
  if (!ABFT) nitems = (a.batch + K::SPT - 1) / K::SPT;
  else if (a.abft.mode == 0) nitems = (a.abft.nwin + K::SPT - 1) / K::SPT;
  else nitems = a.abft.nwin * a.abft.pieces;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > nitems) grid = nitems;
  if (grid < 1) return 0;
  kern<<<(unsigned)grid, K::NT, K::SMEM, st>>>(a);
  return (int)cudaGetLastError();
}

#ifdef TFFT_TUNING
static int g_variant = -1;
}  // namespace tfft
extern "C" void tfft_tune_set_variant(int v) { tfft::g_variant = v; }
namespace tfft {
template <typename T, int L>
constexpr bool tuned_size() { return L == 8 || L == 10 || L == 12 || L == 13; }
#endif

template <typename T, int L, bool INV, bool ABFT>
static int launch_sel(const K1Args& a, int num_sms, cudaStream_t st) {
#ifdef TFFT_TUNING
  if constexpr (tuned_size<T, L>() && !INV) {
    switch (g_variant) {
      case 0: return launch_one<T, L, INV, ABFT, 0>(a, num_sms, st);
      case 1: return launch_one<T, L, INV, ABFT, 1>(a, num_sms, st);
      case 2: return launch_one<T, L, INV, ABFT, 2>(a, num_sms, st);
      case 3: return launch_one<T, L, INV, ABFT, 3>(a, num_sms, st);
      case 4: return launch_one<T, L, INV, ABFT, 4>(a, num_sms, st);
      case 5: return launch_one<T, L, INV, ABFT, 5>(a, num_sms, st);
      case 6: return launch_one<T, L, INV, ABFT, 6>(a, num_sms, st);
      case 7: return launch_one<T, L, INV, ABFT, 7>(a, num_sms, st);
      default: break;
    }
  }
#endif
  return launch_one<T, L, INV, ABFT, prod_variant<T, L>()>(a, num_sms, st);
}

template <typename T, bool INV, bool ABFT>
static int dispatch(int logn, const K1Args& a, int num_sms, cudaStream_t st) {
  switch (logn) {
#define TFFT_CASE(L) \
  case L: return launch_sel<T, L, INV, ABFT>(a, num_sms, st);
    TFFT_CASE(1) TFFT_CASE(2) TFFT_CASE(3) TFFT_CASE(4) TFFT_CASE(5) TFFT_CASE(6) TFFT_CASE(7)
    TFFT_CASE(8) TFFT_CASE(9) TFFT_CASE(10) TFFT_CASE(11) TFFT_CASE(12)
#undef TFFT_CASE
    case 13:
      if constexpr (sizeof(T) == 4) return launch_sel<T, 13, INV, ABFT>(a, num_sms, st);
      return (int)cudaErrorInvalidValue;
    default:
      return (int)cudaErrorInvalidValue;
  }
}

int k1_supported(int prec, int logn) { return logn >= 1 && logn <= (prec == 0 ? 13 : 12); }

int launch_k1(int prec, int logn, bool inverse, bool abft, const K1Args& a, int num_sms, cudaStream_t st) {
  if (!k1_supported(prec, logn)) return (int)cudaErrorInvalidValue;
  if (prec == 0) {
    if (abft) return dispatch<float, false, true>(logn, a, num_sms, st);
    return inverse ? dispatch<float, true, false>(logn, a, num_sms, st) : dispatch<float, false, false>(logn, a, num_sms, st);
  }
  if (abft) return dispatch<double, false, true>(logn, a, num_sms, st);
  return inverse ? dispatch<double, true, false>(logn, a, num_sms, st) : dispatch<double, false, false>(logn, a, num_sms, st);
}

template <typename T, int L>
static int slots_of() {
#ifdef TFFT_TUNING
  if constexpr (tuned_size<T, L>()) {
    switch (g_variant) {
      case 0: return K1<T, L, false, true, 0>::SPT;
      case 1: return K1<T, L, false, true, 1>::SPT;
      case 2: return K1<T, L, false, true, 2>::SPT;
      case 3: return K1<T, L, false, true, 3>::SPT;
      case 4: return K1<T, L, false, true, 4>::SPT;
      case 5: return K1<T, L, false, true, 5>::SPT;
      case 6: return K1<T, L, false, true, 6>::SPT;
      case 7: return K1<T, L, false, true, 7>::SPT;
      default: break;
    }
  }
#endif
  return K1<T, L, false, true, prod_variant<T, L>()>::SPT;
}

int k1_slots(int prec, int logn) {
  switch (logn) {
#define TFFT_SL(L) \
  case L: return prec == 0 ? slots_of<float, L>() : slots_of<double, L>();
    TFFT_SL(1) TFFT_SL(2) TFFT_SL(3) TFFT_SL(4) TFFT_SL(5) TFFT_SL(6) TFFT_SL(7)
    TFFT_SL(8) TFFT_SL(9) TFFT_SL(10) TFFT_SL(11) TFFT_SL(12) TFFT_SL(13)
#undef TFFT_SL
    default: return 1;
  }
}

}  // namespace tfft
