// K5: warp-specialised single-pass batched FFT (N <= 2^13 FP32, 2^12 FP64).
//
// Same transform as K1 (tfft_k1.cu) on the same engine (tfft_fft.cuh), with
// the K4 execution model instead of K1's "every thread is a consumer, thread
// 0 also produces" loop:
//   * one producer warp lands each tile (SPT consecutive signals) with 1-D
//     bulk async copies (the TMA engine) into an S-deep ring of padded slots
//     and never touches the radix work;
//   * NT consumer threads (TPS per signal, tau fastest) run the in-place
//     Stockham passes with named barriers that exclude the producer, release
//     the slot to the producer as soon as their last shared-memory read is
//     done, and store the outputs straight from registers (coalesced);
//   * small CTAs (128 consumers where a signal allows it) so two CTAs share an
//     SM and one's exchange barriers overlap the other's arithmetic;
//   * per-pass twiddle tables live in shared memory (conflict-free reads)
//     when the w_N table is <= 64 KB.
// Bitwise identical to K1 on every input: same passes, same twiddles, same
// *_rn arithmetic.
#include <algorithm>

#include "tfft_fft.cuh"
#include "tfft_internal.h"

namespace tfft {

template <typename T, int LOGN, bool INV, bool ABFT>
struct K5 {
  static constexpr int N = 1 << LOGN;
  static constexpr int BPC = (int)sizeof(C<T>);
  // same radix schedule, ring and twiddle placement with and without ABFT: a
  // fault-free protected run must be bitwise equal to the plain transform
  // (tests/test_abft.py:197-206)
  static constexpr int EMAX = 16;
  static constexpr int TPS0 = N / (EMAX < N ? EMAX : N);
  static constexpr int NT = TPS0 > 128 ? TPS0 : 128;  // consumer threads
  static constexpr int SLOT0 = N + (N >> 4);           // engine NPAD
  static constexpr int SPT0 = NT / TPS0;
  static constexpr int TILE_BYTES0 = SPT0 * SLOT0 * BPC;
  static constexpr int S0 = 100 * 1024 / TILE_BYTES0;
  static constexpr int S = S0 < 2 ? 2 : (S0 > 4 ? 4 : S0);
  static constexpr bool TWS = N * BPC <= 65536 && S * TILE_BYTES0 + N * BPC <= 210 * 1024;
  // group-mode exchanges: a signal's TPS threads sync among themselves only
  using F = Fft<T, N, EMAX, INV, false, -1, TWS>;
  static constexpr int E = F::E;
  static constexpr int TPS = F::TPS;
  static constexpr int SPT = NT / TPS;  // signals per tile
  // slot g's signal lands at g * SLOT (linear, by the bulk copy) and the
  // passes re-lay it out padded inside the same NPAD elements; SLOT keeps the
  // bulk-copy destinations 16-byte aligned
  static constexpr int SLOT = (F::NPAD + (16 / BPC) - 1) / (16 / BPC) * (16 / BPC);
  static constexpr int TILE = SPT * SLOT;
  static constexpr int TILE_BYTES = TILE * BPC;
  // FP32 N = 4096 keeps two 288-thread CTAs per SM (<= 112 registers) with ABFT too
  static constexpr int MINB = (NT <= 128 || (ABFT && sizeof(T) == 4 && NT == 256)) ? 2 : 1;
  static constexpr int NTHR = NT + 32;
  static constexpr int NWARP_SLOT = TPS >= 32 ? TPS / 32 : 1;
  // per-signal partials: 2 tile parities x SPT slots x warps x 5 doubles + arrival counters
  static constexpr int RED_BYTES = ABFT ? (2 * SPT * NWARP_SLOT * 5 * 8 + 2 * SPT * 4 + 8) : 0;
  static constexpr int SMEM = S * TILE_BYTES + (TWS ? N * BPC : 0) + RED_BYTES + 2 * S * 8 + 64;
  // ---- ABFT accumulators in tensor memory: per consumer thread (its own TMEM
  // lane) three arrays of E complex values — s_in (window sum of w_j x_j at the
  // thread's input positions), s_out (sum of w_j y_j at its output positions)
  // and its slice of the left checksum row. A warpgroup's four warps cover the
  // 128 lanes; warpgroup q uses column block q.
  static constexpr int WPC = BPC / 4;              // 32-bit TMEM words per complex value
  static constexpr int ARR = E * WPC;              // words per array (32 FP32, 64 FP64)
  static constexpr int BLK = 3 * ARR;              // columns per warpgroup
  static constexpr int NBLK = NT / 128;
  static constexpr int COLS_USED = BLK * NBLK;
  static constexpr int TCOLS = COLS_USED <= 32 ? 32 : COLS_USED <= 64 ? 64 : COLS_USED <= 128 ? 128
                             : COLS_USED <= 256 ? 256 : 512;
  static_assert(!ABFT || (TPS >= 32 && E == 16 && NT % 128 == 0 && COLS_USED <= 512),
                "TMEM-fused ABFT needs whole-warp signals (N >= 512)");
};

__device__ __forceinline__ void k5_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// TMEM word <-> working-precision values (one complex = WPC words)
template <typename T> __device__ __forceinline__ C<T> tw_get(const uint32_t* r, int q);
template <> __device__ __forceinline__ float2 tw_get<float>(const uint32_t* r, int q) {
  return make_float2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
}
template <> __device__ __forceinline__ double2 tw_get<double>(const uint32_t* r, int q) {
  return make_double2(__hiloint2double((int)r[4 * q + 1], (int)r[4 * q]),
                      __hiloint2double((int)r[4 * q + 3], (int)r[4 * q + 2]));
}
__device__ __forceinline__ void tw_put(uint32_t* r, int q, float2 v) {
  r[2 * q] = __float_as_uint(v.x);
  r[2 * q + 1] = __float_as_uint(v.y);
}
__device__ __forceinline__ void tw_put(uint32_t* r, int q, double2 v) {
  r[4 * q] = (uint32_t)__double2loint(v.x);
  r[4 * q + 1] = (uint32_t)__double2hiint(v.x);
  r[4 * q + 2] = (uint32_t)__double2loint(v.y);
  r[4 * q + 3] = (uint32_t)__double2hiint(v.y);
}

// acc[k] += w * v[k] for the E complex values of one TMEM array (read-modify-
// write in 16-word chunks; warp-collective)
template <typename T, int E>
__device__ __forceinline__ void tmem_axpy(uint32_t taddr, T w, const C<T> (&v)[E]) {
  constexpr int PER = 16 / ((int)sizeof(C<T>) / 4);  // complex values per chunk
#pragma unroll
  for (int ch = 0; ch < E / PER; ++ch) {
    uint32_t r[16];
    tmem_ld16(taddr + ch * 16, r);
    tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      C<T> a = tw_get<T>(r, q);
      const C<T> x = v[ch * PER + q];
      a = mk<T>(rfma(w, x.x, a.x), rfma(w, x.y, a.y));
      tw_put(r, q, a);
    }
    tmem_st16(taddr + ch * 16, r);
  }
}

template <typename T, int E>
__device__ __forceinline__ void tmem_fill(uint32_t taddr, const C<T> (&v)[E]) {
  constexpr int PER = 16 / ((int)sizeof(C<T>) / 4);
#pragma unroll
  for (int ch = 0; ch < E / PER; ++ch) {
    uint32_t r[16];
#pragma unroll
    for (int q = 0; q < PER; ++q) tw_put(r, q, v[ch * PER + q]);
    tmem_st16(taddr + ch * 16, r);
  }
}

template <typename T, int E>
__device__ __forceinline__ void tmem_read(uint32_t taddr, C<T> (&v)[E]) {
  constexpr int PER = 16 / ((int)sizeof(C<T>) / 4);
#pragma unroll
  for (int ch = 0; ch < E / PER; ++ch) {
    uint32_t r[16];
    tmem_ld16(taddr + ch * 16, r);
    tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < PER; ++q) v[ch * PER + q] = tw_get<T>(r, q);
  }
}

// Work decomposition.
// Plain: tile t = SPT consecutive signals, tiles dealt round-robin to CTAs.
// ABFT (abft.py:592-665 fused): CTA c owns the contiguous signal range
// [c B / G, (c+1) B / G), cut at window boundaries (W = T bs signals) into
// segments; a segment is walked in tiles of SPT signals (slot g takes signal
// s0 + g). Per signal, c_in = row . x, ||x||^2 and s_in += w_j x_j come from
// the pass-0 registers before any strike; c_out = e . y and s_out += w_j y_j
// from the output registers. s_in / s_out / the row live in TMEM. At a
// segment end every slot writes its partial sums to ws[(c MAXSEG + j) SPT +
// g][2][N]; tfft_api.cu then adds a window's partials in (CTA, slot) order
// (seg_combine_kernel), FFTs the window sums and forms the group divergence.
template <typename T, int LOGN, bool INV, bool ABFT>
__global__ void __launch_bounds__(K5<T, LOGN, INV, ABFT>::NTHR, K5<T, LOGN, INV, ABFT>::MINB)
    k5_kernel(K1Args a) {
  using K = K5<T, LOGN, INV, ABFT>;
  using F = typename K::F;
  using CT = C<T>;
  constexpr int N = K::N, E = K::E, TPS = K::TPS, SPT = K::SPT, S = K::S, NT = K::NT;

  extern __shared__ __align__(128) unsigned char smem[];
  CT* ring = reinterpret_cast<CT*>(smem);
  CT* tws = ring + S * K::TILE;
  double* red = reinterpret_cast<double*>(tws + (K::TWS ? N : 0));
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(red) + K::RED_BYTES);
  uint64_t* empty = full + S;
  uint32_t* tmem_base = reinterpret_cast<uint32_t*>(empty + S);

  const int tid = threadIdx.x;
  const int64_t B = a.batch;
  const int64_t W = ABFT ? a.abft.win_signals : 1;
  // ABFT: this CTA's contiguous signal range
  const int64_t lo = ABFT ? (int64_t)blockIdx.x * B / gridDim.x : 0;
  const int64_t hi = ABFT ? ((int64_t)blockIdx.x + 1) * B / gridDim.x : 0;
  const CT* __restrict__ x = static_cast<const CT*>(a.x);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NT / 32);
    }
    fence_mbar_init();
  }
  if constexpr (ABFT) {
    if (tid < 32) tmem_alloc(tmem_base, K::TCOLS);
    int* cnt = reinterpret_cast<int*>(red + 2 * SPT * K::NWARP_SLOT * 5);
    for (int i = tid; i < 2 * SPT; i += K::NTHR) cnt[i] = 0;
    tmem_fence_before();
  }
  if constexpr (K::TWS) F::build_pass_tables(tws, static_cast<const CT*>(a.tw), tid, K::NTHR);
  __syncthreads();
  if constexpr (ABFT) tmem_fence_after();
  const CT* tw = K::TWS ? tws : static_cast<const CT*>(a.tw);

  // tile sequence (identical in producer and consumers): plain = round robin;
  // ABFT = the segments of [lo, hi) in order, each in tiles of SPT signals
  if (tid >= NT) {
    // ------------------------------------------------------------ producer
    if (tid != NT) return;
    int it = 0;
    auto land = [&](int64_t s0, int nsig) {
      const int s = it % S;
      if (it >= S) mbar_wait_sleep(&empty[s], ((it / S) & 1) ^ 1);
      CT* dst = ring + s * K::TILE;
      mbar_expect_tx(&full[s], (uint32_t)(nsig * N * K::BPC));
      for (int gg = 0; gg < nsig; ++gg) bulk_g2s(dst + gg * K::SLOT, x + (s0 + gg) * N, N * K::BPC, &full[s]);
      ++it;
    };
    if constexpr (!ABFT) {
      const int64_t ntiles = (B + SPT - 1) / SPT;
#pragma unroll 1
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t s0 = t * SPT;
        land(s0, (int)min((int64_t)SPT, B - s0));
      }
    } else {
#pragma unroll 1
      for (int64_t ss = lo; ss < hi;) {
        const int64_t se = min(hi, (ss / W + 1) * W);
#pragma unroll 1
        for (int64_t s0 = ss; s0 < se; s0 += SPT) land(s0, (int)min((int64_t)SPT, se - s0));
        ss = se;
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g = tid / TPS;
  const int tau = tid % TPS;
  CT* __restrict__ y = static_cast<CT*>(a.y);
  bool bad = false;
  // this thread's TMEM arrays: lane quadrant = warp % 4, column block = warpgroup
  const uint32_t tbase = ABFT ? (*tmem_base + ((uint32_t)(((tid >> 5) & 3) * 32) << 16) +
                                 (uint32_t)((tid >> 7) * K::BLK))
                              : 0u;
  const uint32_t t_sin = tbase, t_sout = tbase + K::ARR, t_row = tbase + 2 * K::ARR;
  if constexpr (ABFT) {
    CT r[E];
    const CT* gr = static_cast<const CT*>(a.abft.row);
#pragma unroll
    for (int k = 0; k < E; ++k) r[k] = gr[tau + TPS * k];
    tmem_fill<T, E>(t_row, r);
  }
  int it = 0;
  // one tile: SPT signals from s0 (nsig valid); accumulate when ABFT
  auto tile = [&](int64_t s0, int nsig) {
    const int s = it % S;
    mbar_wait(&full[s], (it / S) & 1);
    ++it;
    CT* buf = ring + s * K::TILE + g * K::SLOT;
    const int64_t sig = s0 + g;
    const bool valid = g < nsig;
    CT v[E];
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = buf[tau + TPS * k];
    if (valid) {
#pragma unroll
      for (int k = 0; k < E; ++k) bad |= !finite2<T>(v[k]);
    }
    double red5[5] = {0, 0, 0, 0, 0};
    if constexpr (ABFT) {
      if (valid) {  // warp-uniform (TPS >= 32)
        // c_in = row . x, ||x||^2 and s_in += w x from the clean input
        // registers (abft.py:656-659, :602-606), before any strike
        tmem_wait_st();
        const T w = (T)(a.weight0 + sig + 1);
        CT r[E];
        tmem_read<T, E>(t_row, r);
        T cr = 0, cim = 0, fl = 0;
#pragma unroll
        for (int k = 0; k < E; ++k) {
          cr = rfma(r[k].x, v[k].x, rfma(-r[k].y, v[k].y, cr));
          cim = rfma(r[k].x, v[k].y, rfma(r[k].y, v[k].x, cim));
          fl = rfma(v[k].x, v[k].x, rfma(v[k].y, v[k].y, fl));
        }
        tmem_axpy<T, E>(t_sin, w, v);
        red5[0] = (double)cr;
        red5[1] = (double)cim;
        red5[2] = (double)fl;
      }
    }
    // stage-0 strikes: flip the freshly loaded element (fault.py:99-107)
    if (a.nfaults > 0 && valid) {
      for (int f = 0; f < a.nfaults; ++f) {
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
    F::run(buf, v, tau, tw, 2 + g);
    // this warp's reads of the slot are complete: hand it back to the
    // producer (generic-proxy writes ordered before the next bulk copy)
    fence_proxy_async();
    __syncwarp();
    if ((tid & 31) == 0) k5_arrive(&empty[s]);
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
        CT co;
        if (a.abft.enc == ENC_JOU) {
          co = mk<T>(0, 0);
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const CT e = __ldg(static_cast<const CT*>(a.tw) + tau + TPS * F::out_pos(k));  // omega_N^k
            co = cadd<T>(co, cmul<T>(e, v[k]));
          }
        } else {
          // wang: e_k = omega_3^(k mod 3). Output register k sits at k' = tau +
          // TPS j_k, so k' mod 3 = (tau + r_k) mod 3 with r_k = TPS j_k mod 3
          // known at compile time: sum the registers per class r, then one
          // rotation per class (ones: a plain sum)
          CT A[3] = {mk<T>(0, 0), mk<T>(0, 0), mk<T>(0, 0)};
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const int r = (int)(((long long)TPS * F::out_pos(k)) % 3);
            A[r] = cadd<T>(A[r], v[k]);
          }
          if (a.abft.enc == ENC_ONES) {
            co = cadd<T>(cadd<T>(A[0], A[1]), A[2]);
          } else {
            const T h = (T)0.86602540378443864676372317075294;  // sin(2 pi/3)
            const CT w1 = mk<T>((T)-0.5, -h), w2 = mk<T>((T)-0.5, h);
            const int t3 = tau % 3;
            CT acc = mk<T>(0, 0);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              const int m = (t3 + r) % 3;
              acc = cadd<T>(acc, m == 0 ? A[r] : cmul<T>(m == 1 ? w1 : w2, A[r]));
            }
            co = acc;
          }
        }
        tmem_axpy<T, E>(t_sout, w, v);
        red5[3] = (double)co.x;
        red5[4] = (double)co.y;
      }
      // per-signal totals without a CTA barrier: xor-shuffle tree inside each
      // warp (working precision); for TPS > 32 the slot's warps publish
      // partials and the last one to arrive (shared-memory counter) adds them
      // in warp order in FP64
      constexpr int W0 = TPS < 32 ? TPS : 32;
      {
        T r5[5] = {(T)red5[0], (T)red5[1], (T)red5[2], (T)red5[3], (T)red5[4]};
#pragma unroll
        for (int off = W0 / 2; off >= 1; off >>= 1)
#pragma unroll
          for (int kk = 0; kk < 5; ++kk) r5[kk] = radd(r5[kk], __shfl_xor_sync(0xffffffffu, r5[kk], off));
#pragma unroll
        for (int kk = 0; kk < 5; ++kk) red5[kk] = (double)r5[kk];
      }
      bool fin = valid && tau == 0;
      if constexpr (TPS > 32) {
        constexpr int NW = TPS / 32;
        const int par = (it - 1) & 1;
        double* rp = red + ((par * SPT + g) * NW) * 5;
        fin = false;
        if ((tau & 31) == 0) {
#pragma unroll
          for (int kk = 0; kk < 5; ++kk) rp[(tau >> 5) * 5 + kk] = red5[kk];
          __threadfence_block();
          int* cnt = reinterpret_cast<int*>(red + 2 * SPT * NW * 5) + par * SPT + g;
          if (atomicAdd(cnt, 1) == NW - 1) {
            __threadfence_block();
#pragma unroll
            for (int kk = 0; kk < 5; ++kk) {
              double acc = rp[kk];
              for (int i = 1; i < NW; ++i) acc += rp[i * 5 + kk];
              red5[kk] = acc;
            }
            *cnt = 0;
            fin = valid;
          }
        }
      }
      if (fin) {
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
        atomicMax(&a.counters->max_div_bits, (unsigned long long)__double_as_longlong(dv));
      }
    }
  };

  if constexpr (!ABFT) {
    const int64_t ntiles = (B + SPT - 1) / SPT;
#pragma unroll 1
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t s0 = t * SPT;
      tile(s0, (int)min((int64_t)SPT, B - s0));
    }
  } else {
    const int64_t maxseg = a.abft.pieces;  // segments per CTA (host: ceil(ceil(B/G)/W) + 1)
    const int64_t w_first = lo / W;
    CT zero[E];
#pragma unroll
    for (int k = 0; k < E; ++k) zero[k] = mk<T>(0, 0);
#pragma unroll 1
    for (int64_t ss = lo; ss < hi;) {
      const int64_t wnd = ss / W;
      const int64_t se = min(hi, (wnd + 1) * W);
      tmem_fill<T, E>(t_sin, zero);
      tmem_fill<T, E>(t_sout, zero);
#pragma unroll 1
      for (int64_t s0 = ss; s0 < se; s0 += SPT) tile(s0, (int)min((int64_t)SPT, se - s0));
      // segment end: this slot's partial window sums -> ws (coalesced over tau)
      tmem_wait_st();
      CT* ws = static_cast<CT*>(a.abft.ws) + (((int64_t)blockIdx.x * maxseg + (wnd - w_first)) * SPT + g) * 2 * N;
      CT acc[E];
      tmem_read<T, E>(t_sin, acc);
#pragma unroll
      for (int k = 0; k < E; ++k) ws[tau + TPS * k] = acc[k];
      tmem_read<T, E>(t_sout, acc);
#pragma unroll
      for (int k = 0; k < E; ++k) ws[N + tau + TPS * F::out_pos(k)] = acc[k];
      ss = se;
    }
    // release tensor memory: every consumer warp is past its last TMEM access
    tmem_wait_st();
    tmem_fence_before();
    fft_sync<NT>();
    tmem_fence_after();
    if (tid < 32) tmem_dealloc(*tmem_base, K::TCOLS);
  }
  if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0 && a.counters) atomicOr(&a.counters->nonfinite, 1ull);
}

// configured grid of a K5 instantiation on the current device (the fused
// ABFT's per-CTA signal ranges, and so its partial-sum layout, depend on it)
template <typename T, int LOGN, bool INV, bool ABFT>
static int k5_grid_t(int num_sms, int64_t batch, int64_t* grid_out) {
  using K = K5<T, LOGN, INV, ABFT>;
  auto kern = k5_kernel<T, LOGN, INV, ABFT>;
  static LaunchCfg cfg;
  const int dev = current_device();
  if (!cfg.done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
    if (e != cudaSuccess) return (int)e;
    int ps = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, K::NTHR, K::SMEM);
    if (e != cudaSuccess) return (int)e;
    // ABFT: the TMEM columns of the CTAs sharing an SM must fit its 512
    if (ABFT) ps = std::min(ps, 512 / K::TCOLS);
    cfg.per_sm[dev] = ps < 1 ? 1 : ps;
    cfg.done[dev] = true;
  }
  const int64_t nitems = ABFT ? batch : (batch + K::SPT - 1) / K::SPT;
  int64_t grid = (int64_t)num_sms * cfg.per_sm[dev];
  *grid_out = grid > nitems ? nitems : grid;
  return 0;
}

template <typename T, int LOGN, bool INV, bool ABFT>
static int launch_k5_t(const K1Args& a, int num_sms, cudaStream_t st) {
  using K = K5<T, LOGN, INV, ABFT>;
  int64_t grid = 0;
  int e = k5_grid_t<T, LOGN, INV, ABFT>(num_sms, a.batch, &grid);
  if (e) return e;
  if (grid < 1) return 0;
  k5_kernel<T, LOGN, INV, ABFT><<<(unsigned)grid, K::NTHR, K::SMEM, st>>>(a);
  return (int)cudaGetLastError();
}

template <typename T, bool INV>
static int dispatch_k5(int logn, const K1Args& a, int num_sms, cudaStream_t st) {
  switch (logn) {
#define TFFT_K5(L) \
  case L: return launch_k5_t<T, L, INV, false>(a, num_sms, st);
    TFFT_K5(1) TFFT_K5(2) TFFT_K5(3) TFFT_K5(4) TFFT_K5(5) TFFT_K5(6) TFFT_K5(7)
    TFFT_K5(8) TFFT_K5(9) TFFT_K5(10) TFFT_K5(11) TFFT_K5(12)
#undef TFFT_K5
    case 13:
      if constexpr (sizeof(T) == 4) return launch_k5_t<T, 13, INV, false>(a, num_sms, st);
      return (int)cudaErrorInvalidValue;
    default:
      return (int)cudaErrorInvalidValue;
  }
}

int launch_k5(int prec, int logn, bool inverse, const K1Args& a, int num_sms, cudaStream_t st) {
  if (!k1_supported(prec, logn)) return (int)cudaErrorInvalidValue;
  if (prec == 0)
    return inverse ? dispatch_k5<float, true>(logn, a, num_sms, st) : dispatch_k5<float, false>(logn, a, num_sms, st);
  return inverse ? dispatch_k5<double, true>(logn, a, num_sms, st) : dispatch_k5<double, false>(logn, a, num_sms, st);
}

int k5_abft_supported(int prec, int logn) { return logn >= 9 && logn <= (prec == 0 ? 13 : 12); }

// fused-ABFT instantiations: N = 2^9 .. 2^12 (FP64) / 2^13 (FP32); query = grid only
template <typename T>
static int dispatch_k5_abft(int logn, const K1Args* a, int num_sms, cudaStream_t st, int64_t batch, int64_t* grid,
                            int* spt) {
  switch (logn) {
#define TFFT_K5A(L)                                                              \
  case L:                                                                        \
    if (spt) *spt = K5<T, L, false, true>::SPT;                                  \
    if (grid) return k5_grid_t<T, L, false, true>(num_sms, batch, grid);         \
    return launch_k5_t<T, L, false, true>(*a, num_sms, st);
    TFFT_K5A(9) TFFT_K5A(10) TFFT_K5A(11) TFFT_K5A(12)
#undef TFFT_K5A
    case 13:
      if constexpr (sizeof(T) == 4) {
        if (spt) *spt = K5<T, 13, false, true>::SPT;
        if (grid) return k5_grid_t<T, 13, false, true>(num_sms, batch, grid);
        return launch_k5_t<T, 13, false, true>(*a, num_sms, st);
      }
      return (int)cudaErrorInvalidValue;
    default:
      return (int)cudaErrorInvalidValue;
  }
}

int launch_k5_abft(int prec, int logn, const K1Args& a, int num_sms, cudaStream_t st) {
  if (!k5_abft_supported(prec, logn)) return (int)cudaErrorInvalidValue;
  return prec == 0 ? dispatch_k5_abft<float>(logn, &a, num_sms, st, 0, nullptr, nullptr)
                   : dispatch_k5_abft<double>(logn, &a, num_sms, st, 0, nullptr, nullptr);
}

int k5_abft_layout(int prec, int logn, int num_sms, int64_t batch, int64_t* grid, int* spt) {
  if (!k5_abft_supported(prec, logn)) return (int)cudaErrorInvalidValue;
  return prec == 0 ? dispatch_k5_abft<float>(logn, nullptr, num_sms, 0, batch, grid, spt)
                   : dispatch_k5_abft<double>(logn, nullptr, num_sms, 0, batch, grid, spt);
}

}  // namespace tfft
