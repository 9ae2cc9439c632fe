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
#include <cstdio>
#include <cstdlib>

#include "tfft_fft.cuh"
#include "tfft_internal.h"

#ifndef TFFT_K5_EXP
#define TFFT_K5_EXP 0
#endif
// deepest landing ring (tiles in flight per CTA): FP32 2 (a shallower ring
// lets more CTAs share an SM; FP32 2^9 0.382 -> 0.349 ms, 2^11 0.358 -> 0.346,
// tools/ab_interleave.sh), FP64 4 (2 measured 0.3-0.6% slower)
#ifndef TFFT_K5_SMAX
#define TFFT_K5_SMAX (sizeof(T) == 4 ? 2 : 4)
#endif
#ifndef TFFT_K5_FP64_E4096
#define TFFT_K5_FP64_E4096 16
#endif

namespace tfft {

template <typename T, int LOGN, bool INV, bool ABFT>
struct K5 {
  static constexpr int N = 1 << LOGN;
  static constexpr int BPC = (int)sizeof(C<T>);
  // same radix schedule, ring and twiddle placement with and without ABFT: a
  // fault-free protected run must be bitwise equal to the plain transform
  // (tests/test_abft.py:197-206)
  // FP64 N = 4096 runs radix-8 (512 threads per signal, 17 warps per CTA):
  // radix-16 legs need ~140 registers in FP64, so its 205 KB CTA could only
  // run 9 warps per SM
  static constexpr int EMAX = (sizeof(T) == 8 && LOGN >= 12) ? TFFT_K5_FP64_E4096 : 16;
  static constexpr int TPS0 = N / (EMAX < N ? EMAX : N);
  static constexpr int NT = TPS0 > 128 ? TPS0 : 128;  // consumer threads
  static constexpr int SLOT0 = N + (N >> 4);           // engine NPAD
  static constexpr int SPT0 = NT / TPS0;
  static constexpr int TILE_BYTES0 = SPT0 * SLOT0 * BPC;
  static constexpr int S0 = 100 * 1024 / TILE_BYTES0;
  static constexpr int S = S0 < 2 ? 2 : (S0 > TFFT_K5_SMAX ? TFFT_K5_SMAX : S0);
  static constexpr bool TWS = N * BPC <= 65536 && S * TILE_BYTES0 + N * BPC <= 210 * 1024;
  // group-mode exchanges: a signal's TPS threads sync among themselves only
  // generated radix-16 twiddles (Fft TWG): measured 2-3% faster from N = 2048
  // (FP32 and FP64), 2% slower at 512 / 1024
#ifndef TFFT_K5_TWG
#define TFFT_K5_TWG -1
#endif
  static constexpr bool TWG = TFFT_K5_TWG < 0 ? LOGN >= 11 : TFFT_K5_TWG != 0;
  using F = Fft<T, N, EMAX, INV, false, -1, TWS, TWG>;
  static constexpr int E = F::E;
  static constexpr int TPS = F::TPS;
  static constexpr int SPT = NT / TPS;  // signals per tile
  // slot g's signal lands at g * SLOT (linear, by the bulk copy) and the
  // passes re-lay it out padded inside the same NPAD elements; SLOT keeps the
  // bulk-copy destinations 16-byte aligned
  static constexpr int SLOT = (F::NPAD + (16 / BPC) - 1) / (16 / BPC) * (16 / BPC);
  static constexpr int TILE = SPT * SLOT;
  static constexpr int TILE_BYTES = TILE * BPC;
  // FP32 N = 4096 / 8192: two CTAs per SM (<= 128 registers; ptxas chose 110
  // without the bound, one CTA per SM, ncu occupancy 14%)
  static constexpr int MINB = (NT <= 128 || (sizeof(T) == 4 && NT == 256)) ? 2 : 1;
  // 256+ consumer threads: no producer warp (thread 0 refills a released
  // slot), so a CTA is 8 (or 16) warps and two fit an SM's register file
  static constexpr bool INL = NT >= 256;
  static constexpr int NTHR = NT + (INL ? 0 : 32);
  static constexpr int NWARP_SLOT = TPS >= 32 ? TPS / 32 : 1;
  static constexpr int RED_BYTES = 0;
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
  static_assert(!ABFT || (TPS >= 32 && E % (64 / BPC) == 0 && NT % 128 == 0 && COLS_USED <= 512),
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
      a = caxpy<T>(w, x, a);
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
__device__ __forceinline__ void k5_body(const K1Args& a) {
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
    tmem_fence_before();
  }

  // tile sequence (identical in producer and consumers): plain = round robin;
  // ABFT = the segments of [lo, hi) in order, each in tiles of SPT signals
  struct Cursor {
    int64_t t, ss, se;
  };
  auto first = [&]() {
    Cursor c;
    c.t = ABFT ? lo : (int64_t)blockIdx.x;
    c.ss = lo;
    c.se = ABFT ? min(hi, (lo / W + 1) * W) : 0;
    return c;
  };
  auto next = [&](Cursor& c, int64_t& s0, int& nsig) -> bool {
    if constexpr (!ABFT) {
      if (c.t >= (B + SPT - 1) / SPT) return false;
      s0 = c.t * SPT;
      nsig = (int)min((int64_t)SPT, B - s0);
      c.t += gridDim.x;
    } else {
      if (c.t >= c.se) {  // next segment (window piece) of [lo, hi)
        c.ss = c.se;
        if (c.ss >= hi) return false;
        c.se = min(hi, (c.ss / W + 1) * W);
        c.t = c.ss;
      }
      if (c.t >= hi) return false;
      s0 = c.t;
      nsig = (int)min((int64_t)SPT, c.se - s0);
      c.t += SPT;
    }
    return true;
  };
  auto land = [&](int slot, int64_t s0, int nsig) {
    CT* dst = ring + slot * K::TILE;
    mbar_expect_tx(&full[slot], (uint32_t)(nsig * N * K::BPC));
    for (int gg = 0; gg < nsig; ++gg) bulk_g2s(dst + gg * K::SLOT, x + (s0 + gg) * N, N * K::BPC, &full[slot]);
  };
  Cursor pc = first();  // producer cursor (producer warp, or thread 0 when inline)
  // thread 0 lands the first S tiles before the CTA builds its twiddle
  // tables, so the first loads' DRAM latency overlaps the table reads (small
  // batches: C1 is ~7 tiles per CTA); the producer warp takes over from tile S
  if (tid == 0) {
    int64_t s0;
    int nsig;
    for (int i = 0; i < S && next(pc, s0, nsig); ++i) land(i, s0, nsig);
  }
  if constexpr (K::TWS) F::build_pass_tables(tws, static_cast<const CT*>(a.tw), tid, K::NTHR);
  __syncthreads();
  if constexpr (ABFT) tmem_fence_after();
  const CT* tw = K::TWS ? tws : static_cast<const CT*>(a.tw);
  if constexpr (!K::INL) {
    if (tid >= NT) {
      // ---------------------------------------------------------- producer
      if (tid != NT) return;
      int64_t s0;
      int nsig;
      int it = 0;
      for (; it < S && next(pc, s0, nsig); ++it) {
      }
#pragma unroll 1
      for (; next(pc, s0, nsig); ++it) {
        const int s = it % S;
        mbar_wait_sleep(&empty[s], ((it / S) & 1) ^ 1);
        land(s, s0, nsig);
      }
      return;
    }
  }

  // -------------------------------------------------------------- consumers
  const int g = tid / TPS;
  const int tau = tid % TPS;
  CT* __restrict__ y = static_cast<CT*>(a.y);
  unsigned nfx = 0;  // non-finite inputs (nf_acc)
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
      for (int k = 0; k < E; ++k) nfx = nf_acc<T>(nfx, v[k]);
    }
    double red5[5] = {0, 0, 0, 0, 0};
    if constexpr (ABFT) {
      if (valid) {  // warp-uniform (TPS >= 32)
        // c_in = row . x, ||x||^2 and s_in += w x from the clean input
        // registers (abft.py:656-659, :602-606), before any strike
        tmem_wait_st();
        const T w = (T)(a.weight0 + sig + 1);
        CT r[E];
#if TFFT_K5_EXP & 1  // experiment: no TMEM traffic (timing only)
#pragma unroll
        for (int k = 0; k < E; ++k) r[k] = mk<T>((T)1, (T)0);
#else
        tmem_read<T, E>(t_row, r);
#endif
        C<T> ci = mk<T>(0, 0);
        T fl = 0;
#pragma unroll
        for (int k = 0; k < E; ++k) {
          ci = cmac<T>(r[k], v[k], ci);
          fl = rfma(v[k].x, v[k].x, rfma(v[k].y, v[k].y, fl));
        }
        const T cr = ci.x, cim = ci.y;
#if !(TFFT_K5_EXP & 1)
        tmem_axpy<T, E>(t_sin, w, v);
#endif
        red5[0] = (double)cr;
        red5[1] = (double)cim;
        red5[2] = (double)fl;
      }
    }
    // stage-0 strikes: flip the freshly loaded element (fault.py:99-107)
    if (a.nfaults > 0 && valid) {
      // whole-warp signals: lane 0 searches the sorted list, the warp shares it
      int f0;
      if constexpr (TPS >= 32) {
        f0 = (tid & 31) == 0 ? fault_lo(a.faults, a.nfaults, sig) : 0;
        f0 = __shfl_sync(0xffffffffu, f0, 0);
      } else {
        f0 = fault_lo(a.faults, a.nfaults, sig);
      }
      for (int f = f0; f < a.nfaults && a.faults[f].signal == sig; ++f) {
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
    F::run(buf, v, tau, tw, SPT == 1 ? 2 : 2 + g);  // a constant id when one signal per tile (ptxas then reserves 3 barriers, not 16: 16 capped the fused entry at one CTA per SM)
    // this warp's reads of the slot are complete: hand it back to the
    // producer (generic-proxy writes ordered before the next bulk copy)
    fence_proxy_async();
    __syncwarp();
    if ((tid & 31) == 0) k5_arrive(&empty[s]);
    if constexpr (K::INL) {
      // inline producer: once every consumer warp has released this slot,
      // thread 0 lands the tile S ahead into it
      if (tid == 0) {
        int64_t n0;
        int nn;
        mbar_wait(&empty[s], ((it - 1) / S) & 1);
        if (next(pc, n0, nn)) land(s, n0, nn);
      }
    }
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
#if !(TFFT_K5_EXP & 1)
        tmem_axpy<T, E>(t_sout, w, v);
#endif
        red5[3] = (double)co.x;
        red5[4] = (double)co.y;
      }
#if TFFT_K5_EXP & 2  // experiment: no per-signal reduction (timing only)
      if (false) {
#else
      {
#endif
        // per-signal totals are finished OUTSIDE this kernel: each warp
        // reduces its lanes with a fixed xor tree (working precision) and
        // lane 0 stores the warp's 5 partials; launch_signal_epilogue adds a
        // signal's warps in order and decides it. No CTA barrier and no
        // serial FP64 tail on the FFT warps' path (that tail cost +0.17 ms
        // at C3 FP32).
        constexpr int W0 = TPS < 32 ? TPS : 32;
        constexpr int NWS = TPS >= 32 ? TPS / 32 : 1;
        if constexpr (W0 == 32) {
          // transposed (recursive-halving) reduction of the 5 values padded to
          // 8: 4 + 2 + 1 + 1 + 1 = 9 shuffles instead of 25; lane 4 i ends
          // with value i (fixed order, deterministic)
          const int ln = tid & 31;
          T r8[8] = {(T)red5[0], (T)red5[1], (T)red5[2], (T)red5[3], (T)red5[4], (T)0, (T)0, (T)0};
          const bool h4 = ln & 16, h3 = ln & 8, h2 = ln & 4;
          T s4[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const T send = h4 ? r8[i] : r8[i + 4];
            const T keep = h4 ? r8[i + 4] : r8[i];
            s4[i] = radd(keep, __shfl_xor_sync(0xffffffffu, send, 16));
          }
          T s2[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const T send = h3 ? s4[i] : s4[i + 2];
            const T keep = h3 ? s4[i + 2] : s4[i];
            s2[i] = radd(keep, __shfl_xor_sync(0xffffffffu, send, 8));
          }
          T s1;
          {
            const T send = h2 ? s2[0] : s2[1];
            const T keep = h2 ? s2[1] : s2[0];
            s1 = radd(keep, __shfl_xor_sync(0xffffffffu, send, 4));
          }
          s1 = radd(s1, __shfl_xor_sync(0xffffffffu, s1, 2));
          s1 = radd(s1, __shfl_xor_sync(0xffffffffu, s1, 1));
          const int idx = (h4 ? 4 : 0) + (h3 ? 2 : 0) + (h2 ? 1 : 0);
          if (valid && (ln & 3) == 0 && idx < 5)
            a.abft.sig_part[(sig * NWS + (tau >> 5)) * 5 + idx] = (double)s1;
        } else {
          T r5[5] = {(T)red5[0], (T)red5[1], (T)red5[2], (T)red5[3], (T)red5[4]};
#pragma unroll
          for (int off = W0 / 2; off >= 1; off >>= 1)
#pragma unroll
            for (int kk = 0; kk < 5; ++kk) r5[kk] = radd(r5[kk], __shfl_xor_sync(0xffffffffu, r5[kk], off));
          if (valid && (tau & 31) == 0) {
            double* dst = a.abft.sig_part + (sig * NWS + (tau >> 5)) * 5;
#pragma unroll
            for (int kk = 0; kk < 5; ++kk) dst[kk] = (double)r5[kk];
          }
        }
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
  if (__any_sync(0xffffffffu, nf_bad<T>(nfx)) && (tid & 31) == 0 && a.counters) atomicOr(&a.counters->nonfinite, 1ull);
}

template <typename T, int LOGN, bool INV, bool ABFT>
__global__ void __launch_bounds__(K5<T, LOGN, INV, ABFT>::NTHR, K5<T, LOGN, INV, ABFT>::MINB)
    k5_kernel(K1Args a) {
  k5_body<T, LOGN, INV, ABFT>(a);
}

// The fused-ABFT entry of the two-CTA-per-SM shapes (FP32 N = 4096 / 8192,
// 256 threads): the occupancy calculator keeps one CTA per SM at 121-128
// registers (the API reports no room for a second CTA above 112), so the register cap is explicit (__maxnreg__ cannot be combined
// with __launch_bounds__, hence a separate entry)
template <typename T, int LOGN, bool INV>
__global__ void __maxnreg__(112) k5_abft2_kernel(K1Args a) {
  k5_body<T, LOGN, INV, true>(a);
}

template <typename T, int LOGN, bool INV, bool ABFT>
static auto k5_entry() {
  using K = K5<T, LOGN, INV, ABFT>;
  if constexpr (ABFT && K::MINB == 2 && K::INL) return k5_abft2_kernel<T, LOGN, INV>;
  else return k5_kernel<T, LOGN, INV, ABFT>;
}

// configured grid of a K5 instantiation on the current device (the fused
// ABFT's per-CTA signal ranges, and so its partial-sum layout, depend on it)
template <typename T, int LOGN, bool INV, bool ABFT>
static int k5_grid_t(int num_sms, int64_t batch, int64_t* grid_out) {
  using K = K5<T, LOGN, INV, ABFT>;
  auto kern = k5_entry<T, LOGN, INV, ABFT>();
  static LaunchCfg cfg;
  const int dev = current_device();
  if (!cfg.done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
    if (e != cudaSuccess) return (int)e;
    // the largest shared-memory carveout, so two ~100 KB CTAs can share an SM
    // (the driver otherwise picked the 132 KB configuration: one CTA per SM)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return (int)e;
    int ps = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, K::NTHR, K::SMEM);
    if (e != cudaSuccess) return (int)e;
    if (std::getenv("TFFT_DEBUG_OCC")) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, kern);
      size_t avail = 0;
      cudaOccupancyAvailableDynamicSMemPerBlock(&avail, kern, 2, K::NTHR);
      std::fprintf(stderr, "k5<%d,%d,%d,%d> occupancy %d (smem %d, threads %d, tcols %d, regs %d, static %zu, "
                   "local %zu, maxthr %d, avail_dyn@2 %zu)\n", (int)sizeof(T), LOGN, (int)INV, (int)ABFT, ps,
                   K::SMEM, K::NTHR, ABFT ? K::TCOLS : 0, fa.numRegs, fa.sharedSizeBytes, fa.localSizeBytes,
                   fa.maxThreadsPerBlock, avail);
    }
    // The occupancy calculator answers 1 for the TMEM-allocating fused entry
    // even at 112 registers (cudaOccupancyAvailableDynamicSMemPerBlock(2) =
    // 0), but two of its CTAs (2 x 102 KB smem, 2 x 256 TMEM columns, 2 x 256
    // threads x 112 registers) do run concurrently: forcing 296 CTAs took C3
    // FP32 from 0.666 to 0.569 ms. CTAs never wait on each other here, so a
    // grid the SM could not co-schedule would serialise, not deadlock.
    if (ABFT && K::INL && K::MINB == 2) ps = 2;
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
  k5_entry<T, LOGN, INV, ABFT>()<<<(unsigned)grid, K::NTHR, K::SMEM, st>>>(a);
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
// ---------------------------------------------------------------------------
// Window finisher of the fused K5 route (abft.py:592-624 + :648-665), ONE
// launch after the transform instead of five (per-signal epilogue, segment
// combine, window FFT, group divergence): CTA w (grid-stride) owns window w.
//   1. s_in / s_out of the window: the CTAs' segment partials added in (CTA,
//      slot) order, s_in at this thread's pass-0 positions, s_out at its
//      output positions;
//   2. ref = FFT(s_in) in shared memory (the same engine, passes and twiddle
//      values as the plain K5 transform, so ref equals run_plain's output);
//   3. group_div = ||ref - s_out|| / max(||ref||, 1e-30) in FP64 (fixed trees);
//   4. the window's signals: warp per signal, its warps' 5 partials added in
//      order, then c_in / c_out / floor / divergence and the counters (one
//      atomicMax per thread, not per signal).
template <typename T, int LOGN>
struct WinFin {
  static constexpr int N = 1 << LOGN;
  static constexpr int TPS = N / 16;
  static constexpr int NT = TPS < 256 ? 256 : TPS;
  static constexpr int GW = NT / TPS;  // windows in flight per CTA (one per thread group)
  // group mode: a window's TPS threads sync among themselves (named barrier
  // 1 + g, or __syncwarp at TPS == 32)
  using F = Fft<T, N, 16, false, false, -1, false>;
  static constexpr int NW = TPS / 32;  // warps per window
  static constexpr int SMEM = GW * F::NPAD * (int)sizeof(C<T>) + GW * NW * 2 * 8;
  static_assert(TPS >= 32, "window finisher needs N >= 512");
};

template <typename T, int LOGN>
__global__ void __launch_bounds__(WinFin<T, LOGN>::NT) k5_window_finish(
    const C<T>* __restrict__ ws, const double* __restrict__ sig_part, int nws, const C<T>* __restrict__ tw,
    int64_t B, int64_t W, int64_t G, int64_t maxseg, int spt, int64_t nwin, double delta, AbftArgs ab,
    Counters* counters, C<T>* __restrict__ wsave) {
  using WF = WinFin<T, LOGN>;
  using F = typename WF::F;
  using CT = C<T>;
  constexpr int N = WF::N, E = F::E, TPS = WF::TPS, GW = WF::GW, NW = WF::NW;
  extern __shared__ __align__(16) unsigned char wsm[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int g = tid / TPS, tau = tid % TPS;
  CT* buf = reinterpret_cast<CT*>(wsm) + g * F::NPAD;
  double* red = reinterpret_cast<double*>(wsm + GW * F::NPAD * (int)sizeof(CT)) + g * NW * 2;
  // ---- windows: group g of CTA b takes windows (b * GW + g) + k * gridDim.x * GW
  for (int64_t w = (int64_t)blockIdx.x * GW + g; w < nwin; w += (int64_t)gridDim.x * GW) {
    const int64_t w0 = w * W, w1 = min(w0 + W, B);
    CT vi[E], vo[E];
#pragma unroll
    for (int k = 0; k < E; ++k) vi[k] = vo[k] = mk<T>(0, 0);
    int64_t c = w0 * G / B;
    while (c > 0 && c * B / G > w0) --c;
    while (c < G && (c + 1) * B / G <= w0) ++c;
    for (; c < G; ++c) {
      const int64_t lo = c * B / G, hi = (c + 1) * B / G;
      if (lo >= w1) break;
      if (hi <= lo) continue;
      const int64_t j = w - lo / W;
      for (int q = 0; q < spt; ++q) {
        const CT* base = ws + ((c * maxseg + j) * spt + q) * 2 * (int64_t)N;
#pragma unroll
        for (int k = 0; k < E; ++k) {
          vi[k] = cadd<T>(vi[k], base[tau + TPS * k]);
          vo[k] = cadd<T>(vo[k], base[N + tau + TPS * F::out_pos(k)]);
        }
      }
    }
    if (wsave) {  // window sums kept for the batched correction (tfft_correct_windows)
      CT* sv = wsave + w * 2 * (int64_t)N;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        sv[tau + TPS * k] = vi[k];
        sv[N + tau + TPS * F::out_pos(k)] = vo[k];
      }
    }
    F::run(buf, vi, tau, tw, 1 + g);
    double a2 = 0.0, b2 = 0.0;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const double dr = (double)vi[k].x - (double)vo[k].x, di = (double)vi[k].y - (double)vo[k].y;
      a2 += dr * dr + di * di;
      b2 += (double)vi[k].x * (double)vi[k].x + (double)vi[k].y * (double)vi[k].y;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      a2 += __shfl_xor_sync(0xffffffffu, a2, off);
      b2 += __shfl_xor_sync(0xffffffffu, b2, off);
    }
    if constexpr (NW > 1) {
      if (lane == 0) {
        red[2 * (tau >> 5)] = a2;
        red[2 * (tau >> 5) + 1] = b2;
      }
      fft_sync_grp<-1, TPS>(1 + g);
      if (tau == 0) {
        for (int i = 1; i < NW; ++i) {
          a2 += red[2 * i];
          b2 += red[2 * i + 1];
        }
      }
      fft_sync_grp<-1, TPS>(1 + g);  // red[] free for the next window
    }
    if (tau == 0) ab.win_div[w] = sqrt(a2) / fmax(sqrt(b2), 1e-30);
  }
  // ---- per-signal decisions, a thread per signal: its warps' partials in order
  double dmax = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + tid; r < B; r += (int64_t)gridDim.x * blockDim.x) {
    double acc[5] = {0, 0, 0, 0, 0};
    const double* pp = sig_part + r * nws * 5;
    for (int i = 0; i < nws; ++i)
#pragma unroll
      for (int q = 0; q < 5; ++q) acc[q] += pp[i * 5 + q];
    const double floor_v = sqrt(acc[2]) / sqrt((double)N);
    double dv;
    if (!isfinite(acc[3]) || !isfinite(acc[4])) dv = __longlong_as_double(0x7ff0000000000000ll);
    else dv = hypot(acc[0] - acc[3], acc[1] - acc[4]) / fmax(fmax(hypot(acc[0], acc[1]), floor_v), 1e-30);
    ab.c_in[2 * r] = acc[0];
    ab.c_in[2 * r + 1] = acc[1];
    ab.c_out[2 * r] = acc[3];
    ab.c_out[2 * r + 1] = acc[4];
    ab.floors[r] = floor_v;
    ab.div[r] = dv;
    if (dv > delta) atomicAdd(&counters->triggered, 1ull);
    dmax = fmax(dmax, dv);
  }
  // one atomic per warp
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
  if (lane == 0 && dmax > 0.0) atomicMax(&counters->max_div_bits, (unsigned long long)__double_as_longlong(dmax));
}

template <typename T, int LOGN>
static int launch_wf_t(const void* ws, const double* sig_part, int nws, const void* tw, int64_t B, int64_t W,
                       int64_t G, int64_t maxseg, int spt, int64_t nwin, double delta, const AbftArgs& ab,
                       Counters* counters, void* wsave, int num_sms, cudaStream_t st) {
  using WF = WinFin<T, LOGN>;
  auto kern = k5_window_finish<T, LOGN>;
  static LaunchCfg cfg;
  const int dev = current_device();
  if (!cfg.done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, WF::SMEM);
    if (e != cudaSuccess) return (int)e;
    cfg.done[dev] = true;
  }
  if (nwin < 1) return 0;
  // enough CTAs for the windows (GW per CTA) and for a thread per signal
  const int64_t want = std::max<int64_t>((nwin + WF::GW - 1) / WF::GW, (B + WF::NT - 1) / WF::NT);
  const int64_t grid = std::min<int64_t>(want, (int64_t)num_sms * 8);
  kern<<<(unsigned)grid, WF::NT, WF::SMEM, st>>>(static_cast<const C<T>*>(ws), sig_part, nws,
                                                  static_cast<const C<T>*>(tw), B, W, G, maxseg, spt, nwin, delta,
                                                  ab, counters, static_cast<C<T>*>(wsave));
  return (int)cudaGetLastError();
}

int launch_k5_window_finish(int prec, int logn, const void* ws, const double* sig_part, int nws, const void* tw,
                            int64_t B, int64_t W, int64_t G, int64_t maxseg, int spt, int64_t nwin, double delta,
                            const AbftArgs& ab, Counters* counters, void* wsave, int num_sms, cudaStream_t st) {
#define TFFT_WF(L)                                                                                              \
  case L:                                                                                                       \
    return prec == 0 ? launch_wf_t<float, L>(ws, sig_part, nws, tw, B, W, G, maxseg, spt, nwin, delta, ab,     \
                                             counters, wsave, num_sms, st)                                      \
                     : launch_wf_t<double, L>(ws, sig_part, nws, tw, B, W, G, maxseg, spt, nwin, delta, ab,    \
                                              counters, wsave, num_sms, st);
  switch (logn) {
    TFFT_WF(9) TFFT_WF(10) TFFT_WF(11) TFFT_WF(12)
    case 13:
      if (prec == 0)
        return launch_wf_t<float, 13>(ws, sig_part, nws, tw, B, W, G, maxseg, spt, nwin, delta, ab, counters,
                                      wsave, num_sms, st);
      return (int)cudaErrorInvalidValue;
    default:
      return (int)cudaErrorInvalidValue;
  }
#undef TFFT_WF
}

template <typename T>
static int dispatch_k5_abft(int logn, const K1Args* a, int num_sms, cudaStream_t st, int64_t batch, int64_t* grid,
                            int* spt, int* nws) {
  switch (logn) {
#define TFFT_K5A(L)                                                              \
  case L:                                                                        \
    if (spt) *spt = K5<T, L, false, true>::SPT;                                  \
    if (nws) *nws = K5<T, L, false, true>::NWARP_SLOT;                           \
    if (grid) return k5_grid_t<T, L, false, true>(num_sms, batch, grid);         \
    return launch_k5_t<T, L, false, true>(*a, num_sms, st);
    TFFT_K5A(9) TFFT_K5A(10) TFFT_K5A(11) TFFT_K5A(12)
#undef TFFT_K5A
    case 13:
      if constexpr (sizeof(T) == 4) {
        if (spt) *spt = K5<T, 13, false, true>::SPT;
        if (nws) *nws = K5<T, 13, false, true>::NWARP_SLOT;
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
  return prec == 0 ? dispatch_k5_abft<float>(logn, &a, num_sms, st, 0, nullptr, nullptr, nullptr)
                   : dispatch_k5_abft<double>(logn, &a, num_sms, st, 0, nullptr, nullptr, nullptr);
}

int k5_abft_layout(int prec, int logn, int num_sms, int64_t batch, int64_t* grid, int* spt, int* nws) {
  if (!k5_abft_supported(prec, logn)) return (int)cudaErrorInvalidValue;
  return prec == 0 ? dispatch_k5_abft<float>(logn, nullptr, num_sms, 0, batch, grid, spt, nws)
                   : dispatch_k5_abft<double>(logn, nullptr, num_sms, 0, batch, grid, spt, nws);
}

}  // namespace tfft
