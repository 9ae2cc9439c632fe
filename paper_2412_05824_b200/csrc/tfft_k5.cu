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
#include "tfft_fft.cuh"
#include "tfft_internal.h"

namespace tfft {

template <typename T, int LOGN, bool INV, bool ABFT>
struct K5 {
  static constexpr int N = 1 << LOGN;
  static constexpr int BPC = (int)sizeof(C<T>);
  // same radix schedule with and without ABFT: a fault-free protected run
  // must be bitwise equal to the plain transform (tests/test_abft.py:197-206)
  static constexpr int EMAX = 16;
  static constexpr int TPS0 = N / (EMAX < N ? EMAX : N);
  static constexpr int NT = TPS0 > 128 ? TPS0 : 128;  // consumer threads
  static constexpr int SLOT0 = N + (N >> 4);           // engine NPAD
  // slot buffers: S-deep ring + (ABFT) one window buffer; twiddle tables in
  // shared memory when everything fits
  static constexpr int SPT0 = NT / TPS0;
  static constexpr int TILE_BYTES0 = SPT0 * SLOT0 * BPC;
  static constexpr int S0 = 100 * 1024 / TILE_BYTES0;
  static constexpr int S = S0 < 2 ? 2 : (S0 > 4 ? 4 : S0);
  static constexpr bool TWS = N * BPC <= 65536 && (S + (ABFT ? 1 : 0)) * TILE_BYTES0 + N * BPC <= 210 * 1024;
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
  // ABFT keeps two window accumulators (E complex each) per thread beside the
  // E legs: FP64 needs the whole register file of one CTA per SM for them
  static constexpr int MINB = (ABFT && sizeof(T) == 8) ? 1 : (NT <= 128 ? 2 : 1);
  // FP64 ABFT with a 256-thread signal: no separate producer warp (thread 0
  // refills the freed stage after a consumer barrier, as K1 does), so the
  // eight consumer warps keep the whole 255-register budget for the legs and
  // the two window accumulators
  static constexpr bool INL = ABFT && sizeof(T) == 8 && NT >= 256;
  static constexpr int NTHR = NT + (INL ? 0 : 32);
  static constexpr int NWARP_SLOT = TPS >= 32 ? TPS / 32 : 1;
  // per-signal partials: 2 tile parities x SPT slots x warps x 5 doubles + arrival counters
  static constexpr int RED_BYTES = ABFT ? (2 * SPT * NWARP_SLOT * 5 * 8 + 2 * SPT * 4 + 8) : 0;
  static constexpr bool ROWS = ABFT && (S + 1) * TILE_BYTES + (TWS ? 2 : 1) * N * BPC + RED_BYTES <= 200 * 1024;
  static constexpr int SMEM =
      (S + (ABFT ? 1 : 0)) * TILE_BYTES + (TWS ? N * BPC : 0) + (ROWS ? N * BPC : 0) + RED_BYTES + 2 * S * 8 + 64;
};

__device__ __forceinline__ void k5_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// deterministic reduction of NV doubles over the TPS threads of a slot (fixed
// xor-shuffle tree, then the slot's warps in order); result valid in the
// slot's tau == 0 thread. Contains consumer barriers when TPS > 32.
template <int TPS, int NV, int NT>
__device__ __forceinline__ void k5_slot_reduce(double (&r)[NV], double* red, int g, int tau) {
  constexpr int W0 = TPS < 32 ? TPS : 32;
#pragma unroll
  for (int off = W0 / 2; off >= 1; off >>= 1)
#pragma unroll
    for (int k = 0; k < NV; ++k) r[k] += __shfl_xor_sync(0xffffffffu, r[k], off);
  if constexpr (TPS > 32) {
    constexpr int NW = TPS / 32;
    const int w = tau >> 5;
    if ((tau & 31) == 0)
#pragma unroll
      for (int k = 0; k < NV; ++k) red[(g * NW + w) * NV + k] = r[k];
    fft_sync<NT>();
    if (tau == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        double acc = red[(g * NW) * NV + k];
        for (int i = 1; i < NW; ++i) acc += red[(g * NW + i) * NV + k];
        r[k] = acc;
      }
    }
    fft_sync<NT>();
  }
}

// Work decomposition. Plain: tile t = SPT consecutive signals, tiles dealt
// round-robin to CTAs. ABFT (abft.py:592-665 fused): item = one piece of a
// verification window (the window's W signals split into P pieces of PL
// signals, PL a multiple of SPT); slot g of tile i of a piece takes signal
// piece_start + i * SPT + g. Each slot accumulates s_in = sum w_j x_j and
// s_out = sum w_j y_j over its signals in registers; at the piece end the
// slots are combined in order; a window split into P > 1 pieces is finished
// by its last-arriving piece, which adds the piece partials in piece order.
template <typename T, int LOGN, bool INV, bool ABFT>
__global__ void __launch_bounds__(K5<T, LOGN, INV, ABFT>::NTHR, K5<T, LOGN, INV, ABFT>::MINB)
    k5_kernel(K1Args a) {
  using K = K5<T, LOGN, INV, ABFT>;
  using F = typename K::F;
  using CT = C<T>;
  constexpr int N = K::N, E = K::E, TPS = K::TPS, SPT = K::SPT, S = K::S, NT = K::NT;

  extern __shared__ __align__(128) unsigned char smem[];
  CT* ring = reinterpret_cast<CT*>(smem);
  CT* wbuf = ring + S * K::TILE;                // ABFT window buffer (one tile)
  CT* tws = wbuf + (ABFT ? K::TILE : 0);
  CT* rows = tws + (K::TWS ? N : 0);          // ABFT left checksum row (shared copy)
  double* red = reinterpret_cast<double*>(rows + (K::ROWS ? N : 0));
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(red) + K::RED_BYTES);
  uint64_t* empty = full + S;
  int* flag = reinterpret_cast<int*>(empty + S);

  const int tid = threadIdx.x;
  const int64_t B = a.batch;
  // items and their tiles
  const int64_t W = ABFT ? a.abft.win_signals : 1;
  const int64_t P = ABFT ? a.abft.pieces : 1;
  const int64_t PL = ABFT ? ((W + P - 1) / P + SPT - 1) / SPT * SPT : SPT;  // piece length (signals)
  const int64_t nitems = ABFT ? a.abft.nwin * P : (B + SPT - 1) / SPT;
  auto piece = [&](int64_t item, int64_t& ps, int64_t& pe) {  // signal range of an item
    if (!ABFT) {
      ps = item * SPT;
      pe = min(ps + SPT, B);
    } else {
      const int64_t w = item / P, pi = item % P;
      const int64_t w0 = w * W, w1 = min(w0 + W, B);
      ps = min(w0 + pi * PL, w1);
      pe = min(ps + PL, w1);
    }
  };
  const CT* __restrict__ x = static_cast<const CT*>(a.x);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NT / 32);
    }
    fence_mbar_init();
  }
  if constexpr (K::TWS) F::build_pass_tables(tws, static_cast<const CT*>(a.tw), tid, K::NTHR);
  if constexpr (K::ROWS) {
    const CT* gr = static_cast<const CT*>(a.abft.row);
    for (int i = tid; i < N; i += K::NTHR) rows[i] = gr[i];
  }
  if constexpr (ABFT) {
    int* cnt = reinterpret_cast<int*>(red + 2 * SPT * K::NWARP_SLOT * 5);
    for (int i = tid; i < 2 * SPT; i += K::NTHR) cnt[i] = 0;
  }
  __syncthreads();
  const CT* tw = K::TWS ? tws : static_cast<const CT*>(a.tw);

  // the it-th tile this CTA loads: item cursor (p_item, p_i); lands in stage it % S
  int64_t p_item = blockIdx.x, p_i = 0;
  int p_it = 0;
  auto produce_next = [&]() {  // one thread
#pragma unroll 1
    while (p_item < nitems) {
      int64_t ps, pe;
      piece(p_item, ps, pe);
      // at least one tile per item: an empty piece (short last window) still
      // has to arrive for its window to be finished
      const int64_t ntl = pe > ps ? (pe - ps + SPT - 1) / SPT : 1;
      if (p_i >= ntl) {
        p_item += gridDim.x;
        p_i = 0;
        continue;
      }
      const int s = p_it % S;
      const int64_t s0 = ps + p_i * SPT;
      const int nsig = (int)(pe - s0 <= 0 ? 0 : (pe - s0 < SPT ? pe - s0 : SPT));
      CT* dst = ring + s * K::TILE;
      if (nsig == 0) {
        k5_arrive(&full[s]);
      } else {
        mbar_expect_tx(&full[s], (uint32_t)(nsig * N * K::BPC));
        for (int gg = 0; gg < nsig; ++gg) bulk_g2s(dst + gg * K::SLOT, x + (s0 + gg) * N, N * K::BPC, &full[s]);
      }
      ++p_i;
      ++p_it;
      return;
    }
  };
  if constexpr (K::INL) {
    if (tid == 0)
      for (int i = 0; i < S; ++i) produce_next();
  } else if (tid >= NT) {
    // ------------------------------------------------------------ producer
    if (tid != NT) return;
#pragma unroll 1
    while (p_item < nitems) {
      if (p_it >= S) mbar_wait_sleep(&empty[p_it % S], ((p_it / S) & 1) ^ 1);
      produce_next();
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g = tid / TPS;
  const int tau = tid % TPS;
  CT* __restrict__ y = static_cast<CT*>(a.y);
  const CT* rowp = K::ROWS ? rows : static_cast<const CT*>(a.abft.row);
  bool bad = false;
  CT s_in[ABFT ? E : 1], s_out[ABFT ? E : 1];
  if constexpr (ABFT) {
#pragma unroll
    for (int k = 0; k < E; ++k) s_in[k] = s_out[k] = mk<T>(0, 0);
  }
  int it = 0;
#pragma unroll 1
  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
    int64_t ps, pe;
    piece(item, ps, pe);
#pragma unroll 1
    for (int64_t s0 = ps;; s0 += SPT) {
      const int s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      ++it;
      CT* buf = ring + s * K::TILE + g * K::SLOT;
      const int64_t sig = s0 + g;
      const bool valid = sig < pe;
      CT v[E];
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = buf[tau + TPS * k];
      if (valid) {
#pragma unroll
        for (int k = 0; k < E; ++k) bad |= !finite2<T>(v[k]);
      }
      double red5[5] = {0, 0, 0, 0, 0};
      if constexpr (ABFT) {
        if (valid) {
          // c_in = row . x, ||x||^2 and the window sum s_in, all from the clean
          // input registers (abft.py:656-659, :602-606): fused multiply-adds
          T cr = 0, cim = 0, fl = 0;
          const T w = (T)(a.weight0 + sig + 1);
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const CT r = rowp[tau + TPS * k];
            cr = rfma(r.x, v[k].x, rfma(-r.y, v[k].y, cr));
            cim = rfma(r.x, v[k].y, rfma(r.y, v[k].x, cim));
            fl = rfma(v[k].x, v[k].x, rfma(v[k].y, v[k].y, fl));
            s_in[k] = mk<T>(rfma(w, v[k].x, s_in[k].x), rfma(w, v[k].y, s_in[k].y));
          }
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
      if constexpr (K::INL) {
        fft_sync<NT>();  // every consumer is done with stage s: refill it
        if (tid == 0) produce_next();
      } else {
        __syncwarp();
        if ((tid & 31) == 0) k5_arrive(&empty[s]);
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
#pragma unroll
          for (int k = 0; k < E; ++k)
            s_out[k] = mk<T>(rfma(w, v[k].x, s_out[k].x), rfma(w, v[k].y, s_out[k].y));
          red5[3] = (double)co.x;
          red5[4] = (double)co.y;
        }
        // per-signal totals without a CTA barrier: xor-shuffle tree inside each
        // warp; for TPS > 32 the slot's warps publish partials and the last one
        // to arrive (shared-memory counter) adds them in warp order
        constexpr int W0 = TPS < 32 ? TPS : 32;
        {
          // lane tree in working precision (the partials are working precision
          // already; halves the shuffles for FP32), then FP64 across warps
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
      if (s0 + SPT >= pe) break;
    }
    if constexpr (ABFT) {
      // ---- piece end: combine the slots' partials in slot order (s_out is
      // held at output positions: stored to wbuf at those positions)
      const int64_t wid = item / P;
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int pos = tau + TPS * (pass == 0 ? k : F::out_pos(k));
          wbuf[g * K::SLOT + pos] = pass == 0 ? s_in[k] : s_out[k];
        }
        fft_sync<NT>();
        if (g == 0) {
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const int pos = tau + TPS * k;
            CT acc = wbuf[pos];
            for (int gg = 1; gg < SPT; ++gg) acc = cadd<T>(acc, wbuf[gg * K::SLOT + pos]);
            if (pass == 0) s_in[k] = acc;
            else s_out[k] = acc;  // now at natural positions tau + TPS k
          }
        }
        fft_sync<NT>();
      }
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
        fft_sync<NT>();
        if (tid == 0) {
          const unsigned prev = atomicAdd(&a.abft.win_count[wid], 1u);
          *flag = (prev == (unsigned)(P - 1));
        }
        fft_sync<NT>();
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
      if (last) {
        // in-CTA FFT of s_in (working precision, as _fft_column) vs s_out
        const bool have = g == 0;
        CT vv[E];
#pragma unroll
        for (int k = 0; k < E; ++k) vv[k] = have ? s_in[k] : mk<T>(0, 0);
        CT* wb = wbuf + g * K::SLOT;
        F::run(wb, vv, tau, tw, 2 + g);
        // s_out of slot 0 is at natural positions: fetch the ones matching the
        // output positions through the (now free) window buffer
        fft_sync<NT>();
        if (have) {
#pragma unroll
          for (int k = 0; k < E; ++k) wb[tau + TPS * k] = s_out[k];
        }
        fft_sync<NT>();
        double r2[2] = {0, 0};
        if (have) {
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const CT so = wb[tau + TPS * F::out_pos(k)];
            const double dr = (double)vv[k].x - (double)so.x;
            const double di = (double)vv[k].y - (double)so.y;
            r2[0] += dr * dr + di * di;
            r2[1] += (double)vv[k].x * (double)vv[k].x + (double)vv[k].y * (double)vv[k].y;
          }
        }
        k5_slot_reduce<TPS, 2, NT>(r2, red, g, tau);
        if (have && tau == 0) a.abft.win_div[wid] = sqrt(r2[0]) / fmax(sqrt(r2[1]), 1e-30);
        fft_sync<NT>();
      }
#pragma unroll
      for (int k = 0; k < E; ++k) s_in[k] = s_out[k] = mk<T>(0, 0);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0 && a.counters) atomicOr(&a.counters->nonfinite, 1ull);
}

template <typename T, int LOGN, bool INV, bool ABFT>
static int launch_k5_t(const K1Args& a, int num_sms, cudaStream_t st) {
  using K = K5<T, LOGN, INV, ABFT>;
  auto kern = k5_kernel<T, LOGN, INV, ABFT>;
  static bool configured = false;
  static int per_sm = 1;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
    if (e != cudaSuccess) return (int)e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K::NTHR, K::SMEM);
    if (e != cudaSuccess) return (int)e;
    if (per_sm < 1) per_sm = 1;
    configured = true;
  }
  const int64_t nitems = ABFT ? a.abft.nwin * a.abft.pieces : (a.batch + K::SPT - 1) / K::SPT;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > nitems) grid = nitems;
  if (grid < 1) return 0;
  kern<<<(unsigned)grid, K::NTHR, K::SMEM, st>>>(a);
  return (int)cudaGetLastError();
}

template <typename T, bool INV, bool ABFT>
static int dispatch_k5(int logn, const K1Args& a, int num_sms, cudaStream_t st) {
  switch (logn) {
#define TFFT_K5(L) \
  case L: return launch_k5_t<T, L, INV, ABFT>(a, num_sms, st);
    TFFT_K5(1) TFFT_K5(2) TFFT_K5(3) TFFT_K5(4) TFFT_K5(5) TFFT_K5(6) TFFT_K5(7)
    TFFT_K5(8) TFFT_K5(9) TFFT_K5(10) TFFT_K5(11) TFFT_K5(12)
#undef TFFT_K5
    case 13:
      if constexpr (sizeof(T) == 4) return launch_k5_t<T, 13, INV, ABFT>(a, num_sms, st);
      return (int)cudaErrorInvalidValue;
    default:
      return (int)cudaErrorInvalidValue;
  }
}

int launch_k5(int prec, int logn, bool inverse, const K1Args& a, int num_sms, cudaStream_t st) {
  if (!k1_supported(prec, logn)) return (int)cudaErrorInvalidValue;
  if (prec == 0)
    return inverse ? dispatch_k5<float, true, false>(logn, a, num_sms, st)
                   : dispatch_k5<float, false, false>(logn, a, num_sms, st);
  return inverse ? dispatch_k5<double, true, false>(logn, a, num_sms, st)
                 : dispatch_k5<double, false, false>(logn, a, num_sms, st);
}

int launch_k5_abft(int prec, int logn, const K1Args& a, int num_sms, cudaStream_t st) {
  if (!k1_supported(prec, logn)) return (int)cudaErrorInvalidValue;
  return prec == 0 ? dispatch_k5<float, false, true>(logn, a, num_sms, st)
                   : dispatch_k5<double, false, true>(logn, a, num_sms, st);
}

template <typename T, int L>
static void k5_shape_t(int abft, int* spt, int* ctas_per_sm) {
  if (abft) {
    *spt = K5<T, L, false, true>::SPT;
    *ctas_per_sm = K5<T, L, false, true>::MINB;
  } else {
    *spt = K5<T, L, false, false>::SPT;
    *ctas_per_sm = K5<T, L, false, false>::MINB;
  }
}

void k5_shape(int prec, int logn, int abft, int* spt, int* ctas_per_sm) {
  *spt = 1;
  *ctas_per_sm = 1;
  switch (logn) {
#define TFFT_K5S(L) \
  case L: return prec == 0 ? k5_shape_t<float, L>(abft, spt, ctas_per_sm) : k5_shape_t<double, L>(abft, spt, ctas_per_sm);
    TFFT_K5S(1) TFFT_K5S(2) TFFT_K5S(3) TFFT_K5S(4) TFFT_K5S(5) TFFT_K5S(6) TFFT_K5S(7)
    TFFT_K5S(8) TFFT_K5S(9) TFFT_K5S(10) TFFT_K5S(11) TFFT_K5S(12)
#undef TFFT_K5S
    case 13:
      if (prec == 0) k5_shape_t<float, 13>(abft, spt, ctas_per_sm);
      return;
    default:
      return;
  }
}

}  // namespace tfft
