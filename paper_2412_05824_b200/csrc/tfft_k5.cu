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

template <typename T, int LOGN, bool INV>
struct K5 {
  static constexpr int N = 1 << LOGN;
  static constexpr int BPC = (int)sizeof(C<T>);
  static constexpr bool TWS = N * BPC <= 65536;  // per-pass twiddle tables in shared memory
  static constexpr int TPS0 = N / (16 < N ? 16 : N);
  static constexpr int NT = TPS0 > 128 ? TPS0 : 128;  // consumer threads
  using F = Fft<T, N, 16, INV, false, NT, TWS>;
  static constexpr int E = F::E;
  static constexpr int TPS = F::TPS;
  static constexpr int SPT = NT / TPS;  // signals per tile
  // slot g's signal lands at g * SLOT (linear, by the bulk copy) and the
  // passes re-lay it out padded inside the same NPAD elements; SLOT keeps the
  // bulk-copy destinations 16-byte aligned
  static constexpr int SLOT = (F::NPAD + (16 / BPC) - 1) / (16 / BPC) * (16 / BPC);
  static constexpr int TILE = SPT * SLOT;
  static constexpr int TILE_BYTES = TILE * BPC;
  // ring depth: as many stages as fit ~100 KB (two CTAs per SM), at least 2
  static constexpr int S0 = 100 * 1024 / TILE_BYTES;
  static constexpr int S = S0 < 2 ? 2 : (S0 > 4 ? 4 : S0);
  static constexpr int MINB = NT <= 128 ? 2 : 1;
  static constexpr int SMEM = S * TILE_BYTES + (TWS ? N * BPC : 0) + 2 * S * 8 + 64;
};

__device__ __forceinline__ void k5_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename T, int LOGN, bool INV>
__global__ void __launch_bounds__(K5<T, LOGN, INV>::NT + 32, K5<T, LOGN, INV>::MINB) k5_kernel(K1Args a) {
  using K = K5<T, LOGN, INV>;
  using F = typename K::F;
  using CT = C<T>;
  constexpr int N = K::N, E = K::E, TPS = K::TPS, SPT = K::SPT, S = K::S, NT = K::NT;

  extern __shared__ __align__(128) unsigned char smem[];
  CT* ring = reinterpret_cast<CT*>(smem);
  CT* tws = ring + S * K::TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(tws + (K::TWS ? N : 0));
  uint64_t* empty = full + S;

  const int tid = threadIdx.x;
  const int64_t B = a.batch;
  const int64_t ntiles = (B + SPT - 1) / SPT;
  const CT* __restrict__ x = static_cast<const CT*>(a.x);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NT / 32);
    }
    fence_mbar_init();
  }
  if constexpr (K::TWS) F::build_pass_tables(tws, static_cast<const CT*>(a.tw), tid, NT + 32);
  __syncthreads();
  const CT* tw = K::TWS ? tws : static_cast<const CT*>(a.tw);

  if (tid >= NT) {
    // ------------------------------------------------------------ producer
    if (tid != NT) return;
#pragma unroll 1
    for (int it = 0;; ++it) {
      const int64_t t = blockIdx.x + (int64_t)it * gridDim.x;
      if (t >= ntiles) return;
      const int s = it % S;
      if (it >= S) mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
      const int64_t sig0 = t * SPT;
      const int nsig = (int)(B - sig0 < SPT ? B - sig0 : SPT);
      mbar_expect_tx(&full[s], (uint32_t)(nsig * N * K::BPC));
      CT* dst = ring + s * K::TILE;
      for (int g = 0; g < nsig; ++g) bulk_g2s(dst + g * K::SLOT, x + (sig0 + g) * N, N * K::BPC, &full[s]);
    }
  }

  // -------------------------------------------------------------- consumers
  const int g = tid / TPS;
  const int tau = tid % TPS;
  CT* __restrict__ y = static_cast<CT*>(a.y);
  bool bad = false;
#pragma unroll 1
  for (int it = 0;; ++it) {
    const int64_t t = blockIdx.x + (int64_t)it * gridDim.x;
    if (t >= ntiles) break;
    const int s = it % S;
    mbar_wait(&full[s], (it / S) & 1);
    CT* buf = ring + s * K::TILE + g * K::SLOT;
    const int64_t sig = t * SPT + g;
    const bool valid = sig < B;
    CT v[E];
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = buf[tau + TPS * k];
    if (valid) {
#pragma unroll
      for (int k = 0; k < E; ++k) bad |= !finite2<T>(v[k]);
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
    F::run(buf, v, tau, tw);
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
  }
  if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0 && a.counters) atomicOr(&a.counters->nonfinite, 1ull);
}

template <typename T, int LOGN, bool INV>
static int launch_k5_t(const K1Args& a, int num_sms, cudaStream_t st) {
  using K = K5<T, LOGN, INV>;
  auto kern = k5_kernel<T, LOGN, INV>;
  static bool configured = false;
  static int per_sm = 1;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
    if (e != cudaSuccess) return (int)e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K::NT + 32, K::SMEM);
    if (e != cudaSuccess) return (int)e;
    if (per_sm < 1) per_sm = 1;
    configured = true;
  }
  const int64_t ntiles = (a.batch + K::SPT - 1) / K::SPT;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > ntiles) grid = ntiles;
  if (grid < 1) return 0;
  kern<<<(unsigned)grid, K::NT + 32, K::SMEM, st>>>(a);
  return (int)cudaGetLastError();
}

template <typename T, bool INV>
static int dispatch_k5(int logn, const K1Args& a, int num_sms, cudaStream_t st) {
  switch (logn) {
#define TFFT_K5(L) \
  case L: return launch_k5_t<T, L, INV>(a, num_sms, st);
    TFFT_K5(1) TFFT_K5(2) TFFT_K5(3) TFFT_K5(4) TFFT_K5(5) TFFT_K5(6) TFFT_K5(7)
    TFFT_K5(8) TFFT_K5(9) TFFT_K5(10) TFFT_K5(11) TFFT_K5(12)
#undef TFFT_K5
    case 13:
      if constexpr (sizeof(T) == 4) return launch_k5_t<T, 13, INV>(a, num_sms, st);
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

}  // namespace tfft
