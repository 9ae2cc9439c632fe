// Rare-path and boundary kernels.
//
//  * stockham_pass  — one radix-2/4 DIT Stockham pass over a row block with the
//    reference's exact index contract and twiddle arithmetic (w^2 = w*w,
//    w^3 = w^2*w; _kernels.pyx:38-71). It backs the plugin-boundary
//    `stockham_pass` entry point and the stage-strike path, which replays a
//    faulted transaction pass by pass so stage-k strikes hit the canonical
//    intermediate exactly where the reference's injector does (fft_core.py:271).
//  * flip_element   — the strike itself (fault.py:99-107).
//  * row_checksums  — per-signal c_in / c_out / floor / divergence for a row
//    range (abft.py:648-665); used after a strike-path rerun and on recompute.
//  * weighted_cols  — per-transaction (or per-range) location-weighted columns
//    sum_j w_j x_j (abft.py:668-677), accumulated in FP64.
//  * vec ops, group divergence and the fused correction step (abft.py:297-330,
//    392-418) for the replay engine.
#include "tfft_common.cuh"
#include "tfft_internal.h"
#include "tfft_aux.h"

namespace tfft {

// Single-column work of the replay runs at full width: CTA c owns the
// 8192-element chunk c and writes its partials; a one-warp finisher combines
// the chunks in order (deterministic). The partials come from the stream-
// ordered allocator (cudaMallocAsync / cudaFreeAsync on the caller's stream),
// so calls on different streams never share them.
constexpr int64_t kChunk = 8192;

struct ChunkScratch {
  double* p = nullptr;
  cudaStream_t st;
  ChunkScratch(int64_t n, cudaStream_t s) : st(s) {
    const size_t bytes = (size_t)((n + kChunk - 1) / kChunk) * 2 * sizeof(double);
    if (cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, st) != cudaSuccess) p = nullptr;
  }
  ~ChunkScratch() {
    if (p) cudaFreeAsync(p, st);
  }
};


// ---------------------------------------------------------------------------

template <typename T, bool INV>
__global__ void stockham_pass_kernel(const C<T>* __restrict__ src, C<T>* __restrict__ dst, int64_t rows, int64_t n,
                                     int64_t s, int r, const C<T>* __restrict__ base, int64_t base_stride) {
  using CT = C<T>;
  const int64_t nb = n / r;  // butterflies per row
  const int64_t m = n / (s * r);
  const int64_t total = rows * nb;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = id / nb;
    const int64_t j = id - row * nb;  // j = p*s + q
    const int64_t q = j % s, p = j / s;
    const CT* in = src + row * n;
    CT* out = dst + row * n;
    const CT w = base[q * base_stride];
    const int64_t sm = s * m;
    const int64_t i0 = p * s + q;
    if (r == 2) {
      const CT u0 = in[i0];
      const CT u1 = cmul<T>(in[i0 + sm], w);
      out[2 * p * s + q] = cadd<T>(u0, u1);
      out[2 * p * s + q + s] = csub<T>(u0, u1);
    } else {
      const CT w2 = cmul<T>(w, w);
      const CT w3 = cmul<T>(w2, w);
      const CT u0 = in[i0];
      const CT u1 = cmul<T>(in[i0 + sm], w);
      const CT u2 = cmul<T>(in[i0 + 2 * sm], w2);
      const CT u3 = cmul<T>(in[i0 + 3 * sm], w3);
      const CT A = cadd<T>(u0, u2), Bv = csub<T>(u0, u2);
      const CT Cv = cadd<T>(u1, u3), D = rot90<T, INV>(csub<T>(u1, u3));
      const int64_t o0 = 4 * p * s + q;
      out[o0] = cadd<T>(A, Cv);
      out[o0 + s] = cadd<T>(Bv, D);
      out[o0 + 2 * s] = csub<T>(A, Cv);
      out[o0 + 3 * s] = csub<T>(Bv, D);
    }
  }
}

int launch_stockham_pass(int prec, const void* src, void* dst, int64_t rows, int64_t n, int64_t s, int r,
                         const void* base, int64_t base_stride, int inverse, cudaStream_t st) {
  const int64_t total = rows * (n / r);
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  if (prec == 0) {
    if (inverse)
      stockham_pass_kernel<float, true><<<(unsigned)blocks, 256, 0, st>>>((const float2*)src, (float2*)dst, rows, n, s, r,
                                                                         (const float2*)base, base_stride);
    else
      stockham_pass_kernel<float, false><<<(unsigned)blocks, 256, 0, st>>>((const float2*)src, (float2*)dst, rows, n, s, r,
                                                                          (const float2*)base, base_stride);
  } else {
    if (inverse)
      stockham_pass_kernel<double, true><<<(unsigned)blocks, 256, 0, st>>>((const double2*)src, (double2*)dst, rows, n, s, r,
                                                                          (const double2*)base, base_stride);
    else
      stockham_pass_kernel<double, false><<<(unsigned)blocks, 256, 0, st>>>((const double2*)src, (double2*)dst, rows, n, s,
                                                                           r, (const double2*)base, base_stride);
  }
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------

template <typename T>
__global__ void flip_element_kernel(C<T>* buf, int64_t index, int part, int bit) {
  C<T> v = buf[index];
  if (part == 0) v.x = flip_bits(v.x, bit);
  else v.y = flip_bits(v.y, bit);
  buf[index] = v;
}

__global__ void base_table_kernel(float2* f, double2* d, int64_t s, int r, int inverse) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < s; q += (int64_t)gridDim.x * blockDim.x) {
    double sn, cs;
    sincospi(-2.0 * (double)q / ((double)s * r), &sn, &cs);
    if (q == 0) {
      sn = 0;
      cs = 1;
    }
    if (inverse) sn = -sn;
    if (f) f[q] = make_float2((float)cs, (float)sn);
    else d[q] = make_double2(cs, sn);
  }
}

// omega_(s r)^q for q < s (conj for inverse), FP64 sincospi rounded once
int launch_base_table(int prec, int64_t s, int r, int inverse, void* dst, cudaStream_t st) {
  int64_t blocks = (s + 255) / 256;
  if (blocks > 1024) blocks = 1024;
  base_table_kernel<<<(unsigned)blocks, 256, 0, st>>>(prec == 0 ? (float2*)dst : nullptr,
                                                        prec == 0 ? nullptr : (double2*)dst, s, r, inverse);
  return (int)cudaGetLastError();
}

int launch_flip(int prec, void* buf, int64_t index, int part, int bit, cudaStream_t st) {
  if (prec == 0) flip_element_kernel<float><<<1, 1, 0, st>>>((float2*)buf, index, part, bit);
  else flip_element_kernel<double><<<1, 1, 0, st>>>((double2*)buf, index, part, bit);
  return (int)cudaGetLastError();
}

template <typename T>
__global__ void scale_kernel(C<T>* buf, int64_t count, T s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = cscale<T>(buf[i], s);
}

int launch_scale(int prec, void* buf, int64_t count, double s, cudaStream_t st) {
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (prec == 0) scale_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((float2*)buf, count, (float)s);
  else scale_kernel<double><<<(unsigned)blocks, 256, 0, st>>>((double2*)buf, count, s);
  return (int)cudaGetLastError();
}

template <typename T>
__global__ void nonfinite_kernel(const C<T>* __restrict__ buf, int64_t count, Counters* counters) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !finite2<T>(__ldcs(buf + i));
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&counters->nonfinite, 1ull);
}

int launch_nonfinite(int prec, const void* buf, int64_t count, Counters* counters, cudaStream_t st) {
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (prec == 0) nonfinite_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((const float2*)buf, count, counters);
  else nonfinite_kernel<double><<<(unsigned)blocks, 256, 0, st>>>((const double2*)buf, count, counters);
  return (int)cudaGetLastError();
}

// Window sums of the TMEM-fused K5 ABFT: window w's s_in / s_out = the sum of
// the partials of every (CTA segment, slot) that covers part of it, added in
// CTA then slot order (deterministic; tfft_k5.cu writes ws[(c*maxseg + j)*spt
// + g][2][n] for CTA c's j-th segment).
template <typename T>
__global__ void seg_combine_kernel(const C<T>* __restrict__ ws, int64_t n, int64_t B, int64_t W, int64_t G,
                                   int64_t maxseg, int spt, C<T>* __restrict__ s_in, C<T>* __restrict__ s_out) {
  const int64_t w = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t w0 = w * W, w1 = min(w0 + W, B);
  int64_t c = w0 * G / B;
  while (c > 0 && c * B / G > w0) --c;
  while (c < G && (c + 1) * B / G <= w0) ++c;
  C<T> ai = mk<T>(0, 0), ao = mk<T>(0, 0);
  for (; c < G; ++c) {
    const int64_t lo = c * B / G, hi = (c + 1) * B / G;
    if (lo >= w1) break;
    if (hi <= lo) continue;
    const int64_t j = w - lo / W;
    for (int g = 0; g < spt; ++g) {
      const C<T>* base = ws + ((c * maxseg + j) * spt + g) * 2 * n;
      ai = cadd<T>(ai, base[i]);
      ao = cadd<T>(ao, base[n + i]);
    }
  }
  s_in[w * n + i] = ai;
  s_out[w * n + i] = ao;
}

int launch_seg_combine(int prec, const void* ws, int64_t n, int64_t B, int64_t W, int64_t G, int64_t maxseg, int spt,
                       int64_t nwin, void* s_in, void* s_out, cudaStream_t st) {
  const dim3 grid((unsigned)((n + 255) / 256), (unsigned)nwin);
  if (prec == 0)
    seg_combine_kernel<float><<<grid, 256, 0, st>>>((const float2*)ws, n, B, W, G, maxseg, spt, (float2*)s_in,
                                                     (float2*)s_out);
  else
    seg_combine_kernel<double><<<grid, 256, 0, st>>>((const double2*)ws, n, B, W, G, maxseg, spt, (double2*)s_in,
                                                      (double2*)s_out);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// block-wide deterministic FP64 sum (fixed tree), 256 threads

template <int NV>
__device__ __forceinline__ void block_sum256(double (&r)[NV], double* sh) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
    for (int k = 0; k < NV; ++k) r[k] += __shfl_xor_sync(0xffffffffu, r[k], off);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) sh[w * NV + k] = r[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double acc = sh[k];
      for (int i = 1; i < 8; ++i) acc += sh[i * NV + k];
      r[k] = acc;
    }
  }
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ C<T> enc_value(int enc, int64_t k, int64_t n, const C<T>* tw) {
  if (enc == ENC_WANG) {
    const int m = (int)(k % 3);
    const T h = (T)0.86602540378443864676372317075294;
    return m == 0 ? mk<T>(1, 0) : (m == 1 ? mk<T>((T)-0.5, -h) : mk<T>((T)-0.5, h));
  }
  if (enc == ENC_ONES) return mk<T>(1, 0);
  return tw[k];
}

// one CTA per signal row: c_in, c_out, floor, div; bumps the counters
template <typename T>
__global__ void __launch_bounds__(256) row_checksums_kernel(const C<T>* __restrict__ x, const C<T>* __restrict__ y,
                                                            int64_t n, int64_t row0, const C<T>* __restrict__ row,
                                                            const C<T>* __restrict__ tw, int enc, double delta,
                                                            double* c_in, double* c_out, double* floors, double* div,
                                                            Counters* counters, int count) {
  __shared__ double sh[8 * 5];
  const int64_t r = row0 + blockIdx.x;
  const C<T>* xr = x + r * n;
  const C<T>* yr = y + r * n;
  C<T> ci = mk<T>(0, 0), co = mk<T>(0, 0);
  T fl = 0;
  for (int64_t k = threadIdx.x; k < n; k += 256) {
    const C<T> xv = xr[k], yv = yr[k];
    ci = cadd<T>(ci, cmul<T>(row[k], xv));
    fl = rfma(xv.x, xv.x, rfma(xv.y, xv.y, fl));
    co = cadd<T>(co, cmul<T>(enc_value<T>(enc, k, n, tw), yv));
  }
  double acc[5] = {(double)ci.x, (double)ci.y, (double)fl, (double)co.x, (double)co.y};
  block_sum256<5>(acc, sh);
  if (threadIdx.x == 0) {
    const double floor_v = sqrt(acc[2]) / sqrt((double)n);
    double dv;
    if (!isfinite(acc[3]) || !isfinite(acc[4])) dv = __longlong_as_double(0x7ff0000000000000ll);
    else dv = hypot(acc[0] - acc[3], acc[1] - acc[4]) / fmax(fmax(hypot(acc[0], acc[1]), floor_v), 1e-30);
    c_in[2 * r] = acc[0];
    c_in[2 * r + 1] = acc[1];
    c_out[2 * r] = acc[3];
    c_out[2 * r + 1] = acc[4];
    floors[r] = floor_v;
    div[r] = dv;
    if (count) {
      if (dv > delta) atomicAdd(&counters->triggered, 1ull);
      atomicMax(&counters->max_div_bits, (unsigned long long)__double_as_longlong(dv));
    }
  }
}

int launch_row_checksums(int prec, const void* x, const void* y, int64_t n, int64_t row0, int64_t nrows,
                         const void* row, const void* tw, int enc, double delta, const AbftArgs& ab, Counters* counters,
                         int count, cudaStream_t st) {
  if (nrows <= 0) return 0;
  if (prec == 0)
    row_checksums_kernel<float><<<(unsigned)nrows, 256, 0, st>>>((const float2*)x, (const float2*)y, n, row0,
                                                                (const float2*)row, (const float2*)tw, enc, delta,
                                                                ab.c_in, ab.c_out, ab.floors, ab.div, counters, count);
  else
    row_checksums_kernel<double><<<(unsigned)nrows, 256, 0, st>>>((const double2*)x, (const double2*)y, n, row0,
                                                                 (const double2*)row, (const double2*)tw, enc, delta,
                                                                 ab.c_in, ab.c_out, ab.floors, ab.div, counters, count);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// weighted column sums: out[g][k] = sum_{j in group g} (weight0 + j + 1) * src[j][k]
// groups are consecutive row ranges of `gsize` rows starting at row0 (last short)

template <typename T>
__global__ void weighted_cols_kernel(const C<T>* __restrict__ src, int64_t n, int64_t row0, int64_t row1,
                                     int64_t gsize, int64_t weight0, C<T>* __restrict__ out) {
  const int64_t ngroups = (row1 - row0 + gsize - 1) / gsize;
  const int64_t total = ngroups * n;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gidx = id / n, k = id - gidx * n;
    const int64_t a = row0 + gidx * gsize, b = min(a + gsize, row1);
    double re = 0, im = 0;
    for (int64_t j = a; j < b; ++j) {
      const C<T> v = src[j * n + k];
      const double w = (double)(weight0 + j + 1);
      re = fma(w, (double)v.x, re);
      im = fma(w, (double)v.y, im);
    }
    out[id] = mk<T>((T)re, (T)im);
  }
}

int launch_weighted_cols(int prec, const void* src, int64_t n, int64_t row0, int64_t row1, int64_t gsize,
                         int64_t weight0, void* out, cudaStream_t st) {
  const int64_t ngroups = (row1 - row0 + gsize - 1) / gsize;
  int64_t blocks = (ngroups * n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) return 0;
  if (prec == 0)
    weighted_cols_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((const float2*)src, n, row0, row1, gsize, weight0,
                                                                 (float2*)out);
  else
    weighted_cols_kernel<double><<<(unsigned)blocks, 256, 0, st>>>((const double2*)src, n, row0, row1, gsize, weight0,
                                                                  (double2*)out);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Batched online correction of single-trigger windows (tfft_correct_windows).
// Item i: transaction rows [r0, r1) holding the triggered signal k, window
// rows [w0, w1), weight w = weight0 + k + 1, floor, c_in (desc / par arrays).

// out[i][k] = sum_{j in [ra_i, rb_i)} (weight0 + j + 1) src[j][k]; same
// arithmetic as weighted_cols_kernel (FP64 fma, rounded once)
template <typename T>
__global__ void wsum_list_kernel(const C<T>* __restrict__ src, int64_t n, const int64_t* __restrict__ desc, int lo,
                                 int hi, int64_t weight0, C<T>* __restrict__ out) {
  const int64_t i = blockIdx.y;
  const int64_t ra = desc[i * 6 + lo], rb = desc[i * 6 + hi];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    double re = 0, im = 0;
    for (int64_t j = ra; j < rb; ++j) {
      const C<T> v = src[j * n + k];
      const double w = (double)(weight0 + j + 1);
      re = fma(w, (double)v.x, re);
      im = fma(w, (double)v.y, im);
    }
    out[i * n + k] = mk<T>((T)re, (T)im);
  }
}

int launch_wsum_list(int prec, const void* src, int64_t n, const int64_t* desc_dev, int lo, int hi, int64_t count,
                     int64_t weight0, void* out, cudaStream_t st) {
  if (count < 1) return 0;
  unsigned bx = (unsigned)((n + 255) / 256);
  if (bx > 64) bx = 64;
  const dim3 grid(bx, (unsigned)count);
  if (prec == 0)
    wsum_list_kernel<float><<<grid, 256, 0, st>>>((const float2*)src, n, desc_dev, lo, hi, weight0, (float2*)out);
  else
    wsum_list_kernel<double><<<grid, 256, 0, st>>>((const double2*)src, n, desc_dev, lo, hi, weight0, (double2*)out);
  return (int)cudaGetLastError();
}

// rows src[idx_i] (n each) -> dst[i]: gathers window sums into a batch
template <typename T>
__global__ void gather_rows_kernel(const C<T>* __restrict__ src, int64_t stride, const int64_t* __restrict__ desc,
                                   int col, int64_t n, C<T>* __restrict__ dst) {
  const int64_t i = blockIdx.y, r = desc[i * 6 + col];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    dst[i * n + k] = src[r * stride + k];
}

int launch_gather_rows(int prec, const void* src, int64_t stride, const int64_t* desc_dev, int col, int64_t count,
                       int64_t n, void* dst, cudaStream_t st) {
  if (count < 1) return 0;
  unsigned bx = (unsigned)((n + 255) / 256);
  if (bx > 64) bx = 64;
  const dim3 grid(bx, (unsigned)count);
  if (prec == 0)
    gather_rows_kernel<float><<<grid, 256, 0, st>>>((const float2*)src, stride, desc_dev, col, n, (float2*)dst);
  else
    gather_rows_kernel<double><<<grid, 256, 0, st>>>((const double2*)src, stride, desc_dev, col, n, (double2*)dst);
  return (int)cudaGetLastError();
}

// col_i = (t_out_i - ref_i) / w_i in FP64, cast (abft.py:297-317); chunk
// partials {non-finite count, max|col|} per (item, chunk)
template <typename T, typename R>
__global__ void __launch_bounds__(256) corr_cols_kernel(const C<T>* __restrict__ tout, const R* __restrict__ ref,
                                                        const double* __restrict__ par, int64_t n, int64_t nc,
                                                        C<T>* __restrict__ col, double* __restrict__ part) {
  __shared__ double sh[8 * 2];
  const int64_t i = blockIdx.y, c = blockIdx.x;
  const double w = par[i * 4];
  double acc[2] = {0, 0};
  const int64_t k0 = c * kChunk, k1 = min(k0 + kChunk, n);
  for (int64_t k = k0 + threadIdx.x; k < k1; k += 256) {
    const C<T> to = tout[i * n + k];
    const R rf = ref[i * n + k];
    double re, im;
    if (sizeof(T) == 4) {  // FP32 data: the column is formed in FP64
      re = ((double)to.x - (double)rf.x) / w;
      im = ((double)to.y - (double)rf.y) / w;
    } else {  // FP64: working precision, divided by the weight in it
      re = (double)(((T)to.x - (T)rf.x) / (T)w);
      im = (double)(((T)to.y - (T)rf.y) / (T)w);
    }
    const C<T> v = mk<T>((T)re, (T)im);
    col[i * n + k] = v;
    if (!isfinite((double)v.x) || !isfinite((double)v.y)) acc[0] += 1.0;
    else acc[1] = fmax(acc[1], hypot((double)v.x, (double)v.y));
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], off);
    acc[1] = fmax(acc[1], __shfl_xor_sync(0xffffffffu, acc[1], off));
  }
  if ((threadIdx.x & 31) == 0) {
    sh[(threadIdx.x >> 5) * 2] = acc[0];
    sh[(threadIdx.x >> 5) * 2 + 1] = acc[1];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bad = 0, mx = 0;
    for (int q = 0; q < 8; ++q) {
      bad += sh[2 * q];
      mx = fmax(mx, sh[2 * q + 1]);
    }
    part[(i * nc + c) * 2] = bad;
    part[(i * nc + c) * 2 + 1] = mx;
  }
}

// usable_i = all finite && max|col| <= 16 log2N floor sqrt(N) (abft.py:320-330)
__global__ void corr_usable_kernel(const double* part, int64_t nc, int64_t count, const double* par, double limit_scale,
                                   double* res) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  double bad = 0, mx = 0;
  for (int64_t c = 0; c < nc; ++c) {
    bad += part[(i * nc + c) * 2];
    mx = fmax(mx, part[(i * nc + c) * 2 + 1]);
  }
  res[i * 4 + 0] = (bad == 0 && mx <= limit_scale * par[i * 4 + 1]) ? 1.0 : 0.0;
  res[i * 4 + 3] = bad == 0 ? mx : __longlong_as_double(0x7ff0000000000000ll);
}

// re-verify: c_out' = (y_k - col) . enc in working precision per thread,
// chunk partials in FP64 (patch_row_kernel's arithmetic) -- y is not written
template <typename T>
__global__ void __launch_bounds__(256) corr_reverify_kernel(const C<T>* __restrict__ y, const C<T>* __restrict__ col,
                                                            const int64_t* __restrict__ desc, int64_t n, int64_t nc,
                                                            int enc, const C<T>* __restrict__ tw,
                                                            double* __restrict__ part) {
  __shared__ double sh[8 * 2];
  const int64_t i = blockIdx.y, c = blockIdx.x;
  const C<T>* yk = y + desc[i * 6] * n;
  C<T> co = mk<T>(0, 0);
  const int64_t k0 = c * kChunk, k1 = min(k0 + kChunk, n);
  for (int64_t k = k0 + threadIdx.x; k < k1; k += 256) {
    const C<T> v = csub<T>(yk[k], col[i * n + k]);
    co = cadd<T>(co, cmul<T>(enc_value<T>(enc, k, n, tw), v));
  }
  double acc[2] = {(double)co.x, (double)co.y};
  block_sum256<2>(acc, sh);
  if (threadIdx.x == 0) {
    part[(i * nc + c) * 2] = acc[0];
    part[(i * nc + c) * 2 + 1] = acc[1];
  }
}

// detect(c_in, c_out', delta, floor) (abft.py:155-167); res[i*4+1] = divergence,
// res[i*4+0] = 1 only when usable and the re-verify holds
__global__ void corr_decide_kernel(const double* part, int64_t nc, int64_t count, const double* par, double delta,
                                   double* res) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  double a = 0, b = 0;
  for (int64_t c = 0; c < nc; ++c) {
    a += part[(i * nc + c) * 2];
    b += part[(i * nc + c) * 2 + 1];
  }
  const double cr = par[i * 4 + 2], ci = par[i * 4 + 3], fl = par[i * 4 + 1];
  double dv;
  if (!isfinite(a) || !isfinite(b)) dv = __longlong_as_double(0x7ff0000000000000ll);
  else dv = hypot(cr - a, ci - b) / fmax(fmax(hypot(cr, ci), fl), 1e-30);
  res[i * 4 + 1] = dv;
  if (!(dv <= delta)) res[i * 4 + 0] = 0.0;
}

// commit for the items that passed: y_k -= col; s_out_i -= w col (working precision)
template <typename T>
__global__ void corr_commit_kernel(C<T>* __restrict__ y, const C<T>* __restrict__ col, const int64_t* __restrict__ desc,
                                   const double* __restrict__ par, const double* __restrict__ res, int64_t n,
                                   C<T>* __restrict__ s_out) {
  const int64_t i = blockIdx.y;
  if (res[i * 4] != 1.0) return;
  C<T>* yk = y + desc[i * 6] * n;
  const T w = (T)par[i * 4];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const C<T> cv = col[i * n + k];
    yk[k] = csub<T>(yk[k], cv);
    const C<T> so = s_out[i * n + k];
    s_out[i * n + k] = csub<T>(so, mk<T>(w * cv.x, w * cv.y));
  }
}

int launch_correct_items(int prec, void* y, const int64_t* desc_dev, const double* par_dev, int64_t count, int64_t n,
                         const void* tout, const void* ref64_or_ref, void* col, int enc, const void* tw, double delta,
                         void* s_out, double* part, double* res_dev, cudaStream_t st) {
  if (count < 1) return 0;
  const int64_t nc = (n + kChunk - 1) / kChunk;
  const dim3 g2((unsigned)nc, (unsigned)count);
  double lg = 0;
  for (int64_t v = n; v > 1; v >>= 1) lg += 1.0;
  const double limit_scale = 16.0 * lg * sqrt((double)n);
  const unsigned gb = (unsigned)((count + 127) / 128);
  if (prec == 0) {
    corr_cols_kernel<float, double2><<<g2, 256, 0, st>>>((const float2*)tout, (const double2*)ref64_or_ref, par_dev,
                                                         n, nc, (float2*)col, part);
  } else {
    corr_cols_kernel<double, double2><<<g2, 256, 0, st>>>((const double2*)tout, (const double2*)ref64_or_ref,
                                                          par_dev, n, nc, (double2*)col, part);
  }
  corr_usable_kernel<<<gb, 128, 0, st>>>(part, nc, count, par_dev, limit_scale, res_dev);
  if (prec == 0)
    corr_reverify_kernel<float><<<g2, 256, 0, st>>>((const float2*)y, (const float2*)col, desc_dev, n, nc, enc,
                                                    (const float2*)tw, part);
  else
    corr_reverify_kernel<double><<<g2, 256, 0, st>>>((const double2*)y, (const double2*)col, desc_dev, n, nc, enc,
                                                     (const double2*)tw, part);
  corr_decide_kernel<<<gb, 128, 0, st>>>(part, nc, count, par_dev, delta, res_dev);
  unsigned bx = (unsigned)((n + 255) / 256);
  if (bx > 64) bx = 64;
  const dim3 g3(bx, (unsigned)count);
  if (prec == 0)
    corr_commit_kernel<float><<<g3, 256, 0, st>>>((float2*)y, (const float2*)col, desc_dev, par_dev, res_dev, n,
                                                  (float2*)s_out);
  else
    corr_commit_kernel<double><<<g3, 256, 0, st>>>((double2*)y, (const double2*)col, desc_dev, par_dev, res_dev, n,
                                                   (double2*)s_out);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// one-sweep ABFT sums for the two-pass sizes: a CTA owns (window w, chunk of
// CH = 256 * V = 1024 (FP32) / 512 (FP64) elements) and walks the window's signals once, reading x and y
// exactly once per element. It accumulates the window sums s_in / s_out for
// its chunk (working precision, as the reference's GEMV) and, per signal, the chunk's
// partial c_in = row . x, ||x||^2 and c_out = e . y (working precision per
// thread, FP64 xor tree per warp), written to part[signal][chunk][warp][5]
// with no barrier in the signal loop; sweep_epilogue adds the partials in
// (chunk, warp) order per signal.

template <typename T, int V, int D, int MINB>
__global__ void __launch_bounds__(256, MINB) window_sweep_kernel(const C<T>* __restrict__ x, const C<T>* __restrict__ y,
                                                        int64_t n, int64_t batch, int64_t W, int64_t weight0,
                                                        const C<T>* __restrict__ row, const C<T>* __restrict__ tw,
                                                        int enc, C<T>* __restrict__ s_in, C<T>* __restrict__ s_out,
                                                        double* __restrict__ part) {
  constexpr int CH = 256 * V;
  const int64_t nchunk = (n + CH - 1) / CH;
  const int64_t w = blockIdx.x / nchunk, c = blockIdx.x % nchunk;
  const int64_t j0 = w * W, j1 = min(j0 + W, batch);
  const int64_t kb = c * CH + threadIdx.x;
  // window sums in working precision, as the reference's GEMV (abft.py:605-606)
  C<T> a_in[V], a_out[V], rw[V], ev[V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    a_in[i] = a_out[i] = mk<T>(0, 0);
    const int64_t k = kb + 256 * i;
    rw[i] = k < n ? row[k] : mk<T>(0, 0);
    ev[i] = k < n ? enc_value<T>(enc, k, n, tw) : mk<T>(0, 0);
  }
  // register ring of D signals: signal j's slot is refilled with j + D right
  // after j is reduced, so D signals' loads are in flight per thread
  C<T> xb[D][V], yb[D][V];
  auto load = [&](int64_t j, C<T>(&xa)[V], C<T>(&ya)[V]) {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int64_t k = kb + 256 * i;
      xa[i] = (j < j1 && k < n) ? __ldcs(x + j * n + k) : mk<T>(0, 0);
      ya[i] = (j < j1 && k < n) ? __ldcs(y + j * n + k) : mk<T>(0, 0);
    }
  };
#pragma unroll
  for (int d = 0; d < D; ++d) load(j0 + d, xb[d], yb[d]);
#pragma unroll 1
  for (int64_t jb = j0; jb < j1; jb += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int64_t j = jb + d;
      if (j < j1) {
        const T wj = (T)(weight0 + j + 1);
        C<T> ci = mk<T>(0, 0), co = mk<T>(0, 0);
        T fl = 0;
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const C<T> xv = xb[d][i], yv = yb[d][i];
          ci = cadd<T>(ci, cmul<T>(rw[i], xv));
          fl = rfma(xv.x, xv.x, rfma(xv.y, xv.y, fl));
          co = cadd<T>(co, cmul<T>(ev[i], yv));
          a_in[i] = mk<T>(rfma(wj, xv.x, a_in[i].x), rfma(wj, xv.y, a_in[i].y));
          a_out[i] = mk<T>(rfma(wj, yv.x, a_out[i].x), rfma(wj, yv.y, a_out[i].y));
        }
        // warp partials: fixed xor tree in working precision (the products are
        // working precision already), no CTA barrier inside the signal loop
        T acc[5] = {ci.x, ci.y, fl, co.x, co.y};
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
          for (int q = 0; q < 5; ++q) acc[q] = radd(acc[q], __shfl_xor_sync(0xffffffffu, acc[q], off));
        if ((threadIdx.x & 31) == 0)
#pragma unroll
          for (int q = 0; q < 5; ++q) part[((j * nchunk + c) * 8 + (threadIdx.x >> 5)) * 5 + q] = (double)acc[q];
      }
      load(j + D, xb[d], yb[d]);
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int64_t k = kb + 256 * i;
    if (k < n) {
      s_in[w * n + k] = a_in[i];
      s_out[w * n + k] = a_out[i];
    }
  }
}

// one warp per signal: lanes take (chunk, warp) partials i = lane, lane + 32,
// ... in order, then a fixed xor tree
__global__ void sweep_epilogue_kernel(const double* __restrict__ part, int64_t nparts, int64_t n, int64_t batch,
                                      double delta, double* c_in, double* c_out, double* floors, double* div,
                                      Counters* counters) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  double dmax = 0.0;  // one atomicMax per warp, not per signal
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < batch; r += nwarps) {
    double acc[5] = {0, 0, 0, 0, 0};
    for (int64_t i = lane; i < nparts; i += 32)
#pragma unroll
      for (int q = 0; q < 5; ++q) acc[q] += part[(r * nparts + i) * 5 + q];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
      for (int q = 0; q < 5; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
    if (lane != 0) continue;
    const double floor_v = sqrt(acc[2]) / sqrt((double)n);
    double dv;
    if (!isfinite(acc[3]) || !isfinite(acc[4])) dv = __longlong_as_double(0x7ff0000000000000ll);
    else dv = hypot(acc[0] - acc[3], acc[1] - acc[4]) / fmax(fmax(hypot(acc[0], acc[1]), floor_v), 1e-30);
    c_in[2 * r] = acc[0];
    c_in[2 * r + 1] = acc[1];
    c_out[2 * r] = acc[3];
    c_out[2 * r + 1] = acc[4];
    floors[r] = floor_v;
    div[r] = dv;
    if (dv > delta) atomicAdd(&counters->triggered, 1ull);
    dmax = fmax(dmax, dv);
  }
  if (lane == 0 && dmax > 0.0) atomicMax(&counters->max_div_bits, (unsigned long long)__double_as_longlong(dmax));
}

int launch_signal_epilogue(const double* part, int64_t nparts, int64_t n, int64_t batch, double delta,
                           const AbftArgs& ab, Counters* counters, cudaStream_t st) {
  int64_t eb = (batch + 7) / 8;
  if (eb > 148 * 16) eb = 148 * 16;
  if (eb < 1) return 0;
  sweep_epilogue_kernel<<<(unsigned)eb, 256, 0, st>>>(part, nparts, n, batch, delta, ab.c_in, ab.c_out, ab.floors,
                                                      ab.div, counters);
  return (int)cudaGetLastError();
}

int64_t window_sweep_chunks(int64_t n) { return (n + 511) / 512; }  // upper bound (FP64 V = 2 -> 512 per chunk)

int launch_window_sweep(int prec, const void* x, const void* y, int64_t n, int64_t batch, int64_t W, int64_t weight0,
                        const void* row, const void* tw, int enc, void* s_in, void* s_out, double* part,
                        const AbftArgs& ab, double delta, Counters* counters, cudaStream_t st) {
  const int64_t nwin = (batch + W - 1) / W;
  // (V, D) = FP32 (4, 3), FP64 (2, 3): best of (8,1) (4,4) (2,6) / (1,6) (1,4)
  // (2,4) on B200 (tools/abft_ab.py with the sweep route, 1 GiB, T = 8)
  const int V = prec == 0 ? 4 : 2;
  const int64_t nchunk = (n + 256 * V - 1) / (256 * V);
  const int64_t blocks = nwin * nchunk;
  if (blocks <= 0) return 0;
  if (prec == 0)
    window_sweep_kernel<float, 4, 3, 2><<<(unsigned)blocks, 256, 0, st>>>(
        (const float2*)x, (const float2*)y, n, batch, W, weight0, (const float2*)row, (const float2*)tw, enc,
        (float2*)s_in, (float2*)s_out, part);
  else
    window_sweep_kernel<double, 2, 3, 2><<<(unsigned)blocks, 256, 0, st>>>(
        (const double2*)x, (const double2*)y, n, batch, W, weight0, (const double2*)row, (const double2*)tw, enc,
        (double2*)s_in, (double2*)s_out, part);
  int e = (int)cudaGetLastError();
  if (e) return e;
  int64_t eb = (batch + 7) / 8;
  if (eb > 148 * 16) eb = 148 * 16;
  sweep_epilogue_kernel<<<(unsigned)eb, 256, 0, st>>>(part, nchunk * 8, n, batch, delta, ab.c_in, ab.c_out,
                                                      ab.floors, ab.div, counters);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// z = a*x + b*y (complex scalars a, b given in FP64; x or y may be null)

template <typename T>
__global__ void axpby_kernel(C<T>* z, int64_t n, double ar, double ai, const C<T>* x, double br, double bi,
                             const C<T>* y) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    C<T> acc = mk<T>(0, 0);
    if (x) acc = cadd<T>(acc, cmul<T>(mk<T>((T)ar, (T)ai), x[k]));
    if (y) acc = cadd<T>(acc, cmul<T>(mk<T>((T)br, (T)bi), y[k]));
    z[k] = acc;
  }
}

int launch_axpby(int prec, void* z, int64_t n, double ar, double ai, const void* x, double br, double bi,
                 const void* y, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) return 0;
  if (prec == 0)
    axpby_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((float2*)z, n, ar, ai, (const float2*)x, br, bi,
                                                         (const float2*)y);
  else
    axpby_kernel<double><<<(unsigned)blocks, 256, 0, st>>>((double2*)z, n, ar, ai, (const double2*)x, br, bi,
                                                          (const double2*)y);
  return (int)cudaGetLastError();
}

// plain sum a = a + b in working precision (the replay's s_in += t_in)
template <typename T>
__global__ void vadd_kernel(C<T>* a, const C<T>* b, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    a[k] = cadd<T>(a[k], b[k]);
}

int launch_vadd(int prec, void* a, const void* b, int64_t n, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) return 0;
  if (prec == 0) vadd_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((float2*)a, (const float2*)b, n);
  else vadd_kernel<double><<<(unsigned)blocks, 256, 0, st>>>((double2*)a, (const double2*)b, n);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// group divergence ||ref - s_out||_2 / max(||ref||_2, 1e-30) (abft.py:502-507)

template <typename T>
__global__ void __launch_bounds__(256) group_div_kernel(const C<T>* ref, const C<T>* s_out, int64_t n, double* out) {
  __shared__ double sh[8 * 2];
  ref += blockIdx.x * n;
  s_out += blockIdx.x * n;
  out += blockIdx.x;
  double acc[2] = {0, 0};
  for (int64_t k = threadIdx.x; k < n; k += 256) {
    const double dr = (double)ref[k].x - (double)s_out[k].x;
    const double di = (double)ref[k].y - (double)s_out[k].y;
    acc[0] += dr * dr + di * di;
    acc[1] += (double)ref[k].x * (double)ref[k].x + (double)ref[k].y * (double)ref[k].y;
  }
  block_sum256<2>(acc, sh);
  if (threadIdx.x == 0) *out = sqrt(acc[0]) / fmax(sqrt(acc[1]), 1e-30);
}

int launch_group_div(int prec, const void* ref, const void* s_out, int64_t n, double* out, cudaStream_t st) {
  if (n >= 65536) {  // one long row: chunk partials at full width, combined in order
    ChunkScratch scratch(n, st);
    double* part = scratch.p;
    if (!part) return (int)cudaErrorMemoryAllocation;
    return launch_group_div_chunked(prec, ref, s_out, n, 1, out, part, st);
  }
  return launch_group_div_batched(prec, ref, s_out, n, 1, out, st);
}

// chunked group divergence for long rows: partials per (window, 8192-element
// chunk), then one warp per window adds them in chunk order
template <typename T>
__global__ void __launch_bounds__(256) group_div_part_kernel(const C<T>* __restrict__ ref, const C<T>* __restrict__ s_out,
                                                             int64_t n, int64_t nchunk, double* part) {
  __shared__ double sh[8 * 2];
  const int64_t w = blockIdx.x / nchunk, c = blockIdx.x % nchunk;
  const int64_t k0 = c * 8192, k1 = min(k0 + 8192, n);
  double acc[2] = {0, 0};
  for (int64_t k = k0 + threadIdx.x; k < k1; k += 256) {
    const C<T> r = __ldcs(ref + w * n + k), so = __ldcs(s_out + w * n + k);
    const double dr = (double)r.x - (double)so.x, di = (double)r.y - (double)so.y;
    acc[0] += dr * dr + di * di;
    acc[1] += (double)r.x * (double)r.x + (double)r.y * (double)r.y;
  }
  block_sum256<2>(acc, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 2] = acc[0];
    part[blockIdx.x * 2 + 1] = acc[1];
  }
}

__global__ void group_div_fin_kernel(const double* part, int64_t nchunk, int64_t count, double* out) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= count) return;
  double a = 0, b = 0;
  for (int64_t c = 0; c < nchunk; ++c) {
    a += part[(w * nchunk + c) * 2];
    b += part[(w * nchunk + c) * 2 + 1];
  }
  out[w] = sqrt(a) / fmax(sqrt(b), 1e-30);
}

int launch_group_div_chunked(int prec, const void* ref, const void* s_out, int64_t n, int64_t count, double* out,
                             double* part, cudaStream_t st) {
  if (count < 1) return 0;
  const int64_t nchunk = (n + 8191) / 8192;
  const int64_t blocks = count * nchunk;
  if (prec == 0)
    group_div_part_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((const float2*)ref, (const float2*)s_out, n, nchunk,
                                                                   part);
  else
    group_div_part_kernel<double><<<(unsigned)blocks, 256, 0, st>>>((const double2*)ref, (const double2*)s_out, n,
                                                                    nchunk, part);
  int e = (int)cudaGetLastError();
  if (e) return e;
  group_div_fin_kernel<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(part, nchunk, count, out);
  return (int)cudaGetLastError();
}

// one CTA per window: row w of ref / s_out -> out[w]
int launch_group_div_batched(int prec, const void* ref, const void* s_out, int64_t n, int64_t count, double* out,
                             cudaStream_t st) {
  if (count < 1) return 0;
  for (int64_t w0 = 0; w0 < count; w0 += 65535) {
    const int64_t cnt = count - w0 < 65535 ? count - w0 : 65535;
    if (prec == 0)
      group_div_kernel<float><<<(unsigned)cnt, 256, 0, st>>>((const float2*)ref + w0 * n, (const float2*)s_out + w0 * n,
                                                            n, out + w0);
    else
      group_div_kernel<double><<<(unsigned)cnt, 256, 0, st>>>((const double2*)ref + w0 * n,
                                                             (const double2*)s_out + w0 * n, n, out + w0);
  }
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// correction column (abft.py:297-330): col = (snap_out - ref64) / w_k, formed in
// FP64 (ref64 is the FP64 transform of the snapshot input), cast to working
// precision; report finiteness and max|col| so the host applies the usability
// rule. Then, if asked, patch y_k -= col and re-form c_out = y_k . enc.
// res: [0] all finite (1/0), [1] max |col|, [2] c_out re, [3] c_out im

template <typename T>
__global__ void __launch_bounds__(256) correction_column_kernel(const C<T>* snap_out, const double2* ref64, int64_t n,
                                                                double weight, C<T>* col, double* part) {
  __shared__ double sh[8 * 2];
  double acc[2] = {0, 0};  // [0] non-finite count, [1] max |col|
  const int64_t k0 = blockIdx.x * kChunk, k1 = min(k0 + kChunk, n);
  for (int64_t k = k0 + threadIdx.x; k < k1; k += 256) {
    const double re = ((double)snap_out[k].x - ref64[k].x) / weight;
    const double im = ((double)snap_out[k].y - ref64[k].y) / weight;
    const C<T> c = mk<T>((T)re, (T)im);
    col[k] = c;
    if (!isfinite((double)c.x) || !isfinite((double)c.y)) acc[0] += 1.0;
    else acc[1] = fmax(acc[1], hypot((double)c.x, (double)c.y));
  }
  // max-reduction (order independent) for acc[1]; sum for acc[0]
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], off);
    acc[1] = fmax(acc[1], __shfl_xor_sync(0xffffffffu, acc[1], off));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sh[w * 2] = acc[0];
    sh[w * 2 + 1] = acc[1];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bad = 0, mx = 0;
    for (int i = 0; i < 8; ++i) {
      bad += sh[2 * i];
      mx = fmax(mx, sh[2 * i + 1]);
    }
    part[2 * blockIdx.x] = bad;
    part[2 * blockIdx.x + 1] = mx;
  }
}

// mode 0: res[0] = all finite, res[1] = max; mode 1: res[2..3] = sums
__global__ void chunk_finish_kernel(const double* part, int64_t nchunk, int mode, double* res) {
  if (threadIdx.x != 0) return;
  double a = 0, b = 0;
  for (int64_t c = 0; c < nchunk; ++c) {
    if (mode == 0) {
      a += part[2 * c];
      b = fmax(b, part[2 * c + 1]);
    } else {
      a += part[2 * c];
      b += part[2 * c + 1];
    }
  }
  if (mode == 0) {
    res[0] = a == 0 ? 1.0 : 0.0;
    res[1] = b;
  } else {
    res[2] = a;
    res[3] = b;
  }
}

// FP64 data: the reference subtracts in working precision (abft.py:315-317);
// the column is (snap_out - ref) / w with ref in the same precision.
int launch_correction_column(int prec, const void* snap_out, const void* ref64, int64_t n, double weight, void* col,
                             double* res, cudaStream_t st) {
  ChunkScratch scratch(n, st);
  double* part = scratch.p;
  if (!part) return (int)cudaErrorMemoryAllocation;
  const int64_t nc = (n + kChunk - 1) / kChunk;
  if (prec == 0)
    correction_column_kernel<float><<<(unsigned)nc, 256, 0, st>>>((const float2*)snap_out, (const double2*)ref64, n,
                                                                  weight, (float2*)col, part);
  else
    correction_column_kernel<double><<<(unsigned)nc, 256, 0, st>>>((const double2*)snap_out, (const double2*)ref64, n,
                                                                   weight, (double2*)col, part);
  chunk_finish_kernel<<<1, 32, 0, st>>>(part, nc, 0, res);
  return (int)cudaGetLastError();
}

template <typename T>
__global__ void __launch_bounds__(256) patch_row_kernel(C<T>* yk, const C<T>* col, int64_t n, int enc,
                                                        const C<T>* tw, double* part) {
  __shared__ double sh[8 * 2];
  C<T> co = mk<T>(0, 0);
  const int64_t k0 = blockIdx.x * kChunk, k1 = min(k0 + kChunk, n);
  for (int64_t k = k0 + threadIdx.x; k < k1; k += 256) {
    const C<T> v = csub<T>(yk[k], col[k]);
    yk[k] = v;
    co = cadd<T>(co, cmul<T>(enc_value<T>(enc, k, n, tw), v));
  }
  double acc[2] = {(double)co.x, (double)co.y};
  block_sum256<2>(acc, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = acc[0];
    part[2 * blockIdx.x + 1] = acc[1];
  }
}

int launch_patch_row(int prec, void* yk, const void* col, int64_t n, int enc, const void* tw, double* res,
                     cudaStream_t st) {
  ChunkScratch scratch(n, st);
  double* part = scratch.p;
  if (!part) return (int)cudaErrorMemoryAllocation;
  const int64_t nc = (n + kChunk - 1) / kChunk;
  if (prec == 0)
    patch_row_kernel<float><<<(unsigned)nc, 256, 0, st>>>((float2*)yk, (const float2*)col, n, enc, (const float2*)tw,
                                                         part);
  else
    patch_row_kernel<double><<<(unsigned)nc, 256, 0, st>>>((double2*)yk, (const double2*)col, n, enc,
                                                          (const double2*)tw, part);
  chunk_finish_kernel<<<1, 32, 0, st>>>(part, nc, 1, res);
  return (int)cudaGetLastError();
}

__global__ void promote_kernel(const float2* in, double2* out, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    out[k] = make_double2(in[k].x, in[k].y);
}

int launch_promote(const void* in, void* out, int64_t n, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) return 0;
  promote_kernel<<<(unsigned)blocks, 256, 0, st>>>((const float2*)in, (double2*)out, n);
  return (int)cudaGetLastError();
}

// Jou encoding input variant x' = 2 x_k + x_{k+1 mod n} (abft.py:333-334) and
// its undo y /= (2 + e^{2 pi i j / n}) (abft.py:337-339)
template <typename T>
__global__ void jou_variant_kernel(const C<T>* x, C<T>* out, int64_t rows, int64_t n) {
  const int64_t total = rows * n;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = id / n, k = id - r * n;
    const C<T> a = x[id], b = x[r * n + (k + 1 == n ? 0 : k + 1)];
    out[id] = cadd<T>(cscale<T>(a, (T)2), b);
  }
}

template <typename T>
__global__ void jou_undo_kernel(C<T>* y, int64_t rows, int64_t n, const C<T>* tw_inv) {
  const int64_t total = rows * n;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = id % n;
    const C<T> w = tw_inv[k];  // e^{+2 pi i k / n}
    const double dr = 2.0 + (double)w.x, di = (double)w.y;
    const double den = dr * dr + di * di;
    const C<T> v = y[id];
    const double re = ((double)v.x * dr + (double)v.y * di) / den;
    const double im = ((double)v.y * dr - (double)v.x * di) / den;
    y[id] = mk<T>((T)re, (T)im);
  }
}

int launch_jou(int prec, int undo, const void* x, void* out, int64_t rows, int64_t n, const void* tw_inv,
               cudaStream_t st) {
  int64_t blocks = (rows * n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) return 0;
  if (prec == 0) {
    if (undo) jou_undo_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((float2*)out, rows, n, (const float2*)tw_inv);
    else jou_variant_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((const float2*)x, (float2*)out, rows, n);
  } else {
    if (undo) jou_undo_kernel<double><<<(unsigned)blocks, 256, 0, st>>>((double2*)out, rows, n, (const double2*)tw_inv);
    else jou_variant_kernel<double><<<(unsigned)blocks, 256, 0, st>>>((const double2*)x, (double2*)out, rows, n);
  }
  return (int)cudaGetLastError();
}

}  // namespace tfft
