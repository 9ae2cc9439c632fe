// C-ABI layer of libtfft.so (declared in include/tfft.h): plans, dispatch to the
// K1 single-pass / K3 two-pass kernels, the stage-strike path and the
// replay-engine primitives.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <string>
#include <vector>

#include "../../include/tfft.h"
#include "tfft_aux.h"
#include "tfft_internal.h"
#include "tfft_k3.h"

using namespace tfft;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(int e, const char* what) {
  if (e == 0) return TFFT_OK;
  g_err = std::string(what) + ": " + cudaGetErrorString((cudaError_t)e);
  return e == (int)cudaErrorMemoryAllocation ? TFFT_ENOMEM : TFFT_ECUDA;
}

#define TFFT_TRY(expr, what)                          \
  do {                                                \
    int _e = (expr);                                  \
    g_launches.fetch_add(1, std::memory_order_relaxed); \
    if (_e) return cuda_fail(_e, what);               \
  } while (0)

bool is_pow2(int64_t v) { return v >= 1 && (v & (v - 1)) == 0; }
int ilog2_64(int64_t v) {
  int r = 0;
  while ((int64_t(1) << r) < v) ++r;
  return r;
}

// omega_N^k = exp(-2 pi i k / N) in extended precision, rounded once
void fill_twiddles(std::vector<long double>& re, std::vector<long double>& im, int64_t n) {
  re.resize(n);
  im.resize(n);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int64_t k = 0; k < n; ++k) {
    // reduce to the first octant for accuracy, then use symmetry
    const long double a = two_pi * (long double)k / (long double)n;
    re[k] = cosl(a);
    im[k] = -sinl(a);
  }
  // exact values where they are exact
  for (int64_t k = 0; k < n; k += std::max<int64_t>(n / 4, 1)) {
    const int64_t q = (k * 4) / n;
    const long double cs[4] = {1, 0, -1, 0}, sn[4] = {0, -1, 0, 1};
    if (n % 4 == 0 || k == 0) {
      re[k] = cs[q];
      im[k] = sn[q];
    }
  }
  if (n >= 2) {
    re[n / 2] = -1;
    im[n / 2] = 0;
  }
}

template <typename T>
void pack(const std::vector<long double>& re, const std::vector<long double>& im, bool conj, std::vector<T>& out) {
  out.resize(2 * re.size());
  for (size_t k = 0; k < re.size(); ++k) {
    out[2 * k] = (T)re[k];
    out[2 * k + 1] = (T)(conj ? -im[k] : im[k]);
  }
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return (int)e;
    cap = bytes;
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace

namespace tfft {
// error reporting for the other C-ABI translation units (tfft_dist.cu)
int set_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace tfft

struct tfft_plan {
  int64_t n = 0;
  int logn = 0;
  int prec = 0;
  int64_t bs = 1;
  std::vector<int64_t> spans;
  std::vector<int32_t> radices;
  struct Pass {
    int64_t s;
    int r;
    int stage;
  };
  std::vector<Pass> passes;  // the reference's radix-4/2 lowering (fft_core.py:137-202)
  int num_sms = 148;
  int device = 0;
  bool k1 = false;
  bool k5 = false;  // plain single-pass transforms run on the warp-specialised K5
  int mode = 0;              // 0: K1 single pass, 1: K3 two pass, 2: reference-order multipass
  DevBuf tw_fwd, tw_inv;     // omega_N^k, conj (K1 and ABFT encodings)
  DevBuf enc_tab[2];         // omega_N^k / conj for K3/multipass Jou encoding (lazy)
  DevBuf wsum;               // unfused window sums (s_in, s_out, FFT(s_in))
  DevBuf part;               // per-(signal, chunk) ABFT partials of the one-sweep path
  DevBuf rows[3];            // left checksum rows per encoding kind
  bool row_ready[3] = {false, false, false};
  DevBuf counters;           // default counters
  DevBuf faults;
  DevBuf ws, win_count;
  DevBuf sigpart;                     // K5 fused ABFT: per-warp per-signal partials
  DevBuf winsave;                     // K5 fused ABFT: the last call's window sums [nwin][2][n]
  int sums_kind = 0;                  // window sums of the last protected call: 0 none, 1 winsave, 2 wsum
  int64_t sums_nwin = 0;
  DevBuf cw_desc, cw_par, cw_res, cw_tin, cw_tout, cw_ref, cw_col, cw_sin, cw_sout, cw_gref;  // batched correction
  DevBuf scratch_a, scratch_b, base;  // strike path
  DevBuf col_a, col_b, col64;         // single-column work
  K3Plan* k3 = nullptr;               // two-pass machinery (N beyond K1)
  StagePlan* stg = nullptr;           // three-stage plans: one pass per reference stage
  tfft_plan* promoted = nullptr;      // FP64 twin for FP32 correction columns
};

namespace {

size_t cbytes(int prec) { return prec == 0 ? 8 : 16; }

// the reference's radix lowering: micro radix 2^g -> [4]*(g//2) + [2]*(g%2),
// repeated while the remaining span >= micro, then the remainder
void lower(tfft_plan* p) {
  p->passes.clear();
  int64_t s = 1;
  for (size_t si = 0; si < p->spans.size(); ++si) {
    auto micro = [](int64_t radix, std::vector<int>& out) {
      int g = ilog2_64(radix);
      for (int i = 0; i < g / 2; ++i) out.push_back(4);
      if (g % 2) out.push_back(2);
    };
    std::vector<int> f;
    int64_t rest = p->spans[si];
    while (rest >= p->radices[si]) {
      micro(p->radices[si], f);
      rest /= p->radices[si];
    }
    if (rest > 1) micro(rest, f);
    for (int r : f) {
      p->passes.push_back({s, r, (int)si});
      s *= r;
    }
  }
}

int upload(DevBuf& b, const void* host, size_t bytes) {
  int e = b.ensure(bytes);
  if (e) return e;
  return (int)cudaMemcpy(b.p, host, bytes, cudaMemcpyHostToDevice);
}

int ensure_row(tfft_plan* p, int enc) {
  if (p->row_ready[enc]) return 0;
  std::vector<unsigned char> host(p->n * cbytes(p->prec));
  int rc = tfft_left_row(enc, p->n, p->prec, host.data());
  if (rc) return rc;
  int e = upload(p->rows[enc], host.data(), host.size());
  if (e) return cuda_fail(e, "left row upload");
  p->row_ready[enc] = true;
  return 0;
}

// faulted transactions outside K1/K3's in-kernel strike reach: replay them pass
// by pass through the reference-order kernels (fault.py:99-107 semantics)
int strike_path(tfft_plan* p, const void* x, void* y, int64_t batch, int inverse, int64_t signal_offset,
                const std::vector<tfft_fault>& fl, cudaStream_t st, std::vector<int64_t>* touched_rows) {
  const size_t cb = cbytes(p->prec);
  std::vector<int64_t> done;
  for (const tfft_fault& f : fl) {
    const int64_t tx = f.transaction;
    if (std::find(done.begin(), done.end(), tx) != done.end()) continue;
    done.push_back(tx);
    const int64_t a = std::max<int64_t>(tx * p->bs - signal_offset, 0);
    const int64_t b = std::min<int64_t>((tx + 1) * p->bs - signal_offset, batch);
    if (a >= b) continue;
    const int64_t rows = b - a;
    int e = p->scratch_a.ensure(rows * p->n * cb);
    if (!e) e = p->scratch_b.ensure(rows * p->n * cb);
    if (!e) e = p->base.ensure(p->n * cb);
    if (e) return cuda_fail(e, "strike scratch");
    TFFT_TRY((int)cudaMemcpyAsync(p->scratch_a.p, (const char*)x + a * p->n * cb, rows * p->n * cb,
                                  cudaMemcpyDeviceToDevice, st),
             "strike copy-in");
    void* cur = p->scratch_a.p;
    void* nxt = p->scratch_b.p;
    size_t pi = 0;
    for (size_t si = 0; si < p->spans.size(); ++si) {
      for (const tfft_fault& g : fl) {
        if (g.transaction != tx || g.stage != (int)si) continue;
        const int64_t r = g.signal - signal_offset - a;
        if (r < 0 || r >= rows) continue;
        TFFT_TRY(launch_flip(p->prec, cur, r * p->n + g.element, g.part, g.bit, st), "strike flip");
      }
      while (pi < p->passes.size() && p->passes[pi].stage == (int)si) {
        const auto& ps = p->passes[pi];
        // base table omega_(s r)^q = omega_N^(q N/(s r)) read with a stride
        const DevBuf& tw = inverse ? p->tw_inv : p->tw_fwd;
        const void* base = nullptr;
        int64_t stride = 0;
        if (tw.p) {
          base = tw.p;
          stride = p->n / (ps.s * ps.r);
        } else {
          TFFT_TRY(launch_base_table(p->prec, ps.s, ps.r, inverse, p->base.p, st), "strike base table");
          base = p->base.p;
          stride = 1;
        }
        TFFT_TRY(launch_stockham_pass(p->prec, cur, nxt, rows, p->n, ps.s, ps.r, base, stride, inverse, st),
                 "strike pass");
        std::swap(cur, nxt);
        ++pi;
      }
    }
    if (inverse) TFFT_TRY(launch_scale(p->prec, cur, rows * p->n, 1.0 / (double)p->n, st), "strike scale");
    TFFT_TRY((int)cudaMemcpyAsync((char*)y + a * p->n * cb, cur, rows * p->n * cb, cudaMemcpyDeviceToDevice, st),
             "strike copy-out");
    if (touched_rows) {
      touched_rows->push_back(a);
      touched_rows->push_back(b);
    }
  }
  return 0;
}

int zero_counters(tfft_plan* p, uint64_t*& counters, cudaStream_t st) {
  if (!counters) {
    // the plan's default counters are allocated once at their full size (8
    // words: 4 for the caller-visible block, 4 for internal window FFTs), so a
    // later ensure() never reallocates a buffer an earlier launch still uses
    int e = p->counters.ensure(8 * sizeof(uint64_t));
    if (e) return cuda_fail(e, "counters");
    counters = (uint64_t*)p->counters.p;
  }
  TFFT_TRY((int)cudaMemsetAsync(counters, 0, 4 * sizeof(uint64_t), st), "counters memset");
  return 0;
}

int split_faults(tfft_plan* p, const tfft_fault* faults, int nfaults, int64_t signal_offset, int64_t batch,
                 std::vector<DevFault>& dev, std::vector<tfft_fault>& slow, bool k3_split_ok) {
  for (int i = 0; i < nfaults; ++i) {
    const tfft_fault& f = faults[i];
    const int64_t r = f.signal - signal_offset;
    if (r < 0 || r >= batch) continue;
    if (f.element < 0 || f.element >= p->n || f.stage < 0 || f.stage >= (int)p->spans.size() || f.bit < 0 ||
        f.bit >= (p->prec == 0 ? 32 : 64) || (f.part != 0 && f.part != 1))
      return fail(TFFT_EINVAL, "fault spec out of range");
    const bool in_kernel = (p->mode == 2 && p->stg) ||
                           (p->mode != 2 && (f.stage == 0 || (k3_split_ok && f.stage == 1 && p->mode == 1 &&
                                                              k3_strikes_stage1(p->k3))));
    if (in_kernel) dev.push_back({r, f.element, f.stage, f.part, f.bit, 0});
    else slow.push_back(f);
  }
  return 0;
}

int upload_faults(tfft_plan* p, std::vector<DevFault>& dev, cudaStream_t st) {
  if (dev.empty()) return 0;
  // sorted by signal (stable: same-signal faults keep their order) for fault_lo
  std::stable_sort(dev.begin(), dev.end(), [](const DevFault& a, const DevFault& b) { return a.signal < b.signal; });
  int e = p->faults.ensure(dev.size() * sizeof(DevFault));
  if (e) return cuda_fail(e, "fault buffer");
  TFFT_TRY((int)cudaMemcpyAsync(p->faults.p, dev.data(), dev.size() * sizeof(DevFault), cudaMemcpyHostToDevice, st),
           "fault upload");
  return 0;
}

// sizes beyond the fused kernels: the reference's own radix-4/2 pass list, one
// device sweep per pass (correct for any N up to 2^29; not the fast path)
int multipass(tfft_plan* p, const void* x, void* y, int64_t batch, int inverse, uint64_t* counters,
              cudaStream_t st) {
  const size_t cb = cbytes(p->prec);
  // the fused kernels flag non-finite input while loading it; here one
  // reduction over x sets the same counter (fft_core.py:305 raises on it)
  if (counters) TFFT_TRY(launch_nonfinite(p->prec, x, batch * p->n, (Counters*)counters, st), "multipass finite check");
  int e = p->scratch_b.ensure((size_t)batch * p->n * cb);
  if (!e) e = p->base.ensure((size_t)p->n * cb);
  if (e) return cuda_fail(e, "multipass scratch");
  const size_t np = p->passes.size();
  void* bufs[2] = {y, p->scratch_b.p};
  const void* cur = x;
  for (size_t i = 0; i < np; ++i) {
    const auto& ps = p->passes[i];
    void* out = bufs[(np - 1 - i) % 2];
    TFFT_TRY(launch_base_table(p->prec, ps.s, ps.r, inverse, p->base.p, st), "multipass base table");
    TFFT_TRY(launch_stockham_pass(p->prec, cur, out, batch, p->n, ps.s, ps.r, p->base.p, 1, inverse, st),
             "multipass pass");
    cur = out;
  }
  if (inverse) TFFT_TRY(launch_scale(p->prec, y, batch * p->n, 1.0 / (double)p->n, st), "multipass scale");
  return 0;
}

// omega_N^k (conj for inv) for the Jou encoding of plans without K1's table;
// built once, on the caller's stream (stream-ordered before every use on that
// stream; no device-wide synchronisation, graph-capturable after first use)
int enc_table(tfft_plan* p, bool inv, cudaStream_t st, const void** out) {
  if (p->k1) {
    *out = inv ? p->tw_inv.p : p->tw_fwd.p;
    return 0;
  }
  DevBuf& b = p->enc_tab[inv ? 1 : 0];
  if (!b.p) {
    int e = b.ensure((size_t)p->n * cbytes(p->prec));
    if (e) return cuda_fail(e, "encoding table");
    e = launch_base_table(p->prec, p->n, 1, inv ? 1 : 0, b.p, st);
    if (e) {
      b.release();
      return cuda_fail(e, "encoding table launch");
    }
  }
  *out = b.p;
  return 0;
}

int run_plain(tfft_plan* p, const void* x, void* y, int64_t batch, int inverse, int64_t signal_offset,
              const std::vector<DevFault>& dev, uint64_t* counters, cudaStream_t st) {
  if (p->k1) {
    K1Args a{};
    a.x = x;
    a.y = y;
    a.batch = batch;
    a.weight0 = signal_offset;
    a.tw = inverse ? p->tw_inv.p : p->tw_fwd.p;
    a.faults = (const DevFault*)p->faults.p;
    a.nfaults = (int)dev.size();
    a.counters = (Counters*)counters;
    if (p->k5)
      TFFT_TRY(launch_k5(p->prec, p->logn, inverse != 0, a, p->num_sms, st), "k5 launch");
    else
      TFFT_TRY(launch_k1(p->prec, p->logn, inverse != 0, false, a, p->num_sms, st), "k1 launch");
    return 0;
  }
  if (p->mode == 1) {
    int rc = k3_execute(p->k3, x, y, batch, inverse, (const DevFault*)p->faults.p, (int)dev.size(),
                        (Counters*)counters, nullptr, st);
    g_launches.fetch_add(k3_launches(p->k3), std::memory_order_relaxed);
    return rc ? cuda_fail(rc, "k3 launch") : 0;
  }
  if (p->stg) {
    int e = p->scratch_b.ensure((size_t)batch * p->n * cbytes(p->prec));
    if (e) return cuda_fail(e, "stage scratch");
    int rc = stage_execute(p->stg, x, y, p->scratch_b.p, batch, inverse, (const DevFault*)p->faults.p,
                           (int)dev.size(), (Counters*)counters, st);
    g_launches.fetch_add(stage_count(p->stg), std::memory_order_relaxed);
    return rc ? cuda_fail(rc, "stage pass launch") : 0;
  }
  return multipass(p, x, y, batch, inverse, counters, st);
}

// protected sizes with a fused kernel: fused (checksums inside the transform)
// or unfused (plain transform + one checksum sweep over x and y).
// TFFT_ABFT_SWEEP=1 / =0 force either; the default is the measured-faster one.
bool abft_force_sweep() {
  const char* e = std::getenv("TFFT_ABFT_SWEEP");
  return e && e[0] == '1';
}
bool abft_use_sweep(const tfft_plan* p) {
  if (const char* e = std::getenv("TFFT_ABFT_SWEEP")) return e[0] == '1';
  // B200, 1 GiB inputs, T = 8 (tools/abft_ab.py): from 2^11 up the fused
  // kernels lose to plain + sweep (FP32 4096: 1.03 vs 0.87 ms, FP64 4096:
  // 1.44 vs 0.93 ms); below it the window sums of the sweep path (small
  // windows: bs = 1 at 2^10) cost more than the fused kernel's occupancy loss
  return p->logn >= 11;
}

}  // namespace

extern "C" {

int tfft_version(void) { return 1; }
const char* tfft_last_error(void) { return g_err.c_str(); }
uint64_t tfft_launch_count(void) { return g_launches.load(); }

int tfft_plan_create(int64_t n, int precision, int nstages, const int64_t* spans, const int32_t* radices,
                     int64_t bs, tfft_plan** out) {
  if (!out) return fail(TFFT_EINVAL, "null plan out-pointer");
  *out = nullptr;
  if (precision != 0 && precision != 1) return fail(TFFT_EINVAL, "precision must be 0 (single) or 1 (double)");
  if (!is_pow2(n) || n < 2 || n > (int64_t(1) << 29)) return fail(TFFT_EINVAL, "n must be a power of two in [2, 2^29]");
  if (nstages < 1 || nstages > 3 || bs < 1) return fail(TFFT_EINVAL, "plans have 1..3 stages and bs >= 1");
  int64_t prod = 1;
  for (int i = 0; i < nstages; ++i) {
    if (!is_pow2(spans[i]) || spans[i] < 2) return fail(TFFT_EINVAL, "stage span must be a power of two >= 2");
    if (!is_pow2(radices[i]) || radices[i] < 2 || radices[i] > 32 || radices[i] > spans[i])
      return fail(TFFT_EINVAL, "invalid micro radix");
    prod *= spans[i];
  }
  if (prod != n) return fail(TFFT_EINVAL, "stage spans do not multiply to n");
  tfft_plan* p = new tfft_plan();
  p->n = n;
  p->logn = ilog2_64(n);
  p->prec = precision;
  p->bs = bs;
  p->spans.assign(spans, spans + nstages);
  p->radices.assign(radices, radices + nstages);
  lower(p);
  cudaGetDevice(&p->device);
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, p->device);
  p->k1 = k1_supported(precision, p->logn) != 0;
  // K5 measured faster than K1 from N = 512 up; K1's wide 256-thread CTAs
  // (16 signals per tile) still win at N <= 256 (profiles/r1s2_k5)
  p->k5 = p->k1 && p->logn >= 9 && std::getenv("TFFT_NO_K5") == nullptr;
  if (p->k1) {
    std::vector<long double> re, im;
    fill_twiddles(re, im, n);
    int e = 0;
    if (precision == 0) {
      std::vector<float> f, fi;
      pack(re, im, false, f);
      pack(re, im, true, fi);
      e = upload(p->tw_fwd, f.data(), f.size() * 4);
      if (!e) e = upload(p->tw_inv, fi.data(), fi.size() * 4);
    } else {
      std::vector<double> d, di;
      pack(re, im, false, d);
      pack(re, im, true, di);
      e = upload(p->tw_fwd, d.data(), d.size() * 8);
      if (!e) e = upload(p->tw_inv, di.data(), di.size() * 8);
    }
    if (e) {
      tfft_plan_destroy(p);
      return cuda_fail(e, "twiddle upload");
    }
  } else {
    int rc = k3_create(n, precision, p->spans.data(), (int)p->spans.size(), p->num_sms, &p->k3);
    if (rc == (int)cudaErrorInvalidValue) {
      p->mode = 2;
      p->k3 = nullptr;
      // three-stage plans: one stage pass per reference stage when every span
      // is in the pass kernel's range, else the reference-order radix-4/2 passes
      if (std::getenv("TFFT_NO_STAGES") == nullptr) {
        int rs = stage_create(n, precision, p->spans.data(), (int)p->spans.size(), p->num_sms, &p->stg);
        if (rs && rs != (int)cudaErrorInvalidValue) {
          tfft_plan_destroy(p);
          return cuda_fail(rs, "stage plan");
        }
        if (rs) p->stg = nullptr;
      }
    } else if (rc) {
      tfft_plan_destroy(p);
      return cuda_fail(rc, "k3 plan");
    } else {
      // (two-stage plans keep the fused two-pass kernels: stage passes measured
      // 1.5-2x slower at 2^17..2^22, the span-2048 passes load 32-byte runs)
      p->mode = 1;
    }
  }
  *out = p;
  return TFFT_OK;
}

int tfft_plan_destroy(tfft_plan* p) {
  if (!p) return TFFT_OK;
  DevBuf* all[] = {&p->winsave, &p->cw_desc, &p->cw_par, &p->cw_res, &p->cw_tin, &p->cw_tout, &p->cw_ref,
                   &p->cw_col, &p->cw_sin, &p->cw_sout, &p->cw_gref, &p->sigpart, &p->part, &p->tw_fwd, &p->tw_inv, &p->enc_tab[0], &p->enc_tab[1], &p->wsum, &p->rows[0], &p->rows[1], &p->rows[2], &p->counters, &p->faults,
                   &p->ws, &p->win_count, &p->scratch_a, &p->scratch_b, &p->base, &p->col_a, &p->col_b, &p->col64};
  for (DevBuf* b : all) b->release();
  if (p->k3) k3_destroy(p->k3);
  if (p->stg) stage_destroy(p->stg);
  if (p->promoted) tfft_plan_destroy(p->promoted);
  delete p;
  return TFFT_OK;
}

int tfft_debug_skew_twiddle(tfft_plan* p) {
  if (!p) return fail(TFFT_EINVAL, "null plan");
  if (!p->k1 || p->n < 2) return fail(TFFT_EUNSUPPORTED, "skew hook: single-pass plans only");
  for (DevBuf* b : {&p->tw_fwd, &p->tw_inv}) {
    if (p->prec == 0) {
      float v[2];
      TFFT_TRY((int)cudaMemcpy(v, (float*)b->p + 2, sizeof(v), cudaMemcpyDeviceToHost), "skew read");
      v[0] *= 1.001f;
      v[1] *= 1.001f;
      TFFT_TRY((int)cudaMemcpy((float*)b->p + 2, v, sizeof(v), cudaMemcpyHostToDevice), "skew write");
    } else {
      double v[2];
      TFFT_TRY((int)cudaMemcpy(v, (double*)b->p + 2, sizeof(v), cudaMemcpyDeviceToHost), "skew read");
      v[0] *= 1.001;
      v[1] *= 1.001;
      TFFT_TRY((int)cudaMemcpy((double*)b->p + 2, v, sizeof(v), cudaMemcpyHostToDevice), "skew write");
    }
  }
  return TFFT_OK;
}

int tfft_execute(tfft_plan* p, const void* x, void* y, int64_t batch, int inverse, int64_t signal_offset,
                 const tfft_fault* faults, int nfaults, uint64_t* counters, void* stream) {
  if (!p || !x || !y || batch < 1) return fail(TFFT_EINVAL, "invalid execute arguments");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = zero_counters(p, counters, st);
  if (rc) return rc;
  std::vector<DevFault> dev;
  std::vector<tfft_fault> slow;
  rc = split_faults(p, faults, nfaults, signal_offset, batch, dev, slow, true);
  if (rc) return rc;
  rc = upload_faults(p, dev, st);
  if (rc) return rc;
  rc = run_plain(p, x, y, batch, inverse, signal_offset, dev, counters, st);
  if (rc) return rc;
  if (!slow.empty()) return strike_path(p, x, y, batch, inverse, signal_offset, slow, st, nullptr);
  return TFFT_OK;
}

int tfft_protected(tfft_plan* p, const void* x, void* y, int64_t batch, int64_t signal_offset, int enc,
                   double delta, int64_t T, const tfft_fault* faults, int nfaults, const tfft_sums* sums,
                   uint64_t* counters, void* stream) {
  if (!p || !x || !y || batch < 1 || !sums || T < 1 || enc < 0 || enc > 2 || !(delta > 0))
    return fail(TFFT_EINVAL, "invalid protected arguments");
  const int64_t W = T * p->bs;
  if (signal_offset % W) return fail(TFFT_EINVAL, "signal_offset must be a multiple of group_size * bs");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = zero_counters(p, counters, st);
  if (rc) return rc;
  rc = ensure_row(p, enc);
  if (rc) return rc;
  std::vector<DevFault> dev;
  std::vector<tfft_fault> slow;
  rc = split_faults(p, faults, nfaults, signal_offset, batch, dev, slow, true);
  if (rc) return rc;
  rc = upload_faults(p, dev, st);
  if (rc) return rc;
  const int64_t ntx = (batch + p->bs - 1) / p->bs;
  const int64_t nwin = (ntx + T - 1) / T;
  AbftArgs ab{};
  ab.row = p->rows[enc].p;
  ab.enc = enc;
  ab.delta = delta;
  ab.c_in = sums->c_in;
  ab.c_out = sums->c_out;
  ab.floors = sums->floors;
  ab.div = sums->div;
  ab.win_div = sums->win_div;
  ab.win_signals = W;
  ab.nwin = nwin;
  // K5 with the window sums in tensor memory (N = 2^9..2^12/13), K1's fused
  // kernel below that, the plain transform + one checksum sweep otherwise
  const bool k5abft = p->k5 && k5_abft_supported(p->prec, p->logn) && std::getenv("TFFT_NO_K5_ABFT") == nullptr &&
                      !abft_force_sweep();
  const bool sweep = !k5abft && abft_use_sweep(p);
  if (k5abft) {
    int64_t grid = 0;
    int spt = 1, nws = 1;
    int e = k5_abft_layout(p->prec, p->logn, p->num_sms, batch, &grid, &spt, &nws);
    if (e) return cuda_fail(e, "k5 abft layout");
    const int64_t per_cta = (batch + grid - 1) / grid;
    const int64_t maxseg = (per_cta + W - 1) / W + 1;
    const size_t cb = cbytes(p->prec);
    e = p->ws.ensure((size_t)grid * maxseg * spt * 2 * p->n * cb);
    if (!e) e = p->sigpart.ensure((size_t)batch * nws * 5 * sizeof(double));
    if (!e) e = p->winsave.ensure((size_t)nwin * 2 * p->n * cb);
    if (e) return cuda_fail(e, "abft workspace");
    p->sums_kind = 1;
    p->sums_nwin = nwin;
    ab.mode = 2;
    ab.pieces = maxseg;
    ab.ws = p->ws.p;
    ab.sig_part = (double*)p->sigpart.p;
    K1Args a{};
    a.x = x;
    a.y = y;
    a.batch = batch;
    a.weight0 = signal_offset;
    a.tw = p->tw_fwd.p;
    a.faults = (const DevFault*)p->faults.p;
    a.nfaults = (int)dev.size();
    a.counters = (Counters*)counters;
    a.abft = ab;
    TFFT_TRY(launch_k5_abft(p->prec, p->logn, a, p->num_sms, st), "k5 abft launch");
    TFFT_TRY(launch_k5_window_finish(p->prec, p->logn, p->ws.p, (const double*)p->sigpart.p, nws, p->tw_fwd.p, batch,
                                     W, grid, maxseg, spt, nwin, delta, ab, (Counters*)counters, p->winsave.p,
                                     p->num_sms, st),
             "abft window finish");
  } else if (p->k1 && !sweep) {
    p->sums_kind = 0;
    const int spt = k1_slots(p->prec, p->logn);
    if (W <= 4) {
      ab.mode = 0;
      ab.pieces = 1;
    } else {
      ab.mode = 1;
      const int64_t piece = (int64_t)spt * 16;
      ab.pieces = (W + piece - 1) / piece;
    }
    if (ab.mode == 1 && ab.pieces > 1) {
      int e = p->ws.ensure((size_t)nwin * ab.pieces * 2 * p->n * cbytes(p->prec));
      if (e) return cuda_fail(e, "abft workspace");
      const size_t cnt_bytes = (size_t)nwin * sizeof(unsigned);
      if (p->win_count.cap < cnt_bytes) {
        e = p->win_count.ensure(cnt_bytes);
        if (e) return cuda_fail(e, "window counters");
        TFFT_TRY((int)cudaMemsetAsync(p->win_count.p, 0, p->win_count.cap, st), "window counter memset");
      }
      ab.ws = p->ws.p;
      ab.win_count = (unsigned*)p->win_count.p;
    }
    K1Args a{};
    a.x = x;
    a.y = y;
    a.batch = batch;
    a.weight0 = signal_offset;
    a.tw = p->tw_fwd.p;
    a.faults = (const DevFault*)p->faults.p;
    a.nfaults = (int)dev.size();
    a.counters = (Counters*)counters;
    a.abft = ab;
    TFFT_TRY(launch_k1(p->prec, p->logn, false, true, a, p->num_sms, st), "k1 abft launch");
  } else {
    const size_t cb = cbytes(p->prec);
    // three-stage plans, opt-in (TFFT_STAGE_ABFT=1): the checksums and window
    // sums fused into the first and last stage passes, FFT(s_in) carried along
    // as pseudo-signals. Correct (the C4 decision tests pass with it on) but
    // slower than the plain passes + one sweep: the per-item accumulators and
    // row slices spill the pass kernels (64-255 registers, 0.4-1.6 KB spills)
    // and at W = 1 (bs = 1, T = 1: 2^24, 2^25) the row is re-read per window.
    if (p->mode == 2 && p->stg && slow.empty() && !abft_force_sweep() && enc != ENC_JOU &&
        std::getenv("TFFT_STAGE_ABFT") != nullptr) {
      int64_t parts = 0, gper = 0;
      int e = stage_protected_parts(p->stg, &parts, &gper);
      if (!e) e = p->scratch_b.ensure((size_t)batch * p->n * cb);
      if (!e) e = p->scratch_a.ensure((size_t)2 * nwin * p->n * cb);
      if (!e) e = p->sigpart.ensure((size_t)batch * parts * 5 * sizeof(double));
      if (!e) e = p->part.ensure((size_t)nwin * gper * 2 * sizeof(double));
      if (e) return cuda_fail(e, "stage abft workspace");
      char* pa = (char*)p->scratch_a.p;
      char* pb = pa + (size_t)nwin * p->n * cb;
      int rk = stage_protected(p->stg, x, y, p->scratch_b.p, batch, signal_offset, (const DevFault*)p->faults.p,
                               (int)dev.size(), (Counters*)counters, W, enc, p->rows[enc].p, pa, pb,
                               (double*)p->sigpart.p, (double*)p->part.p, sums->win_div, st);
      if (rk != (int)cudaErrorNotSupported) {
        if (rk) return cuda_fail(rk, "stage abft launch");
        g_launches.fetch_add(stage_count(p->stg) + 2, std::memory_order_relaxed);
        p->sums_kind = 0;
        TFFT_TRY(launch_signal_epilogue((const double*)p->sigpart.p, parts, p->n, batch, delta, ab,
                                        (Counters*)counters, st),
                 "abft signal epilogue");
        return TFFT_OK;
      }
    }
    // two-pass sizes on K4, opt-in (TFFT_K4_ABFT=1): the checksums fused into
    // the transform's launch (C tiles over L2-resident x and y), then the
    // window FFT, the group divergence and the per-signal decisions. Correct
    // (the GPU suite passes with it on) but measured slower than plain K4 +
    // one sweep at C5 (2.0-2.4 vs 1.45 ms): the C tiles' re-reads evict the
    // L2 ring (5.2 GB DRAM at 32-signal groups) or, with one window per group,
    // the schedule loses its parallelism (2.3 ms at 3.2 GB). DESIGN.md (d).
    if (p->mode == 1 && slow.empty() && !abft_force_sweep() && std::getenv("TFFT_K4_ABFT") != nullptr) {
      int e = p->wsum.ensure((size_t)3 * nwin * p->n * cb);
      const int64_t nchunk_max = p->n / 256;
      if (!e) e = p->sigpart.ensure((size_t)batch * nchunk_max * 5 * sizeof(double));
      if (!e) e = p->part.ensure((size_t)nwin * ((p->n + 8191) / 8192) * 2 * sizeof(double));
      if (!e) e = p->counters.ensure(8 * sizeof(uint64_t));
      if (e) return cuda_fail(e, "fused abft workspace");
      char* s_in = (char*)p->wsum.p;
      char* s_out = s_in + (size_t)nwin * p->n * cb;
      char* ref = s_out + (size_t)nwin * p->n * cb;
      int64_t nparts = 0;
      int rk = k3_protected(p->k3, x, y, batch, signal_offset, (const DevFault*)p->faults.p, (int)dev.size(),
                            (Counters*)counters, ab, p->rows[enc].p, s_in, s_out, (double*)p->sigpart.p, &nparts,
                            st);
      if (rk != (int)cudaErrorNotSupported) {
        if (rk) return cuda_fail(rk, "fused k4 abft launch");
        p->sums_kind = 2;
        p->sums_nwin = nwin;
        g_launches.fetch_add(1, std::memory_order_relaxed);
        TFFT_TRY(launch_signal_epilogue((const double*)p->sigpart.p, nparts, p->n, batch, delta, ab,
                                        (Counters*)counters, st),
                 "abft signal epilogue");
        std::vector<DevFault> none;
        rc = run_plain(p, s_in, ref, nwin, 0, 0, none, (uint64_t*)p->counters.p + 4, st);
        if (rc) return rc;
        TFFT_TRY(launch_group_div_chunked(p->prec, ref, s_out, p->n, nwin, sums->win_div, (double*)p->part.p, st),
                 "window group div");
        return TFFT_OK;
      }
    }
    // other two-pass / multipass sizes: transform (strikes included), then
    // checksum and window sweeps over x and y on the device
    rc = run_plain(p, x, y, batch, 0, signal_offset, dev, counters, st);
    if (rc) return rc;
    if (!slow.empty()) {
      rc = strike_path(p, x, y, batch, 0, signal_offset, slow, st, nullptr);
      if (rc) return rc;
    }
    int e = p->wsum.ensure((size_t)3 * nwin * p->n * cb);
    if (!e) e = p->part.ensure((size_t)batch * window_sweep_chunks(p->n) * 8 * 5 * sizeof(double));
    if (e) return cuda_fail(e, "window sums");
    char* s_in = (char*)p->wsum.p;
    char* s_out = s_in + (size_t)nwin * p->n * cb;
    char* ref = s_out + (size_t)nwin * p->n * cb;
    const void* etab = nullptr;
    rc = enc_table(p, false, st, &etab);
    if (rc) return rc;
    TFFT_TRY(launch_window_sweep(p->prec, x, y, p->n, batch, W, signal_offset, p->rows[enc].p, etab,
                                 enc, s_in, s_out, (double*)p->part.p, ab, delta, (Counters*)counters, st),
             "abft sweep");
    p->sums_kind = slow.empty() ? 2 : 0;  // strike-path rows changed after the sweep: recompute sums
    p->sums_nwin = nwin;
    std::vector<DevFault> none;
    int e2 = p->counters.ensure(8 * sizeof(uint64_t));
    if (e2) return cuda_fail(e2, "counters");
    rc = run_plain(p, s_in, ref, nwin, 0, 0, none, (uint64_t*)p->counters.p + 4, st);
    if (rc) return rc;
    // the per-signal partials are consumed (epilogue ran): reuse them for the window partials
    TFFT_TRY(launch_group_div_chunked(p->prec, ref, s_out, p->n, nwin, sums->win_div, (double*)p->part.p, st),
             "window group div");
    return TFFT_OK;
  }
  if (slow.empty()) return TFFT_OK;
  p->sums_kind = 0;  // y changes below: kept window sums no longer match it
  // strike path for the faults the fused kernel cannot reach, then refresh
  // the affected rows' checksums and their windows' group divergences
  std::vector<int64_t> touched;
  rc = strike_path(p, x, y, batch, 0, signal_offset, slow, st, &touched);
  if (rc) return rc;
  const size_t cb = cbytes(p->prec);
  const void* etab = nullptr;
  rc = enc_table(p, false, st, &etab);
  if (rc) return rc;
  for (size_t i = 0; i < touched.size(); i += 2) {
    const int64_t a = touched[i], b = touched[i + 1];
    TFFT_TRY(launch_row_checksums(p->prec, x, y, p->n, a, b - a, p->rows[enc].p, etab, enc, delta, ab,
                                  (Counters*)counters, 1, st),
             "strike row checksums");
    const int64_t w = a / W;
    const int64_t w0 = w * W, w1 = std::min<int64_t>(w0 + W, batch);
    int e = p->col_a.ensure(p->n * cb);
    if (!e) e = p->col_b.ensure(p->n * cb);
    if (!e) e = p->col64.ensure(p->n * cb);
    if (e) return cuda_fail(e, "window columns");
    TFFT_TRY(launch_weighted_cols(p->prec, x, p->n, w0, w1, W, signal_offset, p->col_a.p, st), "window s_in");
    TFFT_TRY(launch_weighted_cols(p->prec, y, p->n, w0, w1, W, signal_offset, p->col_b.p, st), "window s_out");
    std::vector<DevFault> none;
    uint64_t* c2 = nullptr;
    int e2 = p->counters.ensure(8 * sizeof(uint64_t));
    if (e2) return cuda_fail(e2, "counters");
    c2 = (uint64_t*)p->counters.p + 4;
    rc = run_plain(p, p->col_a.p, p->col64.p, 1, 0, 0, none, c2, st);
    if (rc) return rc;
    TFFT_TRY(launch_group_div(p->prec, p->col64.p, p->col_b.p, p->n, sums->win_div + w, st), "window group div");
  }
  return TFFT_OK;
}

int tfft_stockham_pass(const void* src, void* dst, int64_t rows, int64_t n, int64_t s, int r, const void* base,
                       int inverse, int precision, void* stream) {
  if (!src || !dst || !base || rows < 1 || n < 2 || s < 1 || (r != 2 && r != 4) || n % (s * r))
    return fail(TFFT_EINVAL, r != 2 && r != 4 ? "kernel supports radix 2 and 4" : "invalid stockham_pass arguments");
  TFFT_TRY(launch_stockham_pass(precision, src, dst, rows, n, s, r, base, 1, inverse, (cudaStream_t)stream),
           "stockham_pass");
  return TFFT_OK;
}

int tfft_left_row(int enc, int64_t n, int precision, void* out_host) {
  if (!out_host || n < 1 || enc < 0 || enc > 2 || (precision != 0 && precision != 1))
    return fail(TFFT_EINVAL, "invalid left-row arguments");
  std::vector<long double> re(n, 0.0L), im(n, 0.0L);
  if (enc == ENC_ONES) {
    re[0] = (long double)n;
  } else if (enc == ENC_JOU) {
    re[n - 1] = (long double)n;
  } else {
    // row[j] = (1 - w3^n) / (1 - w3 w_n^j), w3 = e^{-2 pi i/3}; the pole phase
    // (1/3 + j/n) is reduced exactly as the integer m = (n + 3j) mod 3n
    const long double two_pi = 6.283185307179586476925286766559005768L;
    const int64_t nm3 = n % 3;
    const long double a = two_pi * (long double)nm3 / 3.0L;  // w3^n = e^{-i a}
    const long double num_re = 1.0L - cosl(a), num_im = sinl(a);
    for (int64_t j = 0; j < n; ++j) {
      const int64_t m = (n + 3 * j) % (3 * n);
      const long double th = two_pi * (long double)m / (3.0L * (long double)n);
      const long double sh = sinl(th / 2);
      const long double den_re = 2.0L * sh * sh, den_im = sinl(th);  // 1 - e^{-i th}
      const long double dd = den_re * den_re + den_im * den_im;
      re[j] = (num_re * den_re + num_im * den_im) / dd;
      im[j] = (num_im * den_re - num_re * den_im) / dd;
    }
  }
  if (precision == 0) {
    float* o = (float*)out_host;
    for (int64_t j = 0; j < n; ++j) {
      o[2 * j] = (float)re[j];
      o[2 * j + 1] = (float)im[j];
    }
  } else {
    double* o = (double*)out_host;
    for (int64_t j = 0; j < n; ++j) {
      o[2 * j] = (double)re[j];
      o[2 * j + 1] = (double)im[j];
    }
  }
  return TFFT_OK;
}

int tfft_weighted_columns(int precision, const void* src, int64_t n, int64_t row0, int64_t row1, int64_t group,
                          int64_t weight0, void* out, void* stream) {
  if (!src || !out || row1 < row0 || group < 1) return fail(TFFT_EINVAL, "invalid weighted_columns arguments");
  TFFT_TRY(launch_weighted_cols(precision, src, n, row0, row1, group, weight0, out, (cudaStream_t)stream),
           "weighted columns");
  return TFFT_OK;
}

int tfft_vec_add(int precision, void* a, const void* b, int64_t n, void* stream) {
  TFFT_TRY(launch_vadd(precision, a, b, n, (cudaStream_t)stream), "vec add");
  return TFFT_OK;
}

int tfft_vec_axpby(int precision, void* z, int64_t n, double ar, double ai, const void* x, double br, double bi,
                   const void* y, void* stream) {
  TFFT_TRY(launch_axpby(precision, z, n, ar, ai, x, br, bi, y, (cudaStream_t)stream), "axpby");
  return TFFT_OK;
}

int tfft_group_divergence(int precision, const void* ref, const void* s_out, int64_t n, double* out_dev,
                          void* stream) {
  TFFT_TRY(launch_group_div(precision, ref, s_out, n, out_dev, (cudaStream_t)stream), "group divergence");
  return TFFT_OK;
}

int tfft_correction_column(tfft_plan* p, const void* snap_in, const void* snap_out, double weight, void* col,
                           double* res_dev, void* stream) {
  if (!p) return fail(TFFT_EINVAL, "null plan");
  cudaStream_t st = (cudaStream_t)stream;
  tfft_plan* p64 = p;
  const void* in64 = snap_in;
  if (p->prec == 0) {
    if (!p->promoted) {
      int rc = tfft_plan_create(p->n, 1, (int)p->spans.size(), p->spans.data(), p->radices.data(), p->bs, &p->promoted);
      if (rc) return rc;
    }
    p64 = p->promoted;
    int e = p->col64.ensure(p->n * 16);
    if (e) return cuda_fail(e, "promote buffer");
    TFFT_TRY(launch_promote(snap_in, p->col64.p, p->n, st), "promote");
    in64 = p->col64.p;
  }
  int e = p64->col_a.ensure(p->n * 16);
  if (e) return cuda_fail(e, "ref buffer");
  std::vector<DevFault> none;
  int e2 = p64->counters.ensure(8 * sizeof(uint64_t));
  if (e2) return cuda_fail(e2, "counters");
  int rc = run_plain(p64, in64, p64->col_a.p, 1, 0, 0, none, (uint64_t*)p64->counters.p + 4, st);
  if (rc) return rc;
  TFFT_TRY(launch_correction_column(p->prec, snap_out, p64->col_a.p, p->n, weight, col, res_dev, st),
           "correction column");
  return TFFT_OK;
}

static int correct_windows_chunk(tfft_plan* p, const void* x, void* y, int64_t signal_offset, int64_t count,
                                 const int64_t* desc_host, const double* par_host, int enc, double delta,
                                 double* out_host, cudaStream_t st);

int tfft_correct_windows(tfft_plan* p, const void* x, void* y, int64_t signal_offset, int64_t count,
                         const int64_t* desc_host, const double* par_host, int enc, double delta, double* out_host,
                         void* stream) {
  if (!p || !x || !y || count < 0 || (count && (!desc_host || !par_host || !out_host)))
    return fail(TFFT_EINVAL, "invalid correct_windows arguments");
  if (count == 0) return TFFT_OK;
  // items in chunks of <= 256 MB of working vectors (7 per item)
  int64_t per = ((int64_t)256 << 20) / (p->n * 16);
  if (per < 1) per = 1;
  for (int64_t i0 = 0; i0 < count; i0 += per) {
    const int64_t c = count - i0 < per ? count - i0 : per;
    int rc = correct_windows_chunk(p, x, y, signal_offset, c, desc_host + 6 * i0, par_host + 4 * i0, enc, delta,
                                   out_host + 4 * i0, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return TFFT_OK;
}

static int correct_windows_chunk(tfft_plan* p, const void* x, void* y, int64_t signal_offset, int64_t count,
                                 const int64_t* desc_host, const double* par_host, int enc, double delta,
                                 double* out_host, cudaStream_t st) {
  if (enc != ENC_WANG && enc != ENC_ONES) return fail(TFFT_EUNSUPPORTED, "batched correction: wang / ones only");
  const int64_t n = p->n;
  const size_t cb = cbytes(p->prec);
  const size_t vec = (size_t)count * n * cb;
  int e = p->cw_desc.ensure((size_t)count * 6 * sizeof(int64_t));
  if (!e) e = p->cw_par.ensure((size_t)count * 5 * sizeof(double));
  if (!e) e = p->cw_res.ensure((size_t)count * 4 * sizeof(double));
  if (!e) e = p->cw_tin.ensure(vec);
  if (!e) e = p->cw_tout.ensure(vec);
  if (!e) e = p->cw_ref.ensure((size_t)count * n * 16);
  if (!e) e = p->cw_col.ensure(vec);
  if (!e) e = p->cw_sin.ensure(vec);
  if (!e) e = p->cw_sout.ensure(vec);
  if (!e) e = p->cw_gref.ensure(vec);
  if (!e) e = p->part.ensure((size_t)count * ((n + 8191) / 8192) * 2 * sizeof(double));
  if (!e) e = p->counters.ensure(8 * sizeof(uint64_t));
  if (e) return cuda_fail(e, "batched correction workspace");
  const int64_t* desc = (const int64_t*)p->cw_desc.p;
  double* par = (double*)p->cw_par.p;
  double* res = (double*)p->cw_res.p;
  TFFT_TRY((int)cudaMemcpyAsync(p->cw_desc.p, desc_host, (size_t)count * 6 * sizeof(int64_t),
                                cudaMemcpyHostToDevice, st), "desc upload");
  TFFT_TRY((int)cudaMemcpyAsync(p->cw_par.p, par_host, (size_t)count * 4 * sizeof(double), cudaMemcpyHostToDevice,
                                st), "par upload");
  // the triggering transaction's snapshot (abft.py:668-677): desc = {k, r0, r1, w, w0, w1} (local rows)
  TFFT_TRY(launch_wsum_list(p->prec, x, n, desc, 1, 2, count, signal_offset, p->cw_tin.p, st), "t_in");
  TFFT_TRY(launch_wsum_list(p->prec, y, n, desc, 1, 2, count, signal_offset, p->cw_tout.p, st), "t_out");
  // the window sums: kept by the last protected call, else formed here
  const int64_t nw = p->sums_nwin;
  if (p->sums_kind == 1) {
    TFFT_TRY(launch_gather_rows(p->prec, p->winsave.p, 2 * n, desc, 3, count, n, p->cw_sin.p, st), "s_in gather");
    TFFT_TRY(launch_gather_rows(p->prec, (const char*)p->winsave.p + n * cb, 2 * n, desc, 3, count, n, p->cw_sout.p,
                                st), "s_out gather");
  } else if (p->sums_kind == 2) {
    TFFT_TRY(launch_gather_rows(p->prec, p->wsum.p, n, desc, 3, count, n, p->cw_sin.p, st), "s_in gather");
    TFFT_TRY(launch_gather_rows(p->prec, (const char*)p->wsum.p + (size_t)nw * n * cb, n, desc, 3, count, n,
                                p->cw_sout.p, st), "s_out gather");
  } else {
    TFFT_TRY(launch_wsum_list(p->prec, x, n, desc, 4, 5, count, signal_offset, p->cw_sin.p, st), "s_in");
    TFFT_TRY(launch_wsum_list(p->prec, y, n, desc, 4, 5, count, signal_offset, p->cw_sout.p, st), "s_out");
  }
  // FFT(t_in): FP64 for single precision (abft.py:304-314), working precision otherwise
  std::vector<DevFault> none;
  tfft_plan* p64 = p;
  const void* in64 = p->cw_tin.p;
  if (p->prec == 0) {
    if (!p->promoted) {
      int rc = tfft_plan_create(p->n, 1, (int)p->spans.size(), p->spans.data(), p->radices.data(), p->bs,
                                &p->promoted);
      if (rc) return rc;
    }
    p64 = p->promoted;
    e = p->cw_gref.ensure((size_t)count * n * 16);
    if (e) return cuda_fail(e, "promote buffer");
    TFFT_TRY(launch_promote(p->cw_tin.p, p->cw_gref.p, count * n, st), "promote");
    in64 = p->cw_gref.p;
    int e2 = p64->counters.ensure(8 * sizeof(uint64_t));
    if (e2) return cuda_fail(e2, "counters");
  }
  int rc = run_plain(p64, in64, p->cw_ref.p, count, 0, 0, none, (uint64_t*)p64->counters.p + 4, st);
  if (rc) return rc;
  const void* etab = nullptr;
  rc = enc_table(p, false, st, &etab);
  if (rc) return rc;
  TFFT_TRY(launch_correct_items(p->prec, y, desc, par, count, n, p->cw_tout.p, p->cw_ref.p, p->cw_col.p, enc, etab,
                                delta, p->cw_sout.p, (double*)p->part.p, res, st),
           "batched correction");
  // the windows' verification after decontamination (abft.py:502-507)
  rc = run_plain(p, p->cw_sin.p, p->cw_gref.p, count, 0, 0, none, (uint64_t*)p->counters.p + 4, st);
  if (rc) return rc;
  double* gd = par + 4 * count;  // group divergences (the par tail)
  TFFT_TRY(launch_group_div_chunked(p->prec, p->cw_gref.p, p->cw_sout.p, n, count, gd, (double*)p->part.p, st),
           "batched group div");
  std::vector<double> hres((size_t)count * 4), hgd(count);
  TFFT_TRY((int)cudaMemcpyAsync(hres.data(), res, hres.size() * sizeof(double), cudaMemcpyDeviceToHost, st),
           "result download");
  TFFT_TRY((int)cudaMemcpyAsync(hgd.data(), gd, hgd.size() * sizeof(double), cudaMemcpyDeviceToHost, st),
           "group div download");
  TFFT_TRY((int)cudaStreamSynchronize(st), "batched correction sync");
  for (int64_t i = 0; i < count; ++i) {
    out_host[i * 4 + 0] = hres[i * 4 + 0];  // 1: corrected (usable and re-verified)
    out_host[i * 4 + 1] = hres[i * 4 + 1];  // re-verify divergence
    out_host[i * 4 + 2] = hgd[i];           // window group divergence after decontamination
    out_host[i * 4 + 3] = hres[i * 4 + 3];  // max |col| (inf if non-finite)
  }
  return TFFT_OK;
}

int tfft_patch_row(tfft_plan* p, void* y_row, const void* col, int enc, double* res_dev, void* stream) {
  if (!p) return fail(TFFT_EINVAL, "null plan");
  const void* etab = nullptr;
  int rc = enc_table(p, false, (cudaStream_t)stream, &etab);
  if (rc) return rc;
  TFFT_TRY(launch_patch_row(p->prec, y_row, col, p->n, enc, etab, res_dev, (cudaStream_t)stream), "patch row");
  return TFFT_OK;
}

int tfft_row_checksums(tfft_plan* p, const void* x, const void* y, int64_t row0, int64_t nrows, int enc,
                       double delta, const tfft_sums* sums, uint64_t* counters, int count, void* stream) {
  if (!p || !sums) return fail(TFFT_EINVAL, "invalid row_checksums arguments");
  int rc = ensure_row(p, enc);
  if (rc) return rc;
  AbftArgs ab{};
  ab.c_in = sums->c_in;
  ab.c_out = sums->c_out;
  ab.floors = sums->floors;
  ab.div = sums->div;
  if (!counters) {
    int e = p->counters.ensure(8 * sizeof(uint64_t));
    if (e) return cuda_fail(e, "counters");
    counters = (uint64_t*)p->counters.p;
  }
  const void* etab = nullptr;
  rc = enc_table(p, false, (cudaStream_t)stream, &etab);
  if (rc) return rc;
  TFFT_TRY(launch_row_checksums(p->prec, x, y, p->n, row0, nrows, p->rows[enc].p, etab, enc, delta, ab,
                                (Counters*)counters, count, (cudaStream_t)stream),
           "row checksums");
  return TFFT_OK;
}

int tfft_jou_variant(tfft_plan* p, const void* x, void* out, int64_t rows, void* stream) {
  if (!p) return fail(TFFT_EINVAL, "null plan");
  TFFT_TRY(launch_jou(p->prec, 0, x, out, rows, p->n, nullptr, (cudaStream_t)stream), "jou variant");
  return TFFT_OK;
}

int tfft_jou_undo(tfft_plan* p, void* y, int64_t rows, void* stream) {
  if (!p) return fail(TFFT_EINVAL, "null plan");
  const void* twi = nullptr;
  int rc = enc_table(p, true, (cudaStream_t)stream, &twi);
  if (rc) return rc;
  TFFT_TRY(launch_jou(p->prec, 1, nullptr, y, rows, p->n, twi, (cudaStream_t)stream), "jou undo");
  return TFFT_OK;
}

}  // extern "C"
