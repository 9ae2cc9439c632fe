// Internal (library-private) launch parameter blocks shared between the kernel
// translation units and the C-ABI layer (tfft_api.cu). Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tfft {

// one armed fault, already mapped to this launch (signal index relative to x)
struct DevFault {
  int64_t signal;   // row in the launch's batch
  int64_t element;  // element of the stage-boundary intermediate
  int32_t stage;    // only stage 0 is applied by K1; K3 applies 0 and its split stage
  int32_t part;     // 0 = re, 1 = im
  int32_t bit;
  int32_t pad;
};

// Fault lists are uploaded sorted by signal (upload_faults): the first entry
// of `sig` by binary search, so a kernel tile costs O(log nfaults) per
// signal instead of a scan of every armed fault (one fault per window at C3
// is 128 faults per launch).
__host__ __device__ __forceinline__ int fault_lo(const DevFault* f, int n, int64_t sig) {
  int a = 0, b = n;
  while (a < b) {
    const int m = (a + b) >> 1;
    if (f[m].signal < sig) a = m + 1;
    else b = m;
  }
  return a;
}

enum EncKind : int { ENC_WANG = 0, ENC_ONES = 1, ENC_JOU = 2 };

// status words (device): [0] non-finite input seen, [1] triggered signals,
// [2] max divergence (bit pattern of a non-negative double), [3] spare
struct Counters {
  unsigned long long nonfinite;
  unsigned long long triggered;
  unsigned long long max_div_bits;
  unsigned long long spare;
};

struct AbftArgs {
  const void* row;          // left checksum row e^T W, working precision, length N
  int enc;                  // EncKind
  double delta;
  double* c_in;             // [2*B]  complex128 per signal
  double* c_out;            // [2*B]
  double* floors;           // [B]
  double* div;              // [B]
  double* win_div;          // [nwin] group divergence of each verification window
  int64_t win_signals;      // W = T * bs signals per window (last may be short)
  int64_t nwin;
  int mode;                 // K1: 0 one window per slot (small W); 1 windows split into pieces
  int64_t pieces;           // K1: pieces per window (mode 1); K5: segments per CTA
  void* ws;                 // K1: [nwin*pieces][2][N]; K5: [grid][pieces][SPT][2][N] partial window sums
  unsigned int* win_count;  // [nwin] arrival counters (mode 1, pieces > 1), zero on entry
  double* sig_part;         // K5: [B][warps per signal][5] per-warp partials (c_in, ||x||^2, c_out)
};

struct K1Args {
  const void* x;
  void* y;
  int64_t batch;
  int64_t weight0;          // global index of row 0 (weights are weight0 + j + 1)
  const void* tw;           // omega_N^k (conj for inverse), length N
  const DevFault* faults;
  int nfaults;
  Counters* counters;
  AbftArgs abft;
};

// launchers (return cudaError_t as int)
int launch_k1(int prec, int logn, bool inverse, bool abft, const K1Args& a, int num_sms, cudaStream_t st);
int k1_supported(int prec, int logn);
// K5: warp-specialised single-pass kernel (same sizes and results as K1's plain path)
int launch_k5(int prec, int logn, bool inverse, const K1Args& a, int num_sms, cudaStream_t st);
// K5 with the fused two-sided ABFT (forward, N = 2^9..2^12 FP64 / 2^13 FP32):
// window sums in tensor memory, per-(CTA segment, slot) partials written to
// a.abft.ws ([grid][pieces][SPT][2][N], pieces = segments per CTA)
int k5_abft_supported(int prec, int logn);
int launch_k5_abft(int prec, int logn, const K1Args& a, int num_sms, cudaStream_t st);
// the grid and signals per tile the fused-ABFT launch will use for `batch`
int k5_abft_layout(int prec, int logn, int num_sms, int64_t batch, int64_t* grid, int* spt, int* nws);
int launch_k5_window_finish(int prec, int logn, const void* ws, const double* sig_part, int nws, const void* tw,
                            int64_t B, int64_t W, int64_t G, int64_t maxseg, int spt, int64_t nwin, double delta,
                            const AbftArgs& ab, Counters* counters, void* wsave, int num_sms, cudaStream_t st);

}  // namespace tfft

namespace tfft {
int k1_slots(int prec, int logn);

// Per-device launch configuration cache: cudaFuncSetAttribute and the
// occupancy query are per device, so a launcher's "configured" state is kept
// per device ordinal (a function-static flag set on device 0 would
// skip the attribute on device k).
constexpr int kMaxDevices = 64;
struct LaunchCfg {
  bool done[kMaxDevices] = {};
  int per_sm[kMaxDevices] = {};
};
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 ? 0 : (d >= kMaxDevices ? kMaxDevices - 1 : d);
}
}
