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
  int mode;                 // 0: one window per slot (small W); 1: windows split into pieces
  int64_t pieces;           // pieces per window (mode 1)
  void* ws;                 // [nwin*pieces][2][N] working-precision partials (mode 1, pieces > 1)
  unsigned int* win_count;  // [nwin] arrival counters (mode 1, pieces > 1), zero on entry
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
// K5 with the fused two-sided ABFT (forward only); a.abft.pieces = pieces per window
int launch_k5_abft(int prec, int logn, const K1Args& a, int num_sms, cudaStream_t st);
// signals per tile and CTAs per SM of a K5 instantiation (host-side work split)
void k5_shape(int prec, int logn, int abft, int* spt, int* ctas_per_sm);

}  // namespace tfft

namespace tfft {
int k1_slots(int prec, int logn);
}
