// K4: fused two-pass batched FFT with an L2-resident intermediate ring
// (tfft_k4.cu). Library-private.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tfft_internal.h"

namespace tfft {

// (log2 N1, log2 N2) splits with a compiled K4 instantiation: the reference's
// balanced two-stage splits for 2^13..2^22 (plan.py _stage_exponents) plus the
// curated 2^17 row (256, 512)
#define TFFT_K4_PAIRS \
  TFFT_K4(7, 6) TFFT_K4(7, 7) TFFT_K4(8, 7) TFFT_K4(8, 8) TFFT_K4(8, 9) TFFT_K4(9, 9) TFFT_K4(10, 9) \
  TFFT_K4(10, 10) TFFT_K4(11, 10) TFFT_K4(11, 11)

struct K4Args {
  const void* x;
  void* y;
  void* z;               // intermediate ring: 3 slots of group * N elements
  int64_t batch;
  int64_t group;         // G signals per group
  int64_t ngroups;
  int64_t ta, tb;        // pass-A / pass-B tiles of a full group
  int64_t ta_last, tb_last;  // ... of the last group
  const void* tw1;       // omega_N1^m (conj for inverse)
  const void* tw2;       // omega_N2^m
  const void* hi;        // omega_N^{h 2^lo_bits}
  const void* lo;        // omega_N^l
  int lo_bits;
  const DevFault* faults;
  int nfaults;
  int strike_stage;      // 1 when pass A's output is the reference's stage-1 boundary, else -1
  Counters* counters;
  unsigned long long* ticket;  // zeroed before the launch
  unsigned* done_a;      // [ngroups] finished pass-A tiles, zeroed before the launch
  unsigned* done_b;      // [ngroups]
  unsigned* line_cnt;    // K7: [batch][N1/8] finished pass-B tiles per ring line group (null: no discards)
  // ---- fused two-sided ABFT (K4 only; abft = 0: plain transform). After the
  // B tiles of each group come its C tiles: (window, position chunk) items
  // that read x and y of the window's signals while they are still in L2 and
  // form the window sums s_in / s_out (complete: G % win == 0) and per
  // (signal, chunk) checksum partials (abft.py:648-665, :592-624).
  int abft;
  int enc;               // ENC_WANG / ENC_ONES
  int64_t win;           // W = T * bs signals per verification window
  int64_t tc, tc_last;   // C tiles of a full / the last group
  int64_t nchunk;        // position chunks per signal (one C tile each)
  int64_t weight0;       // global index of row 0 (location weights weight0 + j + 1)
  const void* row;       // left checksum row (working precision)
  void* s_in;            // [nwin][N]
  void* s_out;           // [nwin][N]
  double* sig_part;      // [B][nchunk][5]
  unsigned* done_w;      // [nwin] finished B tiles per window, zeroed before the launch
};

bool k4_supported(int prec, int l1, int l2);
int k4_columns_per_tile(int prec, int logl, int lmax);
int launch_k4(int prec, bool inverse, int l1, int l2, const K4Args& a, int num_sms, cudaStream_t st);
// fused-ABFT K4 (forward): C-tile chunk width in elements and consumer warps
int k4_abft_chunk(int prec, int l1, int l2);
int launch_k4_abft(int prec, int l1, int l2, const K4Args& a, int num_sms, cudaStream_t st);
// K7: FP64 K4 variant with warp-local columns (columns <= 512 points); the
// intermediate ring is p-major instead of K4's column-blocked layout
bool k7_supported(int prec, int l1, int l2);
// pass-A / pass-B columns per K7 tile
int k7_columns_per_tile(int prec, int logl);
// pass-B tiles narrower than a ring line: line groups discarded by the releaser (K4Args::line_cnt)
bool k7_line_discard(int prec, int l1, int l2);
int launch_k7(int prec, bool inverse, int l1, int l2, const K4Args& a, int num_sms, cudaStream_t st);

}  // namespace tfft
