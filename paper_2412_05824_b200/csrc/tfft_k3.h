// K3 / K4: two-pass (four-step) batched FFT for N beyond the single-pass range,
// optionally with the fused ABFT epilogue. Library-private.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tfft_internal.h"

namespace tfft {

struct K3Plan;

int k3_create(int64_t n, int prec, const int64_t* spans, int nstages, int num_sms, K3Plan** out);
void k3_destroy(K3Plan* p);
int k3_execute(K3Plan* p, const void* x, void* y, int64_t batch, int inverse, const DevFault* faults, int nfaults,
               Counters* counters, void* reserved, cudaStream_t st);
// fused two-sided ABFT on the K4 schedule (forward); cudaErrorNotSupported
// when not applicable. Outputs s_in / s_out [nwin][n] and [B][*nparts][5]
// per-signal checksum partials (launch_signal_epilogue decides them).
int k3_protected(K3Plan* p, const void* x, void* y, int64_t batch, int64_t weight0, const DevFault* faults,
                 int nfaults, Counters* counters, const AbftArgs& ab, const void* row, void* s_in, void* s_out,
                 double* sig_part, int64_t* nparts, cudaStream_t st);
// omega_(s r)^q for q < s into dst (working precision, conj for inverse)
int k3_base_table(K3Plan* p, int prec, int64_t s, int r, int inverse, void* dst, cudaStream_t st);
// true when the two-pass split equals the reference's first stage span, so
// stage-1 strikes land in-kernel on the canonical intermediate
bool k3_strikes_stage1(const K3Plan* p);
// kernel launches one k3_execute makes (1 with the fused K4 schedule)
int k3_launches(const K3Plan* p);
// omega_N^k / conj tables (built lazily; only the Jou encoding reads them)
const void* k3_enc_table(K3Plan* p);
const void* k3_enc_table_inv(K3Plan* p);

// Stage passes (three-stage plans, N = 2^23..2^25): one launch per reference
// stage, each a radix-span Stockham pass over the batch, so every stage
// boundary is a kernel boundary (strikes of any stage land in-kernel) and
// the transform costs nstages HBM round trips instead of one per radix-4 pass.
struct StagePlan;
int stage_create(int64_t n, int prec, const int64_t* spans, int nstages, int num_sms, StagePlan** out);
void stage_destroy(StagePlan* p);
// x -> y through tmp (batch * n elements); faults of any stage (signal rows local)
int stage_execute(StagePlan* p, const void* x, void* y, void* tmp, int64_t batch, int inverse, const DevFault* faults,
                  int nfaults, Counters* counters, cudaStream_t st);
int stage_count(const StagePlan* p);
// Fused two-sided ABFT over the stage passes (forward): checksums and window
// sums in the first / last stage, FFT(s_in) carried as pseudo-signals through
// pa / pb ([nwin][n] each). Outputs per-signal partials [B][*parts][5] (for
// launch_signal_epilogue) and win_div. cudaErrorNotSupported when not applicable.
int stage_protected_parts(const StagePlan* p, int64_t* parts, int64_t* gper);
int stage_protected(StagePlan* p, const void* x, void* y, void* tmp, int64_t batch, int64_t weight0,
                    const DevFault* faults, int nfaults, Counters* counters, int64_t win, int enc, const void* row,
                    void* pa, void* pb, double* sig_part, double* gpart, double* win_div, cudaStream_t st);

}  // namespace tfft
