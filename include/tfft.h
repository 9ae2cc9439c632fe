/*
 * tfft.h — C ABI of libtfft.so, the B200 (sm_100a) batched 1-D complex FFT with
 * fused two-sided ABFT and in-kernel fault injection.
 *
 * This is the drop-in boundary for the reference package `resilient-fft` 0.1.0
 * (/root/reference/pkg/src/resilient_fft). The reference's plugin point is the
 * backend registry (backend.py:21-66) whose modules export one Stockham pass,
 * `stockham_pass(src, dst, s, r, base, inverse)` (_kernels.pyx:74-84); its
 * callers (_run_transaction fft_core.py:255-280, execute_plan :296-329,
 * run_protected abft.py:690-752) loop over transactions in Python. Here the
 * whole plan runs per call, on device buffers, and the Python host
 * (paper_2412_05824_b200/) keeps the reference's API and decision logic.
 *
 * Conventions: plain C types only. Signal data is interleaved complex
 * (complex64 = 2 x float, complex128 = 2 x double), B rows of N samples,
 * row-major, exactly numpy's layout. Pointers named `x`, `y`, `buf`, `col`,
 * `ref`, `res_dev`, `counters` are DEVICE pointers; `out_host` is host memory.
 * `stream` is a cudaStream_t (NULL = legacy default stream). Calls are
 * asynchronous on `stream` unless stated otherwise. A plan is reentrant only
 * on one stream at a time (it owns scratch buffers).
 *
 * Return codes: 0 ok, 1 invalid argument, 2 non-finite input, 3 CUDA error,
 * 4 out of memory, 5 unsupported size; tfft_last_error() gives the message.
 */
#ifndef TFFT_H
#define TFFT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TFFT_OK 0
#define TFFT_EINVAL 1
#define TFFT_ENONFINITE 2
#define TFFT_ECUDA 3
#define TFFT_ENOMEM 4
#define TFFT_EUNSUPPORTED 5

#define TFFT_SINGLE 0 /* complex64  (fft_core.py:22 "single") */
#define TFFT_DOUBLE 1 /* complex128 (fft_core.py:22 "double") */

#define TFFT_ENC_WANG 0 /* abft.py:93-94  omega_3^(k mod 3) */
#define TFFT_ENC_ONES 1 /* abft.py:88-89 */
#define TFFT_ENC_JOU 2  /* abft.py:90-92  omega_N^k, with the x' = 2x_k + x_(k+1) variant */

typedef struct tfft_plan tfft_plan;

/* One armed single-event upset (reference FaultSpec, fault.py:52-63). Indices
 * are GLOBAL (transaction = signal / bs over the whole, unsharded batch).
 * part: 0 = re, 1 = im. Stage k strikes the canonical stage-boundary
 * intermediate before stage k's first pass (fft_core.py:271-272). */
typedef struct {
  int64_t transaction;
  int64_t signal;
  int64_t element;
  int32_t stage;
  int32_t part;
  int32_t bit;
  int32_t reserved;
} tfft_fault;

/* Device outputs of a protected run (abft.py:264-272 _BatchSums + windows). */
typedef struct {
  double* c_in;    /* [2*B] complex128 left checksums of the inputs */
  double* c_out;   /* [2*B] complex128 checksums of the outputs */
  double* floors;  /* [B]   ||x||_2 / sqrt(N) */
  double* div;     /* [B]   relative divergence, +inf for non-finite c_out */
  double* win_div; /* [ceil(ceil(B/bs)/T)] group divergence of each window */
} tfft_sums;

/* Device counters, 4 x uint64: [0] non-finite input seen, [1] signals with
 * div > delta, [2] bit pattern of max div (non-negative double), [3] spare.
 * Zeroed by every tfft_execute / tfft_protected call. */

int tfft_version(void);
const char* tfft_last_error(void);
/* number of kernels this library launched since load (evidence counter) */
uint64_t tfft_launch_count(void);

/* Plan = reference build_plan(PlanParams) (plan.py:148-152 -> fft_core.py:185-202):
 * stage spans/radices fix the transaction size bs and the stage boundaries at
 * which stage-k faults strike. The kernels choose their own radix schedule. */
int tfft_plan_create(int64_t n, int precision, int nstages, const int64_t* spans, const int32_t* radices,
                     int64_t bs, tfft_plan** out);
int tfft_plan_destroy(tfft_plan* plan);

/* Debug hook of the CLI self-test (reference cli.py:254-264 `_skew_plan`):
 * multiplies the plan's w_N^1 twiddle (forward and inverse tables) by
 * (1 + 1e-3) so the oracle and checksum checks must fail. Never used by a
 * transform; destroy the plan afterwards. */
int tfft_debug_skew_twiddle(tfft_plan* plan);

/* Plain transform of `batch` rows, out of place; replaces execute_plan's
 * transaction loop (fft_core.py:296-329) and _run_transaction (:255-280),
 * including armed fault strikes and inverse x 1/N. `signal_offset` is the
 * global index of row 0 (batch sharding). Non-finite input sets counters[0]. */
int tfft_execute(tfft_plan* plan, const void* x, void* y, int64_t batch, int inverse, int64_t signal_offset,
                 const tfft_fault* faults, int nfaults, uint64_t* counters, void* stream);

/* Fused protected transform (abft.py:690-752 up to the decision replay): the
 * forward transform plus per-signal checksums and per-window group
 * divergences in the same kernel. `group_size` = T transactions per window;
 * `signal_offset` must be a multiple of T*bs. */
int tfft_protected(tfft_plan* plan, const void* x, void* y, int64_t batch, int64_t signal_offset, int enc_kind,
                   double delta, int64_t group_size, const tfft_fault* faults, int nfaults, const tfft_sums* sums,
                   uint64_t* counters, void* stream);

/* The reference plugin kernel itself (_kernels.pyx:74-84): one radix-2/4 DIT
 * Stockham pass over `rows` rows; base = omega_(s r)^q, q < s (conj for inverse). */
int tfft_stockham_pass(const void* src, void* dst, int64_t rows, int64_t n, int64_t s, int r, const void* base,
                       int inverse, int precision, void* stream);

/* Left checksum row e^T W of a named encoding (abft.py:116-147), closed form
 * with integer phase reduction in extended precision, rounded to `precision`;
 * writes n complex values to out_host. Synchronous, host only. */
int tfft_left_row(int enc_kind, int64_t n, int precision, void* out_host);

/* ---- replay-engine primitives (abft.py:342-585), all on device ----------- */

/* out[g] = sum_{j in group g} (weight0 + j + 1) * src[j] for consecutive groups
 * of `group` rows in [row0, row1) (abft.py:668-677), FP64 accumulation. */
int tfft_weighted_columns(int precision, const void* src, int64_t n, int64_t row0, int64_t row1, int64_t group,
                          int64_t weight0, void* out, void* stream);
int tfft_vec_add(int precision, void* a, const void* b, int64_t n, void* stream);
int tfft_vec_axpby(int precision, void* z, int64_t n, double ar, double ai, const void* x, double br, double bi,
                   const void* y, void* stream);
/* ||ref - s_out|| / max(||ref||, 1e-30) -> *out_dev (abft.py:502-507) */
int tfft_group_divergence(int precision, const void* ref, const void* s_out, int64_t n, double* out_dev,
                          void* stream);
/* col = (snap_out - FFT(snap_in)) / weight with the FFT in FP64 for single
 * precision plans (abft.py:297-317); res_dev[0] = all finite, [1] = max|col|. */
int tfft_correction_column(tfft_plan* plan, const void* snap_in, const void* snap_out, double weight, void* col,
                           double* res_dev, void* stream);
/* Batched online correction of windows holding exactly one triggered signal
 * (abft.py:392-418 + :493-551, the replay's common case, all items at once):
 * item i has desc_host[6i..6i+5] = {k, r0, r1, w, w0, w1} (local rows: the
 * signal, its transaction [r0, r1), its window index and rows [w0, w1)) and
 * par_host[4i..4i+3] = {weight w_k, floor_k, Re c_in_k, Im c_in_k}. For each:
 * t_in / t_out of the transaction, col = (t_out - FFT(t_in)) / w_k (FFT in FP64
 * for single precision), usable = finite && max|col| <= 16 log2N floor sqrt N;
 * when usable and the re-verify detect(c_in, (y_k - col) . enc) holds, y_k -=
 * col and the window's s_out -= w_k col; then the window's group divergence.
 * out_host[4i..4i+3] = {corrected (1/0), re-verify divergence, group divergence,
 * max|col|}. y is untouched for items not corrected. Window sums come from the
 * last tfft_protected call on this plan when it kept them. Synchronous. */
int tfft_correct_windows(tfft_plan* plan, const void* x, void* y, int64_t signal_offset, int64_t count,
                         const int64_t* desc_host, const double* par_host, int enc_kind, double delta,
                         double* out_host, void* stream);
/* y_row -= col; res_dev[2..3] = y_row . enc (abft.py:404-406) */
int tfft_patch_row(tfft_plan* plan, void* y_row, const void* col, int enc_kind, double* res_dev, void* stream);
/* per-row checksums for rows [row0, row0+nrows) of x/y into `sums`
 * (abft.py:648-665); count != 0 also bumps counters[1..2]. */
int tfft_row_checksums(tfft_plan* plan, const void* x, const void* y, int64_t row0, int64_t nrows, int enc_kind,
                       double delta, const tfft_sums* sums, uint64_t* counters, int count, void* stream);
/* Jou encoding input variant and output undo (abft.py:333-339) */
int tfft_jou_variant(tfft_plan* plan, const void* x, void* out, int64_t rows, void* stream);
int tfft_jou_undo(tfft_plan* plan, void* y, int64_t rows, void* stream);

/* ---- multi-GPU (batch sharding) -------------------------- */

/* The one collective of a sharded protected run: sums_dev[0..nsums) (int64:
 * signal sweeps, verifications, corrections, recomputations, events) are
 * SUM-reduced and max_dev[0] (max divergence, double) MAX-reduced across the
 * ranks of `nccl_comm` (an ncclComm_t), in one ncclGroupStart/End on `stream`.
 * NCCL comes from the libnccl.so.2 already loaded in the process (the one that
 * made the communicator). Replaces the reference's single-process counters
 * (abft.py:201-218, RunStats) for a batch split over GPUs. */
int tfft_allreduce_stats(int64_t* sums_dev, int nsums, double* max_dev, void* nccl_comm, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TFFT_H */
