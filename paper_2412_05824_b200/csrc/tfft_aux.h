// Launchers for the rare-path / boundary kernels in tfft_aux.cu (library-private).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tfft_internal.h"

namespace tfft {

int launch_stockham_pass(int prec, const void* src, void* dst, int64_t rows, int64_t n, int64_t s, int r,
                         const void* base, int64_t base_stride, int inverse, cudaStream_t st);
int launch_flip(int prec, void* buf, int64_t index, int part, int bit, cudaStream_t st);
int launch_scale(int prec, void* buf, int64_t count, double s, cudaStream_t st);
// counters->nonfinite |= any element of buf[0, count) (complex) is not finite
int launch_nonfinite(int prec, const void* buf, int64_t count, Counters* counters, cudaStream_t st);
int launch_row_checksums(int prec, const void* x, const void* y, int64_t n, int64_t row0, int64_t nrows,
                         const void* row, const void* tw, int enc, double delta, const AbftArgs& ab, Counters* counters,
                         int count, cudaStream_t st);
int launch_weighted_cols(int prec, const void* src, int64_t n, int64_t row0, int64_t row1, int64_t gsize,
                         int64_t weight0, void* out, cudaStream_t st);
// one read of x and y: per-signal ABFT sums (via chunk partials + epilogue) and the window sums
int64_t window_sweep_chunks(int64_t n);
int launch_window_sweep(int prec, const void* x, const void* y, int64_t n, int64_t batch, int64_t W, int64_t weight0,
                        const void* row, const void* tw, int enc, void* s_in, void* s_out, double* part,
                        const AbftArgs& ab, double delta, Counters* counters, cudaStream_t st);
// window sums from the fused K5's per-(CTA segment, slot) partials
// per-signal c_in / c_out / floor / divergence from [batch][nparts][5] partials
// (summed in a fixed order), counting triggers and the max divergence
int launch_signal_epilogue(const double* part, int64_t nparts, int64_t n, int64_t batch, double delta,
                           const AbftArgs& ab, Counters* counters, cudaStream_t st);
int launch_wsum_list(int prec, const void* src, int64_t n, const int64_t* desc_dev, int lo, int hi, int64_t count,
                     int64_t weight0, void* out, cudaStream_t st);
int launch_gather_rows(int prec, const void* src, int64_t stride, const int64_t* desc_dev, int col, int64_t count,
                       int64_t n, void* dst, cudaStream_t st);
int launch_correct_items(int prec, void* y, const int64_t* desc_dev, const double* par_dev, int64_t count, int64_t n,
                         const void* tout, const void* ref64_or_ref, void* col, int enc, const void* tw, double delta,
                         void* s_out, double* part, double* res_dev, cudaStream_t st);
int launch_seg_combine(int prec, const void* ws, int64_t n, int64_t B, int64_t W, int64_t G, int64_t maxseg, int spt,
                       int64_t nwin, void* s_in, void* s_out, cudaStream_t st);
// group divergence of `count` long rows through chunk partials (part: count * ceil(n / 8192) * 2 doubles)
int launch_group_div_chunked(int prec, const void* ref, const void* s_out, int64_t n, int64_t count, double* out,
                             double* part, cudaStream_t st);
int launch_axpby(int prec, void* z, int64_t n, double ar, double ai, const void* x, double br, double bi,
                 const void* y, cudaStream_t st);
int launch_vadd(int prec, void* a, const void* b, int64_t n, cudaStream_t st);
int launch_group_div(int prec, const void* ref, const void* s_out, int64_t n, double* out, cudaStream_t st);
int launch_group_div_batched(int prec, const void* ref, const void* s_out, int64_t n, int64_t count, double* out,
                             cudaStream_t st);
int launch_base_table(int prec, int64_t s, int r, int inverse, void* dst, cudaStream_t st);
int launch_correction_column(int prec, const void* snap_out, const void* ref64, int64_t n, double weight, void* col,
                             double* res, cudaStream_t st);
int launch_patch_row(int prec, void* yk, const void* col, int64_t n, int enc, const void* tw, double* res,
                     cudaStream_t st);
int launch_promote(const void* in, void* out, int64_t n, cudaStream_t st);
int launch_jou(int prec, int undo, const void* x, void* out, int64_t rows, int64_t n, const void* tw_inv,
               cudaStream_t st);

}  // namespace tfft
