// Common device building blocks for the sm_100a batched FFT kernels.
//
// Every arithmetic op on signal data goes through the *_rn intrinsics below, so
// nvcc never contracts across them: the plain kernels and their ABFT twins run
// the identical instruction sequence on y, which is what makes a fault-free
// run_protected bitwise equal to execute_plan (reference abft.py:694-696,
// tests/test_abft.py:197-206).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tfft {

template <typename T> struct cplx;
template <> struct cplx<float> { using type = float2; };
template <> struct cplx<double> { using type = double2; };
template <typename T> using C = typename cplx<T>::type;

__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float rfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rfma(double a, double b, double c) { return __fma_rn(a, b, c); }

template <typename T> __device__ __forceinline__ C<T> mk(T re, T im) { C<T> r; r.x = re; r.y = im; return r; }
template <typename T> __device__ __forceinline__ C<T> cadd(C<T> a, C<T> b) { return mk<T>(radd(a.x, b.x), radd(a.y, b.y)); }
template <typename T> __device__ __forceinline__ C<T> csub(C<T> a, C<T> b) { return mk<T>(rsub(a.x, b.x), rsub(a.y, b.y)); }
// (a.x b.x - a.y b.y, a.x b.y + a.y b.x) with one rounding on the fused term
template <typename T> __device__ __forceinline__ C<T> cmul(C<T> a, C<T> b) {
  return mk<T>(rfma(a.x, b.x, -rmul(a.y, b.y)), rfma(a.x, b.y, rmul(a.y, b.x)));
}

// FP32 complex arithmetic on the packed f32x2 pipe of sm_100 (FADD2 / FMUL2 /
// FFMA2: both lanes in one instruction, operand swaps, broadcasts and per-lane
// negation folded into the operands): half the FP32 instructions of the
// scalar forms, with the same roundings per component, so every result is
// bitwise the scalar version's.
#define TFFT_F2(v) "f"(v.x), "f"(v.y)
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(r.x), "=f"(r.y) : TFFT_F2(a), TFFT_F2(b));
  return r;
}
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(r.x), "=f"(r.y) : TFFT_F2(a), TFFT_F2(b));
  return r;
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(r.x), "=f"(r.y) : TFFT_F2(a), TFFT_F2(b));
  return r;
}
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(r.x), "=f"(r.y) : TFFT_F2(a), TFFT_F2(b), TFFT_F2(c));
  return r;
}
#undef TFFT_F2
#ifndef TFFT_NO_F32X2  // (experiment switch: the scalar forms)
template <> __device__ __forceinline__ float2 cadd<float>(float2 a, float2 b) { return f2_add(a, b); }
template <> __device__ __forceinline__ float2 csub<float>(float2 a, float2 b) { return f2_sub(a, b); }
// t = (a.y b.y, a.y b.x) rounded; (a.x b.x - t.x, a.x b.y + t.y) in one fused op
template <> __device__ __forceinline__ float2 cmul<float>(float2 a, float2 b) {
  const float2 t = f2_mul(make_float2(a.y, a.y), make_float2(b.y, b.x));
  return f2_fma(make_float2(a.x, a.x), b, make_float2(-t.x, t.y));
}
#endif
// multiply by -i (forward) or +i (inverse)
template <typename T, bool INV> __device__ __forceinline__ C<T> rot90(C<T> a) {
  return INV ? mk<T>(-a.y, a.x) : mk<T>(a.y, -a.x);
}
// acc + w x (checksum window sums) and acc + r v (checksum dot products),
// one rounding per fused term; FP32: packed (FFMA2), same roundings per lane
template <typename T> __device__ __forceinline__ C<T> caxpy(T w, C<T> x, C<T> acc) {
  return mk<T>(rfma(w, x.x, acc.x), rfma(w, x.y, acc.y));
}
template <typename T> __device__ __forceinline__ C<T> cmac(C<T> r, C<T> v, C<T> acc) {
  return mk<T>(rfma(r.x, v.x, rfma(-r.y, v.y, acc.x)), rfma(r.x, v.y, rfma(r.y, v.x, acc.y)));
}
template <typename T> __device__ __forceinline__ C<T> cscale(C<T> a, T s) { return mk<T>(rmul(a.x, s), rmul(a.y, s)); }
#ifndef TFFT_NO_F32X2
template <> __device__ __forceinline__ float2 cscale<float>(float2 a, float s) { return f2_mul(a, make_float2(s, s)); }
template <> __device__ __forceinline__ float2 caxpy<float>(float w, float2 x, float2 acc) {
  return f2_fma(make_float2(w, w), x, acc);
}
template <> __device__ __forceinline__ float2 cmac<float>(float2 r, float2 v, float2 acc) {
  return f2_fma(make_float2(r.x, r.x), v, f2_fma(make_float2(-r.y, r.y), make_float2(v.y, v.x), acc));
}
#endif

// Twiddle run w_j = base * step^j, j = 0, 1, ... in ascending order, as four
// interleaved product chains (w_{j+4} = w_j * step^4): a dependency depth of
// about j/4 + 2 complex products instead of the j of the single recurrence,
// which left the four-step twiddle epilogues latency-bound. next(j) returns
// w_j and must be called with j = 0, 1, 2, ... (unrolled, compile-time j).
template <typename T>
struct TwRun {
  C<T> c[4], s4;
  __device__ __forceinline__ TwRun(C<T> base, C<T> step) {
    const C<T> s2 = cmul<T>(step, step);
    c[0] = base;
    c[1] = cmul<T>(base, step);
    c[2] = cmul<T>(base, s2);
    c[3] = cmul<T>(c[1], s2);
    s4 = cmul<T>(s2, s2);
  }
  __device__ __forceinline__ C<T> next(int j) {
    const C<T> w = c[j & 3];
    c[j & 3] = cmul<T>(c[j & 3], s4);
    return w;
  }
};

// ---------------------------------------------------------------------------
// constant twiddles omega_R^k = exp(-+2 pi i k / R) for the in-register codelets

template <typename T, int R, int K, bool INV>
__device__ __forceinline__ C<T> wconst_mul(C<T> a) {
  constexpr int k = ((K % R) + R) % R;
  if constexpr (k == 0) {
    return a;
  } else if constexpr (4 * k == R) {
    return rot90<T, INV>(a);
  } else if constexpr (2 * k == R) {
    return mk<T>(-a.x, -a.y);
  } else if constexpr (4 * k == 3 * R) {
    return rot90<T, !INV>(a);
  } else if constexpr (8 * k == R || 8 * k == 3 * R || 8 * k == 5 * R || 8 * k == 7 * R) {
    // (+-1 +- i)/sqrt2: two adds and two muls
    const T h = (T)0.70710678118654752440084436210485;
    // w = (cx + i sy) / sqrt2 with cx, sy in {+1, -1}
    constexpr int cx = (8 * k == R || 8 * k == 7 * R) ? 1 : -1;
    constexpr int sy0 = (8 * k == R || 8 * k == 3 * R) ? -1 : 1;  // forward sign
    constexpr int sy = INV ? -sy0 : sy0;
    // (a.x + i a.y)(cx + i sy) = (cx a.x - sy a.y) + i (sy a.x + cx a.y)
    T re = (cx == 1) ? (sy == 1 ? rsub(a.x, a.y) : radd(a.x, a.y)) : (sy == 1 ? -radd(a.x, a.y) : rsub(a.y, a.x));
    T im = (cx == 1) ? (sy == 1 ? radd(a.x, a.y) : rsub(a.y, a.x)) : (sy == 1 ? rsub(a.x, a.y) : -radd(a.x, a.y));
    return mk<T>(rmul(re, h), rmul(im, h));
  } else {
    // remaining angles of the radix-16 codelet: k odd, omega_16^k = exp(-i pi k / 8)
    static_assert(R == 16, "codelets stop at radix 16");
    const T c1 = (T)0.92387953251128675612818318939678829;  // cos(pi/8)
    const T s1 = (T)0.38268343236508977172845998403039887;  // sin(pi/8)
    T c, s;  // forward omega = c + i s
    if constexpr (k == 1) { c = c1; s = -s1; }
    else if constexpr (k == 3) { c = s1; s = -c1; }
    else if constexpr (k == 5) { c = -s1; s = -c1; }
    else if constexpr (k == 7) { c = -c1; s = -s1; }
    else if constexpr (k == 9) { c = -c1; s = s1; }
    else if constexpr (k == 11) { c = -s1; s = c1; }
    else if constexpr (k == 13) { c = s1; s = c1; }
    else { c = c1; s = s1; }
    if constexpr (INV) s = -s;
    return cmul<T>(a, mk<T>(c, s));
  }
}


// ---------------------------------------------------------------------------
// in-register DFT codelets, natural order in and out (forward: omega = e^{-2 pi i/R})

template <typename T, bool INV>
__device__ __forceinline__ void dft2(C<T>& a0, C<T>& a1) {
  C<T> t = a0;
  a0 = cadd<T>(t, a1);
  a1 = csub<T>(t, a1);
}

template <typename T, bool INV>
__device__ __forceinline__ void dft4(C<T>& a0, C<T>& a1, C<T>& a2, C<T>& a3) {
  C<T> A = cadd<T>(a0, a2), B = csub<T>(a0, a2);
  C<T> Cc = cadd<T>(a1, a3), D = rot90<T, INV>(csub<T>(a1, a3));
  a0 = cadd<T>(A, Cc);
  a2 = csub<T>(A, Cc);
  a1 = cadd<T>(B, D);
  a3 = csub<T>(B, D);
}

template <typename T, int R, bool INV>
__device__ __forceinline__ void dft(C<T>* a) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    dft2<T, INV>(a[0], a[1]);
  } else if constexpr (R == 4) {
    dft4<T, INV>(a[0], a[1], a[2], a[3]);
  } else if constexpr (R == 8) {
    dft4<T, INV>(a[0], a[2], a[4], a[6]);
    dft4<T, INV>(a[1], a[3], a[5], a[7]);
    a[3] = wconst_mul<T, 8, 1, INV>(a[3]);
    a[5] = wconst_mul<T, 8, 2, INV>(a[5]);
    a[7] = wconst_mul<T, 8, 3, INV>(a[7]);
    // even half sits at a[0,2,4,6] (bins 0..3), odd half at a[1,3,5,7]
    C<T> e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6];
    C<T> o0 = a[1], o1 = a[3], o2 = a[5], o3 = a[7];
    a[0] = cadd<T>(e0, o0); a[4] = csub<T>(e0, o0);
    a[1] = cadd<T>(e1, o1); a[5] = csub<T>(e1, o1);
    a[2] = cadd<T>(e2, o2); a[6] = csub<T>(e2, o2);
    a[3] = cadd<T>(e3, o3); a[7] = csub<T>(e3, o3);
  } else if constexpr (R == 16) {
    // n = 4 n1 + n2; inner 4-point DFTs over n1, twiddle omega_16^{n2 k1}, outer over n2
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4<T, INV>(a[n2], a[4 + n2], a[8 + n2], a[12 + n2]);
    // a[4 k1 + n2] now holds B[n2][k1]
    a[5] = wconst_mul<T, 16, 1, INV>(a[5]);
    a[6] = wconst_mul<T, 16, 2, INV>(a[6]);
    a[7] = wconst_mul<T, 16, 3, INV>(a[7]);
    a[9] = wconst_mul<T, 16, 2, INV>(a[9]);
    a[10] = wconst_mul<T, 16, 4, INV>(a[10]);
    a[11] = wconst_mul<T, 16, 6, INV>(a[11]);
    a[13] = wconst_mul<T, 16, 3, INV>(a[13]);
    a[14] = wconst_mul<T, 16, 6, INV>(a[14]);
    a[15] = wconst_mul<T, 16, 9, INV>(a[15]);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<T, INV>(a[4 * k1], a[4 * k1 + 1], a[4 * k1 + 2], a[4 * k1 + 3]);
    // a[4 k1 + k2] holds X[k1 + 4 k2]: transpose the 4x4 index map into natural order
    C<T> t[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) t[k1 + 4 * k2] = a[4 * k1 + k2];
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = t[k];
  } else {
    static_assert(R <= 16, "radix > 16");
  }
}

// ---------------------------------------------------------------------------
// IEEE bit flip (reference fault.py:25-38) on one component of a complex value

__device__ __forceinline__ float flip_bits(float v, int bit) {
  return __uint_as_float(__float_as_uint(v) ^ (1u << bit));
}
__device__ __forceinline__ double flip_bits(double v, int bit) {
  return __longlong_as_double(__double_as_longlong(v) ^ (1ll << bit));
}

// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA 1-D) helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TFFT_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TFFT_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// wait with back-off, for the producer / releaser warps: a tight try_wait
// loop would take issue slots from the consumer warps of the same SM sub-partition
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint: the hardware parks the thread until the
// phase completes (or ~1 ms passes), so an idle producer costs no issue slots
__device__ __forceinline__ bool mbar_try_suspend(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_suspend(bar, parity)) {
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// streaming (evict-first) global store of one complex value
__device__ __forceinline__ void st_cs(float2* p, float2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs(double2* p, double2 v) { __stcs(p, v); }

template <typename T> __device__ __forceinline__ bool finite2(C<T> v) { return isfinite(v.x) && isfinite(v.y); }


// Non-finite detection on the integer pipe (isfinite of a double is two DSETP
// on the half-rate FP64 pipe per element): nf_acc keeps the largest exponent
// field seen, which is all-ones exactly when some value was Inf or NaN
template <typename T> __device__ __forceinline__ unsigned nf_acc(unsigned acc, C<T> v) {
  if constexpr (sizeof(T) == 8)
    return __vimax3_u32(acc, (unsigned)__double2hiint(v.x) & 0x7ff00000u, (unsigned)__double2hiint(v.y) & 0x7ff00000u);
  else
    return __vimax3_u32(acc, __float_as_uint(v.x) & 0x7f800000u, __float_as_uint(v.y) & 0x7f800000u);
}
template <typename T> __device__ __forceinline__ bool nf_bad(unsigned acc) {
  return acc == (sizeof(T) == 8 ? 0x7ff00000u : 0x7f800000u);
}

// XOR swizzle (element units) so Stockham scatter writes hit distinct banks:
// 16 float2 / 8 double2 slots per 128-byte bank row.
template <typename T> __device__ __forceinline__ int swz(int a) {
  if constexpr (sizeof(T) == 4) return a ^ ((a >> 4) & 15);
  else return a ^ ((a >> 3) & 7);
}

// ---------------------------------------------------------------------------
// Tensor memory (TMEM) as a per-thread accumulator store (sm_100a tcgen05).
// A warp reaches the 32 TMEM lanes of its quadrant (warp id % 4); with the
// 32x32b shape thread l of the warp reads/writes columns [col, col + 16) of
// lane 32 * (warp % 4) + l. Used by the fused-ABFT K5 for the window sums, so
// the FFT keeps its register budget (the accumulators never occupy registers
// or shared memory bandwidth).

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {  // one full warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // the allocating warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

}  // namespace tfft
