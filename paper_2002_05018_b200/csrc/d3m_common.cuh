// d3m_common.cuh -- shared device helpers for the D3M sm_100a kernels.
//
// Complex numbers are interleaved (re, im) doubles, i.e. numpy complex128 /
// cuDoubleComplex layout (double2).  Two families of arithmetic live here:
//
//  * "exact" helpers (x_mul, x_sub, x_div_py, x_div_np, glibc_hypot) use
//    explicit round-to-nearest intrinsics so nvcc can never contract them into
//    FMAs.  They reproduce, bit for bit, the operation order of the
//    reference's numba kernels (kernels.py:36-202 under accel.py:36-40,
//    fastmath=False): complex multiply (ac-bd, ad+bc), CPython scalar
//    division for scalars and fused array expressions, the numpy ufunc
//    Smith division for in-place '/=', and glibc 2.39 hypot for the modulus.
//    They are used where the pivot decisions are made (dense BK kernel).
//  * plain operators for the tensor-core / FMA paths (GEMM, TRSM, solves),
//    whose parity with the reference is to tolerance.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

namespace d3m {

// Host: true the first time first() is called for the current device (one
// instance per call site, e.g. a kernel's shared-memory attribute, which is
// per device); thread-safe.
struct PerDeviceOnce {
  std::atomic<unsigned long long> done{0};
  bool first() {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    return !(done.fetch_or(bit) & bit);
  }
};

using cplx = double2;

__device__ __forceinline__ cplx mk(double re, double im) { return make_double2(re, im); }

// ---- exact (non-contracted) complex arithmetic ---------------------------
__device__ __forceinline__ cplx x_add(cplx a, cplx b) {
  return mk(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ cplx x_sub(cplx a, cplx b) {
  return mk(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
// numba complex_mul_impl: (ac - bd) + (ad + bc) i, four roundings then two.
__device__ __forceinline__ cplx x_mul(cplx a, cplx b) {
  double ac = __dmul_rn(a.x, b.x), bd = __dmul_rn(a.y, b.y);
  double ad = __dmul_rn(a.x, b.y), bc = __dmul_rn(a.y, b.x);
  return mk(__dsub_rn(ac, bd), __dadd_rn(ad, bc));
}
// numba complex_div_impl == CPython _Py_c_quot (scalar '/', fused array exprs).
__device__ __forceinline__ cplx x_div_py(cplx a, cplx b) {
  if (fabs(b.x) >= fabs(b.y)) {
    if (b.x == 0.0) return mk(nan(""), nan(""));
    double ratio = __ddiv_rn(b.y, b.x);
    double denom = __dadd_rn(b.x, __dmul_rn(b.y, ratio));
    return mk(__ddiv_rn(__dadd_rn(a.x, __dmul_rn(a.y, ratio)), denom),
              __ddiv_rn(__dsub_rn(a.y, __dmul_rn(a.x, ratio)), denom));
  }
  if (b.y == 0.0) return mk(nan(""), nan(""));
  double ratio = __ddiv_rn(b.x, b.y);
  double denom = __dadd_rn(__dmul_rn(b.x, ratio), b.y);
  return mk(__ddiv_rn(__dadd_rn(__dmul_rn(a.x, ratio), a.y), denom),
            __ddiv_rn(__dsub_rn(__dmul_rn(a.y, ratio), a.x), denom));
}
// numba np_complex_div_impl (in-place array '/='): Smith with reciprocal scale.
__device__ __forceinline__ cplx x_div_np(cplx a, cplx b) {
  double br = fabs(b.x), bi = fabs(b.y);
  if (br >= bi) {
    if (br == 0.0 && bi == 0.0) return mk(__ddiv_rn(a.x, br), __ddiv_rn(a.y, bi));
    double rat = __ddiv_rn(b.y, b.x);
    double scl = __ddiv_rn(1.0, __dadd_rn(b.x, __dmul_rn(b.y, rat)));
    return mk(__dmul_rn(__dadd_rn(a.x, __dmul_rn(a.y, rat)), scl),
              __dmul_rn(__dsub_rn(a.y, __dmul_rn(a.x, rat)), scl));
  }
  double rat = __ddiv_rn(b.x, b.y);
  double scl = __ddiv_rn(1.0, __dadd_rn(b.y, __dmul_rn(b.x, rat)));
  return mk(__dmul_rn(__dadd_rn(__dmul_rn(a.x, rat), a.y), scl),
            __dmul_rn(__dsub_rn(__dmul_rn(a.y, rat), a.x), scl));
}
// re^2 + im^2 without contraction (kernels.py:46,110,130).
__device__ __forceinline__ double x_abs2(cplx z) {
  return __dadd_rn(__dmul_rn(z.x, z.x), __dmul_rn(z.y, z.y));
}

// glibc 2.39 __hypot (sysdeps/ieee754/dbl-64/e_hypot.c, non-FMA kernel;
// Borges 2019, "An improved algorithm for hypot(a,b)").  Pinned bit-exact
// against host libm hypot by tests/test_hypot.py.
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
  double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= __dmul_rn(2.0, ay)) {
    double delta = __dsub_rn(h, ay);
    t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
    t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
  } else {
    double delta = __dsub_rn(h, ax);
    t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
    t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
  }
  return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}
__device__ __forceinline__ double glibc_hypot(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) {
    if (isinf(x) || isinf(y)) return __longlong_as_double(0x7ff0000000000000LL);
    return __dadd_rn(x, y);
  }
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x, ay = x < y ? x : y;
  const double SCALE = 0x1p-600, LARGE_VAL = 0x1p+511, TINY_VAL = 0x1p-459, EPS = 0x1p-54;
  if (ax > LARGE_VAL) {
    if (ay <= __dmul_rn(ax, EPS)) return __dadd_rn(ax, ay);
    return __ddiv_rn(hypot_kernel(__dmul_rn(ax, SCALE), __dmul_rn(ay, SCALE)), SCALE);
  }
  if (ay < TINY_VAL) {
    if (ax >= __ddiv_rn(ay, EPS)) return __dadd_rn(ax, ay);
    return __dmul_rn(hypot_kernel(__ddiv_rn(ax, SCALE), __ddiv_rn(ay, SCALE)), SCALE);
  }
  if (ay <= __dmul_rn(ax, EPS)) return __dadd_rn(ax, ay);
  return hypot_kernel(ax, ay);
}
__device__ __forceinline__ double x_abs(cplx z) { return glibc_hypot(z.x, z.y); }

// numpy 2.x np.abs on complex128 arrays (the SIMD loop in
// loops_unary_complex.dispatch.c.src, FMA-dispatched on AVX-512 hosts):
// larger * sqrt(fma(r, r, 1)), r = smaller / larger.  dense_ldlt_bk takes
// its pivot-threshold scale and its symmetry check from this function
// (factor.py:94-98), so info/threshold parity needs it bit-exact.
__device__ __forceinline__ double np_abs(cplx z) {
  double r = fabs(z.x), m = fabs(z.y);
  if (isinf(r) || isinf(m)) return __longlong_as_double(0x7ff0000000000000LL);
  if (isnan(r) || isnan(m)) return nan("");
  double L = r > m ? r : m, S = r > m ? m : r;
  if (L == 0.0) return 0.0;
  double q = __ddiv_rn(S, L);
  return __dmul_rn(__dsqrt_rn(fma(q, q, 1.0)), L);
}

// ---- plain (FMA-friendly) complex arithmetic ------------------------------
__device__ __forceinline__ cplx c_add(cplx a, cplx b) { return mk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cplx c_sub(cplx a, cplx b) { return mk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cplx c_mul(cplx a, cplx b) {
  return mk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc += a*b
__device__ __forceinline__ void c_fma(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc -= a*b
__device__ __forceinline__ void c_fms(cplx& acc, cplx a, cplx b) {
  acc.x = fma(-a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(-a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}

// D^{-1} application for one 1x1 pivot (in-place '/=', ufunc division) or
// one 2x2 pivot (kernels.py:161-202).  The 2x2 form is a fused numba array
// expression, so its divisions are the scalar CPython form.
__device__ __forceinline__ void dinv_pair(cplx a, cplx b, cplx c, cplx& x0, cplx& x1) {
  cplx akm1 = x_div_py(a, b), ak = x_div_py(c, b);
  cplx denom = x_sub(x_mul(akm1, ak), mk(1.0, 0.0));
  cplx t1 = x_div_py(x0, b), t2 = x_div_py(x1, b);
  x0 = x_div_py(x_sub(x_mul(ak, t1), t2), denom);
  x1 = x_div_py(x_sub(x_mul(akm1, t2), t1), denom);
}

// ---- warp / block reductions ----------------------------------------------
// argmax with first-index tie break (np.argmax): larger value wins, equal
// values keep the smaller index.
__device__ __forceinline__ void argmax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}
__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    argmax_merge(v, i, v2, i2);
  }
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Pivot threshold of a BK factorisation: pivot_tol * scale (factor.py:99,
// scale = np.abs(W).max() computed on the device), or pivot_tol itself when
// it is an absolute threshold (BkArgs::abs_tol: kernels.bk_factor(W, tol_abs)
// bindings pass the caller's tol_abs unchanged instead of round-tripping it
// through tol_abs / scale * scale, which can move it by an ulp).
__device__ __forceinline__ double bk_threshold(double pivot_tol, double scale, bool abs_tol) {
  return abs_tol ? pivot_tol : __dmul_rn(pivot_tol, scale);
}

// ---- pivot-decision margins (diagnostic, BkArgs::margin) --------------------
// Relative distance of a pivot test "lhs >= rhs" (kernels.py:59-77) to its
// threshold: |lhs - rhs| / max(lhs, rhs); 1 when both sides are 0.  A kernel
// whose arithmetic differs from the reference's by rounding (FMA, another
// update order) takes the same decision whenever this is well above the
// relative rounding of the operands (~1e-15).
__device__ __forceinline__ double test_margin(double lhs, double rhs) {
  const double m = fmax(lhs, rhs);
  return m > 0.0 ? fabs(lhs - rhs) / m : 1.0;
}
// The per-step margins of one pivot decision, in the reference's test order:
// the singularity test, |a_kk| >= alpha colmax, then (rowmax path)
// |a_kk| rowmax >= alpha colmax^2 and |a_imax,imax| >= alpha rowmax as far as
// they are evaluated.  stage: 1 = decided by the first test, 2 = by the
// second, 3 = by the third (or the 2x2 fall-through).
__device__ __forceinline__ double decision_margin(double tol_abs, double absakk, double colmax, double rowmax,
                                                  double absimax, double alpha, int stage) {
  double m = test_margin(tol_abs, fmax(absakk, colmax));
  m = fmin(m, test_margin(absakk, alpha * colmax));
  if (stage >= 2) m = fmin(m, test_margin(absakk * rowmax, alpha * colmax * colmax));
  if (stage >= 3) m = fmin(m, test_margin(absimax, alpha * rowmax));
  return m;
}
// Running top-2 of a first-index argmax: (v, i) the winner, v2 the largest
// value of any other index (ties with the winner give v2 == v: gap 0).
__device__ __forceinline__ void top2_merge(double& v, int& i, double& v2, double w, int wi) {
  if (w > v || (w == v && wi < i)) { v2 = fmax(v2, v); v = w; i = wi; }
  else v2 = fmax(v2, w);
}
// relative gap of the argmax winner v1 over the runner-up v2
__device__ __forceinline__ double argmax_gap(double v1, double v2) {
  return (v1 > 0.0 && v2 >= 0.0) ? (v1 - v2) / v1 : 1.0;
}

}  // namespace d3m
