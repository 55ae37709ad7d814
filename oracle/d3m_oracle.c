/*
 * d3m_oracle.c -- CPU restatement of the reference's dense inner kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the sm_100a
 * product path; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product package
 * never links or calls it.
 *
 * It restates, operation for operation, the five numba kernels of
 * /root/reference/pkg/src/ddsolve/kernels.py as the numba 0.65 JIT backend
 * (accel.py:36-40, fastmath=False) executes them:
 *
 *   - complex multiply  (a+bi)(c+di) = (ac-bd) + (ad+bc)i, no FMA
 *     (numba/cpython/numbers.py complex_mul_impl);
 *   - scalar complex '/' = CPython's _Py_c_quot (numbers.py complex_div_impl);
 *   - in-place array '/=' (np.true_divide ufunc) = Smith with a reciprocal
 *     scale (numba/np/npyfuncs.py np_complex_div_impl), while a fused array
 *     expression such as 'B[k, :] / b' lowers to the scalar CPython form;
 *   - abs(complex) / np.abs = libm hypot (glibc 2.39 in this image).
 *
 * Compile with -ffp-contract=off so no multiply-add is fused: the reference
 * JIT code contains no FMA instructions.
 *
 * Storage contract (kernels.py:7-22): W is n x n row-major with leading
 * dimension lda; only the lower triangle is read or written.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef struct { double re, im; } cplx;

static inline cplx c_mk(double re, double im) { cplx z = {re, im}; return z; }
static inline cplx c_add(cplx a, cplx b) { return c_mk(a.re + b.re, a.im + b.im); }
static inline cplx c_sub(cplx a, cplx b) { return c_mk(a.re - b.re, a.im - b.im); }
static inline cplx c_mul(cplx a, cplx b) {
  double ac = a.re * b.re, bd = a.im * b.im, ad = a.re * b.im, bc = a.im * b.re;
  return c_mk(ac - bd, ad + bc);
}
/* Scalar division: CPython algorithm as lowered by numba (numbers.py:1094-1120). */
static inline cplx c_div_scalar(cplx a, cplx b) {
  if (fabs(b.re) >= fabs(b.im)) {
    if (b.re == 0.0) return c_mk(NAN, NAN);
    double ratio = b.im / b.re;
    double denom = b.re + b.im * ratio;
    return c_mk((a.re + a.im * ratio) / denom, (a.im - a.re * ratio) / denom);
  }
  if (b.im == 0.0) return c_mk(NAN, NAN);
  double ratio = b.re / b.im;
  double denom = b.re * ratio + b.im;
  return c_mk((a.re * ratio + a.im) / denom, (a.im * ratio - a.re) / denom);
}
/* Ufunc division: Smith with reciprocal scale (npyfuncs.py:292-362). */
static inline cplx c_div_ufunc(cplx a, cplx b) {
  double br = fabs(b.re), bi = fabs(b.im);
  if (br >= bi) {
    if (br == 0.0 && bi == 0.0) return c_mk(a.re / br, a.im / bi);
    double rat = b.im / b.re;
    double scl = 1.0 / (b.re + b.im * rat);
    return c_mk((a.re + a.im * rat) * scl, (a.im - a.re * rat) * scl);
  }
  double rat = b.re / b.im;
  double scl = 1.0 / (b.im + b.re * rat);
  return c_mk((a.re * rat + a.im) * scl, (a.im * rat - a.re) * scl);
}
static inline double c_abs(cplx z) { return hypot(z.re, z.im); }
static inline double c_abs2(cplx z) { return z.re * z.re + z.im * z.im; }

#define AT(W, i, j) ((W)[(int64_t)(i) * lda + (j)])

/* (1+sqrt(17))/8, kernels.py:33 */
double d3m_oracle_bk_alpha(void) { return (1.0 + sqrt(17.0)) / 8.0; }

/* Relative distance of a pivot test lhs >= rhs to its threshold (the
 * margin diagnostic of the GPU kernels, d3m_common.cuh test_margin). */
static double test_margin(double lhs, double rhs) {
  double m = lhs > rhs ? lhs : rhs;
  return m > 0.0 ? fabs(lhs - rhs) / m : 1.0;
}
static double fmin2(double a, double b) { return a < b ? a : b; }

/*
 * Bunch-Kaufman LDL^T, kernels.py:36-146.  Returns info (-1 = success,
 * else the failing elimination step); perm/tags/n2x2/growth as the reference.
 * margin (NULL = not tracked): [0] the minimum relative distance of every
 * evaluated test of kernels.py:59-77 to its threshold, [1] the minimum
 * relative gap of the colmax winner over the runner-up (checker of the GPU
 * kernels' BkArgs::margin diagnostic).
 */
int64_t d3m_oracle_bk_factor_m(cplx* W, int64_t n, int64_t lda, double tol_abs,
                               int64_t* perm, int8_t* tags, int64_t* n2x2_out,
                               double* growth_out, double* margin) {
  const double alpha = d3m_oracle_bk_alpha();
  double mdec = 1.0, mgap = 1.0;
  int64_t n2x2 = 0, info = -1;
  double growth = 1.0;
  for (int64_t i = 0; i < n; ++i) { perm[i] = i; tags[i] = 0; }
  if (n == 0) { *n2x2_out = 0; *growth_out = 1.0; return -1; }
  /* kernels.py:45-46: initial trailing max over tril(W) (zeros included). */
  double tm2 = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j <= i; ++j) { double v = c_abs2(AT(W, i, j)); if (v > tm2) tm2 = v; }
  double trail_max = sqrt(tm2);
  int64_t k = 0;
  while (k < n) {
    int64_t kstep = 1, kp, imax = k;
    double absakk = c_abs(AT(W, k, k)), colmax = 0.0;
    if (k + 1 < n) {                     /* first maximiser (np.argmax) */
      double second = -1.0;
      imax = k + 1; colmax = c_abs(AT(W, k + 1, k));
      for (int64_t i = k + 2; i < n; ++i) {
        double v = c_abs(AT(W, i, k));
        if (v > colmax) { second = colmax; colmax = v; imax = i; }
        else if (v > second) second = v;
      }
      if (margin && colmax > 0.0 && second >= 0.0) mgap = fmin2(mgap, (colmax - second) / colmax);
    }
    double amax = absakk > colmax ? absakk : colmax;
    if (margin) mdec = fmin2(mdec, test_margin(tol_abs, amax));
    if (amax <= tol_abs) { info = k; break; }
    if (margin) mdec = fmin2(mdec, test_margin(absakk, alpha * colmax));
    if (absakk >= alpha * colmax) {
      kp = k;
    } else {
      double rowmax = c_abs(AT(W, imax, k));
      for (int64_t j = k + 1; j < imax; ++j) { double v = c_abs(AT(W, imax, j)); if (v > rowmax) rowmax = v; }
      if (imax + 1 < n) {
        double v2 = c_abs(AT(W, imax + 1, imax));
        for (int64_t i = imax + 2; i < n; ++i) { double v = c_abs(AT(W, i, imax)); if (v > v2) v2 = v; }
        if (v2 > rowmax) rowmax = v2;
      }
      if (margin) mdec = fmin2(mdec, test_margin(absakk * rowmax, alpha * colmax * colmax));
      if (absakk * rowmax >= alpha * colmax * colmax) kp = k;
      else {
        if (margin) mdec = fmin2(mdec, test_margin(c_abs(AT(W, imax, imax)), alpha * rowmax));
        if (c_abs(AT(W, imax, imax)) >= alpha * rowmax) kp = imax;
        else { kp = imax; kstep = 2; }
      }
    }
    int64_t kk = k + kstep - 1;
    if (kp != kk) {                      /* kernels.py:79-101 */
      cplx t;
      for (int64_t i = kp + 1; i < n; ++i) { t = AT(W, i, kk); AT(W, i, kk) = AT(W, i, kp); AT(W, i, kp) = t; }
      for (int64_t i = kk + 1; i < kp; ++i) { t = AT(W, i, kk); AT(W, i, kk) = AT(W, kp, i); AT(W, kp, i) = t; }
      t = AT(W, kk, kk); AT(W, kk, kk) = AT(W, kp, kp); AT(W, kp, kp) = t;
      if (kstep == 2) { t = AT(W, kk, k); AT(W, kk, k) = AT(W, kp, k); AT(W, kp, k) = t; }
      for (int64_t j = 0; j < k; ++j) { t = AT(W, kk, j); AT(W, kk, j) = AT(W, kp, j); AT(W, kp, j) = t; }
      int64_t p = perm[kk]; perm[kk] = perm[kp]; perm[kp] = p;
    }
    double step_sq = 0.0;
    if (kstep == 1) {                    /* kernels.py:103-113 */
      tags[k] = 1;
      cplx piv = AT(W, k, k);
      for (int64_t j = k + 1; j < n; ++j) {
        cplx lj = c_div_scalar(AT(W, j, k), piv);
        double cm = 0.0;
        for (int64_t i = j; i < n; ++i) {
          AT(W, i, j) = c_sub(AT(W, i, j), c_mul(AT(W, i, k), lj));
          double v = c_abs2(AT(W, i, j)); if (v > cm) cm = v;
        }
        if (cm > step_sq) step_sq = cm;
      }
      for (int64_t i = k + 1; i < n; ++i) AT(W, i, k) = c_div_ufunc(AT(W, i, k), piv);
    } else {                             /* kernels.py:114-134 */
      tags[k] = 2; tags[k + 1] = 0; ++n2x2;
      cplx d21 = AT(W, k + 1, k);
      cplx d11 = c_div_scalar(AT(W, k + 1, k + 1), d21);
      cplx d22 = c_div_scalar(AT(W, k, k), d21);
      cplx t2 = c_div_scalar(c_mk(1.0, 0.0), c_sub(c_mul(d11, d22), c_mk(1.0, 0.0)));
      cplx d21s = c_div_scalar(t2, d21);
      for (int64_t j = k + 2; j < n; ++j) {
        cplx wk = c_mul(d21s, c_sub(c_mul(d11, AT(W, j, k)), AT(W, j, k + 1)));
        cplx wkp = c_mul(d21s, c_sub(c_mul(d22, AT(W, j, k + 1)), AT(W, j, k)));
        double cm = 0.0;
        for (int64_t i = j; i < n; ++i) {
          cplx u = c_add(c_mul(AT(W, i, k), wk), c_mul(AT(W, i, k + 1), wkp));
          AT(W, i, j) = c_sub(AT(W, i, j), u);
          double v = c_abs2(AT(W, i, j)); if (v > cm) cm = v;
        }
        if (cm > step_sq) step_sq = cm;
        AT(W, j, k) = wk; AT(W, j, k + 1) = wkp;
      }
    }
    int64_t kn = k + kstep;
    if (kn < n) {                        /* kernels.py:135-144 */
      double step_max = sqrt(step_sq);
      if (trail_max > 0.0) {
        double r = step_max / trail_max;
        if (kstep == 2) r = sqrt(r);
        if (r > growth) growth = r;
      }
      trail_max = step_max;
    }
    k = kn;
  }
  *n2x2_out = n2x2; *growth_out = growth;
  if (margin) { margin[0] = mdec; margin[1] = mgap; }
  return info;
}

int64_t d3m_oracle_bk_factor(cplx* W, int64_t n, int64_t lda, double tol_abs,
                             int64_t* perm, int8_t* tags, int64_t* n2x2_out,
                             double* growth_out) {
  return d3m_oracle_bk_factor_m(W, n, lda, tol_abs, perm, tags, n2x2_out, growth_out, 0);
}

/* B <- L^{-1} B, unit lower (kernels.py:149-152).  B is n x m, ldb. */
void d3m_oracle_solve_unit_lower(const cplx* L, int64_t n, int64_t lda, cplx* B,
                                 int64_t m, int64_t ldb) {
  for (int64_t k = 0; k + 1 < n; ++k)
    for (int64_t i = k + 1; i < n; ++i) {
      cplx l = AT(L, i, k);
      for (int64_t c = 0; c < m; ++c)
        B[i * ldb + c] = c_sub(B[i * ldb + c], c_mul(l, B[k * ldb + c]));
    }
}

/* B <- L^{-T} B (kernels.py:155-158): row k minus the ascending sum over i>k. */
void d3m_oracle_solve_unit_lower_t(const cplx* L, int64_t n, int64_t lda, cplx* B,
                                   int64_t m, int64_t ldb) {
  for (int64_t k = n - 2; k >= 0; --k)
    for (int64_t c = 0; c < m; ++c) {
      cplx s = c_mk(0.0, 0.0);
      for (int64_t i = k + 1; i < n; ++i) s = c_add(s, c_mul(AT(L, i, k), B[i * ldb + c]));
      B[k * ldb + c] = c_sub(B[k * ldb + c], s);
    }
}

/* D^{-1} applied from the left (rows) or right (columns), kernels.py:161-202. */
static void dinv_pair(cplx a, cplx b, cplx c, cplx* x0, cplx* x1) {
  cplx akm1 = c_div_scalar(a, b), ak = c_div_scalar(c, b);
  cplx denom = c_sub(c_mul(akm1, ak), c_mk(1.0, 0.0));
  /* 't1 = B[k] / b' and '(...) / denom' are fused numba array expressions,
     which lower to the scalar CPython division, unlike the in-place '/='. */
  cplx t1 = c_div_scalar(*x0, b), t2 = c_div_scalar(*x1, b);
  *x0 = c_div_scalar(c_sub(c_mul(ak, t1), t2), denom);
  *x1 = c_div_scalar(c_sub(c_mul(akm1, t2), t1), denom);
}

void d3m_oracle_apply_dinv_left(const cplx* d, const cplx* e, const int8_t* tags,
                                int64_t n, cplx* B, int64_t m, int64_t ldb) {
  for (int64_t k = 0; k < n;) {
    if (tags[k] == 1) {
      for (int64_t c = 0; c < m; ++c) B[k * ldb + c] = c_div_ufunc(B[k * ldb + c], d[k]);
      k += 1;
    } else {
      for (int64_t c = 0; c < m; ++c) dinv_pair(d[k], e[k], d[k + 1], &B[k * ldb + c], &B[(k + 1) * ldb + c]);
      k += 2;
    }
  }
}

void d3m_oracle_apply_dinv_right(const cplx* d, const cplx* e, const int8_t* tags,
                                 int64_t n, cplx* B, int64_t rows, int64_t ldb) {
  for (int64_t k = 0; k < n;) {
    if (tags[k] == 1) {
      for (int64_t r = 0; r < rows; ++r) B[r * ldb + k] = c_div_ufunc(B[r * ldb + k], d[k]);
      k += 1;
    } else {
      for (int64_t r = 0; r < rows; ++r) dinv_pair(d[k], e[k], d[k + 1], &B[r * ldb + k], &B[r * ldb + k + 1]);
      k += 2;
    }
  }
}

/* glibc hypot, exposed so tests can compare the GPU modulus against libm. */
double d3m_oracle_hypot(double x, double y) { return hypot(x, y); }
void d3m_oracle_hypot_array(const double* x, const double* y, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = hypot(x[i], y[i]);
}
