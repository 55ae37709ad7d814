// bk_exact.cu -- batched complex-symmetric Bunch-Kaufman LDL^T, bit-exact.
//
// One CTA factors one matrix in place (lower triangle, packed storage of
// kernels.py:7-22).  Every arithmetic operation reproduces the reference's
// numba kernel _bk_factor (kernels.py:36-146) in the same order and rounding,
// so the pivot sequence, the tags, the growth factor AND the factor values
// are bit-identical to the CPU reference.  The kernel is used for the
// supernode diagonal blocks of block_ldlt (n ~ 256, on the critical path,
// overlapped with the trailing updates) and for dense_ldlt_bk.
//
// Per elimination step k (all threads of the CTA, __syncthreads between):
//   1. argmax |W[i,k]| over i>k (glibc-hypot modulus, first-index ties)
//   2. if needed, rowmax over row/column imax (kernels.py:66-70)
//   3. the symmetric interchange kk<->kp incl. computed L rows (:79-101)
//   4. stage column k (and k+1) and the multipliers l_j in shared memory
//   5. rank-1 / rank-2 update of the trailing lower triangle, warp per row
//      (coalesced along the row), with the per-step growth max (:102-144).
//
// The prologue also computes numpy's np.abs(W).max() (the pivot-threshold
// scale) and np.abs(W - W.T).max() (the symmetry check) of factor.py:94-98.
#include "d3m_common.cuh"
#include "d3m_kernels.h"

namespace d3m {

constexpr double kBkAlpha = 0.6403882032022076;  // (1 + sqrt(17)) / 8, kernels.py:33


template <int NT>
__device__ __forceinline__ double block_max(double v, double* slots) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) slots[warp] = v;
  __syncthreads();
  double r = slots[0];
#pragma unroll
  for (int w = 1; w < NT / 32; ++w) r = fmax(r, slots[w]);
  return r;
}

template <int NT>
__device__ __forceinline__ void block_argmax(double& v, int& idx, double* vslots, int* islots) {
  warp_argmax(v, idx);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { vslots[warp] = v; islots[warp] = idx; }
  __syncthreads();
  v = vslots[0];
  idx = islots[0];
#pragma unroll
  for (int w = 1; w < NT / 32; ++w) argmax_merge(v, idx, vslots[w], islots[w]);
}

template <int NT>
__global__ void __launch_bounds__(NT) bk_exact_kernel(BkArgs a, int use_smem) {
  const int csym = a.check_sym_dev ? *a.check_sym_dev : a.check_sym;   // per-block device flag (block_ldlt)
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ double red_a[NT / 32], red_b[NT / 32], red_c[NT / 32], red_d[NT / 32];
  __shared__ int red_ai[NT / 32];

  const int b = blockIdx.x;
  const int n = a.n, lda = a.lda;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  cplx* W = a.W + (int64_t)b * a.stride_w;
  int64_t* perm = a.perm + (int64_t)b * n;
  int8_t* tags = a.tags + (int64_t)b * n;
  cplx* stage = use_smem ? reinterpret_cast<cplx*>(dyn_smem) : a.scratch + (int64_t)b * 4 * n;
  cplx* xs = stage;          // column k           (rows k+kstep..n-1, indexed by row)
  cplx* ys = stage + n;      // column k+1         (2x2 only)
  cplx* ls = stage + 2 * n;  // l_j or wk_j
  cplx* ws = stage + 3 * n;  // wkp_j              (2x2 only)

  for (int i = tid; i < n; i += NT) { perm[i] = i; tags[i] = 0; }

  // ---- prologue: numpy scale / symmetry check, initial trailing max -------
  double scale = 0.0, asym = 0.0, tm2 = 0.0;
  for (int64_t idx = tid; idx < (int64_t)n * n; idx += NT) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    const cplx z = W[(int64_t)i * lda + j];
    scale = fmax(scale, np_abs(z));
    if (j <= i) tm2 = fmax(tm2, x_abs2(z));
    if (csym && j < i) asym = fmax(asym, np_abs(x_sub(z, W[(int64_t)j * lda + i])));
  }
  scale = block_max<NT>(scale, red_a);
  asym = block_max<NT>(asym, red_b);
  tm2 = block_max<NT>(tm2, red_c);
  if (tid == 0) { a.scale[b] = scale; a.asym[b] = asym; }
  if (csym && n > 0 && scale > 0.0 && asym > __dmul_rn(1e-12, scale)) {
    if (tid == 0) {
      a.info[b] = -2; a.n2x2[b] = 0; a.growth[b] = 1.0;
      if (a.margin) { a.margin[2 * b] = 1.0; a.margin[2 * b + 1] = 1.0; }
    }
    return;
  }
  const double tol_abs = bk_threshold(a.pivot_tol, scale, a.abs_tol);
  double trail_max = __dsqrt_rn(tm2);
  double growth = 1.0;
  int n2x2 = 0, info = -1;
  const bool track = a.margin != nullptr;
  double mdec = 1.0, mgap = 1.0;
  __syncthreads();

  int k = 0;
  while (k < n) {
    // ---- 1. column search -------------------------------------------------
    const double absakk = x_abs(W[(int64_t)k * lda + k]);
    double colmax = 0.0;
    int imax = k;
    if (k + 1 < n) {
      double v = -1.0, v2 = -1.0;
      int vi = 0x7fffffff;
      for (int i = k + 1 + tid; i < n; i += NT) top2_merge(v, vi, v2, x_abs(W[(int64_t)i * lda + k]), i);
      const double tv = v;
      const int ti = vi;
      block_argmax<NT>(v, vi, red_a, red_ai);
      colmax = v;
      imax = vi;
      if (track) {   // runner-up: every thread's best other than the winner
        __syncthreads();
        const double r2 = block_max<NT>(ti == imax ? v2 : tv, red_c);
        mgap = fmin(mgap, argmax_gap(colmax, r2));
      }
    }
    if (fmax(absakk, colmax) <= tol_abs) {
      if (track) mdec = fmin(mdec, test_margin(tol_abs, fmax(absakk, colmax)));
      info = k;
      break;
    }

    int kstep = 1, kp;
    if (absakk >= __dmul_rn(kBkAlpha, colmax)) {
      kp = k;
      if (track) mdec = fmin(mdec, decision_margin(tol_abs, absakk, colmax, 0.0, 0.0, kBkAlpha, 1));
    } else {
      // ---- 2. rowmax over W[imax, k:imax] and W[imax+1:, imax] -------------
      // every thread reads |W[imax, imax]| before the reduction's barrier, so
      // no thread can observe it after another has started the interchange
      const double absimax = x_abs(W[(int64_t)imax * lda + imax]);
      double rm = 0.0;
      const int cnt1 = imax - k, cnt2 = n - imax - 1;
      for (int t = tid; t < cnt1 + cnt2; t += NT) {
        const cplx z = t < cnt1 ? W[(int64_t)imax * lda + k + t]
                                : W[(int64_t)(imax + 1 + t - cnt1) * lda + imax];
        rm = fmax(rm, x_abs(z));
      }
      const double rowmax = block_max<NT>(rm, red_b);
      int stage = 3;
      if (__dmul_rn(absakk, rowmax) >= __dmul_rn(__dmul_rn(kBkAlpha, colmax), colmax)) {
        kp = k;
        stage = 2;
      } else if (absimax >= __dmul_rn(kBkAlpha, rowmax)) {
        kp = imax;
      } else {
        kp = imax;
        kstep = 2;
      }
      if (track) mdec = fmin(mdec, decision_margin(tol_abs, absakk, colmax, rowmax, absimax, kBkAlpha, stage));
    }

    // ---- 3. symmetric interchange kk <-> kp --------------------------------
    const int kk = k + kstep - 1;
    if (kp != kk) {
      const int c1 = n - kp - 1;             // W[kp+1:, kk] <-> W[kp+1:, kp]
      const int c2 = kp - kk - 1;            // W[kk+1:kp, kk] <-> W[kp, kk+1:kp]
      const int c3 = 1;                      // diagonal
      const int c4 = kstep == 2 ? 1 : 0;     // W[kk, k] <-> W[kp, k]
      const int c5 = k;                      // W[kk, :k] <-> W[kp, :k]
      const int tot = c1 + c2 + c3 + c4 + c5;
      for (int t = tid; t < tot; t += NT) {
        int64_t p, q;
        int u = t;
        if (u < c1) { const int i = kp + 1 + u; p = (int64_t)i * lda + kk; q = (int64_t)i * lda + kp; }
        else if ((u -= c1) < c2) { const int i = kk + 1 + u; p = (int64_t)i * lda + kk; q = (int64_t)kp * lda + i; }
        else if ((u -= c2) < c3) { p = (int64_t)kk * lda + kk; q = (int64_t)kp * lda + kp; }
        else if ((u -= c3) < c4) { p = (int64_t)kk * lda + k; q = (int64_t)kp * lda + k; }
        else { u -= c4; p = (int64_t)kk * lda + u; q = (int64_t)kp * lda + u; }
        const cplx tp = W[p];
        W[p] = W[q];
        W[q] = tp;
      }
      if (tid == 0) { const int64_t t = perm[kk]; perm[kk] = perm[kp]; perm[kp] = t; }
      __syncthreads();
    }

    // ---- 4./5. stage and update ---------------------------------------------
    const int k0 = k + kstep;
    double step_sq = 0.0;
    if (kstep == 1) {
      const cplx piv = W[(int64_t)k * lda + k];
      for (int i = k0 + tid; i < n; i += NT) {
        const cplx x = W[(int64_t)i * lda + k];
        xs[i] = x;
        ls[i] = x_div_py(x, piv);                      // lj = W[j, k] / piv
      }
      __syncthreads();
      for (int i = k0 + warp; i < n; i += NW) {
        const cplx xi = xs[i];
        cplx* row = W + (int64_t)i * lda;
        for (int j = k0 + lane; j <= i; j += 32) {
          const cplx w = x_sub(row[j], x_mul(xi, ls[j]));   // W[j:, j] -= W[j:, k] * lj
          row[j] = w;
          step_sq = fmax(step_sq, x_abs2(w));
        }
        if (lane == 0) row[k] = x_div_np(xi, piv);    // W[k+1:, k] /= piv
      }
      if (tid == 0) tags[k] = 1;
    } else {
      const cplx d21 = W[(int64_t)(k + 1) * lda + k];
      const cplx d11 = x_div_py(W[(int64_t)(k + 1) * lda + k + 1], d21);
      const cplx d22 = x_div_py(W[(int64_t)k * lda + k], d21);
      const cplx t2 = x_div_py(mk(1.0, 0.0), x_sub(x_mul(d11, d22), mk(1.0, 0.0)));
      const cplx d21s = x_div_py(t2, d21);
      for (int i = k0 + tid; i < n; i += NT) {
        const cplx x = W[(int64_t)i * lda + k], y = W[(int64_t)i * lda + k + 1];
        xs[i] = x;
        ys[i] = y;
        ls[i] = x_mul(d21s, x_sub(x_mul(d11, x), y));      // wk
        ws[i] = x_mul(d21s, x_sub(x_mul(d22, y), x));      // wkp
      }
      __syncthreads();
      for (int i = k0 + warp; i < n; i += NW) {
        const cplx xi = xs[i], yi = ys[i];
        cplx* row = W + (int64_t)i * lda;
        for (int j = k0 + lane; j <= i; j += 32) {
          const cplx u = x_add(x_mul(xi, ls[j]), x_mul(yi, ws[j]));
          const cplx w = x_sub(row[j], u);
          row[j] = w;
          step_sq = fmax(step_sq, x_abs2(w));
        }
        if (lane == 0) { row[k] = ls[i]; row[k + 1] = ws[i]; }
      }
      if (tid == 0) { tags[k] = 2; tags[k + 1] = 0; }
      ++n2x2;
    }
    step_sq = block_max<NT>(step_sq, red_d);
    if (k0 < n) {
      const double step_max = __dsqrt_rn(step_sq);
      if (trail_max > 0.0) {
        double r = __ddiv_rn(step_max, trail_max);
        if (kstep == 2) r = __dsqrt_rn(r);
        if (r > growth) growth = r;
      }
      trail_max = step_max;
    }
    k = k0;
  }
  if (tid == 0) {
    a.n2x2[b] = n2x2;
    a.growth[b] = growth;
    a.info[b] = info;
    if (track) { a.margin[2 * b] = mdec; a.margin[2 * b + 1] = mgap; }
  }
}

}  // namespace d3m

extern "C" int d3m_bk_launch(d3m::BkArgs* a, int batch, void* stream) {
  using namespace d3m;
  if (batch <= 0) return 0;
  const size_t stage_bytes = (size_t)4 * a->n * sizeof(cplx);
  const bool use_smem = stage_bytes <= 200 * 1024;
  const size_t smem = use_smem ? stage_bytes : 0;
  if (!use_smem && a->scratch == nullptr) return -22;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (a->n <= 384) {
    cudaFuncSetAttribute(bk_exact_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bk_exact_kernel<512><<<batch, 512, smem, s>>>(*a, use_smem ? 1 : 0);
  } else {
    cudaFuncSetAttribute(bk_exact_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bk_exact_kernel<1024><<<batch, 1024, smem, s>>>(*a, use_smem ? 1 : 0);
  }
  return (int)cudaGetLastError();
}
