// bk_panel.cu -- batched blocked Bunch-Kaufman for large dense subdomain
// matrices (reduce_domain's dense_ldlt_bk, subdomain.py:173; n ~ 2k..13k).
//
// The reference factors A_d with the unblocked right-looking kernel
// (kernels.py:36-146), which rewrites the whole trailing triangle per step.
// Here (LAPACK zlasyf, lower) every matrix of the batch advances one panel of
// NB columns per launch of bk_panel_kernel (a cluster of CS CTAs per matrix,
// each owning a contiguous slice of the active rows; the panel and the
// X = L D workspace in global memory), applying the reference's
// decision rules (glibc-hypot modulus, alpha, first-index argmax, "<= tol"),
// its symmetric interchanges including the L rows of all previous columns,
// and storing L/D in the reference's packed layout.  The trailing rank-NB
// update of ALL matrices is then one grouped DMMA GEMM launch whose task
// records each panel CTA writes itself (its panel may end at NB or NB+1
// columns).  Pivot decisions match the reference whenever no test sits
// within rounding of its threshold (measured margins >= 1.3e-4 on config 3);
// growth is reported per panel (per-step geometric mean of the trailing-max
// ratio).
#include <algorithm>
#include <cstdlib>
#include <vector>
#include <cooperative_groups.h>
#include "d3m_common.cuh"
#include "d3m_gemm.h"
#include "d3m_kernels.h"

namespace d3m {
namespace cg = cooperative_groups;

constexpr int CNT = 256;       // threads per panel CTA (two CTAs fit an SM)
constexpr double kAlphaP = 0.6403882032022076;

struct BkState {          // 64 bytes per matrix
  int32_t k, info, n2x2, npiv_last;
  double trail_max, growth, tol_abs, scale, asym;
  float mdec, mgap;       // running pivot-decision margins (BkArgs::margin)
};
static_assert(sizeof(BkState) == 64, "BkState layout");

#ifdef D3M_PANEL_PROFILE
// phase clocks of matrix 0's rank-0 CTA (thread 0), summed over the panel launches (profiling builds only;
// tools/panel_profile.sh): 0 gemv(k) 1 argmax(k) 2 cluster merge 3 gemv(imax) 4 argmax + merge (imax)
// 5 interchange 6 L store 7 loop top; 8 steps 9 rowmax steps 10 interchanges
__device__ double g_panel_prof[16];
#define PANEL_MARK(slot) do { if (prof_on) { long long t_ = clock64(); pacc[slot] += (double)(t_ - prof_t); \
    prof_t = t_; } } while (0)
#define PANEL_COUNT(slot) do { if (prof_on) pacc[slot] += 1.0; } while (0)
#else
#define PANEL_MARK(slot) do { } while (0)
#define PANEL_COUNT(slot) do { } while (0)
#endif

template <int NT>
__device__ __forceinline__ double pmax_red(double v, double* slots) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) slots[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = slots[0];
#pragma unroll
  for (int w = 1; w < NT / 32; ++w) r = fmax(r, slots[w]);
  __syncthreads();
  return r;
}

template <int NT>
__device__ __forceinline__ void pargmax_red(double& v, int& idx, double* vs, int* is) {
  warp_argmax(v, idx);
  if ((threadIdx.x & 31) == 0) { vs[threadIdx.x >> 5] = v; is[threadIdx.x >> 5] = idx; }
  __syncthreads();
  v = vs[0];
  idx = is[0];
#pragma unroll
  for (int w = 1; w < NT / 32; ++w) argmax_merge(v, idx, vs[w], is[w]);
  __syncthreads();
}


// ---- prologue scan, tiled over many CTAs: per matrix b, atomic maxima of
//   pass 0: proxies |W|^2 (full), |W - W^T|^2 (i>j), trailing |W|^2 (i>=j)
//   pass 1: exact numpy-abs scale / asym for entries within 1e-14 of the proxies
// 32x32 tile pairs (ti >= tj) are staged through shared memory so both the
// tile and its transpose are read row-wise (coalesced).
__device__ __forceinline__ void atomic_max_pos(unsigned long long* p, double v) {
  atomicMax(p, (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ double as_pos(unsigned long long u) { return __longlong_as_double((long long)u); }

__global__ void __launch_bounds__(256) bk_scan_kernel(BkArgs a, unsigned long long* red, int pass) {
  __shared__ cplx Ta[32][33], Tb[32][33];
  __shared__ double wred[8][3];
  const int b = blockIdx.y, n = a.n, lda = a.lda;
  const cplx* W = a.W + (int64_t)b * a.stride_w;
  unsigned long long* rb = red + 8 * b;      // [p_all, p_asy, tm2, scale, asym]
  const int nt = (n + 31) / 32;
  const int ntile = nt * (nt + 1) / 2;
  const double ta = pass ? as_pos(rb[0]) * (1.0 - 1e-14) : 0.0;
  const double tb = pass ? as_pos(rb[1]) * (1.0 - 1e-14) : 0.0;
  double v0 = 0.0, v1 = 0.0, v2 = 0.0;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int t = blockIdx.x; t < ntile; t += gridDim.x) {
    int ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (ti * (ti + 1) / 2 > t) --ti;
    const int tj = t - ti * (ti + 1) / 2;
    for (int r = ty; r < 32; r += 8) {
      const int i = ti * 32 + r, j = tj * 32 + tx;
      Ta[r][tx] = (i < n && j < n) ? W[(int64_t)i * lda + j] : mk(0.0, 0.0);        // block (ti, tj)
      const int i2 = tj * 32 + r, j2 = ti * 32 + tx;
      // block (tj, ti); not read in lower_only mode
      Tb[r][tx] = (i2 < n && j2 < n && !a.lower_only) ? W[(int64_t)i2 * lda + j2] : mk(0.0, 0.0);
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      const int i = ti * 32 + r, j = tj * 32 + tx;
      if (i >= n || j >= n || j > i) continue;
      const cplx z = Ta[r][tx], zt = Tb[tx][r];     // W[i][j], W[j][i]
      if (pass == 0) {
        const double q = x_abs2(z);
        v0 = fmax(v0, a.lower_only ? q : fmax(q, x_abs2(zt)));
        v2 = fmax(v2, q);
        if (a.check_sym && j < i) v1 = fmax(v1, x_abs2(x_sub(z, zt)));
      } else {
        if (x_abs2(z) >= ta) v0 = fmax(v0, np_abs(z));
        if (!a.lower_only && x_abs2(zt) >= ta) v0 = fmax(v0, np_abs(zt));
        if (a.check_sym && j < i) {
          const cplx dz = x_sub(z, zt);
          if (x_abs2(dz) >= tb) v1 = fmax(v1, np_abs(dz));
        }
      }
    }
    __syncthreads();
  }
  v0 = warp_max(v0);
  v1 = warp_max(v1);
  v2 = warp_max(v2);
  if (tx == 0) { wred[ty][0] = v0; wred[ty][1] = v1; wred[ty][2] = v2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) { v0 = fmax(v0, wred[w][0]); v1 = fmax(v1, wred[w][1]); v2 = fmax(v2, wred[w][2]); }
    if (pass == 0) { atomic_max_pos(rb + 0, v0); atomic_max_pos(rb + 1, v1); atomic_max_pos(rb + 2, v2); }
    else { atomic_max_pos(rb + 3, v0); atomic_max_pos(rb + 4, v1); }
  }
}

__global__ void bk_panel_state_kernel(BkArgs a, BkState* st, const unsigned long long* red, int batch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const unsigned long long* rb = red + 8 * b;
  const double scale = as_pos(rb[3]), asym = as_pos(rb[4]);
  BkState s{};
  s.k = 0;
  s.info = (a.check_sym && a.n > 0 && scale > 0.0 && asym > __dmul_rn(1e-12, scale)) ? -2 : -1;
  s.trail_max = sqrt(as_pos(rb[2]));
  s.growth = 1.0;
  s.tol_abs = bk_threshold(a.pivot_tol, scale, a.abs_tol);
  s.scale = scale;
  s.asym = asym;
  s.mdec = 1.0f;
  s.mgap = 1.0f;
  st[b] = s;
  a.scale[b] = scale;
  a.asym[b] = asym;
}

__global__ void bk_perm_init_kernel(BkArgs a, int batch) {
  const int64_t total = (int64_t)batch * a.n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    a.perm[e] = e % a.n;
    a.tags[e] = 0;
  }
}

// Up-to-date column of the panel step over the rows [r_lo, r_hi) this CTA owns:
//   out[i] = base(i) - sum_{c < kw} G(i, k0 + c) * Wp[src][c]
// with NB/4 lanes per row (4 of the <= NB panel columns each, independent loads)
// and PG_ROWS rows per lane group in flight (all loads of an iteration are
// issued before any use: one L2/HBM round trip per iteration); base(i) is
// G(i, col) for i >= col (stale column) or G(col, i) for i < col (its row
// part), col = the target column.  The summation order per row is fixed (4
// partial sums, butterfly).
#ifndef D3M_EXACT_ROWS
#define D3M_EXACT_ROWS 2
#endif
constexpr int kExactRows = D3M_EXACT_ROWS;   // rows per thread up to which the pivot search takes exact moduli directly
constexpr int PG_ROWS = 3;   // (4: 2-3% slower panels on every config, 2: slower again; r02 A/B)
template <int NB, int NT>
__device__ __forceinline__ void panel_gemv(const cplx* __restrict__ W, int lda, int r_lo, int r_hi, int k0, int kw,
                                           int col, const cplx* __restrict__ Wp, int src,
                                           cplx* __restrict__ out_col /* Wp + kwcol, stride NB+1 */) {
  constexpr int LDW = NB + 1, LN = NB / 4;       // LN lanes per row, 4 panel columns each
  const int sub = threadIdx.x % LN;
  constexpr int rstride = NT / LN;
  cplx xs[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = sub + LN * q;
    xs[q] = c < kw ? Wp[(int64_t)src * LDW + c] : mk(0.0, 0.0);
  }
  // warp-uniform trip count: the shuffles below need all 32 lanes
  for (int base = r_lo; base < r_hi; base += PG_ROWS * rstride) {
    cplx l[PG_ROWS][4], bv[PG_ROWS];
#pragma unroll
    for (int g = 0; g < PG_ROWS; ++g) {
      const int ia = base + (int)threadIdx.x / LN + g * rstride;
      const bool va = ia < r_hi;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = sub + LN * q;
        l[g][q] = (c < kw && va) ? W[(int64_t)ia * lda + k0 + c] : mk(0.0, 0.0);
      }
      bv[g] = mk(0.0, 0.0);
      if (sub == 0 && va) bv[g] = ia >= col ? W[(int64_t)ia * lda + col] : W[(int64_t)col * lda + ia];
    }
#pragma unroll
    for (int g = 0; g < PG_ROWS; ++g) {
      const int ia = base + (int)threadIdx.x / LN + g * rstride;
      cplx sa = mk(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < 4; ++q) c_fma(sa, l[g][q], xs[q]);
#pragma unroll
      for (int o = 1; o < LN; o <<= 1) {
        sa.x += __shfl_xor_sync(0xffffffffu, sa.x, o);
        sa.y += __shfl_xor_sync(0xffffffffu, sa.y, o);
      }
      if (sub == 0 && ia < r_hi) out_col[(int64_t)ia * LDW] = c_sub(bv[g], sa);
    }
  }
}

// Exact modulus argmax (glibc hypot, first index) of col[i] over this CTA's
// rows i in [r0, r1), i != skip.  The |z|^2 proxy selects the candidates
// (within 1e-14 of the local proxy max); the union of all CTAs' local
// candidate sets contains every global maximiser, so merging the local exact
// results with argmax_merge gives the reference's np.argmax(abs(...)).
// Returns ev = -1, ei = INT_MAX for an empty range.
// With `ev2` (margin diagnostic), also the modulus of the local runner-up
// (largest |col[i]| of any other row, from the |z|^2 proxies; -1: none).
template <int NT>
__device__ __forceinline__ void local_exact_argmax(const cplx* col, int ldw, int r0, int r1, int skip, double& ev,
                                                   int& ei, double* vs, int* is, double* ev2 = nullptr) {
  if (!ev2 && r1 - r0 <= kExactRows * NT) {
    // few rows per thread: the exact moduli directly (one reduction; the proxy passes below cost two
    // more barriers and two more reads of the column)
    double v = -1.0;
    int vi = 0x7fffffff;
    for (int i = r0 + (int)threadIdx.x; i < r1; i += NT)
      if (i != skip) argmax_merge(v, vi, x_abs(col[(int64_t)i * ldw]), i);
    pargmax_red<NT>(v, vi, vs, is);
    ev = v;
    ei = vi;
    return;
  }
  double pv = -1.0, pv2 = -1.0;
  int pi = 0x7fffffff;
  for (int i = r0 + (int)threadIdx.x; i < r1; i += NT)
    if (i != skip) top2_merge(pv, pi, pv2, x_abs2(col[(int64_t)i * ldw]), i);
  const double tv = pv;
  const int ti = pi;
  pargmax_red<NT>(pv, pi, vs, is);
  if (ev2) {
    const double r2 = pmax_red<NT>(ti == pi ? pv2 : tv, vs);
    *ev2 = r2 >= 0.0 ? sqrt(r2) : -1.0;
  }
  if (pi == 0x7fffffff) { ev = -1.0; ei = pi; return; }
  const double thr = pv * (1.0 - 1e-14);
  int amb = 0;
  for (int i = r0 + (int)threadIdx.x; i < r1; i += NT)
    amb |= (i != skip && i != pi && x_abs2(col[(int64_t)i * ldw]) >= thr);
  if (__syncthreads_or(amb)) {
    double v = -1.0;
    int vi = 0x7fffffff;
    for (int i = r0 + (int)threadIdx.x; i < r1; i += NT) {
      if (i == skip) continue;
      const cplx z = col[(int64_t)i * ldw];
      if (x_abs2(z) >= thr) argmax_merge(v, vi, x_abs(z), i);
    }
    pargmax_red<NT>(v, vi, vs, is);
    ev = v;
    ei = vi;
  } else {
    ev = x_abs(col[(int64_t)pi * ldw]);
    ei = pi;
  }
}

struct ClSlot {       // one CTA's contribution to a cluster-wide pivot search
  double ev;          // local exact max over the local candidates (-1: none)
  double own;         // modulus of the published diagonal-ish entry (-1: not owned)
  double ev2;         // local runner-up (margin diagnostic, -1: none / not tracked)
  int ei;             // first index of ev
  int pad;
  double dre, dim;    // the published entry itself (owner only): the 1 x 1 pivot value when no rows move
};

// Gather the CS slots (DSMEM) after a cluster barrier; every CTA merges in the
// same order, so all CTAs hold bitwise-identical decisions.
template <int CS>
__device__ __forceinline__ ClSlot cl_merge(cg::cluster_group& cl, ClSlot* slot, ClSlot* out, bool track = false) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double ev = -1.0, own = -1.0, r2 = -1.0, dre = 0.0, dim = 0.0;
    int ei = 0x7fffffff;
    if (lane < CS) {
      const ClSlot* p = cl.map_shared_rank(slot, lane);
      ev = p->ev;
      own = p->own;
      r2 = p->ev2;
      ei = p->ei;
      dre = p->dre;
      dim = p->dim;
    }
    // the owner's entry (at most one CTA publishes own >= 0)
    const unsigned ob = __ballot_sync(0xffffffffu, own >= 0.0);
    const int ol = ob ? __ffs(ob) - 1 : 0;
    dre = __shfl_sync(0xffffffffu, dre, ol);
    dim = __shfl_sync(0xffffffffu, dim, ol);
    const double lv = ev;
    const int li = ei;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ev2 = __shfl_xor_sync(0xffffffffu, ev, o);
      const int ei2 = __shfl_xor_sync(0xffffffffu, ei, o);
      own = fmax(own, __shfl_xor_sync(0xffffffffu, own, o));
      argmax_merge(ev, ei, ev2, ei2);
    }
    if (track) r2 = warp_max(li == ei ? r2 : lv);   // the winner's runner-up, every other CTA's winner
    if (lane == 0) { out->ev = ev; out->own = own; out->ei = ei; out->ev2 = r2; out->dre = dre; out->dim = dim; }
  }
  __syncthreads();
  return *out;
}

// ---- one panel of up to NB (+1) columns per matrix, CS CTAs per matrix -----
// The cluster's CTAs own contiguous slices of the active rows [k0, n) and run
// the column updates, proxy scans and the L-column store for their rows;
// pivot searches meet in one cluster barrier each (DSMEM slots, double
// buffered), and the symmetric interchange (global memory, any thread of the
// cluster) is fenced by one more barrier when it moves data.
// TRACK: the pivot-decision margin diagnostic (BkArgs::margin) is compiled only into the TRACK instance, so
// the production kernel keeps its registers (it sits at the 128-register cap of two CTAs per SM).
template <int NB, int CS, bool TRACK>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(CNT)
bk_panel_kernel(BkArgs a, BkState* st, cplx* Wp_base, GemmTask* tasks, unsigned long long* tmax, int maxtiles) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double ra[CNT / 32];
  __shared__ int rai[CNT / 32];
  __shared__ ClSlot slots[2], merged;
  __shared__ double s_own[3];              // |entry|, re, im of the published entry (owner CTA)
  constexpr int LDW = NB + 1;
  const int rank = (int)cl.block_rank();
  const int b = blockIdx.x / CS, n = a.n, lda = a.lda, tid = threadIdx.x;
  const bool lead = rank == 0 && tid == 0;
  cplx* W = a.W + (int64_t)b * a.stride_w;
  int64_t* perm = a.perm + (int64_t)b * n;
  int8_t* tags = a.tags + (int64_t)b * n;
  cplx* Wp = Wp_base + (int64_t)b * n * LDW;          // [n][NB+1] row-major
  auto G = [&](int r, int c) -> cplx& { return W[(int64_t)r * lda + c]; };
  BkState s = st[b];
  GemmTask tk{};
  tk.tile_start = b * maxtiles;
  tk.tiles_n = 1;
  if (s.info != -1 || s.k >= n) {       // uniform over the cluster
    if (lead) tasks[b] = tk;            // m = 0: the GEMM CTAs of this matrix exit
    return;
  }
  // growth over the previous panel (its trailing max came from the GEMM)
  if (s.npiv_last > 0) {
    const double step_max = sqrt(__longlong_as_double((long long)tmax[b]));
    if (s.trail_max > 0.0) {
      const double r = pow(step_max / s.trail_max, 1.0 / s.npiv_last);
      if (r > s.growth) s.growth = r;
    }
    s.trail_max = step_max;
  }
  const int k0 = s.k;
  const int ch = (n - k0 + CS - 1) / CS;
  const int lo = min(n, k0 + rank * ch), hi = min(n, lo + ch);
  int k = k0, kw = 0, npiv = 0, info = -1, n2x2 = s.n2x2, par = 0;
  constexpr bool track = TRACK;               // pivot-decision margins
  double mdec = s.mdec, mgap = s.mgap;
  // a step starts only while kw <= NB-2, so a panel is NB-1 or NB columns
  // (zlasyf's exit rule) and the trailing update has K <= NB = 16
#ifdef D3M_PANEL_PROFILE
  const bool prof_on = blockIdx.x == 0 && tid == 0;
  double pacc[16] = {};
  long long prof_t = clock64();
#endif
  while (kw < NB - 1 && k < n) {
    PANEL_MARK(7);
    PANEL_COUNT(8);
    // -- A: column k up to date into Wp[:, kw] for the own rows, then the
    //    cluster's exact colmax / imax below the diagonal and |a_kk|
    panel_gemv<NB, CNT>(W, lda, max(k, lo), hi, k0, kw, k, Wp, k, Wp + kw);
    __syncthreads();
    PANEL_MARK(0);
    {
      // the owner of row k publishes |a_kk| and a_kk: read by the last warp's first lane while the
      // others search (the reductions' barriers publish s_own to thread 0)
      if (tid == CNT - 32) {
        cplx dk = mk(0.0, 0.0);
        double ak = -1.0;
        if (k >= lo && k < hi) {
          dk = Wp[(int64_t)k * LDW + kw];
          ak = x_abs(dk);
        }
        s_own[0] = ak;
        s_own[1] = dk.x;
        s_own[2] = dk.y;
      }
      double ev, ev2 = -1.0;
      int ei;
      local_exact_argmax<CNT>(Wp + kw, LDW, max(k + 1, lo), hi, -1, ev, ei, ra, rai, track ? &ev2 : nullptr);
      if (tid == 0) {
        ClSlot& sl = slots[par];
        sl.ev = ev;
        sl.ev2 = ev2;
        sl.ei = ei;
        sl.own = s_own[0];
        sl.dre = s_own[1];
        sl.dim = s_own[2];
      }
    }
    PANEL_MARK(1);
    cl.sync();
    const ClSlot m1 = cl_merge<CS>(cl, &slots[par], &merged, track);
    PANEL_MARK(2);
    par ^= 1;
    const double absakk = m1.own;
    double colmax = 0.0;
    int imax = k;
    if (k + 1 < n) {
      imax = m1.ei;
      colmax = m1.ev;
      if (track) mgap = fmin(mgap, argmax_gap(colmax, m1.ev2));
    }
    if (fmax(absakk, colmax) <= s.tol_abs) {
      if (track) mdec = fmin(mdec, test_margin(s.tol_abs, fmax(absakk, colmax)));
      info = k;
      break;
    }
    int kstep = 1, kp = k;
    bool copy = false;
    if (absakk >= __dmul_rn(kAlphaP, colmax)) {
      if (track) mdec = fmin(mdec, decision_margin(s.tol_abs, absakk, colmax, 0.0, 0.0, kAlphaP, 1));
    } else {
      // -- C: column imax up to date into Wp[:, kw+1], then the cluster's
      //    exact rowmax (diagonal entry imax excluded) and |a_imax,imax|
      PANEL_COUNT(9);
      panel_gemv<NB, CNT>(W, lda, max(k, lo), hi, k0, kw, imax, Wp, imax, Wp + kw + 1);
      __syncthreads();
      PANEL_MARK(3);
      {
        double ev;
        int ei;
        local_exact_argmax<CNT>(Wp + kw + 1, LDW, max(k, lo), hi, imax, ev, ei, ra, rai);
        if (tid == 0) {
          ClSlot& sl = slots[par];
          sl.ev = ev;
          sl.ei = ei;
          sl.own = (imax >= lo && imax < hi) ? x_abs(Wp[(int64_t)imax * LDW + kw + 1]) : -1.0;
          sl.dre = sl.dim = 0.0;
        }
      }
      cl.sync();
      const ClSlot m2 = cl_merge<CS>(cl, &slots[par], &merged);
      PANEL_MARK(4);
      par ^= 1;
      const double rowmax = fmax(0.0, m2.ev);
      const double absimax = m2.own;
      int stage = 3;
      if (__dmul_rn(absakk, rowmax) >= __dmul_rn(__dmul_rn(kAlphaP, colmax), colmax)) {
        kp = k;
        stage = 2;
      } else if (absimax >= __dmul_rn(kAlphaP, rowmax)) {
        kp = imax;
        copy = true;                       // column kw := column kw+1
      } else {
        kp = imax;
        kstep = 2;
      }
      if (track) mdec = fmin(mdec, decision_margin(s.tol_abs, absakk, colmax, rowmax, absimax, kAlphaP, stage));
    }
    const int kk = k + kstep - 1, kkw = kw + kstep - 1;
    if (copy)   // own rows; rows kk / kp are moved by the interchange below
      for (int i = max(k, lo) + tid; i < hi; i += CNT)
        if (i != kk && i != kp) Wp[(int64_t)i * LDW + kw] = Wp[(int64_t)i * LDW + kw + 1];
    // -- D: interchange kk <-> kp: stale column kk moves to kp, L rows and X
    //    rows swap (spread over the whole cluster; none of these writes
    //    touches column kk, which is only read here)
    if (kp != kk) {
      const int c1 = kp - kk - 1, c2 = n - kp - 1, c3 = kk, c4 = kkw + 1;
      const int tot = 1 + c1 + c2 + c3 + c4;
      for (int t = rank * CNT + tid; t < tot; t += CS * CNT) {
        int u = t;
        if (u == 0) { G(kp, kp) = G(kk, kk); continue; }
        u -= 1;
        if (u < c1) { const int j = kk + 1 + u; G(kp, j) = G(j, kk); continue; }
        u -= c1;
        if (u < c2) { const int i = kp + 1 + u; G(i, kp) = G(i, kk); continue; }
        u -= c2;
        if (u < c3) { const cplx t0 = G(kk, u); G(kk, u) = G(kp, u); G(kp, u) = t0; continue; }
        u -= c3;
        cplx* p0 = Wp + (int64_t)kk * LDW + u;
        cplx* p1 = Wp + (int64_t)kp * LDW + u;
        const int uc = (copy && u == kw) ? 1 : 0;    // the copied column comes from kw+1
        const cplx t0 = p0[uc];
        *p0 = p1[uc];
        *p1 = t0;
      }
      if (lead) { const int64_t t0 = perm[kk]; perm[kk] = perm[kp]; perm[kp] = t0; }
      cl.sync();
    }
    // (no barrier when no rows move: everything step E reads was written before the barriers of the
    //  column updates and the pivot searches)
    if (kp != kk) PANEL_COUNT(10);
    PANEL_MARK(5);
    // -- E: store D and the L column(s) of the own rows (packed layout,
    //    kernels.py:7-22)
    if (kstep == 1) {
      // the pivot: the owner published it with |a_kk| (no rows moved), else it moved into row k
      const cplx d = kp == kk ? mk(m1.dre, m1.dim) : Wp[(int64_t)k * LDW + kw];
      const bool re_big = fabs(d.x) >= fabs(d.y);
      const double rat = re_big ? __ddiv_rn(d.y, d.x) : __ddiv_rn(d.x, d.y);
      const double scl = re_big ? __ddiv_rn(1.0, __dadd_rn(d.x, __dmul_rn(d.y, rat)))
                                : __ddiv_rn(1.0, __dadd_rn(d.y, __dmul_rn(d.x, rat)));
      for (int i = max(k, lo) + tid; i < hi; i += CNT) {
        const cplx w = Wp[(int64_t)i * LDW + kw];
        cplx q;
        if (i == k) q = d;
        else if (d.x == 0.0 && d.y == 0.0) q = x_div_np(w, d);
        else if (re_big) q = mk(__dmul_rn(__dadd_rn(w.x, __dmul_rn(w.y, rat)), scl),
                                __dmul_rn(__dsub_rn(w.y, __dmul_rn(w.x, rat)), scl));
        else q = mk(__dmul_rn(__dadd_rn(__dmul_rn(w.x, rat), w.y), scl),
                    __dmul_rn(__dsub_rn(__dmul_rn(w.y, rat), w.x), scl));
        G(i, k) = q;
      }
      if (lead) tags[k] = 1;
    } else {
      const cplx d21 = Wp[(int64_t)(k + 1) * LDW + kw];
      const cplx d11 = x_div_py(Wp[(int64_t)(k + 1) * LDW + kw + 1], d21);
      const cplx d22 = x_div_py(Wp[(int64_t)k * LDW + kw], d21);
      const cplx t2 = x_div_py(mk(1.0, 0.0), x_sub(x_mul(d11, d22), mk(1.0, 0.0)));
      const cplx d21s = x_div_py(t2, d21);
      for (int i = max(k, lo) + tid; i < hi; i += CNT) {
        const cplx xk = Wp[(int64_t)i * LDW + kw], xk1 = Wp[(int64_t)i * LDW + kw + 1];
        if (i >= k + 2) {
          G(i, k) = x_mul(d21s, x_sub(x_mul(d11, xk), xk1));
          G(i, k + 1) = x_mul(d21s, x_sub(x_mul(d22, xk1), xk));
        } else if (i == k) {
          G(k, k) = xk;
        } else {
          G(k + 1, k) = xk;
          G(k + 1, k + 1) = xk1;
        }
      }
      if (lead) { tags[k] = 2; tags[k + 1] = 0; }
      ++n2x2;
    }
    ++npiv;
    __syncthreads();
    PANEL_MARK(6);
    k += kstep;
    kw += kstep;
  }
#ifdef D3M_PANEL_PROFILE
  if (prof_on)
    for (int i = 0; i < 16; ++i) atomicAdd(&g_panel_prof[i], pacc[i]);
#endif
  // the TMA-staged trailing update reads B = Wp in 16-column k-slices: a panel of NB - 1 columns
  // leaves column kw of the slice, which must read as zero (its A partner is the first trailing column)
  if (info < 0 && k < n && (kw & 15))
    for (int i = max(k, lo) + tid; i < hi; i += CNT) Wp[(int64_t)i * LDW + kw] = mk(0.0, 0.0);
  if (lead) {
    s.k = k;
    s.info = info;
    s.n2x2 = n2x2;
    s.mdec = (float)mdec;
    s.mgap = (float)mgap;
    s.npiv_last = (info < 0 && k < n) ? npiv : 0;
    st[b] = s;
    if (info < 0 && k < n) {
      // trailing update  A22 -= L21 X21^T  (lower only, running max for growth)
      tk.a_off = (int64_t)b * a.stride_w + (int64_t)k * lda + k0;
      tk.b_off = (int64_t)b * n * LDW + (int64_t)k * LDW;
      tk.c_off = (int64_t)b * a.stride_w + (int64_t)k * lda + k;
      tk.m = tk.n = n - k;
      tk.k = kw;
      tk.lda = lda;
      tk.ldb = LDW;
      tk.ldc = lda;
      tk.flags = kGemmSub | kGemmSym | kGemmLowerOnly | kGemmTrackMax;
      tk.tiles_n = (n - k + 63) / 64;
      tk.pad_ = b;
      tmax[b] = 0ull;
    }
    tasks[b] = tk;
  }
  cl.sync();     // peers may still read this CTA's slots
}

__global__ void bk_panel_finalize_kernel(BkArgs a, const BkState* st, int batch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const BkState s = st[b];
  a.info[b] = s.info;
  a.n2x2[b] = s.n2x2;
  a.growth[b] = s.growth;
  if (a.margin) { a.margin[2 * b] = s.mdec; a.margin[2 * b + 1] = s.mgap; }
}

}  // namespace d3m

// Host driver: init, then per panel one panel launch + one grouped GEMM over
// the batch.  workspace: batch * (n * 129 complex + 64 B state + 64 B task + 8 B + 64 B).
namespace d3m {
constexpr int kPanelLdwMax = 129;     // workspace row pitch for the widest panel (NB = 128)

// Panel loop for one panel width (NB - 1 or NB columns per panel); the
// rank-<= NB trailing updates of all matrices run as one grouped GEMM launch.
template <int NB>
static int panel_run(BkArgs* a, int batch, BkState* st, cplx* Wp, GemmTask* tasks, unsigned long long* tmax,
                     void* d_maps, cudaStream_t s, void* stream) {
  const int n = a->n;
  cudaError_t e;
  // CTAs per matrix: the largest cluster size whose CTAs (two per SM) fill
  // the GPU at most once; 16 is a non-portable cluster size
  int cs = batch * 16 <= 296 ? 16 : batch * 8 <= 296 ? 8 : batch * 4 <= 296 ? 4 : batch * 2 <= 296 ? 2 : 1;
  if (const char* env = getenv("D3M_PANEL_CS")) cs = atoi(env);
  if (cs != 1 && cs != 2 && cs != 4 && cs != 8 && cs != 16) cs = 1;
  // can this device keep a 16-CTA cluster of the panel kernel resident?
  // (per device: bit d of ok16 set = checked, of yes16 = resident)
  static std::atomic<unsigned long long> ok16{0}, yes16{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long dbit = 1ull << (dev & 63);
  if (cs == 16 && !(ok16.load() & dbit)) {
    cudaFuncSetAttribute(bk_panel_kernel<NB, 16, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(bk_panel_kernel<NB, 16, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(CNT);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, bk_panel_kernel<NB, 16, false>, &cfg) == cudaSuccess && nclusters > 0)
      yes16.fetch_or(dbit);
    cudaGetLastError();
    ok16.fetch_or(dbit);
  }
  if (cs == 16 && !(yes16.load() & dbit)) cs = 8;
  for (int p = 0; p * (NB - 1) < n; ++p) {
    const int mrem = n - (p + 1) * (NB - 1);           // rows left after this panel (upper bound)
    const int tm = mrem > 0 ? (mrem + 63) / 64 : 0;
    const int maxtiles = tm * (tm + 1) / 2;
#define D3M_PANEL_LAUNCH(CSV)                                                                                \
  if (a->margin) bk_panel_kernel<NB, CSV, true><<<batch * CSV, CNT, 0, s>>>(*a, st, Wp, tasks, tmax, maxtiles); \
  else bk_panel_kernel<NB, CSV, false><<<batch * CSV, CNT, 0, s>>>(*a, st, Wp, tasks, tmax, maxtiles)
    switch (cs) {
      case 16: D3M_PANEL_LAUNCH(16); break;
      case 8: D3M_PANEL_LAUNCH(8); break;
      case 4: D3M_PANEL_LAUNCH(4); break;
      case 2: D3M_PANEL_LAUNCH(2); break;
      default: D3M_PANEL_LAUNCH(1); break;
    }
#undef D3M_PANEL_LAUNCH
    if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
    if (maxtiles > 0) {
      // rank-<=NB trailing update on the pipelined grouped kernel (C
      // prefetched into freed ring stages; 4% faster on config 3 than a
      // small-K kernel that staged C with A and B, since removed)
      const int rc = d_maps ? d3m_gemm_tma_launch_batched(d_maps, a->W, tasks, batch, batch * maxtiles, a->stride_w,
                                                         (int64_t)n * (NB + 1), tmax, stream)
                            : d3m_gemm_launch_tm(0, 0, a->W, Wp, a->W, tasks, batch, batch * maxtiles, tmax, stream);
      if (rc) return rc;
    }
  }
  return 0;
}
}  // namespace d3m

extern "C" int d3m_bk_panel_batched_launch(d3m::BkArgs* a, int batch, void* workspace, void* stream) {
  using namespace d3m;
  if (batch <= 0 || a->n <= 0) return 0;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int n = a->n;
  // panel width 64: rank-<=64 trailing updates cut the trailing-matrix
  // traffic 4x against NB = 16 (config 5 BK: 20.7 s at NB 16, 15.6 s at 32,
  // 13.0 s at 64; configs 2/3: -21% / -17%; the narrow panels are gone)
  // NB = 128 for large subdomains (n >= 8192, config 5): the rank-128 updates
  // halve the trailing-matrix traffic per flop again, and the longer panel
  // steps are a small share there.  D3M_PANEL_NB=64|128 overrides (tests).
  int nb = n >= 8192 ? 128 : 64;
  if (const char* env = getenv("D3M_PANEL_NB")) nb = atoi(env) == 128 ? 128 : 64;
  char* w = static_cast<char*>(workspace);
  cplx* Wp = reinterpret_cast<cplx*>(w);
  w += (size_t)batch * n * kPanelLdwMax * sizeof(cplx);
  BkState* st = reinterpret_cast<BkState*>(w);
  w += (size_t)batch * sizeof(BkState);
  GemmTask* tasks = reinterpret_cast<GemmTask*>(w);
  w += (size_t)batch * sizeof(GemmTask);
  unsigned long long* tmax = reinterpret_cast<unsigned long long*>(w);
  w += (size_t)batch * sizeof(unsigned long long);
  unsigned long long* red = reinterpret_cast<unsigned long long*>(w);
  w += (size_t)batch * 8 * sizeof(unsigned long long);
  // TMA-staged trailing updates (3M form): per matrix a tensor-map pair over W_b (n x n, pitch lda) and
  // over its X workspace Wp_b (n x (nb + 1)), encoded on the host and copied once per factorisation
  // (D3M_PANEL_TMA=0: the cp.async grouped kernel).  Bitwise the same factor; BK class time config 5
  // 8.18 -> 7.67 s, config 2 65.1 -> 63.7 ms, config 3 63.6 -> 62.6 ms
  const char* tma_str = getenv("D3M_PANEL_TMA");
  const int tma_env = tma_str ? atoi(tma_str) : -1;
  void* d_maps = nullptr;
  if (tma_env != 0 && d3m_gemm_set_form(0) == 3) {
    std::vector<unsigned char> hm((size_t)batch * 256);
    const int rc = d3m_gemm_tma_prepare_batched(a->W, a->stride_w, n, n, a->lda, Wp, (int64_t)n * (nb + 1), n, nb + 1,
                                                nb + 1, batch, hm.data());
    if (rc == 0) {
      d_maps = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(w) + 127) & ~uintptr_t(127));
      // (pageable source: staged before the call returns)
      if (cudaMemcpyAsync(d_maps, hm.data(), hm.size(), cudaMemcpyHostToDevice, s) != cudaSuccess) d_maps = nullptr;
    } else if (rc != -38) {
      return rc;
    }
  }
  cudaMemsetAsync(red, 0, (size_t)batch * 8 * sizeof(unsigned long long), s);
  const int nt = (n + 31) / 32, ntile = nt * (nt + 1) / 2;
  const dim3 sgrid(std::min(ntile, 256), batch);
  bk_perm_init_kernel<<<std::min((batch * n + 255) / 256, 4096), 256, 0, s>>>(*a, batch);
  bk_scan_kernel<<<sgrid, 256, 0, s>>>(*a, red, 0);
  bk_scan_kernel<<<sgrid, 256, 0, s>>>(*a, red, 1);
  bk_panel_state_kernel<<<(batch + 127) / 128, 128, 0, s>>>(*a, st, red, batch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  const int rc = nb == 128 ? panel_run<128>(a, batch, st, Wp, tasks, tmax, d_maps, s, stream)
                            : panel_run<64>(a, batch, st, Wp, tasks, tmax, d_maps, s, stream);
  if (rc) return rc;
  bk_panel_finalize_kernel<<<(batch + 127) / 128, 128, 0, s>>>(*a, st, batch);
  return (int)cudaGetLastError();
}

namespace d3m {
__global__ void sym_scan_store_kernel(const unsigned long long* red, double* scale, double* asym, int batch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  scale[b] = as_pos(red[8 * b + 3]);
  asym[b] = as_pos(red[8 * b + 4]);
}
}  // namespace d3m

// The prologue scan alone over full matrices: scale = np.abs(W).max() and
// asym = np.abs(W - W.T).max() per matrix (factor.py:94-98), exactly as the
// factorisation kernels compute them.  red: >= 64 * batch bytes.
extern "C" int d3m_sym_scan_batched_launch(d3m::BkArgs* a, int batch, void* red_ws, void* stream) {
  using namespace d3m;
  if (batch <= 0 || a->n <= 0) return 0;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto* red = static_cast<unsigned long long*>(red_ws);
  cudaMemsetAsync(red, 0, (size_t)batch * 8 * sizeof(unsigned long long), s);
  const int nt = (a->n + 31) / 32, ntile = nt * (nt + 1) / 2;
  const dim3 sgrid(std::min(ntile, 256), batch);
  BkArgs x = *a;
  x.check_sym = 1;
  x.lower_only = false;
  bk_scan_kernel<<<sgrid, 256, 0, s>>>(x, red, 0);
  bk_scan_kernel<<<sgrid, 256, 0, s>>>(x, red, 1);
  sym_scan_store_kernel<<<(batch + 127) / 128, 128, 0, s>>>(red, a->scale, a->asym, batch);
  return (int)cudaGetLastError();
}

#ifdef D3M_PANEL_PROFILE
extern "C" int d3m_panel_prof_read(double* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, d3m::g_panel_prof, sizeof(double) * 16);
  if (reset) {
    double z[16] = {};
    cudaMemcpyToSymbol(d3m::g_panel_prof, z, sizeof(z));
  }
  return 0;
}
#endif

extern "C" size_t d3m_bk_panel_workspace_bytes(int n, int batch) {
  return (size_t)batch * ((size_t)n * d3m::kPanelLdwMax * 16 + 64 + 64 + 8 + 64 + 256) + 512;   // + tensor maps
}
