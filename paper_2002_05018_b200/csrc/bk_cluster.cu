// bk_cluster.cu -- bit-exact Bunch-Kaufman LDL^T of one dense block per
// thread-block cluster, the lower triangle resident in distributed shared
// memory (the 256-wide diagonal blocks of block_ldlt, factor.py:205-210, on
// the critical path of the block factorisation).
//
// bk_exact.cu runs the reference's unblocked right-looking algorithm
// (kernels.py:36-146) in ONE CTA against global memory; at n = 256 that is
// 256 dependent steps of ~5 us, mostly L2 latency.  Here a cluster of CS CTAs
// holds the packed lower triangle in shared memory, rows distributed
// cyclically (row i on CTA i % CS: balanced triangle), so every per-step
// access is a shared-memory access and the rank-1/rank-2 update is spread
// over CS SMs.  The arithmetic of every entry is the one of bk_exact.cu
// (itself operation-for-operation the numba kernel), so pivots, tags, growth
// AND values stay bit-identical to the CPU reference.
//
// Per step k (cluster barriers marked |):
//   row owners push column k into every CTA's broadcast vector; local exact
//   argmax over the own rows                                          | merge
//   [rowmax phase: push column k+1 and the symmetric column imax      | merge]
//   every CTA derives the post-interchange columns k (and k+1), the pivot
//   and ALL multipliers locally from the broadcast vectors; the interchange
//   is applied row by row by the row owners (the L rows of kk / kp by kk's
//   owner through DSMEM, untouched by anyone else this step); rank-1 / rank-2
//   update of the own rows (warp per row).  The step's max |a_ij|^2 rides on
//   the next step's barrier (growth, kernels.py:102-144).  One cluster
//   barrier per step (two when the rowmax test runs).
#include <cooperative_groups.h>
#include <cstdlib>
#include "d3m_common.cuh"
#include "d3m_kernels.h"

namespace d3m {
namespace cg = cooperative_groups;

constexpr int BKC_NT = 512;
constexpr double kBkcAlpha = 0.6403882032022076;  // (1 + sqrt(17)) / 8, kernels.py:33

struct BkcSlot {
  double v;      // argmax value (exact modulus) or -1
  double own;    // a value only the owner of a row can supply, else -1
  double aux;    // max-reduced payload (rowmax, step max, prologue maxima)
  double aux2;
  int i;         // argmax index
  int pad;
};

// Each CTA posts its slot into every CTA's inbox (DSMEM stores) before the
// cluster barrier; after it every CTA merges its own inbox from local shared
// memory in rank order, so all CTAs hold bitwise-identical decisions.
template <int CS>
__device__ __forceinline__ void bkc_post(cg::cluster_group& cl, BkcSlot* box, int rank, const BkcSlot& v) {
#pragma unroll
  for (int c = 0; c < CS; ++c) *cl.map_shared_rank(box + rank, c) = v;
}

template <int CS>
__device__ __forceinline__ BkcSlot bkc_merge(const BkcSlot* box, BkcSlot* out) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    BkcSlot r{-1.0, -1.0, -1.0, -1.0, 0x7fffffff, 0};
    if (lane < CS) r = box[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, r.v, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, r.i, o);
      r.own = fmax(r.own, __shfl_xor_sync(0xffffffffu, r.own, o));
      r.aux = fmax(r.aux, __shfl_xor_sync(0xffffffffu, r.aux, o));
      r.aux2 = fmax(r.aux2, __shfl_xor_sync(0xffffffffu, r.aux2, o));
      argmax_merge(r.v, r.i, v2, i2);
    }
    if (lane == 0) *out = r;
  }
  __syncthreads();
  return *out;
}

__device__ __forceinline__ double bkc_block_max(double v, double* slots) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) slots[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = slots[0];
#pragma unroll
  for (int w = 1; w < BKC_NT / 32; ++w) r = fmax(r, slots[w]);
  __syncthreads();
  return r;
}

__device__ __forceinline__ void bkc_block_argmax(double& v, int& idx, double* vs, int* is) {
  warp_argmax(v, idx);
  if ((threadIdx.x & 31) == 0) { vs[threadIdx.x >> 5] = v; is[threadIdx.x >> 5] = idx; }
  __syncthreads();
  v = vs[0];
  idx = is[0];
#pragma unroll
  for (int w = 1; w < BKC_NT / 32; ++w) argmax_merge(v, idx, vs[w], is[w]);
  __syncthreads();
}

// packed offset of row i (i % CS == r) inside its CTA: rows q = i / CS of
// lengths q*CS + r + 1 stored back to back
template <int CS>
__device__ __forceinline__ int64_t bkc_off(int i) {
  const int q = i / CS, r = i - q * CS;
  return (int64_t)CS * q * (q - 1) / 2 + (int64_t)q * (r + 1);
}

template <int CS>
__host__ __device__ inline int64_t bkc_entries(int n) {    // per-CTA capacity (largest rank)
  const int nq = (n + CS - 1) / CS;
  return (int64_t)CS * nq * (nq - 1) / 2 + (int64_t)nq * CS;
}

#ifdef D3M_BK_PROFILE
#define BKC_MARK(slot) do { __syncthreads(); if (tid == 0 && rank == 0) { long long t_ = clock64(); \
    prof[slot] += (double)(t_ - prof_t); prof_t = t_; } } while (0)
#else
#define BKC_MARK(slot) do { } while (0)
#endif

template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(BKC_NT) bk_cluster_kernel(BkArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char bkc_smem[];
  __shared__ double rv[BKC_NT / 32];
  __shared__ int ri[BKC_NT / 32];
  __shared__ double rst[BKC_NT / 32];
  __shared__ BkcSlot inbox[2][CS], merged;
  const int rank = (int)cl.block_rank();
  const int b = blockIdx.x / CS;
  const int n = a.n, lda = a.lda, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = BKC_NT / 32;
  const int64_t cap = bkc_entries<CS>(n);
  cplx* Rl = reinterpret_cast<cplx*>(bkc_smem);      // own packed lower rows
  cplx* ls = Rl + cap;                                 // l_j / wk_j of every row (computed locally)
  cplx* ws = ls + n;                                   // wkp_j (2x2)
  cplx* W = a.W + (int64_t)b * a.stride_w;
  int64_t* perm = a.perm + (int64_t)b * n;
  int8_t* tags = a.tags + (int64_t)b * n;
  const bool lead = rank == 0 && tid == 0;
  const int nown = (n - rank + CS - 1) / CS;          // own rows: rank, rank + CS, ...
  auto L = [&](int i, int j) -> cplx& { return Rl[bkc_off<CS>(i) + j]; };   // own row i
  auto Rm = [&](int i, int j) -> cplx& {                                     // any row (DSMEM)
    cplx* base = cl.map_shared_rank(Rl, i % CS);
    return base[bkc_off<CS>(i) + j];
  };
  int par = 0;

  // ---- prologue: numpy scale / symmetry check / trailing max, own rows -> smem
  double scale = 0.0, asym = 0.0, tm2 = 0.0;
  for (int q = warp; q < nown; q += NW) {
    const int i = rank + q * CS;
    const cplx* row = W + (int64_t)i * lda;
    cplx* dst = Rl + bkc_off<CS>(i);
    const int jend = a.check_sym == 2 ? i + 1 : n;     // 2: verified exactly symmetric (lower suffices)
    for (int j = lane; j < jend; j += 32) {
      const cplx z = row[j];
      scale = fmax(scale, np_abs(z));
      if (j <= i) { tm2 = fmax(tm2, x_abs2(z)); dst[j] = z; }
      if (a.check_sym == 1 && j < i) asym = fmax(asym, np_abs(x_sub(z, W[(int64_t)j * lda + i])));
    }
  }
  if (rank == 0)
    for (int i = tid; i < n; i += BKC_NT) { perm[i] = i; tags[i] = 0; }
  scale = bkc_block_max(scale, rv);
  asym = bkc_block_max(asym, rv);
  tm2 = bkc_block_max(tm2, rv);
  if (tid == 0) bkc_post<CS>(cl, inbox[par], rank, BkcSlot{-1.0, scale, asym, tm2, 0x7fffffff, 0});
  cl.sync();
  {
    const BkcSlot m = bkc_merge<CS>(inbox[par], &merged);
    scale = m.own;
    asym = m.aux;
    tm2 = m.aux2;
  }
  par ^= 1;
  if (lead) { a.scale[b] = scale; a.asym[b] = asym; }
  if (a.check_sym == 1 && n > 0 && scale > 0.0 && asym > __dmul_rn(1e-12, scale)) {
    if (lead) { a.info[b] = -2; a.n2x2[b] = 0; a.growth[b] = 1.0; }
    cl.sync();
    return;
  }
  const double tol_abs = __dmul_rn(a.pivot_tol, scale);
  double trail_max = __dsqrt_rn(tm2);
  double growth = 1.0;
  int n2x2 = 0, info = -1;
  double lstep = 0.0;          // this CTA's max |a_ij|^2 of the previous update
  int prev_kstep = 0, prev_k0 = 0;

  // broadcast vectors (double-buffered by step parity; written by the row
  // owners through DSMEM before the step's barrier):
  //   cA: column k (rows >= k)      cB: column k+1 (rows >= k+1, rowmax phase)
  //   cC: symmetric column imax, cC[i] = A[imax][i] (i < imax) / A[i][imax]
  cplx* vec = ws + n;                    // [2][3][n]
  int k = 0, step = 0;
#ifdef D3M_BK_PROFILE
  double* prof = reinterpret_cast<double*>(a.scratch);
  long long prof_t = clock64();
#endif
  // column 0: pushed and searched here; later columns k0 are pushed and
  // searched by the update of the previous step (the lane that writes W[i,k0])
  double sv = -1.0;
  int si = 0x7fffffff;
  for (int q = tid; q < nown; q += BKC_NT) {
    const int i = rank + q * CS;
    const cplx z = L(i, 0);
#pragma unroll
    for (int c = 0; c < CS; ++c) cl.map_shared_rank(vec, c)[i] = z;
    if (i > 0) argmax_merge(sv, si, x_abs(z), i);
  }
  while (k < n) {
    const int p = step & 1;
    cplx* cA = vec + (size_t)(p * 3 + 0) * n;
    cplx* cB = vec + (size_t)(p * 3 + 1) * n;
    cplx* cC = vec + (size_t)(p * 3 + 2) * n;
    cplx* cAn = vec + (size_t)((p ^ 1) * 3 + 0) * n;     // next step's column buffer
    // ---- 1. exact argmax |W[i,k]| over i > k (values from the update) -------
    {
      double v = sv, st = lstep;
      int vi = si;
      warp_argmax(v, vi);
      st = warp_max(st);
      if (lane == 0) { rv[warp] = v; ri[warp] = vi; rst[warp] = st; }
      __syncthreads();
      if (warp == 0) {
        v = lane < NW ? rv[lane] : -1.0;
        vi = lane < NW ? ri[lane] : 0x7fffffff;
        st = lane < NW ? rst[lane] : -1.0;
        warp_argmax(v, vi);
        st = warp_max(st);
        if (lane == 0) bkc_post<CS>(cl, inbox[par], rank, BkcSlot{v, -1.0, st, -1.0, vi, 0});
      }
    }
    BKC_MARK(0);
    cl.sync();
    const BkcSlot m1 = bkc_merge<CS>(inbox[par], &merged);
    par ^= 1;
    BKC_MARK(1);
    if (prev_kstep && prev_k0 < n) {           // growth of the previous step (kernels.py:135-144)
      const double step_max = __dsqrt_rn(m1.aux);
      if (trail_max > 0.0) {
        double r = __ddiv_rn(step_max, trail_max);
        if (prev_kstep == 2) r = __dsqrt_rn(r);
        if (r > growth) growth = r;
      }
      trail_max = step_max;
    }
    const double absakk = x_abs(cA[k]);
    double colmax = 0.0;
    int imax = k;
    if (k + 1 < n) { colmax = m1.v; imax = m1.i; }
    if (fmax(absakk, colmax) <= tol_abs) { info = k; break; }

    int kstep = 1, kp;
    if (absakk >= __dmul_rn(kBkcAlpha, colmax)) {
      kp = k;
    } else {
      // ---- 2. push column k+1 and the symmetric column imax; rowmax over
      //         W[imax, k:imax] and W[imax+1:, imax] --------------------------
      double rm = 0.0;
      if (imax % CS == rank)
        for (int t = k + tid; t <= imax; t += BKC_NT) {
          const cplx z = L(imax, t);
#pragma unroll
          for (int c = 0; c < CS; ++c) cl.map_shared_rank(cC, c)[t] = z;
          if (t < imax) rm = fmax(rm, x_abs(z));
        }
      {
        const int q0 = (k + 1 - rank + CS - 1) / CS > 0 ? (k + 1 - rank + CS - 1) / CS : 0;
        for (int q = q0 + tid; q < nown; q += BKC_NT) {
          const int i = rank + q * CS;
          const cplx y = L(i, k + 1);
#pragma unroll
          for (int c = 0; c < CS; ++c) cl.map_shared_rank(cB, c)[i] = y;
          if (i > imax) {
            const cplx z = L(i, imax);
#pragma unroll
            for (int c = 0; c < CS; ++c) cl.map_shared_rank(cC, c)[i] = z;
            rm = fmax(rm, x_abs(z));
          }
        }
      }
      rm = bkc_block_max(rm, rv);
      if (tid == 0) bkc_post<CS>(cl, inbox[par], rank, BkcSlot{-1.0, -1.0, rm, -1.0, 0x7fffffff, 0});
      cl.sync();
      const BkcSlot m2 = bkc_merge<CS>(inbox[par], &merged);
      par ^= 1;
      const double rowmax = m2.aux, absimax = x_abs(cC[imax]);
      if (__dmul_rn(absakk, rowmax) >= __dmul_rn(__dmul_rn(kBkcAlpha, colmax), colmax)) {
        kp = k;
      } else if (absimax >= __dmul_rn(kBkcAlpha, rowmax)) {
        kp = imax;
      } else {
        kp = imax;
        kstep = 2;
      }
      BKC_MARK(2);
    }

    // ---- 3. symmetric interchange kk <-> kp (kernels.py:79-101), each row by
    //         its owner from the broadcast columns; the L rows (columns < k)
    //         of kk and kp by kk's owner through DSMEM (no one else touches
    //         them this step: loads issued here, stores after the update) ----
    const int kk = k + kstep - 1, k0 = k + kstep;
    const cplx* cK = kstep == 1 ? cA : cB;          // column kk before the swap
    const bool lswap = kp != kk && kk % CS == rank;
    cplx lsv[2] = {mk(0.0, 0.0), mk(0.0, 0.0)};
    if (kp != kk) {
      {   // rows i > kp: W[i, kk] <-> W[i, kp]
        const int q0 = (kp + 1 - rank + CS - 1) / CS > 0 ? (kp + 1 - rank + CS - 1) / CS : 0;
        for (int q = q0 + tid; q < nown; q += BKC_NT) {
          const int i = rank + q * CS;
          const cplx t0 = L(i, kk);
          L(i, kk) = L(i, kp);
          L(i, kp) = t0;
        }
      }
      if (kp % CS == rank)   // row kp: W[kp, kk+1:kp] <- W[kk+1:kp, kk]; W[kp, kp] <- W[kk, kk]
        for (int j = kk + 1 + tid; j <= kp; j += BKC_NT) L(kp, j) = j < kp ? cK[j] : cK[kk];
      if (lswap) {
        if (tid == 0) {
          L(kk, kk) = cC[kp];                      // W[kk, kk] <- W[kp, kp]
          if (kstep == 2) L(kk, k) = cA[kp];       // W[k+1, k] <- W[kp, k]
        }
        const cplx* rkp = &Rm(kp, 0);
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (tid + h * BKC_NT < k) lsv[h] = rkp[tid + h * BKC_NT];   // W[kp, :k], stored below
      }
      if (lead) { const int64_t t0 = perm[kk]; perm[kk] = perm[kp]; perm[kp] = t0; }
    }
    BKC_MARK(3);
    // post-interchange columns k (X) and k+1 (Y) at row i >= k0: sigma swaps kk, kp
    auto Xc = [&](int i) -> cplx {
      if (kstep == 1) return kp == k ? cA[i] : (i == kp ? cC[k] : cC[i]);
      return i == kp ? cA[kk] : cA[i];
    };
    auto Yc = [&](int i) -> cplx { return i == kp ? cC[kk] : cC[i]; };

    // ---- 4. multipliers of every row (each CTA computes all of them) -------
    cplx piv = mk(0.0, 0.0);
    if (kstep == 1) {
      piv = kp == k ? cA[k] : cC[kp];
      for (int j = k0 + tid; j < n; j += BKC_NT) ls[j] = x_div_py(Xc(j), piv);   // lj = W[j, k] / piv
    } else {
      const cplx d21 = cA[kp];                                   // W'[k+1, k]
      const cplx d11 = x_div_py(cC[kp], d21);                    // W'[k+1, k+1] / d21
      const cplx d22 = x_div_py(cA[k], d21);                     // W'[k, k] / d21
      const cplx t2 = x_div_py(mk(1.0, 0.0), x_sub(x_mul(d11, d22), mk(1.0, 0.0)));
      const cplx d21s = x_div_py(t2, d21);
      for (int j = k0 + tid; j < n; j += BKC_NT) {
        const cplx x = Xc(j), y = Yc(j);
        ls[j] = x_mul(d21s, x_sub(x_mul(d11, x), y));            // wk
        ws[j] = x_mul(d21s, x_sub(x_mul(d22, y), x));            // wkp
      }
    }
    __syncthreads();
    BKC_MARK(4);

    // ---- 5. rank-1 / rank-2 update of the own rows (warp per row); the lane
    //         that writes W[i, k0] pushes it and searches it for step k0 -----
    const int qk0 = (k0 - rank + CS - 1) / CS > 0 ? (k0 - rank + CS - 1) / CS : 0;
    double step_sq = 0.0;
    sv = -1.0;
    si = 0x7fffffff;
    for (int q = qk0 + warp; q < nown; q += NW) {
      const int i = rank + q * CS;
      cplx* row = Rl + bkc_off<CS>(i);
      const cplx xi = Xc(i);
      const cplx yi = kstep == 2 ? Yc(i) : mk(0.0, 0.0);
      for (int j0 = k0; j0 <= i; j0 += 64) {
        const int ja = j0 + lane, jb = ja + 32;
        cplx wa = mk(0.0, 0.0), wb = mk(0.0, 0.0);
        if (kstep == 1) {
          if (ja <= i) wa = x_sub(row[ja], x_mul(xi, ls[ja]));       // W[j:, j] -= W[j:, k] * lj
          if (jb <= i) wb = x_sub(row[jb], x_mul(xi, ls[jb]));
        } else {
          if (ja <= i) wa = x_sub(row[ja], x_add(x_mul(xi, ls[ja]), x_mul(yi, ws[ja])));
          if (jb <= i) wb = x_sub(row[jb], x_add(x_mul(xi, ls[jb]), x_mul(yi, ws[jb])));
        }
        if (ja <= i) { row[ja] = wa; step_sq = fmax(step_sq, x_abs2(wa)); }
        if (jb <= i) { row[jb] = wb; step_sq = fmax(step_sq, x_abs2(wb)); }
        if (j0 == k0 && lane == 0) {          // W[i, k0]: next step's column
#pragma unroll
          for (int c = 0; c < CS; ++c) cl.map_shared_rank(cAn, c)[i] = wa;
          if (i > k0) argmax_merge(sv, si, x_abs(wa), i);
        }
      }
      if (lane == 0) {
        if (kstep == 1) {
          row[k] = x_div_np(xi, piv);                              // W[k+1:, k] /= piv
        } else {
          row[k] = ls[i];
          row[k + 1] = ws[i];
        }
      }
    }
    if (lswap) {                               // W[kk, :k] <-> W[kp, :k]
      cplx* rkp = &Rm(kp, 0);
      cplx* rkk = &L(kk, 0);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = tid + h * BKC_NT;
        if (u < k) {
          rkp[u] = rkk[u];
          rkk[u] = lsv[h];
        }
      }
    }
    if (lead) {
      if (kstep == 1) tags[k] = 1;
      else { tags[k] = 2; tags[k + 1] = 0; }
    }
    if (kstep == 2) ++n2x2;
    lstep = step_sq;
    prev_kstep = kstep;
    prev_k0 = k0;
    __syncthreads();
    BKC_MARK(5);
    k = k0;
    ++step;
  }
  // ---- write back the own rows (lower triangle) ----------------------------
  for (int q = warp; q < nown; q += NW) {
    const int i = rank + q * CS;
    const cplx* src = Rl + bkc_off<CS>(i);
    cplx* row = W + (int64_t)i * lda;
    for (int j = lane; j <= i; j += 32) row[j] = src[j];
  }
  if (lead) {
    a.n2x2[b] = n2x2;
    a.growth[b] = growth;
    a.info[b] = info;
  }
  cl.sync();     // peers may still read this CTA's shared memory
}

template <int CS>
static int bkc_launch(BkArgs* a, int batch, cudaStream_t s) {
  const size_t smem = sizeof(cplx) * (size_t)(bkc_entries<CS>(a->n) + 8 * (int64_t)a->n);
  if (smem > 200 * 1024) return -22;
  cudaFuncSetAttribute(bk_cluster_kernel<CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bk_cluster_kernel<CS><<<batch * CS, BKC_NT, smem, s>>>(*a);
  return (int)cudaGetLastError();
}

}  // namespace d3m

// Bit-exact BK of `batch` blocks, one cluster each.  Returns -22 when the
// block does not fit the cluster's shared memory (caller falls back).
extern "C" int d3m_bk_cluster_launch(d3m::BkArgs* a, int batch, void* stream) {
  using namespace d3m;
  if (batch <= 0 || a->n <= 0) return 0;
  int cs = 8;
  if (const char* env = getenv("D3M_BKC_CS")) cs = atoi(env);
  auto s = reinterpret_cast<cudaStream_t>(stream);
  int rc = -22;
  switch (cs) {
    case 2: rc = bkc_launch<2>(a, batch, s); break;
    case 4: rc = bkc_launch<4>(a, batch, s); break;
    default: break;
  }
  return rc == -22 ? bkc_launch<8>(a, batch, s) : rc;
}
