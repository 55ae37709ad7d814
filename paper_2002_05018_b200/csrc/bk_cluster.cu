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
// Per step the work splits into a pivot warp (the critical chain: merge,
// decision, interchange, update and publication of the next pivot column) and
// bulk warps (multipliers, L column, trailing update), with a split cluster
// barrier: the pivot warp ARRIVES once column k0 is published and the next
// step WAITS, so the bulk update overlaps the exchange (see the kernel).
#include <cooperative_groups.h>
#include <cstdlib>
#include "d3m_common.cuh"
#include "d3m_kernels.h"

namespace d3m {
namespace cg = cooperative_groups;

constexpr int BKC_NT = 384;
constexpr int BKC_JPT = 2;       // multiplier rows per bulk thread: n <= BKC_JPT * (BKC_NT - 32)
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
    for (int o = CS / 2; o > 0; o >>= 1) {      // lanes >= CS hold neutral slots
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

// split cluster barrier (arrive publishes this thread's prior DSMEM stores;
// wait acquires every peer's)
__device__ __forceinline__ void bkc_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void bkc_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }

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
// per-role phase clocks of CTA 0: slots 0-7 the pivot warp (lane 0), 8-15 the
// first bulk thread; accumulated in registers, written once at the end
#define BKC_MARK(who, slot) do { if (rank == 0 && tid == (who)) { long long t_ = clock64(); \
    pacc[slot] += (double)(t_ - prof_t); prof_t = t_; } } while (0)
#else
#define BKC_MARK(who, slot) do { } while (0)
#endif

// Roles inside each CTA of the cluster (per step k, pivot column k0 = k + kstep):
//   pivot warp (warp 0): merge of the argmax slots -> pivot decision ->
//     interchange of the own rows' columns kk / kp -> update of column k0 of
//     the own rows -> publish it (DSMEM) with its exact argmax, the modulus of
//     the new diagonal entry and the update maximum of step s-1 -> ARRIVE on
//     the cluster barrier.  This chain is the step's critical path.
//   bulk warps (1..NW-1): row kp refill and the L rows of kk / kp, multipliers
//     of every row (each CTA computes all of them) and the L column of the own
//     rows -> ARRIVE -> rank-1 / rank-2 update of the columns > k0 of the own
//     rows, overlapping the barrier and the next step's merge.
// The next step WAITS on the barrier, so one barrier per step (two with the
// rowmax exchange).  Broadcast vectors and inboxes are triple-buffered by step:
// the buffer step s+1 publishes into was last read in step s-2, whose bulk
// every CTA finished before arriving in step s-1.
template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(BKC_NT) bk_cluster_kernel(BkArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char bkc_smem[];
  __shared__ double rv[BKC_NT / 32];
  __shared__ double rst[2][BKC_NT / 32];      // per-warp max |a_ij|^2 of a step's update, by step parity
  __shared__ BkcSlot inbox[3][CS], inboxR[CS], merged;
  const int rank = (int)cl.block_rank();
  const int b = blockIdx.x / CS;
  const int n = a.n, lda = a.lda, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = BKC_NT / 32, NBT = BKC_NT - 32;   // bulk threads
  const int bt = tid - 32;
  const bool pw = warp == 0;                           // pivot warp
  const bool gthread = tid == 32;                      // owns the growth recurrence
  const int64_t cap = bkc_entries<CS>(n);
  cplx* Rl = reinterpret_cast<cplx*>(bkc_smem);      // own packed lower rows
  cplx* ls = Rl + cap;                                 // l_j / wk_j of every row (computed locally)
  cplx* ws = ls + n;                                   // wkp_j (2x2)
  cplx* vec = ws + n;                                  // broadcast vectors [3][3][n]
  int64_t* perm_s = reinterpret_cast<int64_t*>(vec + 9 * (int64_t)n);
  int8_t* tags_s = reinterpret_cast<int8_t*>(perm_s + n);
  cplx* W = a.W + (int64_t)b * a.stride_w;
  const bool lead = rank == 0 && tid == 0;
  const int nown = (n - rank + CS - 1) / CS;          // own rows: rank, rank + CS, ...
  auto L = [&](int i, int j) -> cplx& { return Rl[bkc_off<CS>(i) + j]; };   // own row i
  auto Rm = [&](int i, int j) -> cplx& {                                     // any row (DSMEM)
    cplx* base = cl.map_shared_rank(Rl, i % CS);
    return base[bkc_off<CS>(i) + j];
  };
  auto first_q = [&](int i0) { const int q = (i0 - rank + CS - 1) / CS; return q > 0 ? q : 0; };  // own rows >= i0

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
  for (int i = tid; i < n; i += BKC_NT) { perm_s[i] = i; tags_s[i] = 0; }
  scale = bkc_block_max(scale, rv);
  asym = bkc_block_max(asym, rv);
  tm2 = bkc_block_max(tm2, rv);
  if (tid == 0) bkc_post<CS>(cl, inboxR, rank, BkcSlot{-1.0, scale, asym, tm2, 0x7fffffff, 0});
  cl.sync();
  {
    const BkcSlot m = bkc_merge<CS>(inboxR, &merged);
    scale = m.own;
    asym = m.aux;
    tm2 = m.aux2;
  }
  if (lead) { a.scale[b] = scale; a.asym[b] = asym; }
  if (a.check_sym == 1 && n > 0 && scale > 0.0 && asym > __dmul_rn(1e-12, scale)) {
    if (lead) {
      a.info[b] = -2; a.n2x2[b] = 0; a.growth[b] = 1.0;
      for (int i = 0; i < n; ++i) { a.perm[(int64_t)b * n + i] = i; a.tags[(int64_t)b * n + i] = 0; }
    }
    cl.sync();
    return;
  }
  const double tol_abs = __dmul_rn(a.pivot_tol, scale);
  // growth recurrence (kernels.py:135-144), run by gthread only: a step's
  // update maximum reaches every CTA two steps later, applied in step order
  double trail_max = __dsqrt_rn(tm2);
  double growth = 1.0;
  int n2x2 = 0, info = -1;
  int ks1 = 0, k01 = 0, ks2 = 0, k02 = 0;          // kstep / k0 of steps s-1, s-2
  auto grow = [&](double usq, int kstep, int k0) {
    if (k0 < n) {
      const double step_max = __dsqrt_rn(usq);
      if (trail_max > 0.0) {
        double r = __ddiv_rn(step_max, trail_max);
        if (kstep == 2) r = __dsqrt_rn(r);
        if (r > growth) growth = r;
      }
      trail_max = step_max;
    }
  };

  // ---- column 0: published by the pivot warps ------------------------------
  if (pw) {
    double v = -1.0, own = -1.0;
    int vi = 0x7fffffff;
    for (int q = lane; q < nown; q += 32) {
      const int i = rank + q * CS;
      const cplx z = L(i, 0);
#pragma unroll
      for (int c = 0; c < CS; ++c) cl.map_shared_rank(vec, c)[i] = z;
      const double az = x_abs(z);
      if (i > 0) argmax_merge(v, vi, az, i);
      else own = az;
    }
    warp_argmax(v, vi);
    own = warp_max(own);
    if (lane == 0) bkc_post<CS>(cl, inbox[0], rank, BkcSlot{v, own, -1.0, -1.0, vi, 0});
  }
  bkc_arrive();
#ifdef D3M_BK_PROFILE
  double pacc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) pacc[i] = 0.0;
  long long prof_t = clock64();
#endif
  int k = 0, s = 0;
  double pend_usq = 0.0;
  while (k < n) {
    const int bs = s % 3;
    cplx* cA = vec + (int64_t)(bs * 3 + 0) * n;
    cplx* cB = vec + (int64_t)(bs * 3 + 1) * n;
    cplx* cC = vec + (int64_t)(bs * 3 + 2) * n;
    // ---- 1. wait for column k and the argmax slots; merge ------------------
    bkc_wait();
    BKC_MARK(0, 0);
    BKC_MARK(32, 8);
    const BkcSlot m1 = bkc_merge<CS>(inbox[bs], &merged);   // its __syncthreads also ends the local bulk
    BKC_MARK(0, 1);
    BKC_MARK(32, 9);
    pend_usq = m1.aux;                                       // step s-2's update maximum
    const double absakk = m1.own;                            // |W[k, k]|, from its owner
    double colmax = 0.0;
    int imax = k;
    if (k + 1 < n) { colmax = m1.v; imax = m1.i; }
    if (fmax(absakk, colmax) <= tol_abs) { info = k; break; }

    int kstep = 1, kp;
    if (absakk >= __dmul_rn(kBkcAlpha, colmax)) {
      kp = k;
    } else {
      // ---- 2. push column k+1 and the symmetric column imax; rowmax over
      //         W[imax, k:imax] and W[imax+1:, imax]; |W[imax, imax]| ----------
      double rm = 0.0, aim = -1.0;
      if (imax % CS == rank) {
        for (int t = k + tid; t <= imax; t += BKC_NT) {
          const cplx z = L(imax, t);
#pragma unroll
          for (int c = 0; c < CS; ++c) cl.map_shared_rank(cC, c)[t] = z;
          if (t < imax) rm = fmax(rm, x_abs(z));
          else aim = x_abs(z);
        }
      }
      for (int q = first_q(k + 1) + tid; q < nown; q += BKC_NT) {
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
      rm = bkc_block_max(rm, rv);
      aim = bkc_block_max(aim, rv);
      if (tid == 0) bkc_post<CS>(cl, inboxR, rank, BkcSlot{-1.0, aim, rm, -1.0, 0x7fffffff, 0});
      cl.sync();
      const BkcSlot m2 = bkc_merge<CS>(inboxR, &merged);
      const double rowmax = m2.aux, absimax = m2.own;
      if (__dmul_rn(absakk, rowmax) >= __dmul_rn(__dmul_rn(kBkcAlpha, colmax), colmax)) {
        kp = k;
      } else if (absimax >= __dmul_rn(kBkcAlpha, rowmax)) {
        kp = imax;
      } else {
        kp = imax;
        kstep = 2;
      }
    }
    const int kk = k + kstep - 1, k0 = k + kstep;
    const cplx* cK = kstep == 1 ? cA : cB;          // column kk before the swap
    // post-interchange columns k (X) and k+1 (Y) at row i >= k0: sigma swaps kk, kp
    auto Xc = [&](int i) -> cplx {
      if (kstep == 1) return kp == k ? cA[i] : (i == kp ? cC[k] : cC[i]);
      return i == kp ? cA[kk] : cA[i];
    };
    auto Yc = [&](int i) -> cplx { return i == kp ? cC[kk] : cC[i]; };
    const cplx piv = kstep == 1 ? (kp == k ? cA[k] : cC[kp]) : mk(0.0, 0.0);
    // 2x2 pivot coefficients (kernels.py:115-119), computed by every thread
    cplx d11 = mk(0.0, 0.0), d22 = d11, d21s = d11;
    if (kstep == 2) {
      const cplx d21 = cA[kp];                                   // W'[k+1, k]
      d11 = x_div_py(cC[kp], d21);                               // W'[k+1, k+1] / d21
      d22 = x_div_py(cA[k], d21);                                // W'[k, k] / d21
      const cplx t2 = x_div_py(mk(1.0, 0.0), x_sub(x_mul(d11, d22), mk(1.0, 0.0)));
      d21s = x_div_py(t2, d21);
    }
    const int nb = (s + 1) % 3;
    const int qk0 = first_q(k0);
    double step_sq = 0.0;

    if (pw) {
      // ---- 3P. interchange of the own rows i > kp: W[i, kk] <-> W[i, kp] ----
      if (kp != kk) {
        for (int q = first_q(kp + 1) + lane; q < nown; q += 32) {
          const int i = rank + q * CS;
          const cplx t0 = L(i, kk);
          L(i, kk) = L(i, kp);
          L(i, kp) = t0;
        }
        if (lead) { const int64_t t0 = perm_s[kk]; perm_s[kk] = perm_s[kp]; perm_s[kp] = t0; }
      }
      if (lead) {
        if (kstep == 1) tags_s[k] = 1;
        else { tags_s[k] = 2; tags_s[k + 1] = 0; }
      }
      __syncwarp();
      asm volatile("bar.arrive 1, %0;\n" ::"n"(BKC_NT) : "memory");   // the bulk may read the swapped rows
      BKC_MARK(0, 2);
      // ---- 4P. update of column k0 of the own rows, publish ----------------
      double up = -1.0;
      if (s >= 1) up = warp_max(lane < NW ? rst[(s - 1) & 1][lane] : 0.0);
      double v = -1.0, own = -1.0;
      int vi = 0x7fffffff;
      if (k0 < n) {
        // multipliers of row k0 (the bulk threads compute the same values for rows > k0)
        cplx l0, p0 = mk(0.0, 0.0);
        if (kstep == 1) {
          l0 = x_div_py(Xc(k0), piv);                                        // lj = W[j, k] / piv
        } else {
          const cplx x = Xc(k0), y = Yc(k0);
          l0 = x_mul(d21s, x_sub(x_mul(d11, x), y));                          // wk
          p0 = x_mul(d21s, x_sub(x_mul(d22, y), x));                          // wkp
        }
        BKC_MARK(0, 4);
        cplx* cAn = vec + (int64_t)(nb * 3) * n;
        for (int q = qk0 + lane; q < nown; q += 32) {
          const int i = rank + q * CS;
          cplx* row = Rl + bkc_off<CS>(i);
          // W'[i, k0]: row kp was refilled from column kk (left to the bulk,
          // except this entry)
          const cplx wo = (i == kp && kp != kk) ? (k0 < kp ? cK[k0] : cK[kk]) : row[k0];
          const cplx xi = Xc(i);
          const cplx w = kstep == 1 ? x_sub(wo, x_mul(xi, l0))
                                    : x_sub(wo, x_add(x_mul(xi, l0), x_mul(Yc(i), p0)));
          row[k0] = w;
#pragma unroll
          for (int c = 0; c < CS; ++c) cl.map_shared_rank(cAn, c)[i] = w;
          step_sq = fmax(step_sq, x_abs2(w));
          const double aw = x_abs(w);
          if (i > k0) argmax_merge(v, vi, aw, i);
          else own = aw;
        }
        BKC_MARK(0, 5);
        warp_argmax(v, vi);
        own = warp_max(own);
      }
      step_sq = warp_max(step_sq);
      if (lane == 0) {
        rst[s & 1][0] = step_sq;
        bkc_post<CS>(cl, inbox[nb], rank, BkcSlot{v, own, up, -1.0, vi, 0});
      }
      BKC_MARK(0, 6);
      bkc_arrive();
      BKC_MARK(0, 3);
      if (kstep == 2) ++n2x2;
    } else {
      // ---- 3B. row kp refill W[kp, kk+1:kp] <- W[kk+1:kp, kk], W[kp, kp] <-
      //          W[kk, kk] (entry k0 left to the pivot warp); L rows of kk / kp
      const bool lswap = kp != kk && kk % CS == rank;
      cplx lsv[BKC_JPT];
      if (kp != kk) {
        if (kp % CS == rank)
          for (int j = kk + 1 + bt; j <= kp; j += NBT)
            if (j != k0) L(kp, j) = j < kp ? cK[j] : cK[kk];
        if (lswap) {
          if (bt == 0) {
            L(kk, kk) = cC[kp];                      // W[kk, kk] <- W[kp, kp]
            if (kstep == 2) L(kk, k) = cA[kp];       // W[k+1, k] <- W[kp, k]
          }
#pragma unroll
          for (int h = 0; h < BKC_JPT; ++h)          // W[kp, :k], stored below
            if (bt + h * NBT < k) lsv[h] = Rm(kp, bt + h * NBT);
        }
      }
      // ---- 4B. multipliers of every row > k0 (up to BKC_JPT rows per bulk
      //          thread: the launcher guarantees n <= BKC_JPT * NBT) and the L
      //          column of the own rows, stored after the pivot warp's
      //          interchange is visible -------------------------------------------
      cplx lc0[BKC_JPT], lc1[BKC_JPT];
#pragma unroll
      for (int t = 0; t < BKC_JPT; ++t) {
        const int j = k0 + bt + t * NBT;
        lc0[t] = lc1[t] = mk(0.0, 0.0);
        if (j < n) {
          const cplx x = Xc(j);
          if (kstep == 1) {
            if (j > k0) ls[j] = x_div_py(x, piv);                  // lj = W[j, k] / piv
            if (j % CS == rank) lc0[t] = x_div_np(x, piv);        // W[k+1:, k] /= piv
          } else {
            const cplx y = Yc(j);
            lc0[t] = x_mul(d21s, x_sub(x_mul(d11, x), y));          // wk
            lc1[t] = x_mul(d21s, x_sub(x_mul(d22, y), x));          // wkp
            ls[j] = lc0[t];
            ws[j] = lc1[t];
          }
        }
      }
      if (lswap) {                             // W[kk, :k] <-> W[kp, :k]
#pragma unroll
        for (int h = 0; h < BKC_JPT; ++h) {
          const int u = bt + h * NBT;
          if (u < k) {
            Rm(kp, u) = L(kk, u);
            L(kk, u) = lsv[h];
          }
        }
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(BKC_NT) : "memory");     // swapped rows + multipliers
#pragma unroll
      for (int t = 0; t < BKC_JPT; ++t) {
        const int j = k0 + bt + t * NBT;
        if (j < n && j % CS == rank) {
          L(j, k) = lc0[t];
          if (kstep == 2) L(j, k + 1) = lc1[t];
        }
      }
      bkc_arrive();
      if (gthread && s >= 2) grow(pend_usq, ks2, k02);
      BKC_MARK(32, 10);
      // ---- 5B. rank-1 / rank-2 update of the columns > k0 of the own rows
      //          (warp per row; each chunk loads before it stores) -------------
      for (int q = first_q(k0 + 1) + (warp - 1); q < nown; q += NW - 1) {
        const int i = rank + q * CS;
        cplx* row = Rl + bkc_off<CS>(i);
        const cplx xi = Xc(i);
        if (kstep == 1) {
          for (int j0 = k0 + 1; j0 <= i; j0 += 128) {
            cplx rw[4], lw[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = j0 + lane + 32 * u;
              if (j <= i) { rw[u] = row[j]; lw[u] = ls[j]; }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = j0 + lane + 32 * u;
              if (j <= i) {
                const cplx w = x_sub(rw[u], x_mul(xi, lw[u]));          // W[j:, j] -= W[j:, k] * lj
                row[j] = w;
                step_sq = fmax(step_sq, x_abs2(w));
              }
            }
          }
        } else {
          const cplx yi = Yc(i);
          for (int j0 = k0 + 1; j0 <= i; j0 += 64) {
            cplx rw[2], lw[2], ww[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int j = j0 + lane + 32 * u;
              if (j <= i) { rw[u] = row[j]; lw[u] = ls[j]; ww[u] = ws[j]; }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int j = j0 + lane + 32 * u;
              if (j <= i) {
                const cplx w = x_sub(rw[u], x_add(x_mul(xi, lw[u]), x_mul(yi, ww[u])));
                row[j] = w;
                step_sq = fmax(step_sq, x_abs2(w));
              }
            }
          }
        }
      }
      step_sq = warp_max(step_sq);
      if (lane == 0) rst[s & 1][warp] = step_sq;
      BKC_MARK(32, 11);
    }
    ks2 = ks1; k02 = k01;
    ks1 = kstep; k01 = k0;
    k = k0;
    ++s;
  }
  // ---- growth of the steps whose update maxima are still in flight ---------
  if (info >= 0) {
    // stopped at the top of step s: step s-1's maximum is in rst, not posted
    if (s >= 1) {
      if (pw) {
        const double up = warp_max(lane < NW ? rst[(s - 1) & 1][lane] : 0.0);
        if (lane == 0) bkc_post<CS>(cl, inboxR, rank, BkcSlot{-1.0, -1.0, up, -1.0, 0x7fffffff, 0});
      }
      cl.sync();
      const BkcSlot mf = bkc_merge<CS>(inboxR, &merged);
      if (gthread) {
        if (s >= 2) grow(pend_usq, ks2, k02);
        grow(mf.aux, ks1, k01);
      }
    }
  } else {
    // ran to the end: the last step's arrival carried step s-2's maximum
    bkc_wait();
    const BkcSlot mf = bkc_merge<CS>(inbox[s % 3], &merged);
    if (gthread && s >= 2) grow(mf.aux, ks2, k02);
  }
  // ---- write back the own rows (lower triangle), pivots, stats -------------
  for (int q = warp; q < nown; q += NW) {
    const int i = rank + q * CS;
    const cplx* src = Rl + bkc_off<CS>(i);
    cplx* row = W + (int64_t)i * lda;
    for (int j = lane; j <= i; j += 32) row[j] = src[j];
  }
  if (rank == 0)
    for (int i = tid; i < n; i += BKC_NT) {
      a.perm[(int64_t)b * n + i] = perm_s[i];
      a.tags[(int64_t)b * n + i] = tags_s[i];
    }
  if (lead) {
    a.n2x2[b] = n2x2;
    a.info[b] = info;
  }
  if (rank == 0 && gthread) a.growth[b] = growth;
#ifdef D3M_BK_PROFILE
  if (rank == 0 && (tid == 0 || tid == 32)) {
    double* prof = reinterpret_cast<double*>(a.scratch);
#pragma unroll
    for (int i = 0; i < 8; ++i) prof[(tid == 0 ? 0 : 8) + i] = pacc[(tid == 0 ? 0 : 8) + i];
  }
#endif
  cl.sync();     // peers may still read this CTA's shared memory
}

template <int CS>
static int bkc_launch(BkArgs* a, int batch, cudaStream_t s) {
  // own rows + ls, ws (2n) + broadcast vectors (9n) + perm / tags (< n)
  const size_t smem = sizeof(cplx) * (size_t)(bkc_entries<CS>(a->n) + 12 * (int64_t)a->n);
  if (smem > 200 * 1024 || a->n > BKC_JPT * (BKC_NT - 32)) return -22;
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
