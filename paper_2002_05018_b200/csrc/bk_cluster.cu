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
// Communication: each step's pivot column (and, for the rowmax test, columns
// k+1 and imax) is pushed to every CTA with st.async, which completes on the
// RECEIVER's mbarrier (expected bytes armed by the receiver), together with a
// 32-byte slot carrying each CTA's exact argmax.  There is no cluster barrier
// in the step loop.  The interchange of the L rows left of column k
// (kernels.py:96-98) never crosses CTAs either: every CTA records the step's
// interchange and the L entries are written to their final rows at the end
// (each column's entries move by the interchanges of the later steps).
#include <cooperative_groups.h>
#include <cstdlib>
#include "d3m_common.cuh"
#include "d3m_kernels.h"

namespace d3m {
namespace cg = cooperative_groups;

constexpr int BKC_NT = 384;
constexpr int BKC_JPT = 2;       // multiplier rows per bulk thread: n <= BKC_JPT * (BKC_NT - 32)
constexpr double kBkcAlpha = 0.6403882032022076;  // (1 + sqrt(17)) / 8, kernels.py:33

// prologue exchange (scale, asym, trailing max), through the cluster barrier
struct BkcSlot {
  double v, own, aux, aux2;
  int i, pad;
};

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

// ---- step exchange slot: 48 bytes, three st.async.v2.f64 -------------------
struct XSlot {
  double v;      // exact argmax value or -1
  double own;    // a modulus only the owner of a row can supply, else -1
  double aux;    // max-reduced payload (rowmax, update maximum)
  double i;      // argmax index (int bits)
  double v2;     // runner-up of the argmax (margin diagnostic), else -1
  double pad;
};
constexpr unsigned kSlotBytesMin = 32;          // v, own, aux, i (v2 only when margins are tracked)
__device__ __forceinline__ unsigned slot_bytes(bool track) { return track ? (unsigned)sizeof(XSlot) : kSlotBytesMin; }

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// 16-byte store into a peer's shared memory, completing on the peer's mbarrier
__device__ __forceinline__ void st_async(uint32_t raddr, double x, double y, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n"
               ::"r"(raddr), "d"(x), "d"(y), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t* b, unsigned tx) {       // the single arrival + tx
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n"
               ::"r"(saddr(b)), "r"(tx) : "memory");
}
// bounded wait: a lost transfer traps (kernel error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  for (unsigned it = 0;; ++it) {
    unsigned ok;
    asm volatile("{\n .reg .pred p;\n"
                 " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(saddr(b)), "r"(parity) : "memory");
    if (ok) return;
    if (it > (1u << 26)) __trap();
  }
}

// one slot to CTA `lane` (lanes < CS of the calling warp; all lanes hold x);
// the runner-up v2 travels only when margins are tracked (slot_bytes)
template <int CS>
__device__ __forceinline__ void xpost(const XSlot* box, int rank, const XSlot& x, uint64_t* bar, bool track) {
  const int lane = threadIdx.x & 31;
  if (lane < CS) {
    const uint32_t dst = mapa(saddr(box + rank), lane), rb = mapa(saddr(bar), lane);
    st_async(dst, x.v, x.own, rb);
    st_async(dst + 16, x.aux, x.i, rb);
    if (track) st_async(dst + 32, x.v2, x.pad, rb);
  }
}

// merge of the CS slots of a local inbox (warp 0), broadcast through smem;
// with `track`, also the cluster-wide runner-up of the argmax (v2)
template <int CS>
__device__ __forceinline__ XSlot xmerge(const XSlot* box, XSlot* out, bool track = false) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double v = -1.0, own = -1.0, aux = -1.0, r2 = -1.0;
    int vi = 0x7fffffff;
    if (lane < CS) {
      const XSlot r = box[lane];
      v = r.v;
      own = r.own;
      aux = r.aux;
      r2 = r.v2;
      vi = (int)__double_as_longlong(r.i);
    }
    const double lv = v;
    const int li = vi;
#pragma unroll
    for (int o = CS / 2; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, vi, o);
      own = fmax(own, __shfl_xor_sync(0xffffffffu, own, o));
      aux = fmax(aux, __shfl_xor_sync(0xffffffffu, aux, o));
      argmax_merge(v, vi, v2, i2);
    }
    if (track) {   // the winner's slot offers its own runner-up, every other slot its winner
      double c = li == vi ? r2 : lv;
#pragma unroll
      for (int o = CS / 2; o > 0; o >>= 1) c = fmax(c, __shfl_xor_sync(0xffffffffu, c, o));
      r2 = c;
    }
    if (lane == 0) *out = XSlot{v, own, aux, __longlong_as_double((long long)vi), r2, 0.0};
  }
  __syncthreads();
  return *out;
}
__device__ __forceinline__ int xidx(const XSlot& x) { return (int)__double_as_longlong(x.i); }
__device__ __forceinline__ XSlot xslot(double v, double own, double aux, int i, double v2 = -1.0) {
  return XSlot{v, own, aux, __longlong_as_double((long long)i), v2, 0.0};
}
// runner-up of a warp's first-index argmax: lanes hold their own top-2
// (lv, li, lv2), (v, vi) is the warp winner
__device__ __forceinline__ double warp_runner_up(double lv, int li, double lv2, int vi) {
  return warp_max(li == vi ? lv2 : lv);
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
// first bulk thread; accumulated in registers, written once at the end into
// g_bkc_prof (read by d3m_bkc_prof_read; profiling builds only)
__device__ double g_bkc_prof[32];
#define BKC_MARK(who, slot) do { if (rank == 0 && tid == (who)) { long long t_ = clock64(); \
    pacc[slot] += (double)(t_ - prof_t); prof_t = t_; } } while (0)
#else
#define BKC_MARK(who, slot) do { } while (0)
#endif

// Roles inside each CTA of the cluster (per step k, pivot column k0 = k + kstep):
//   pivot warp (warp 0): merge of the argmax slots -> pivot decision ->
//     interchange of the own rows' columns kk / kp -> update of column k0 of
//     the own rows -> push it with its exact argmax, the modulus of the new
//     diagonal entry and the update maximum of step s-1.  This chain is the
//     step's critical path.
//   bulk warps (1..NW-1): row kp refill, multipliers of every row (each CTA
//     computes all of them) and the L column of the own rows, then the rank-1
//     / rank-2 update of the columns > k0 of the own rows, overlapping the
//     next step's exchange.
// The pivot-column vector and the inboxes are triple-buffered by step: the
// buffer a peer fills during its step s was last read here in step s-2, and
// the peer only reaches step s after this CTA pushed its step s-1 column,
// which follows the end of its step s-2 bulk update.  The rowmax columns
// (k+1, imax) are filled and read inside one step: double-buffered.
// TRACK: the margin diagnostic (BkArgs::margin) is compiled in only in the
// TRACK instance, so the production kernel keeps its registers.
template <int CS, bool TRACK>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(BKC_NT) bk_cluster_kernel(BkArgs a) {
#ifdef D3M_BK_PROFILE
  const long long t_entry = clock64();
#endif
  const int csym = a.check_sym_dev ? *a.check_sym_dev : a.check_sym;   // per-block device flag (block_ldlt)
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char bkc_smem[];
  __shared__ double rv[BKC_NT / 32];
  __shared__ double rst[2][BKC_NT / 32];      // per-warp max |a_ij|^2 of a step's update, by step parity
  __shared__ __align__(16) XSlot inbox[3][CS];
  __shared__ __align__(16) XSlot inboxR[CS];
  __shared__ XSlot xmerged;
  __shared__ BkcSlot pbox[CS], pmerged;
  __shared__ __align__(8) uint64_t mbar[3], mbarR;
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
  cplx* vec = ws + n;                                  // broadcast vectors: A [3][n], B [2][n], C [2][n]
  short* perm_s = reinterpret_cast<short*>(vec + 7 * (int64_t)n);
  short* qmap = perm_s + n;                            // write-back row map
  short* stk = qmap + n;                               // per step: k, kstep, kp (-1: no interchange)
  int8_t* tags_s = reinterpret_cast<int8_t*>(stk + 3 * n);
  cplx* W = a.W + (int64_t)b * a.stride_w;
  const bool lead = rank == 0 && tid == 0;
  const int nown = (n - rank + CS - 1) / CS;          // own rows: rank, rank + CS, ...
  auto L = [&](int i, int j) -> cplx& { return Rl[bkc_off<CS>(i) + j]; };   // own row i
  auto first_q = [&](int i0) { const int q = (i0 - rank + CS - 1) / CS; return q > 0 ? q : 0; };  // own rows >= i0

  if (tid == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&mbar[i]);
    mbar_init(&mbarR);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // ---- prologue: numpy scale / symmetry check / trailing max, own rows -> smem
  double scale = 0.0, asym = 0.0, tm2 = 0.0;
  for (int q = warp; q < nown; q += NW) {
    const int i = rank + q * CS;
    const cplx* row = W + (int64_t)i * lda;
    cplx* dst = Rl + bkc_off<CS>(i);
    const int jend = csym == 2 ? i + 1 : n;     // 2: verified exactly symmetric (lower suffices)
    for (int j = lane; j < jend; j += 32) {
      const cplx z = row[j];
      scale = fmax(scale, np_abs(z));
      if (j <= i) { tm2 = fmax(tm2, x_abs2(z)); dst[j] = z; }
      if (csym == 1 && j < i) asym = fmax(asym, np_abs(x_sub(z, W[(int64_t)j * lda + i])));
    }
  }
  for (int i = tid; i < n; i += BKC_NT) { perm_s[i] = (short)i; tags_s[i] = 0; }
  scale = bkc_block_max(scale, rv);
  asym = bkc_block_max(asym, rv);
  tm2 = bkc_block_max(tm2, rv);
  if (tid == 0) bkc_post<CS>(cl, pbox, rank, BkcSlot{-1.0, scale, asym, tm2, 0x7fffffff, 0});
  cl.sync();                                          // also publishes the mbarrier inits
  {
    const BkcSlot m = bkc_merge<CS>(pbox, &pmerged);
    scale = m.own;
    asym = m.aux;
    tm2 = m.aux2;
  }
  if (lead) { a.scale[b] = scale; a.asym[b] = asym; }
  if (csym == 1 && n > 0 && scale > 0.0 && asym > __dmul_rn(1e-12, scale)) {
    if (lead) {
      a.info[b] = -2; a.n2x2[b] = 0; a.growth[b] = 1.0;
      if (a.margin) { a.margin[2 * b] = 1.0; a.margin[2 * b + 1] = 1.0; }
      for (int i = 0; i < n; ++i) { a.perm[(int64_t)b * n + i] = i; a.tags[(int64_t)b * n + i] = 0; }
    }
    cl.sync();
    return;
  }
  const double tol_abs = bk_threshold(a.pivot_tol, scale, a.abs_tol);
  constexpr bool track = TRACK;                // pivot-decision margins (lead thread)
  double mdec = 1.0, mgap = 1.0;
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

  // ---- column 0, pushed by the pivot warps -----------------------------------
  if (pw) {
    double v = -1.0, own = -1.0, v2 = -1.0;
    int vi = 0x7fffffff;
    for (int q = lane; q < nown; q += 32) {
      const int i = rank + q * CS;
      const cplx z = L(i, 0);
      const uint32_t src = saddr(vec + i), sb = saddr(&mbar[0]);
#pragma unroll
      for (int c = 0; c < CS; ++c) st_async(mapa(src, c), z.x, z.y, mapa(sb, c));
      const double az = x_abs(z);
      if (i > 0) {
        if (track) top2_merge(v, vi, v2, az, i);
        else argmax_merge(v, vi, az, i);
      }
      else own = az;
    }
    const double lv = v;
    const int li = vi;
    warp_argmax(v, vi);
    own = warp_max(own);
    if (track) v2 = warp_runner_up(lv, li, v2, vi);
    xpost<CS>(inbox[0], rank, xslot(v, own, -1.0, vi, v2), &mbar[0], track);
  }
#ifdef D3M_BK_PROFILE
  const long long t_loop0 = clock64();
  double pacc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) pacc[i] = 0.0;
  long long prof_t = clock64();
#endif
  int k = 0, s = 0;
  unsigned rphase = 0;
  double pend_usq = 0.0;
  while (k < n) {
    // column k (cA) is pushed during the previous step: triple-buffered.
    // Columns k+1 / imax (cB, cC) are pushed and read inside step s; a peer
    // reaches step s+2's push only after this CTA's step s+1 merge (which ends
    // the step-s bulk), so two buffers suffice.
    const int bs = s % 3;
    cplx* cA = vec + (int64_t)bs * n;
    cplx* cB = vec + (int64_t)(3 + (s & 1)) * n;
    cplx* cC = vec + (int64_t)(5 + (s & 1)) * n;
    // ---- 1. column k and the argmax slots have landed; merge ---------------
    if (tid == 0) mbar_arm(&mbar[bs], (unsigned)(n - k) * 16u + CS * slot_bytes(track));
    mbar_wait(&mbar[bs], (unsigned)(s / 3) & 1u);
    BKC_MARK(0, 0);
    BKC_MARK(32, 8);
    const XSlot m1 = xmerge<CS>(inbox[bs], &xmerged, track);   // its __syncthreads also ends the local bulk
    BKC_MARK(0, 1);
    BKC_MARK(32, 9);
    pend_usq = m1.aux;                                       // step s-2's update maximum
    const double absakk = m1.own;                            // |W[k, k]|, from its owner
    double colmax = 0.0;
    int imax = k;
    if (k + 1 < n) {
      colmax = m1.v;
      imax = xidx(m1);
      if (track && lead) mgap = fmin(mgap, argmax_gap(colmax, m1.v2));
    }
    if (fmax(absakk, colmax) <= tol_abs) {
      if (track && lead) mdec = fmin(mdec, test_margin(tol_abs, fmax(absakk, colmax)));
      info = k;
      break;
    }

    int kstep = 1, kp;
#ifdef D3M_BK_PROFILE
    bool prof_rm = false;
#endif
    if (absakk >= __dmul_rn(kBkcAlpha, colmax)) {
      kp = k;
      if (track && lead) mdec = fmin(mdec, decision_margin(tol_abs, absakk, colmax, 0.0, 0.0, kBkcAlpha, 1));
    } else {
      // ---- 2. push column k+1 and the symmetric column imax; rowmax over
      //         W[imax, k:imax] and W[imax+1:, imax]; |W[imax, imax]| ----------
      if (tid == 0) mbar_arm(&mbarR, (unsigned)(2 * (n - k) - 1) * 16u + CS * slot_bytes(track));
#ifdef D3M_BK_PROFILE
      if (rank == 0 && tid == 0) pacc[13] += 1.0;
      prof_rm = true;
#endif
      const uint32_t rb = saddr(&mbarR);
      double rm = 0.0, aim = -1.0;
      if (imax % CS == rank) {
        for (int t = k + tid; t <= imax; t += BKC_NT) {
          const cplx z = L(imax, t);
          const uint32_t src = saddr(cC + t);
#pragma unroll
          for (int c = 0; c < CS; ++c) st_async(mapa(src, c), z.x, z.y, mapa(rb, c));
          if (t < imax) rm = fmax(rm, x_abs(z));
          else aim = x_abs(z);
        }
      }
      for (int q = first_q(k + 1) + tid; q < nown; q += BKC_NT) {
        const int i = rank + q * CS;
        const cplx y = L(i, k + 1);
        const uint32_t srcb = saddr(cB + i);
#pragma unroll
        for (int c = 0; c < CS; ++c) st_async(mapa(srcb, c), y.x, y.y, mapa(rb, c));
        if (i > imax) {
          const cplx z = L(i, imax);
          const uint32_t srcc = saddr(cC + i);
#pragma unroll
          for (int c = 0; c < CS; ++c) st_async(mapa(srcc, c), z.x, z.y, mapa(rb, c));
          rm = fmax(rm, x_abs(z));
        }
      }
      rm = bkc_block_max(rm, rv);
      aim = bkc_block_max(aim, rv);
      if (pw) xpost<CS>(inboxR, rank, xslot(-1.0, aim, rm, 0x7fffffff), &mbarR, track);
      mbar_wait(&mbarR, rphase & 1u);
      ++rphase;
      const XSlot m2 = xmerge<CS>(inboxR, &xmerged);
      const double rowmax = m2.aux, absimax = m2.own;
      int stage = 3;
      if (__dmul_rn(absakk, rowmax) >= __dmul_rn(__dmul_rn(kBkcAlpha, colmax), colmax)) {
        kp = k;
        stage = 2;
      } else if (absimax >= __dmul_rn(kBkcAlpha, rowmax)) {
        kp = imax;
      } else {
        kp = imax;
        kstep = 2;
      }
      if (track && lead)
        mdec = fmin(mdec, decision_margin(tol_abs, absakk, colmax, rowmax, absimax, kBkcAlpha, stage));
    }
    const int kk = k + kstep - 1, k0 = k + kstep;
#ifdef D3M_BK_PROFILE
    if (rank == 0 && tid == 0) { pacc[14] += kp != kk ? 1.0 : 0.0; pacc[15] += kstep == 2 ? 1.0 : 0.0; }
#endif
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
#ifdef D3M_BK_PROFILE
    BKC_MARK(0, prof_rm ? 12 : 3);
#endif

    if (pw) {
      // ---- 3P. interchange of the own rows i > kp: W[i, kk] <-> W[i, kp] ----
      if (kp != kk) {
        for (int q = first_q(kp + 1) + lane; q < nown; q += 32) {
          const int i = rank + q * CS;
          const cplx t0 = L(i, kk);
          L(i, kk) = L(i, kp);
          L(i, kp) = t0;
        }
        if (lead) { const short t0 = perm_s[kk]; perm_s[kk] = perm_s[kp]; perm_s[kp] = t0; }
      }
      if (lane == 0) {     // every CTA records the step for the L write-back
        stk[3 * s] = (short)k;
        stk[3 * s + 1] = (short)kstep;
        stk[3 * s + 2] = (short)(kp != kk ? kp : -1);
        if (rank == 0) {
          if (kstep == 1) tags_s[k] = 1;
          else { tags_s[k] = 2; tags_s[k + 1] = 0; }
        }
      }
      __syncwarp();
      asm volatile("bar.arrive 1, %0;\n" ::"n"(BKC_NT) : "memory");   // the bulk may read the swapped rows
#ifdef D3M_BK_PROFILE
      BKC_MARK(0, prof_rm ? 12 : 2);
#endif
      // ---- 4P. update of column k0 of the own rows, push ------------------
      double up = -1.0;
      if (s >= 1) up = warp_max(lane < NW ? rst[(s - 1) & 1][lane] : 0.0);
      BKC_MARK(0, 7);
      double v = -1.0, own = -1.0, v2 = -1.0;
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
        cplx* cAn = vec + (int64_t)nb * n;
        const uint32_t nbar = saddr(&mbar[nb]);
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
          const uint32_t src = saddr(cAn + i);
#pragma unroll
          for (int c = 0; c < CS; ++c) st_async(mapa(src, c), w.x, w.y, mapa(nbar, c));
          step_sq = fmax(step_sq, x_abs2(w));
          const double aw = x_abs(w);
          if (i > k0) {
            if (track) top2_merge(v, vi, v2, aw, i);
            else argmax_merge(v, vi, aw, i);
          }
          else own = aw;
        }
        BKC_MARK(0, 5);
        const double lv = v;
        const int li = vi;
        // the critical butterfly carries only the exact argmax (first-index,
        // order-free); the owner's modulus |W[k0, k0]| comes from lane 0
        // (row k0 is the first own row >= k0), and the update maximum is
        // reduced after the push, off the chain
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double v2_ = __shfl_xor_sync(0xffffffffu, v, o);
          const int i2 = __shfl_xor_sync(0xffffffffu, vi, o);
          argmax_merge(v, vi, v2_, i2);
        }
        own = __shfl_sync(0xffffffffu, own, 0);
        if (track) v2 = warp_runner_up(lv, li, v2, vi);
      }
      xpost<CS>(inbox[nb], rank, xslot(v, own, up, vi, v2), &mbar[nb], track);
      step_sq = warp_max(step_sq);
      if (lane == 0) rst[s & 1][0] = step_sq;
      BKC_MARK(0, 6);
      if (kstep == 2) ++n2x2;
    } else {
      // ---- 3B. row kp refill W[kp, kk+1:kp] <- W[kk+1:kp, kk], W[kp, kp] <-
      //          W[kk, kk] (entry k0 left to the pivot warp); D of row kk
      if (kp != kk) {
        if (kp % CS == rank)
          for (int j = kk + 1 + bt; j <= kp; j += NBT)
            if (j != k0) L(kp, j) = j < kp ? cK[j] : cK[kk];
        if (kk % CS == rank && bt == 0) {
          L(kk, kk) = cC[kp];                      // W[kk, kk] <- W[kp, kp]
          if (kstep == 2) L(kk, k) = cA[kp];       // W[k+1, k] <- W[kp, k]
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
      asm volatile("bar.sync 1, %0;\n" ::"n"(BKC_NT) : "memory");     // swapped rows + multipliers
#pragma unroll
      for (int t = 0; t < BKC_JPT; ++t) {
        const int j = k0 + bt + t * NBT;
        if (j < n && j % CS == rank) {
          L(j, k) = lc0[t];
          if (kstep == 2) L(j, k + 1) = lc1[t];
        }
      }
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
    // stopped at the top of step s: step s-1's maximum is in rst, not pushed
    if (s >= 1) {
      if (tid == 0) mbar_arm(&mbarR, CS * slot_bytes(track));
      if (pw) {
        const double up = warp_max(lane < NW ? rst[(s - 1) & 1][lane] : 0.0);
        xpost<CS>(inboxR, rank, xslot(-1.0, -1.0, up, 0x7fffffff), &mbarR, track);
      }
      mbar_wait(&mbarR, rphase & 1u);
      const XSlot mf = xmerge<CS>(inboxR, &xmerged);
      if (gthread) {
        if (s >= 2) grow(pend_usq, ks2, k02);
        grow(mf.aux, ks1, k01);
      }
    }
  } else {
    // ran to the end: the last step's push carried step s-2's maximum
    if (tid == 0) mbar_arm(&mbar[s % 3], (unsigned)(n - k) * 16u + CS * slot_bytes(track));
    mbar_wait(&mbar[s % 3], (unsigned)(s / 3) & 1u);
    const XSlot mf = xmerge<CS>(inbox[s % 3], &xmerged);
    if (gthread && s >= 2) grow(mf.aux, ks2, k02);
  }
#ifdef D3M_BK_PROFILE
  const long long t_loop1 = clock64();
#endif
  // ---- write back: diagonal / D entries and the trailing part in place; the
  //      L entries of the columns of step t move by the interchanges of the
  //      steps after t (kernels.py:96-98), applied here in reverse order ------
  for (int i = tid; i < n; i += BKC_NT) qmap[i] = (short)i;
  __syncthreads();
  const int kend = info >= 0 ? k : n;                 // columns >= kend: unfactored trailing part
  for (int q = warp; q < nown; q += NW) {
    const int i = rank + q * CS;
    const cplx* src = Rl + bkc_off<CS>(i);
    cplx* row = W + (int64_t)i * lda;
    for (int j = kend + lane; j <= i; j += 32) row[j] = src[j];
  }
  for (int t = s - 1; t >= 0; --t) {
    const int kt = stk[3 * t], kst = stk[3 * t + 1], kpt = stk[3 * t + 2];
    // columns kt (and kt+1) of step t: D entries in place, L entries (rows
    // >= kt + kst) to row qmap[i] (= their row after the interchanges of t+1..)
    const int q0 = first_q(kt);
    for (int e = tid; e < (nown - q0) * kst; e += BKC_NT) {
      const int i = rank + (q0 + e / kst) * CS, c = kt + e % kst;
      if (c > i) continue;
      const int dst = i >= kt + kst ? qmap[i] : i;
      W[(int64_t)dst * lda + c] = Rl[bkc_off<CS>(i) + c];
    }
    if (kpt >= 0) {                                   // qmap <- qmap o tau_t
      __syncthreads();
      if (tid == 0) {
        const int kkt = kt + kst - 1;
        const short t0 = qmap[kkt];
        qmap[kkt] = qmap[kpt];
        qmap[kpt] = t0;
      }
      __syncthreads();
    }
  }
  if (rank == 0)
    for (int i = tid; i < n; i += BKC_NT) {
      a.perm[(int64_t)b * n + i] = (int64_t)perm_s[i];
      a.tags[(int64_t)b * n + i] = tags_s[i];
    }
  if (lead) {
    a.n2x2[b] = n2x2;
    a.info[b] = info;
    if (track) { a.margin[2 * b] = mdec; a.margin[2 * b + 1] = mgap; }
  }
  if (rank == 0 && gthread) a.growth[b] = growth;
#ifdef D3M_BK_PROFILE
  if (rank == 0 && (tid == 0 || tid == 32)) {
    double* prof = g_bkc_prof;
#pragma unroll
    for (int i = 0; i < 8; ++i) prof[(tid == 0 ? 0 : 8) + i] = pacc[(tid == 0 ? 0 : 8) + i];
    if (tid == 0) {   // prologue, step loop, write-back (cycles)
      const long long t_end = clock64();
      prof[16] = (double)(t_loop0 - t_entry);
      prof[17] = (double)(t_loop1 - t_loop0);
      prof[18] = (double)(t_end - t_loop1);
      prof[19] = pacc[13];     // steps with the rowmax exchange
      prof[20] = pacc[14];     // steps with an interchange
      prof[21] = pacc[15];     // 2x2 pivots
      prof[22] = (double)s;    // steps
      prof[23] = pacc[12];     // decide + rowmax + interchange cycles of the rowmax steps
    }
  }
#endif
  cl.sync();     // no CTA exits while a peer may still push into its shared memory
}

template <int CS>
static size_t bkc_smem_bytes(int n) {
  // own rows + ls, ws (2n) + broadcast vectors (7n) complex; perm, row map
  // (int16), step records (3 x int16), tags (int8): 11n bytes
  return sizeof(cplx) * (size_t)(bkc_entries<CS>(n) + 9 * (int64_t)n) + 11 * (size_t)n + 16;
}
constexpr size_t kBkcSmemMax = 220 * 1024;

template <int CS>
static bool bkc_fits(int n) { return bkc_smem_bytes<CS>(n) <= kBkcSmemMax && n <= BKC_JPT * (BKC_NT - 32); }

template <int CS, bool TRACK>
static int bkc_launch_t(BkArgs* a, int batch, cudaStream_t s) {
  const size_t smem = bkc_smem_bytes<CS>(a->n);
  if (!bkc_fits<CS>(a->n)) return -22;   // the CTA owns its SM
  cudaFuncSetAttribute(bk_cluster_kernel<CS, TRACK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (CS == 16) {
    // 16 is a non-portable cluster size: check once per device that a
    // cluster of full-SM CTAs can be resident on this part
    static PerDeviceOnce checked;
    static std::atomic<unsigned long long> yes16{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (checked.first()) {
      cudaFuncSetAttribute(bk_cluster_kernel<CS, TRACK>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(bk_cluster_kernel<CS, TRACK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kBkcSmemMax);
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 16;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(BKC_NT);
      cfg.dynamicSmemBytes = kBkcSmemMax;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, bk_cluster_kernel<CS, TRACK>, &cfg) == cudaSuccess &&
          nclusters > 0)
        yes16.fetch_or(1ull << (dev & 63));
      cudaGetLastError();
      cudaFuncSetAttribute(bk_cluster_kernel<CS, TRACK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    if (!(yes16.load() & (1ull << (dev & 63)))) return -22;
  }
  bk_cluster_kernel<CS, TRACK><<<batch * CS, BKC_NT, smem, s>>>(*a);
  return (int)cudaGetLastError();
}

template <int CS>
static int bkc_launch(BkArgs* a, int batch, cudaStream_t s) {
  return a->margin ? bkc_launch_t<CS, true>(a, batch, s) : bkc_launch_t<CS, false>(a, batch, s);
}

}  // namespace d3m

// Bit-exact BK of `batch` blocks, one cluster each.  Returns -22 when the
// block does not fit the cluster's shared memory (caller falls back).
extern "C" int d3m_bk_cluster_launch_cs(d3m::BkArgs* a, int batch, int cs, void* stream);

extern "C" int d3m_bk_cluster_launch(d3m::BkArgs* a, int batch, void* stream) {
  return d3m_bk_cluster_launch_cs(a, batch, 0, stream);
}

// cs: cluster size (2, 4, 8 or 16); 0 = D3M_BKC_CS or 8.  A block that does
// not fit the requested size's shared memory moves to the next larger
// cluster (8, then 16); -22 when it fits none.
extern "C" int d3m_bk_cluster_launch_cs(d3m::BkArgs* a, int batch, int cs, void* stream) {
  using namespace d3m;
  if (batch <= 0 || a->n <= 0) return 0;
  if (cs == 0) {
    cs = 8;
    if (const char* env = getenv("D3M_BKC_CS")) cs = atoi(env);
  }
  auto s = reinterpret_cast<cudaStream_t>(stream);
  int rc = -22;
  switch (cs) {
    case 2: rc = bkc_launch<2>(a, batch, s); break;
    case 4: rc = bkc_launch<4>(a, batch, s); break;
    case 16: return bkc_launch<16>(a, batch, s);
    default: break;
  }
  if (rc == -22) rc = bkc_launch<8>(a, batch, s);
  return rc == -22 ? bkc_launch<16>(a, batch, s) : rc;
}

// largest n the cluster kernel holds at cluster size cs (0: the largest of any size)
extern "C" int d3m_bk_cluster_max_n(int cs) {
  using namespace d3m;
  int best = 0;
  for (int n = 1; n <= BKC_JPT * (BKC_NT - 32); ++n) {
    const bool f = cs == 2 ? bkc_fits<2>(n) : cs == 4 ? bkc_fits<4>(n) : cs == 8 ? bkc_fits<8>(n)
                 : cs == 16 ? bkc_fits<16>(n) : (bkc_fits<8>(n) || bkc_fits<16>(n));
    if (f) best = n;
  }
  return best;
}

#ifdef D3M_BK_PROFILE
// profiling builds (-DD3M_BK_PROFILE, tools/bkc_profile.sh): the phase clocks of the last cluster BK
extern "C" int d3m_bkc_prof_read(double* host32) {
  return (int)cudaMemcpyFromSymbol(host32, d3m::g_bkc_prof, sizeof(double) * 32);
}
#endif
