// skinny_dmma.cu -- tall-skinny complex GEMM on the FP64 tensor pipe for the
// block substitutions (block_solve, factor.py:271-310) with few RHS.
//
//   C[cmap(r)][c]  op=  sum_k A(r, k) B[bmap(k)][c]      r < M, c < N <= 16 per pass
//
// A(r, k) = A[r*lda + k] (TA = 0: z = Binv b, b_i -= L_ij z) or A[k*lda + r]
// (TA = 1: L_ij^T x_i, Binv^T w).  With 16 RHS every factor entry feeds 16
// complex FMAs (8 flop/B), which the FP64 CUDA-core pipe cannot sustain at
// HBM speed; DMMA m8n8k4 takes 16 RHS as exactly two n-tiles.
//
// CTA tile 16 rows x 16 RHS; its 4 warps split K (64-row slices, each warp
// its own 4-deep cp.async ring, 2 x 2 DMMA sub-tiles with (re, im)
// accumulators) and add their sums in warp order at the end: the dependent
// chain per warp is 4x shorter than one warp walking all of K, and small
// products get 4x more CTAs (8 warps of 32-row slices, one CTA per SM for
// the shared memory, made the dataflow solve 16% slower: fewer items in
// flight for the bulk updates).  gridDim.y > 1 splits K into chunks of kchunk rows; each chunk writes
// its partial sums (no atomics) for an ordered reduction afterwards.  The
// summation order of an output entry depends only on K and the chunking, so a
// k-RHS solve equals k single-RHS solves bit for bit.
#include <algorithm>
#include <cooperative_groups.h>
#include "d3m_common.cuh"
#include "d3m_kernels.h"
#include "../../include/d3m.h"

namespace d3m {

constexpr int SN_BM = 16, SN_BN = 16, SN_BK = 8, SN_ST = 3, SN_PA = SN_BK + 4, SN_PB = SN_BN + 2, SN_NT = 128;
constexpr int SN_NW = SN_NT / 32;
constexpr int SN_KW = 64;                  // K rows per warp and CTA pass (a CTA covers 256 K rows)

struct SnWarpSmem {                        // one warp's private staging ring
  cplx A[SN_ST][SN_BM][SN_PA];
  cplx B[SN_ST][SN_BK][SN_PB];
};
constexpr size_t kSnSmem = sizeof(SnWarpSmem) * SN_NW;

__device__ __forceinline__ void sn_cp16(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void sn_dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// one warp stages A(16 rows x 8 k) and B(8 k x 16 RHS): 4 + 4 chunks per lane
template <bool TA>
__device__ __forceinline__ void sn_load_a(SnWarpSmem& S, int st, const cplx* A, int lda, int M, int m0, int k0,
                                          int kend, int lane) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int e = p * 32 + lane;
    int r, k;
    if (!TA) { r = e >> 3; k = e & 7; }      // 8 lanes per 128-byte row segment
    else { r = e & 15; k = e >> 4; }         // 16 lanes per 256-byte stored row
    const bool ok = (m0 + r < M) && (k0 + k < kend);
    const cplx* g = TA ? A + (int64_t)(k0 + k) * lda + m0 + r : A + (int64_t)(m0 + r) * lda + k0 + k;
    sn_cp16(&S.A[st][r][k], ok ? g : A, ok);
  }
}
__device__ __forceinline__ void sn_load_b(SnWarpSmem& S, int st, const cplx* B, int ldb, const int64_t* bmap, int N,
                                          int k0, int kend, int lane) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int e = p * 32 + lane, k = e >> 4, c = e & 15;
    const bool ok = (k0 + k < kend) && (c < N);
    const int64_t row = bmap ? bmap[ok ? k0 + k : 0] : (int64_t)(k0 + k);
    sn_cp16(&S.B[st][k][c], ok ? B + row * ldb + c : B, ok);
  }
}
template <bool TA>
__device__ __forceinline__ void sn_load(SnWarpSmem& S, int st, const cplx* A, int lda, int M, const cplx* B, int ldb,
                                        const int64_t* bmap, int N, int m0, int k0, int kend, int lane) {
  sn_load_a<TA>(S, st, A, lda, M, m0, k0, kend, lane);
  sn_load_b(S, st, B, ldb, bmap, N, k0, kend, lane);
}

struct SnNoWait {
  __device__ void operator()() const {}
};

// mode: 0 store, 1 subtract, 2 partial (part[(chunk * M + r) * N + c])
// CTA: 16 rows x 16 RHS over K rows [kbeg, kbeg + 256 * passes) of its chunk;
// warp w takes the 64-row slices w, w + 4, ...; the four warp sums are added
// in warp order at the end (fixed order, independent of N).
// One CTA tile (rows [m0, m0+16), K rows [kbeg, kend) of chunk `chunk`);
// shared by the per-product kernel below and the persistent block solve.
// `wait` runs between the prefetch of the first stages' A (factor data, never
// produced in-kernel) and the loads of B (the vectors another CTA may still
// be producing): the dataflow solve waits for its inputs there, so the A
// latency overlaps the dependency wait.  It is called by every thread.
template <bool TA, class W = SnNoWait>
__device__ __forceinline__ void sn_tile(const cplx* __restrict__ A, int lda, int M, const cplx* __restrict__ B,
                                        int ldb, const int64_t* __restrict__ bmap, int N, cplx* C, int ldc,
                                        const int64_t* __restrict__ cmap, int mode, int m0, int chunk, int kbeg,
                                        int kend, unsigned char* sn_smem, W wait = W()) {
  SnWarpSmem* ws = reinterpret_cast<SnWarpSmem*>(sn_smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  SnWarpSmem& S = ws[warp];
  double acc_re[2][2][2], acc_im[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc_re[i][j][0] = acc_re[i][j][1] = acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
  // this warp's k-tiles: slices of SN_KW rows, strided by SN_NW slices
  const int tiles_per_slice = SN_KW / SN_BK;
  const int nslice = (kend - kbeg + SN_KW - 1) / SN_KW;
  const int my_slices = nslice > warp ? (nslice - warp + SN_NW - 1) / SN_NW : 0;
  const int ktiles = my_slices * tiles_per_slice;
  auto tile_k0 = [&](int t) { return kbeg + ((t / tiles_per_slice) * SN_NW + warp) * SN_KW + (t % tiles_per_slice) * SN_BK; };
  // A of stages 0..ST-2 as one group, then B of each stage as its own group:
  // with ST-2 groups in flight the main loop's waits see A_s and B_s landed
#pragma unroll
  for (int s = 0; s < SN_ST - 1; ++s)
    if (s < ktiles) sn_load_a<TA>(S, s, A, lda, M, m0, tile_k0(s), kend, lane);
  asm volatile("cp.async.commit_group;\n" ::);
  wait();
#pragma unroll
  for (int s = 0; s < SN_ST - 1; ++s) {
    if (s < ktiles) sn_load_b(S, s, B, ldb, bmap, N, tile_k0(s), kend, lane);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(SN_ST - 2));
    __syncwarp();
    const int nk = kt + SN_ST - 1;
    if (nk < ktiles) sn_load<TA>(S, nk % SN_ST, A, lda, M, B, ldb, bmap, N, m0, tile_k0(nk), kend, lane);
    asm volatile("cp.async.commit_group;\n" ::);
    const int st = kt % SN_ST;
#pragma unroll
    for (int kk = 0; kk < SN_BK / 4; ++kk) {
      double are[2], aim[2], anim[2], bre[2], bim[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const cplx a = S.A[st][i * 8 + fr][kk * 4 + fc];
        are[i] = a.x;
        aim[i] = a.y;
        anim[i] = -a.y;
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const cplx b = S.B[st][kk * 4 + fc][j * 8 + fr];
        bre[j] = b.x;
        bim[j] = b.y;
      }
      // four passes over all sub-tiles: dependent DMMAs on one accumulator are
      // 8 instructions apart (per-accumulator order unchanged: bitwise same)
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) sn_dmma(acc_re[i][j][0], acc_re[i][j][1], are[i], bre[j]);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) sn_dmma(acc_im[i][j][0], acc_im[i][j][1], are[i], bim[j]);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) sn_dmma(acc_re[i][j][0], acc_re[i][j][1], anim[i], bim[j]);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) sn_dmma(acc_im[i][j][0], acc_im[i][j][1], aim[i], bre[j]);
    }
    __syncwarp();
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  // cross-warp sum in warp order through the (now idle) staging memory
  cplx (*red)[SN_BM][SN_BN] = reinterpret_cast<cplx (*)[SN_BM][SN_BN]>(sn_smem);
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) red[warp][i * 8 + fr][j * 8 + fc * 2 + h] = mk(acc_re[i][j][h], acc_im[i][j][h]);
  __syncthreads();
  for (int e = threadIdx.x; e < SN_BM * SN_BN; e += SN_NT) {
    const int rr = e >> 4, c = e & 15, r = m0 + rr;
    if (r >= M || c >= N) continue;
    cplx v = red[0][rr][c];
#pragma unroll
    for (int w = 1; w < SN_NW; ++w) v = c_add(v, red[w][rr][c]);
    if (mode == 2) {
      C[((int64_t)chunk * M + r) * N + c] = v;
    } else {
      cplx* p = C + (cmap ? cmap[r] : (int64_t)r) * ldc + c;
      *p = mode == 1 ? c_sub(*p, v) : v;
    }
  }
  __syncthreads();                 // the staging memory is reused by the next tile
}

template <bool TA>
__global__ void __launch_bounds__(SN_NT)
skinny_dmma_kernel(const cplx* __restrict__ A, int lda, int M, int K, const cplx* __restrict__ B, int ldb,
                   const int64_t* __restrict__ bmap, int N, cplx* C, int ldc, const int64_t* __restrict__ cmap,
                   int mode, int kchunk) {
  extern __shared__ __align__(128) unsigned char sn_smem[];
  const int chunk = blockIdx.y;
  const int kbeg = chunk * kchunk;
  sn_tile<TA>(A, lda, M, B, ldb, bmap, N, C, ldc, cmap, mode, blockIdx.x * SN_BM, chunk, kbeg, min(K, kbeg + kchunk),
              sn_smem);
}

// out[r * ldo + c] = (base ? base[r * ldb + c] : 0) + sign * sum_{ch < nch} part[(ch * M + r) * np + c]
// (chunks summed in ascending order), r < M, c < np
__global__ void skinny_reduce_kernel(const cplx* base, int ldb, const cplx* part, int nch, int M, int np,
                                     double sign, cplx* out, int ldo) {
  const int64_t len = (int64_t)M * np;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / np), c = (int)(e % np);
    cplx acc = mk(0.0, 0.0);
    for (int ch = 0; ch < nch; ++ch) acc = c_add(acc, part[(int64_t)ch * len + e]);
    const cplx b = base ? base[(int64_t)r * ldb + c] : mk(0.0, 0.0);
    out[(int64_t)r * ldo + c] = mk(b.x + sign * acc.x, b.y + sign * acc.y);
  }
}

// ---- persistent block substitution (block_solve, factor.py:271-310) ------
// One cooperative launch runs both sweeps for <= 16 RHS: the same products as
// the per-product launches (sn_tile, same tiles and summation order, so the
// results are bitwise those of the launch sequence) separated by grid-wide
// barriers instead of kernel boundaries (864 launches of ~14 us latency each
// on config 4).
__global__ void __launch_bounds__(SN_NT, 2) block_solve_persistent(SolvePlanDev p) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char sn_smem[];
  const int G = gridDim.x, cta = blockIdx.x;
  const int N = p.N, ld = p.ldn;
  constexpr int KCH = 256;
  // forward: z = Binv_j b_j; u_j = D_j^-1 z; b_i -= L_ij z
  for (int j = 0; j < p.nb; ++j) {
    const int nj = (int)p.sizes[j];
    if (nj == 0) continue;
    const int R = (int)p.panel_rows[j];
    cplx* bj = p.b + p.row_off[j] * ld + p.c0;
    for (int t = cta; t * SN_BM < nj; t += G)
      sn_tile<false>(p.binv + p.binv_off[j], nj, nj, bj, ld, nullptr, N, p.tmp, N, nullptr, 0, t * SN_BM, 0, 0, nj,
                     sn_smem);
    grid.sync();
    {
      const cplx* F = p.pool + p.diag_off[j];
      const int8_t* tg = p.tags + p.piv_off[j];
      cplx* uj = p.u + p.row_off[j] * ld + p.c0;
      for (int e = cta * SN_NT + threadIdx.x; e < nj * N; e += G * SN_NT) {     // dinv_left_copy
        const int c = e / N, col = e - c * N;
        const int8_t t = tg[c];
        if (t == 1) {
          uj[(int64_t)c * ld + col] = x_div_np(p.tmp[e], F[(int64_t)c * nj + c]);
        } else if (t == 2) {
          cplx x0 = p.tmp[e], x1 = p.tmp[e + N];
          dinv_pair(F[(int64_t)c * nj + c], F[(int64_t)(c + 1) * nj + c], F[(int64_t)(c + 1) * nj + c + 1], x0, x1);
          uj[(int64_t)c * ld + col] = x0;
          uj[(int64_t)(c + 1) * ld + col] = x1;
        }
      }
    }
    for (int t = cta; t * SN_BM < R; t += G)
      sn_tile<false>(p.pool + p.panel_off[j], nj, R, p.tmp, N, nullptr, N, p.b + p.c0, ld, p.gidx + p.gptr[j], 1,
                     t * SN_BM, 0, 0, nj, sn_smem);
    grid.sync();
  }
  // backward: w = u_j - sum_i L_ij^T x_i (split-K partials, ordered reduce); x_j = Binv_j^T w
  for (int j = p.nb - 1; j >= 0; --j) {
    const int nj = (int)p.sizes[j];
    if (nj == 0) continue;
    const int R = (int)p.panel_rows[j];
    const int nch = R > 0 ? (R + KCH - 1) / KCH : 0;
    const int mt = (nj + SN_BM - 1) / SN_BM;
    if (nch > 0) {
      for (int t = cta; t < mt * nch; t += G) {
        const int ch = t / mt, m0 = (t - ch * mt) * SN_BM;
        sn_tile<true>(p.pool + p.panel_off[j], nj, nj, p.x + p.c0, ld, p.gidx + p.gptr[j], N, p.part, N, nullptr, 2,
                      m0, ch, ch * KCH, min(R, ch * KCH + KCH), sn_smem);
      }
      grid.sync();
    }
    const cplx* uj = p.u + p.row_off[j] * ld + p.c0;
    const int64_t len = (int64_t)nj * N;
    for (int64_t e = cta * SN_NT + threadIdx.x; e < len; e += (int64_t)G * SN_NT) {   // skinny_reduce
      const int r = (int)(e / N), c = (int)(e % N);
      cplx acc = mk(0.0, 0.0);
      for (int ch = 0; ch < nch; ++ch) acc = c_add(acc, p.part[(int64_t)ch * len + e]);
      const cplx bb = uj[(int64_t)r * ld + c];
      p.tmp[(int64_t)r * N + c] = mk(bb.x + -1.0 * acc.x, bb.y + -1.0 * acc.y);
    }
    grid.sync();
    for (int t = cta; t * SN_BM < nj; t += G)
      sn_tile<true>(p.binv + p.binv_off[j], nj, nj, p.tmp, N, nullptr, N, p.x + p.row_off[j] * ld + p.c0, ld, nullptr,
                    0, t * SN_BM, 0, 0, nj, sn_smem);
    grid.sync();
  }
}

// ---- dataflow block substitution ---------------------------------------------
// The grid-barrier kernel above runs 720 dependent phases on config 4 (~13 us
// each: 9.3 ms against a 1.4 ms HBM floor; ncu: 43% of the stall samples at
// the grid barrier).  Here the same tiles (same rows, K ranges, split-K and
// summation order, so the results are bitwise those of the barrier kernel)
// are work items of a host-built list (factor.py _solve_flow), taken from a
// global atomic queue by the resident CTAs.  Each item names the counters
// it waits for (>= target) and the counters it increments when done, so only
// true dependencies serialise:
//   FA(j,t)  z_j rows [16t,16t+16) = Binv_j b_j        waits: all updates into b_j
//   FD(j)    u_j = D_j^-1 z_j                           waits: z_j
//   FB(j,r)  b[gidx] -= L_panel(j)[rows r..r+16) z_j    waits: z_j, the previous
//            update of the same 16 rows (per-tile sequence: ascending j, as the
//            phases of the barrier kernel)
//   BC(j,ch,mt)  split-K partial of L_ij^T x_i (chunk ch, 16 rows mt)
//                                                       waits: x_i of the chunk's blocks
//   BR(j,r0,r1)  w_j = u_j - sum_ch partials (ascending ch), in place in u
//                                                       waits: all partials of j, u_j
//   BE(j,t)  x_j rows [16t,16t+16) = Binv_j^T w_j       waits: w_j
// z_j lives in the x rows of block j until BE(j) overwrites them (every reader
// of z_j precedes BE(j) in the dependency order).  The list is a topological
// order, so the smallest unfinished item always has its inputs: with every
// CTA resident (cooperative launch) the queue cannot deadlock.  Waits are
// bounded (a lost dependency traps instead of hanging the GPU).
struct FlowItem {
  int type, j, p0, p1, dep_off, dep_cnt, inc0, inc1;
};
enum { kFA = 0, kFD = 1, kFB = 2, kBC = 3, kBR = 4, kBE = 5 };

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
  return t;
}

// Two queues: the chain items (items[0, nchain): z_j, the parent block's
// update, the parent chunk's partials, the reduce and x_j -- the critical
// path of both sweeps) go to the "chain" CTAs, one per SM on the first
// chain_sms SMs to arrive (the other CTA of such an SM exits), so they never
// share an SM's DMMA pipe; every other CTA takes the rest, items[nchain,
// nitems).  Each list is a subsequence of one topological order, so the
// smallest unfinished item is always held by a CTA of its class that can
// run it: no deadlock.  sched: [0] chain head, [1] bulk head, [2] chain CTA
// count, [4, 4 + kFlowSms) SM tickets, [4 + kFlowSms, 4 + 2 kFlowSms) SM roles.
constexpr int kFlowSms = 1024;

__global__ void __launch_bounds__(SN_NT, 3)
block_solve_dataflow(SolvePlanDev p, const FlowItem* __restrict__ items, int nitems, int nchain, int chain_sms,
                     const int2* __restrict__ deps, const int64_t* __restrict__ part_off, int* cnt, int* sched,
                     long long* trace) {
  extern __shared__ __align__(128) unsigned char sn_smem[];
  __shared__ int s_idx, s_role;
  const int N = p.N, ld = p.ldn;
  constexpr int KCH = 256;
  __shared__ int s_next;
  if (threadIdx.x == 0) {
    int role = 0;                                    // 0 rest, 1 chain, 2 exit
    if (nchain > 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;\n" : "=r"(smid));
      smid &= kFlowSms - 1;
      int* role_of = sched + 4 + kFlowSms;
      if (atomicAdd(sched + 4 + smid, 1) == 0) {
        role = atomicAdd(sched + 2, 1) < chain_sms ? 1 : 0;
        atomicExch(role_of + smid, role + 1);
      } else {
        int r;
        for (unsigned spin = 0; (r = ld_acquire(role_of + smid)) == 0; ++spin)
          if (spin > (1u << 26)) __trap();
        role = r == 2 ? 2 : 0;
      }
    }
    s_role = role;
  }
  __syncthreads();
  if (s_role == 2) return;
  const bool chain = s_role == 1;
  const int q0 = chain ? 0 : nchain;
  const int qn = chain ? nchain : nitems;
  int* next = sched + (chain ? 0 : 1);
  if (threadIdx.x == 0) s_next = q0 + atomicAdd(next, 1);
  for (;;) {
    // the queue index of the item after this one is taken while this one runs
    if (threadIdx.x == 0) {
      s_idx = s_next;
      if (s_idx < qn) s_next = q0 + atomicAdd(next, 1);
    }
    __syncthreads();
    const int idx = s_idx;
    if (idx >= qn) break;
    const FlowItem it = items[idx];
    if (trace && threadIdx.x == 0) trace[3 * (int64_t)idx] = gtimer();
    // inputs ready: thread 0 polls the item's counters, then a CTA barrier;
    // the tile items run it inside sn_tile, after their A prefetch
    auto waitdeps = [&]() {
      if (threadIdx.x == 0) {
        for (int d = 0; d < it.dep_cnt; ++d) {
          const int2 dp = deps[it.dep_off + d];
          for (unsigned spin = 0; ld_acquire(cnt + dp.x) < dp.y; ++spin) {
            if (spin > (1u << 28)) __trap();
            if (spin > 64) __nanosleep(32);
          }
        }
        if (trace) trace[3 * (int64_t)idx + 1] = gtimer();
      }
      __syncthreads();
    };
    const int j = it.j;
    const int nj = (int)p.sizes[j];
    const int64_t ro = p.row_off[j];
    switch (it.type) {
      case kFA:
        sn_tile<false>(p.binv + p.binv_off[j], nj, nj, p.b + ro * ld + p.c0, ld, nullptr, N, p.x + ro * ld + p.c0, ld,
                       nullptr, 0, it.p0 * SN_BM, 0, 0, nj, sn_smem, waitdeps);
        break;
      case kFD: {      // rows [p0, p1) (a 2x2 pair belongs to the piece of its first row)
        waitdeps();
        const cplx* F = p.pool + p.diag_off[j];
        const int8_t* tg = p.tags + p.piv_off[j];
        const cplx* z = p.x + ro * ld + p.c0;
        cplx* uj = p.u + ro * ld + p.c0;
        for (int e = it.p0 * N + threadIdx.x; e < it.p1 * N; e += SN_NT) {
          const int c = e / N, col = e - c * N;
          const int8_t t = tg[c];
          if (t == 1) {
            uj[(int64_t)c * ld + col] = x_div_np(__ldcg(z + (int64_t)c * ld + col), F[(int64_t)c * nj + c]);
          } else if (t == 2) {
            cplx x0 = __ldcg(z + (int64_t)c * ld + col), x1 = __ldcg(z + (int64_t)(c + 1) * ld + col);
            dinv_pair(F[(int64_t)c * nj + c], F[(int64_t)(c + 1) * nj + c], F[(int64_t)(c + 1) * nj + c + 1], x0, x1);
            uj[(int64_t)c * ld + col] = x0;
            uj[(int64_t)(c + 1) * ld + col] = x1;
          }
        }
        break;
      }
      case kFB:
        sn_tile<false>(p.pool + p.panel_off[j] + (int64_t)it.p0 * nj, nj, it.p1, p.x + ro * ld + p.c0, ld, nullptr, N,
                       p.b + p.c0, ld, p.gidx + p.gptr[j] + it.p0, 1, 0, 0, 0, nj, sn_smem, waitdeps);
        break;
      case kBC: {
        const int R = (int)p.panel_rows[j], ch = it.p0;
        sn_tile<true>(p.pool + p.panel_off[j], nj, nj, p.x + p.c0, ld, p.gidx + p.gptr[j], N, p.part + part_off[j], N,
                      nullptr, 2, it.p1 * SN_BM, ch, ch * KCH, min(R, ch * KCH + KCH), sn_smem, waitdeps);
        break;
      }
      case kBR: {      // rows [p0, p1); partials loaded 16 chunks ahead, summed in chunk order
        waitdeps();
        const int R = (int)p.panel_rows[j];
        const int nch = R > 0 ? (R + KCH - 1) / KCH : 0;
        const int64_t len = (int64_t)nj * N;
        const cplx* part = p.part + part_off[j];
        cplx* uj = p.u + ro * ld + p.c0;
        for (int e = it.p0 * N + threadIdx.x; e < it.p1 * N; e += SN_NT) {
          const int r = e / N, c = e - r * N;
          cplx acc = mk(0.0, 0.0);
          for (int c8 = 0; c8 < nch; c8 += 16) {
            cplx v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (c8 + q < nch) v[q] = __ldcg(part + (int64_t)(c8 + q) * len + e);
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (c8 + q < nch) acc = c_add(acc, v[q]);
          }
          const cplx bb = __ldcg(uj + (int64_t)r * ld + c);
          uj[(int64_t)r * ld + c] = mk(bb.x + -1.0 * acc.x, bb.y + -1.0 * acc.y);
        }
        break;
      }
      default:   // kBE
        sn_tile<true>(p.binv + p.binv_off[j], nj, nj, p.u + ro * ld + p.c0, ld, nullptr, N, p.x + ro * ld + p.c0, ld,
                      nullptr, 0, it.p0 * SN_BM, 0, 0, nj, sn_smem, waitdeps);
        break;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      if (it.inc0 >= 0) atomicAdd(cnt + it.inc0, 1);
      if (it.inc1 >= 0) atomicAdd(cnt + it.inc1, 1);
      if (trace) trace[3 * (int64_t)idx + 2] = gtimer();
    }
  }
}

}  // namespace d3m

static long long* g_flow_trace = nullptr;
static int g_flow_trace_n = 0;
// copy the last traced pass's stamps (3 per item) to host memory; returns the item count
extern "C" int d3m_flow_trace(void* host, int max_items) {
  if (!g_flow_trace) return 0;
  const int n = g_flow_trace_n < max_items ? g_flow_trace_n : max_items;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_flow_trace, sizeof(long long) * 3 * (size_t)n, cudaMemcpyDeviceToHost);
  return n;
}

// Dataflow block solve (one cooperative launch per pass of <= 16 RHS; the
// launcher zeroes `cnt` (ncounters ints, the last D3M_FLOW_EXTRA_COUNTERS
// the scheduler's) before each pass).  Returns -22 when the grid cannot be co-resident.
extern "C" int d3m_block_solve_flow_launch(void* plan, const void* items, int nitems, int nchain, const void* deps,
                                           const void* part_off, void* cnt, int ncounters, void* stream) {
  using namespace d3m;
  static int grid = -1;
  if (grid < 0) {
    cudaFuncSetAttribute(block_solve_dataflow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSnSmem);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, block_solve_dataflow, SN_NT, kSnSmem);
    grid = sms * std::min(per, 3);      // three CTAs per SM (two: +0.4-0.8 ms per pass)
    if (grid <= 0) grid = 0;
  }
  if (grid == 0) return -22;
  auto s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(int) * (size_t)ncounters, s);
  if (e != cudaSuccess) return (int)e;
  const SolvePlanDev* pl = static_cast<const SolvePlanDev*>(plan);
  const FlowItem* it = static_cast<const FlowItem*>(items);
  const int2* dp = static_cast<const int2*>(deps);
  const int64_t* po = static_cast<const int64_t*>(part_off);
  int* c = static_cast<int*>(cnt);
  int* sc = c + ncounters - D3M_FLOW_EXTRA_COUNTERS;          // scheduler scratch (see block_solve_dataflow)
  // D3M_FLOW_TRACE=1 (dev aid): per-item globaltimer stamps (taken, inputs
  // ready, done) of the last pass, read back by d3m_flow_trace
  static long long* trace = nullptr;
  static int64_t trace_cap = 0;
  static const char* tenv = getenv("D3M_FLOW_TRACE");
  long long* tr = nullptr;
  if (tenv && tenv[0] == '1') {
    if (trace_cap < 3 * (int64_t)nitems) {
      if (trace) cudaFree(trace);
      if (cudaMalloc(&trace, sizeof(long long) * 3 * (size_t)nitems) != cudaSuccess) return 2;
      trace_cap = 3 * (int64_t)nitems;
    }
    tr = trace;
    g_flow_trace = trace;
    g_flow_trace_n = nitems;
  }
  // chain SMs: 32.  A block column of config 4 puts 48 items on the chain
  // queue per sweep step (16 BC tiles, 16 BR pieces, 16 BE tiles).  With 24
  // chain CTAs the rotation has two stable phases, picked by the start-up
  // race: all 16 BC tiles held before x_{j+1} lands (5.97 ms per 16-RHS
  // pass), or 8 of them taken one round late (7.55 ms, about 40% of the
  // passes; tools/flow_modes.py, tools/solve_mode_probe.py).  32 chain CTAs
  // always hold the 16 BC tiles in time: 5.94-6.06 ms, every pass (16 SMs x
  // 2 CTAs: 6.03; 48: 6.19; 16 x 3: 6.21; 16 x 1: 7.24 ms).
  int csms = 32;
  void* args[] = {const_cast<SolvePlanDev*>(pl), &it, &nitems, &nchain, &csms, &dp, &po, &c, &sc, &tr};
  e = cudaLaunchCooperativeKernel((void*)block_solve_dataflow, dim3(grid), dim3(SN_NT), args, kSnSmem, s);
  return (int)e;
}

// Persistent block solve over device-resident plan arrays (SolvePlanDev
// pointers); one cooperative launch per pass of <= 16 RHS.  Returns -22 when
// the device cannot co-schedule the grid (the caller falls back).
extern "C" int d3m_block_solve_persistent_launch(void* plan, void* stream) {
  using namespace d3m;
  static int grid = -1;
  if (grid < 0) {
    cudaFuncSetAttribute(block_solve_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSnSmem);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, block_solve_persistent, SN_NT, kSnSmem);
    grid = sms * std::min(per, 2);
    if (grid <= 0) grid = 0;
  }
  if (grid == 0) return -22;
  void* args[] = {plan};
  const cudaError_t e = cudaLaunchCooperativeKernel((void*)block_solve_persistent, dim3(grid), dim3(SN_NT), args,
                                                    kSnSmem, reinterpret_cast<cudaStream_t>(stream));
  return (int)e;
}

extern "C" int d3m_skinny_reduce_launch(const void* base, int ldb, const void* part, int nch, int M, int np,
                                        double sign, void* out, int ldo, void* stream) {
  using namespace d3m;
  const int64_t len = (int64_t)M * np;
  if (len <= 0) return 0;
  const int threads = 128;
  const int blocks = (int)std::min<int64_t>((len + threads - 1) / threads, 1024);
  skinny_reduce_kernel<<<blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const cplx*>(base), ldb, static_cast<const cplx*>(part), nch, M, np, sign,
      static_cast<cplx*>(out), ldo);
  return (int)cudaGetLastError();
}

// One pass of <= 16 RHS.  kchunk > 0 with mode 2 splits K (partials of
// ceil(K / kchunk) chunks, M x N each, written to C); returns the chunk count.
extern "C" int d3m_skinny_launch(int ta, const void* A, int lda, int M, int K, const void* B, int ldb,
                                 const void* bmap, int N, void* C, int ldc, const void* cmap, int mode, int kchunk,
                                 void* stream) {
  using namespace d3m;
  if (M <= 0 || N <= 0 || N > SN_BN) return M <= 0 || N <= 0 ? 0 : -22;
  const int kc = kchunk > 0 ? kchunk : (K > 0 ? K : 1);
  const int nch = K > 0 ? (K + kc - 1) / kc : 1;
  const dim3 grid((M + SN_BM - 1) / SN_BM, nch);
  auto s = reinterpret_cast<cudaStream_t>(stream);
  auto a = static_cast<const cplx*>(A);
  auto b = static_cast<const cplx*>(B);
  auto c = static_cast<cplx*>(C);
  auto bm = static_cast<const int64_t*>(bmap);
  auto cm = static_cast<const int64_t*>(cmap);
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(skinny_dmma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSnSmem);
    cudaFuncSetAttribute(skinny_dmma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSnSmem);
    cfg = true;
  }
  if (ta) skinny_dmma_kernel<true><<<grid, SN_NT, kSnSmem, s>>>(a, lda, M, K, b, ldb, bm, N, c, ldc, cm, mode, kc);
  else skinny_dmma_kernel<false><<<grid, SN_NT, kSnSmem, s>>>(a, lda, M, K, b, ldb, bm, N, c, ldc, cm, mode, kc);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? nch : -(int)e;
}
