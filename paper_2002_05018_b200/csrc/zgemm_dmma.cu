// zgemm_dmma.cu -- grouped complex128 GEMM on the B200 FP64 tensor pipe.
//
//   C  op=  A_eff * B_eff^T        (A_eff: M x K, B_eff: N x K, C: M x N)
//
// with op one of  C -= AB (trailing Schur updates, factor.py:213-230),
// C = AB (Schur reduction D^T X, subdomain.py:181-183) or C += AB.
//
// B200 has no tcgen05 FP64 kind (ptxas rejects .kind::f64), so the tensor
// path is the warp-level DMMA: mma.sync.aligned.m8n8k4.f64 lowers to SASS
// DMMA.8x8x4 (36.9 TFLOP/s measured burst, profiles/fp64_peak_r01.txt).
// A complex product is four real DMMAs on the (re, im) planes:
//   acc_re += a_re b_re + (-a_im) b_im,   acc_im += a_re b_im + a_im b_re.
//
// Structure: CTA tile 64 x 64 complex, 4 warps (2 x 2), warp tile 32 x 32
// complex = 4 x 4 DMMA sub-tiles x (re, im) accumulators (128 registers).
// K is staged 8 complex per stage through a 4-deep cp.async (LDGSTS.128)
// ring in shared memory; complex values stay interleaved so one LDS.128
// returns (re, im) of a fragment element.  Row pitch 12 complex (192 B =
// 64 mod 128) makes every quarter-warp fragment load conflict-free.
//
// Scheduling: one CTA per output tile of a flat task list (grouped GEMM).
// Each task carries its own offsets/shape/leading dimensions and the prefix
// sum of tile counts; a CTA finds its task by binary search.  A task flagged
// SYM is a diagonal-block target of the block LDL^T: only lower tiles are
// computed and each lower value u_rc is subtracted at (r, c) and at (c, r),
// which is exactly the reference's tril(upd) + tril(upd, -1)^T rule
// (factor.py:217-220).
#include "d3m_common.cuh"
#include "d3m_gemm.h"
#include "d3m_kernels.h"
#include <algorithm>
#include <cstdlib>
#include <cuda.h>

namespace d3m {

constexpr int BM = 64, BN = 64, BKC = 8, STAGES = 4, PITCH = BKC + 4;
constexpr int NTHREADS = 128;
// k-major pitch of a transposed operand's stage slice: 66 = 2 mod 8, so a quarter warp's fragment
// LDS.128 (4 k-rows x 2 consecutive elements) covers the eight 16-byte bank groups once
constexpr int TPITCH = BM + 2;
static_assert(BKC * TPITCH <= BM * PITCH, "a k-major slice fits the stage's operand slot");
// One ring stage: the A and B k-slices side by side, so a freed stage is one
// contiguous 24 KB block (the epilogue's C prefetch reuses freed stages).
struct GemmStage {
  cplx a[BM][PITCH];
  cplx b[BN][PITCH];
};
constexpr int CP_PITCH = BN + 1;     // odd pitch: conflict-free fragment reads of C
constexpr int CP_ROWS = 22;          // C rows per freed stage (even: row pairs never straddle)
static_assert(CP_ROWS * CP_PITCH <= (int)(sizeof(GemmStage) / sizeof(cplx)), "C chunk exceeds a stage");
static_assert(3 * CP_ROWS >= BM && STAGES == 4, "three freed stages hold the C tile");

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// CTA-scope mbarriers for the 3M kernel's ring (no CTA-wide barrier per k-slice)
__device__ __forceinline__ unsigned smaddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smaddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smaddr(b)) : "memory");
}
// arrives once this thread's earlier cp.async copies have landed (count pre-set by mb_init)
__device__ __forceinline__ void mb_cp_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smaddr(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned parity) {
  for (unsigned it = 0;; ++it) {
    unsigned ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(smaddr(b)), "r"(parity) : "memory");
    if (ok) return;
    if (it > (1u << 28)) __trap();
  }
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Stage loader: tile rows [r0, r0+64) x k-columns [k0, k0+8) of an operand
// whose element (r, k) lives at  P[r*ld + k]  (TRANS=false) or P[k*ld + r].
// NT threads (128 or 256) cover the 512 16-byte elements of a stage slice.
template <bool TRANS, int NT = NTHREADS>
__device__ __forceinline__ void load_tile(cplx (*S)[PITCH], const cplx* P, int ld, int r0, int rows,
                                          int k0, int kdim, const int64_t* gcol = nullptr) {
  const int t = threadIdx.x;
  if (!TRANS) {
    // 8 threads cover one 128-byte row segment; NT/8 rows per pass (gcol: column gather)
    const int kq = t & 7;
    const int64_t col = (k0 + kq < kdim) ? (gcol ? gcol[k0 + kq] : (int64_t)(k0 + kq)) : 0;
#pragma unroll
    for (int p = 0; p < 512 / NT; ++p) {
      const int r = p * (NT / 8) + (t >> 3), k = kq;
      const bool ok = (r0 + r < rows) && (k0 + k < kdim);
      const cplx* g = ok ? P + (int64_t)(r0 + r) * ld + col : P;
      cp_async16(&S[r][k], g, ok);
    }
  } else {
    // 64 threads cover one contiguous 1 KB row of the stored operand, and the stage keeps it k-major
    // (St[k][r], pitch TPITCH): the 64 threads' 16-byte shared-memory writes are contiguous.  (Written
    // as S[r][k] at the 192-byte row pitch they fell into two bank groups -- a 16-way conflict per
    // warp, which bound the transposed launches of the subdomain solves.)
    cplx* St = &S[0][0];
#pragma unroll
    for (int p = 0; p < 512 / NT; ++p) {
      const int r = t & 63, k = p * (NT / 64) + (t >> 6);
      const bool ok = (r0 + r < rows) && (k0 + k < kdim);
      const cplx* g = ok ? P + (int64_t)(k0 + k) * ld + (r0 + r) : P;
      cp_async16(St + k * TPITCH + r, g, ok);
    }
  }
}

// Task of a tile: the last task whose tile_start <= tile, by a 32-ary search
// of warp 0 (one dependent load per round: 2 rounds for ~1000 tasks, against
// ~10 for a binary search), broadcast through shared memory.
__device__ __forceinline__ int find_task(const GemmTask* __restrict__ tasks, int ntasks, int tile) {
  __shared__ int s_task;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int lo = 0, hi = ntasks;               // answer in [lo, hi); tasks[0].tile_start == 0 <= tile
    while (hi - lo > 1) {
      const int step = (hi - lo + 31) >> 5;
      const int idx = lo + lane * step;
      const bool ok = idx < hi && tasks[idx].tile_start <= tile;
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      lo += (31 - __clz(m)) * step;
      hi = min(hi, lo + step);
    }
    if (lane == 0) s_task = lo;
  }
  __syncthreads();
  return s_task;
}

// G3 selects the complex product.  G3 = false: four real DMMAs per complex
// product (4M), 128 threads, 32 x 32 complex warp tiles.  G3 = true: Gauss's
// three-multiplication form (3M),
//   P = A_re B_re,  Q = A_im B_im,  R = (A_re + A_im)(B_re + B_im),
//   re = P - Q,     im = R - P - Q,
// 25% fewer DMMAs; its three accumulators need 48 doubles per 32 x 16 warp
// tile, so the CTA runs 8 warps (2 x 4) and stays at two CTAs per SM.  The
// operand sums are formed in registers from the staged (re, im) pairs.  3M
// is normwise stable (each entry's error is bounded by eps times
// (|a_re|+|a_im|)(|b_re|+|b_im|) summed over k, against the 4M product's
// eps |a||b|), so the results stay within rounding of the reference's ZGEMM.
template <bool TA, bool TB, bool G3, bool MB = false>
__global__ void __launch_bounds__(G3 ? 2 * NTHREADS : NTHREADS, 2)
zgemm_grouped_kernel(const cplx* __restrict__ Abase, const cplx* __restrict__ Bbase, cplx* Cbase,
                     const GemmTask* __restrict__ tasks, int ntasks, unsigned long long* tmax,
                     const int64_t* __restrict__ gperm) {
  constexpr int NT = G3 ? 2 * NTHREADS : NTHREADS;
  constexpr int WJ = G3 ? 2 : 4;             // 8-column DMMA sub-tiles per warp tile
  extern __shared__ __align__(128) unsigned char smem_raw[];
  GemmStage* st = reinterpret_cast<GemmStage*>(smem_raw);

  // ---- locate the task and the tile --------------------------------------
  const int tile = blockIdx.x;
  const GemmTask tk = tasks[find_task(tasks, ntasks, tile)];
  int local = tile - tk.tile_start, tm, tn;
  if (tk.flags & kGemmSym) {
    tm = (int)((sqrt(8.0 * local + 1.0) - 1.0) * 0.5);
    while ((tm + 1) * (tm + 2) / 2 <= local) ++tm;
    while (tm * (tm + 1) / 2 > local) --tm;
    tn = local - tm * (tm + 1) / 2;
  } else {
    tm = local / tk.tiles_n;
    tn = local - tm * tk.tiles_n;
  }
  const cplx* A = Abase + tk.a_off;
  const cplx* B = Bbase + tk.b_off;
  cplx* C = Cbase + tk.c_off;
  const int M = tk.m, N = tk.n, K = tk.k;
  const int m0 = tm * BM, n0 = tn * BN;
  if (m0 >= M || n0 >= N) return;      // device-built tasks may shrink below their tile budget

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = G3 ? (warp >> 2) * 32 : (warp >> 1) * 32;
  const int wn = G3 ? (warp & 3) * 16 : (warp & 1) * 32;
  const int fr = lane >> 2, fc = lane & 3;

  // 4M: acc_re / acc_im.  3M: acc_re = P, acc_im = Q, acc_x = R until the epilogue.
  double acc_re[4][WJ][2], acc_im[4][WJ][2], acc_x[4][WJ][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < WJ; ++j)
      acc_re[i][j][0] = acc_re[i][j][1] = acc_im[i][j][0] = acc_im[i][j][1] = acc_x[i][j][0] =
          acc_x[i][j][1] = 0.0;

  // TriGather: gathered A columns, K cut at the end of the triangular B's
  // nonzero columns for this output column tile (the skipped products are
  // exact zeros: the sum is bitwise that of the full range)
  const bool trig = (tk.flags & kGemmTriGather) != 0 && gperm != nullptr;
  const int64_t* gcol = trig ? gperm + tk.pad_ : nullptr;
  const int Keff = trig ? min(K, n0 + BN) : K;
  const int ktiles = (Keff + BKC - 1) / BKC;
  // MB: the ring is tracked by mbarriers -- full[s] completes when every
  // thread's copies of the stage in slot s have landed, empty[s] when all
  // warps have consumed it -- so a warp waits only for the data it reads and,
  // before refilling a slot, for the slowest warp of the PREVIOUS k-slice
  // (instead of a CTA barrier at every k-slice).
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  if constexpr (MB) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int s = 0; s < STAGES; ++s) {
        mb_init(&full_bar[s], NT);
        mb_init(&empty_bar[s], NT / 32);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) {
      load_tile<TA, NT>(st[s].a, A, tk.lda, m0, M, s * BKC, K, gcol);
      load_tile<TB, NT>(st[s].b, B, tk.ldb, n0, N, s * BKC, K);
      if constexpr (MB) mb_cp_arrive(&full_bar[s]);
    }
    if constexpr (!MB) cp_commit();
  }
  // C prefetch (C -= / += AB targets without mirrored writes): the last STAGES-1 iterations issue
  // no A/B loads, so each frees one ring slot; chunk c of the C tile (rows
  // [22c, 22c+22), pitch CP_PITCH) is fetched into the slot freed at
  // iteration ktiles-3+c and has landed by the epilogue.
  const int mode = tk.flags & kGemmModeMask;
  const bool sym = (tk.flags & kGemmSym) != 0;
  const bool cpre = (!sym || (tk.flags & kGemmLowerOnly)) && mode != kGemmStore && ktiles >= STAGES;

  for (int kt = 0; kt < ktiles; ++kt) {
    if constexpr (MB) {
      mb_wait(&full_bar[kt % STAGES], (unsigned)(kt / STAGES) & 1u);
    } else {
      cp_wait<STAGES - 2>();
      __syncthreads();
    }
    if constexpr (!MB) {
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) {
        const int slot = nk % STAGES;
        load_tile<TA, NT>(st[slot].a, A, tk.lda, m0, M, nk * BKC, K, gcol);
        load_tile<TB, NT>(st[slot].b, B, tk.ldb, n0, N, nk * BKC, K);
      } else if (cpre) {
        const int ch = nk - ktiles, r0 = ch * CP_ROWS;
        const int rows = min(CP_ROWS, BM - r0);
        cplx* dst = reinterpret_cast<cplx*>(&st[(kt + STAGES - 1) % STAGES]);
        for (int e = threadIdx.x; e < rows * BN; e += NT) {
          const int r = e / BN, c = e - r * BN;
          const bool ok = m0 + r0 + r < M && n0 + c < N;
          cp_async16(dst + r * CP_PITCH + c, ok ? C + (int64_t)(m0 + r0 + r) * tk.ldc + n0 + c : C, ok);
        }
      }
      cp_commit();
    }
    const int slot = kt % STAGES;
    // fragment element (tile row r, k) of a staged operand: row-major slices, k-major when transposed
    auto fa = [&](int r, int k) -> cplx {
      if constexpr (TA) return (&st[slot].a[0][0])[k * TPITCH + r];
      else return st[slot].a[r][k];
    };
    auto fb = [&](int r, int k) -> cplx {
      if constexpr (TB) return (&st[slot].b[0][0])[k * TPITCH + r];
      else return st[slot].b[r][k];
    };
    if constexpr (G3) {
#pragma unroll
      for (int kk = 0; kk < BKC / 4; ++kk) {
        double bre[WJ], bim[WJ], bsum[WJ];
#pragma unroll
        for (int j = 0; j < WJ; ++j) {
          const cplx b = fb(wn + j * 8 + fr, kk * 4 + fc);
          bre[j] = b.x;
          bim[j] = b.y;
          bsum[j] = b.x + b.y;
        }
        // per A sub-tile row: P, Q, R for both column sub-tiles; a given
        // accumulator is touched once per k-step (24 DMMAs apart)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const cplx a = fa(wm + i * 8 + fr, kk * 4 + fc);
          const double asum = a.x + a.y;
#pragma unroll
          for (int j = 0; j < WJ; ++j) dmma(acc_re[i][j][0], acc_re[i][j][1], a.x, bre[j]);
#pragma unroll
          for (int j = 0; j < WJ; ++j) dmma(acc_im[i][j][0], acc_im[i][j][1], a.y, bim[j]);
#pragma unroll
          for (int j = 0; j < WJ; ++j) dmma(acc_x[i][j][0], acc_x[i][j][1], asum, bsum[j]);
        }
      }
      if constexpr (MB) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mb_arrive(&empty_bar[slot]);
        const int nk = kt + STAGES - 1;
        const int slot2 = nk % STAGES;
        if (nk < ktiles || cpre) {
          // slot2 last held stage nk - STAGES (= kt - 1): wait until every warp consumed it
          if (nk >= STAGES) mb_wait(&empty_bar[slot2], (unsigned)((nk - STAGES) / STAGES) & 1u);
          if (nk < ktiles) {
            load_tile<TA, NT>(st[slot2].a, A, tk.lda, m0, M, nk * BKC, K, gcol);
            load_tile<TB, NT>(st[slot2].b, B, tk.ldb, n0, N, nk * BKC, K);
            mb_cp_arrive(&full_bar[slot2]);
          } else {
            const int ch = nk - ktiles, r0 = ch * CP_ROWS;
            const int rows = min(CP_ROWS, BM - r0);
            cplx* dst = reinterpret_cast<cplx*>(&st[slot2]);
            for (int e = threadIdx.x; e < rows * BN; e += NT) {
              const int r = e / BN, c = e - r * BN;
              const bool ok = m0 + r0 + r < M && n0 + c < N;
              cp_async16(dst + r * CP_PITCH + c, ok ? C + (int64_t)(m0 + r0 + r) * tk.ldc + n0 + c : C, ok);
            }
          }
        }
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < BKC / 4; ++kk) {
        double are[4], aim[4], anim[4], bre[4], bim[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const cplx a = fa(wm + i * 8 + fr, kk * 4 + fc);
          are[i] = a.x;
          aim[i] = a.y;
          anim[i] = -a.y;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const cplx b = fb(wn + j * 8 + fr, kk * 4 + fc);
          bre[j] = b.x;
          bim[j] = b.y;
        }
        // four passes over all sub-tiles: dependent DMMAs on one accumulator are
        // 32 instructions apart (per-accumulator order unchanged: bitwise same)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc_re[i][j][0], acc_re[i][j][1], are[i], bre[j]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc_im[i][j][0], acc_im[i][j][1], are[i], bim[j]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc_re[i][j][0], acc_re[i][j][1], anim[i], bim[j]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc_im[i][j][0], acc_im[i][j][1], aim[i], bre[j]);
      }
    }
  }
  if constexpr (MB) cp_commit();        // the C chunks of the MB path are not in a committed group yet
  cp_wait<0>();
  if constexpr (G3) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < WJ; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double p = acc_re[i][j][h], q = acc_im[i][j][h];
          acc_re[i][j][h] = p - q;
          acc_im[i][j][h] = (acc_x[i][j][h] - p) - q;
        }
  }

  // ---- epilogue ------------------------------------------------------------
  const bool mirror = sym && !(tk.flags & kGemmLowerOnly);
  const bool track = (tk.flags & kGemmTrackMax) != 0 && tmax != nullptr;
  double tm2 = 0.0;
  const int ldc = tk.ldc;
  if (cpre) {
    __syncthreads();                     // every thread's C chunks have landed
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rl = wm + i * 8 + fr, r = m0 + rl;
      const int ch = rl / CP_ROWS;
      const cplx* crow = reinterpret_cast<const cplx*>(&st[(ktiles + ch) % STAGES]) + (rl - ch * CP_ROWS) * CP_PITCH;
#pragma unroll
      for (int j = 0; j < WJ; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cl = wn + j * 8 + fc * 2 + h, c = n0 + cl;
          if (r >= M || c >= N || (sym && c > r)) continue;      // SYM here is lower-only
          const cplx u = mk(acc_re[i][j][h], acc_im[i][j][h]);
          const cplx w = mode == kGemmSub ? c_sub(crow[cl], u) : c_add(crow[cl], u);
          C[(int64_t)r * ldc + c] = w;
          if (track) tm2 = fmax(tm2, w.x * w.x + w.y * w.y);
        }
    }
  } else {
    // Per fragment row i: issue all 8 C loads (and the mirror loads) before any
    // store.  C is not __restrict__ (the mirror writes land in the same block),
    // so a fused load-op-store per element would serialise 32 memory round
    // trips per thread; batched, the epilogue costs 4.
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = m0 + wm + i * 8 + fr;
      cplx cv[WJ][2], cq[WJ][2];
#pragma unroll
      for (int j = 0; j < WJ; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = n0 + wn + j * 8 + fc * 2 + h;
          const bool ok = r < M && c < N && (!sym || c <= r);
          cv[j][h] = mk(0.0, 0.0);
          cq[j][h] = mk(0.0, 0.0);
          if (ok && mode != kGemmStore) cv[j][h] = C[(int64_t)r * ldc + c];
          if (ok && mirror && c < r) cq[j][h] = C[(int64_t)c * ldc + r];
        }
#pragma unroll
      for (int j = 0; j < WJ; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = n0 + wn + j * 8 + fc * 2 + h;
          if (r >= M || c >= N) continue;
          const cplx u = mk(acc_re[i][j][h], acc_im[i][j][h]);
          if (sym) {
            if (c > r) continue;
            const cplx w = c_sub(cv[j][h], u);
            C[(int64_t)r * ldc + c] = w;
            if (track) tm2 = fmax(tm2, w.x * w.x + w.y * w.y);
            if (mirror && c < r) C[(int64_t)c * ldc + r] = c_sub(cq[j][h], u);
          } else {
            cplx* p = C + (int64_t)r * ldc + c;
            if (mode == kGemmSub) *p = c_sub(cv[j][h], u);
            else if (mode == kGemmStore) *p = u;
            else *p = c_add(cv[j][h], u);
          }
        }
    }
  }
  if (track) {   // non-negative doubles order like their bit patterns: integer max is exact
    tm2 = warp_max(tm2);
    if ((threadIdx.x & 31) == 0) atomicMax(tmax + tk.pad_, (unsigned long long)__double_as_longlong(tm2));
  }
}

constexpr size_t kGemmSmem = sizeof(cplx) * STAGES * (BM + BN) * PITCH;

// Optional per-launch operands: tmax (kGemmTrackMax targets) and gperm (the
// column gather of kGemmTriGather tasks), passed with every launch.
struct LaunchExtra {
  unsigned long long* tmax;
  const int64_t* gperm;
};

template <bool TA, bool TB, bool G3, bool MB = false>
static int launch_g(const cplx* A, const cplx* B, cplx* C, const GemmTask* tasks, int ntasks, int ntiles,
                    const LaunchExtra& x, cudaStream_t s) {
  static PerDeviceOnce configured;
  if (configured.first())
    cudaFuncSetAttribute(zgemm_grouped_kernel<TA, TB, G3, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kGemmSmem);
  zgemm_grouped_kernel<TA, TB, G3, MB><<<ntiles, G3 ? 2 * NTHREADS : NTHREADS, kGemmSmem, s>>>(A, B, C, tasks,
                                                                                               ntasks, x.tmax, x.gperm);
  return (int)cudaGetLastError();
}

// Complex product form of the grouped GEMM: 3M (default) or 4M, a process-wide
// setting (D3M_ZGEMM=3m|4m at the first launch, or d3m_gemm_set_form).
static std::atomic<int> g_form{-1};
static bool use_3m() {
  int f = g_form.load();
  if (f < 0) {
    const char* e = getenv("D3M_ZGEMM");
    int expect = -1;
    g_form.compare_exchange_strong(expect, (e && (e[0] == '4')) ? 4 : 3);
    f = g_form.load();
  }
  return f == 3;
}

// ---- 3M on half tiles: three CTAs per SM -------------------------------------
// Each 64 x 64 task tile runs as two 64 x 32 CTAs (blockIdx.x = 2 * tile +
// half; the task tile maps are unchanged) of 4 warps with the same 32 x 16
// warp tiles: at three 128-thread CTAs per SM the register cap is 170 instead
// of 128, so the A fragments need not reuse the registers of the DMMAs in
// flight.  Per-element accumulation order and form are those of the 64 x 64
// 3M kernel (bitwise equal results).
constexpr int HN = 32, HNT = 128;
struct HStage {
  cplx a[BM][PITCH];
  cplx b[HN][PITCH];
};
constexpr int HCP_PITCH = HN + 1;
static_assert(32 * HCP_PITCH <= (int)(sizeof(HStage) / sizeof(cplx)), "a 32-row C chunk fits a freed stage");
constexpr size_t kHSmem = sizeof(HStage) * STAGES;

template <bool TA, bool TB>
__global__ void __launch_bounds__(HNT, 3)
zgemm3m_half_kernel(const cplx* __restrict__ Abase, const cplx* __restrict__ Bbase, cplx* Cbase,
                    const GemmTask* __restrict__ tasks, int ntasks, unsigned long long* tmax,
                    const int64_t* __restrict__ gperm) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  HStage* st = reinterpret_cast<HStage*>(smem_raw);
  const int tile = blockIdx.x >> 1, half = blockIdx.x & 1;
  const GemmTask tk = tasks[find_task(tasks, ntasks, tile)];
  int local = tile - tk.tile_start, tm, tn;
  const bool sym = (tk.flags & kGemmSym) != 0;
  if (sym) {
    tm = (int)((sqrt(8.0 * local + 1.0) - 1.0) * 0.5);
    while ((tm + 1) * (tm + 2) / 2 <= local) ++tm;
    while (tm * (tm + 1) / 2 > local) --tm;
    tn = local - tm * (tm + 1) / 2;
  } else {
    tm = local / tk.tiles_n;
    tn = local - tm * tk.tiles_n;
  }
  const int M = tk.m, N = tk.n, K = tk.k;
  const int m0 = tm * BM, n0 = tn * BN + half * HN;
  if (m0 >= M || n0 >= N) return;
  const cplx* A = Abase + tk.a_off;
  const cplx* B = Bbase + tk.b_off;
  cplx* C = Cbase + tk.c_off;
  const bool trig = (tk.flags & kGemmTriGather) != 0 && gperm != nullptr;
  const int64_t* gcol = trig ? gperm + tk.pad_ : nullptr;
  const int Keff = trig ? min(K, n0 + HN) : K;
  const int ktiles = (Keff + BKC - 1) / BKC;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 16;
  const int fr = lane >> 2, fc = lane & 3;
  auto load_stage = [&](int slot, int k0) {
    if constexpr (!TA) {
      const int kq = t & 7;
      const int64_t acol = (k0 + kq < K) ? (gcol ? gcol[k0 + kq] : (int64_t)(k0 + kq)) : 0;
#pragma unroll
      for (int p = 0; p < 4; ++p) {     // A: 64 rows, 16 per pass (8 threads per 128-byte row segment)
        const int r = p * 16 + (t >> 3);
        const bool ok = (m0 + r < M) && (k0 + kq < K);
        cp_async16(&st[slot].a[r][kq], ok ? A + (int64_t)(m0 + r) * tk.lda + acol : A, ok);
      }
    } else {
#pragma unroll
      for (int p = 0; p < 4; ++p) {     // A stored K x M: 64 threads per 1 KB row of the stored operand
        const int r = t & 63, k = p * 2 + (t >> 6);
        const bool ok = (m0 + r < M) && (k0 + k < K);
        cp_async16(&st[slot].a[r][k], ok ? A + (int64_t)(k0 + k) * tk.lda + m0 + r : A, ok);
      }
    }
    if constexpr (!TB) {
      const int kq = t & 7;
#pragma unroll
      for (int p = 0; p < 2; ++p) {     // B: 32 rows
        const int r = p * 16 + (t >> 3);
        const bool ok = (n0 + r < N) && (k0 + kq < K);
        cp_async16(&st[slot].b[r][kq], ok ? B + (int64_t)(n0 + r) * tk.ldb + k0 + kq : B, ok);
      }
    } else {
#pragma unroll
      for (int p = 0; p < 2; ++p) {     // B stored K x N: 32 threads per 512-byte row segment
        const int r = t & 31, k = p * 4 + (t >> 5);
        const bool ok = (n0 + r < N) && (k0 + k < K);
        cp_async16(&st[slot].b[r][k], ok ? B + (int64_t)(k0 + k) * tk.ldb + n0 + r : B, ok);
      }
    }
  };
  double P3[4][2][2], Q3[4][2][2], R3[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) P3[i][j][0] = P3[i][j][1] = Q3[i][j][0] = Q3[i][j][1] = R3[i][j][0] = R3[i][j][1] = 0.0;
  const int mode = tk.flags & kGemmModeMask;
  const bool cpre = (!sym || (tk.flags & kGemmLowerOnly)) && mode != kGemmStore && ktiles >= STAGES;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s * BKC);
    cp_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int nk = kt + STAGES - 1;
    if (nk < ktiles) {
      load_stage(nk % STAGES, nk * BKC);
    } else if (cpre && nk - ktiles < 2) {          // C rows [32c, 32c+32) into the freed stage
      const int ch = nk - ktiles;
      cplx* dst = reinterpret_cast<cplx*>(&st[nk % STAGES]);
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int e = p * HNT + t, r = e >> 5, c = e & 31;
        const int gr = m0 + ch * 32 + r;
        const bool ok = gr < M && n0 + c < N;
        cp_async16(dst + r * HCP_PITCH + c, ok ? C + (int64_t)gr * tk.ldc + n0 + c : C, ok);
      }
    }
    cp_commit();
    const HStage& S = st[kt % STAGES];
#pragma unroll
    for (int kk = 0; kk < BKC / 4; ++kk) {
      double bre[2], bim[2], bsum[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const cplx b = S.b[wn + j * 8 + fr][kk * 4 + fc];
        bre[j] = b.x;
        bim[j] = b.y;
        bsum[j] = b.x + b.y;
      }
      cplx a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = S.a[wm + i * 8 + fr][kk * 4 + fc];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double asum = a[i].x + a[i].y;
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(P3[i][j][0], P3[i][j][1], a[i].x, bre[j]);
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(Q3[i][j][0], Q3[i][j][1], a[i].y, bim[j]);
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(R3[i][j][0], R3[i][j][1], asum, bsum[j]);
      }
    }
  }
  cp_wait<0>();
  const bool mirror = sym && !(tk.flags & kGemmLowerOnly);
  const bool track = (tk.flags & kGemmTrackMax) != 0 && tmax != nullptr;
  double tm2 = 0.0;
  const int ldc = tk.ldc;
  if (cpre) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rl = wm + i * 8 + fr, r = m0 + rl, ch = rl >> 5;
      const cplx* crow = reinterpret_cast<const cplx*>(&st[(ktiles + ch) % STAGES]) + (rl & 31) * HCP_PITCH;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cl = wn + j * 8 + fc * 2 + h, c = n0 + cl;
          if (r >= M || c >= N || (sym && c > r)) continue;
          const double p = P3[i][j][h], q = Q3[i][j][h];
          const cplx u = mk(p - q, (R3[i][j][h] - p) - q);
          const cplx w = mode == kGemmSub ? c_sub(crow[cl], u) : c_add(crow[cl], u);
          C[(int64_t)r * ldc + c] = w;
          if (track) tm2 = fmax(tm2, w.x * w.x + w.y * w.y);
        }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = m0 + wm + i * 8 + fr;
      cplx cv[2][2], cq[2][2];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = n0 + wn + j * 8 + fc * 2 + h;
          const bool ok = r < M && c < N && (!sym || c <= r);
          cv[j][h] = mk(0.0, 0.0);
          cq[j][h] = mk(0.0, 0.0);
          if (ok && mode != kGemmStore) cv[j][h] = C[(int64_t)r * ldc + c];
          if (ok && mirror && c < r) cq[j][h] = C[(int64_t)c * ldc + r];
        }
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = n0 + wn + j * 8 + fc * 2 + h;
          if (r >= M || c >= N) continue;
          const double p = P3[i][j][h], q = Q3[i][j][h];
          const cplx u = mk(p - q, (R3[i][j][h] - p) - q);
          if (sym) {
            if (c > r) continue;
            const cplx w = c_sub(cv[j][h], u);
            C[(int64_t)r * ldc + c] = w;
            if (track) tm2 = fmax(tm2, w.x * w.x + w.y * w.y);
            if (mirror && c < r) C[(int64_t)c * ldc + r] = c_sub(cq[j][h], u);
          } else {
            cplx* pc = C + (int64_t)r * ldc + c;
            if (mode == kGemmSub) *pc = c_sub(cv[j][h], u);
            else if (mode == kGemmStore) *pc = u;
            else *pc = c_add(cv[j][h], u);
          }
        }
    }
  }
  if (track) {   // non-negative doubles order like their bit patterns: integer max is exact
    tm2 = warp_max(tm2);
    if (lane == 0) atomicMax(tmax + tk.pad_, (unsigned long long)__double_as_longlong(tm2));
  }
}

template <bool TA, bool TB>
static int launch_half(const cplx* A, const cplx* B, cplx* C, const GemmTask* tasks, int ntasks, int ntiles,
                       const LaunchExtra& x, cudaStream_t s) {
  static PerDeviceOnce configured;
  if (configured.first())
    cudaFuncSetAttribute(zgemm3m_half_kernel<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHSmem);
  zgemm3m_half_kernel<TA, TB><<<2 * ntiles, HNT, kHSmem, s>>>(A, B, C, tasks, ntasks, x.tmax, x.gperm);
  return (int)cudaGetLastError();
}

// ---- 3M half tiles staged by TMA ----------------------------------------------
// The trailing updates of block LDL^T read whole panels (X_j in the xbuf ring,
// L_j in the pool; lda = ldb = K = n_j), so one 2-D tensor map per panel
// describes every task's operand tile: a task's A tile is the box at (k0,
// a_off / lda + m0).  One elected thread issues the stage's two bulk tensor
// copies (cp.async.bulk.tensor.2d, SASS UTMALDG) against a per-stage mbarrier;
// the other 127 threads issue no staging instructions at all (the cp.async
// ring spends 6 LDGSTS plus their address / predicate math per thread and
// k-slice).  Rows past a task's block are whatever follows in the panel (they
// only feed accumulator rows that are never written); rows past the panel and
// k >= n_j are zero-filled by TMA.  The per-element product order is that of
// zgemm3m_half_kernel, so the results are bitwise equal.
//
// Shared-memory layout per stage: two 8-wide k-slices (one CTA barrier per 16 k: 43.0 against 41.9 TF/s
// at K = 256 with one slice per stage and four stages), tile bases 1024-byte aligned; per slice
//   a  64 x 8 complex, 128-byte rows, SWIZZLE_128B: 16-byte chunk c of row r at chunk c ^ (r & 7)
//   b  32 x 8 complex, same
// A DMMA fragment row fr (lane >> 2) is mapped to tile row pr = (fr >> 1) |
// ((fr & 1) << 2) of its 8-row group: a quarter warp's LDS.128 then covers the
// rows {q, q + 4} x 4 chunks, which the swizzle puts in different 64-byte
// halves (conflict-free).  The same map applies to B's rows, i.e. to the
// columns of C: accumulator (i, j, h) of a lane is C(wm + 8i + pr, wn + 8j +
// fc + 4h), so a store instruction writes 64 contiguous bytes per row.
// A stage holds two 8-wide k-slices (one CTA barrier per 16 k), three stages in the ring.
constexpr int TSTAGES = 3, TKS = 2;
struct alignas(1024) TStage {
  cplx a[TKS][BM][BKC];
  cplx b[TKS][HN][BKC];
};
static_assert(32 * HCP_PITCH * sizeof(cplx) <= sizeof(TStage), "a 32-row C chunk fits a freed stage");
constexpr size_t kTSmem = sizeof(TStage) * TSTAGES + 1024;      // + manual 1024-byte alignment

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smaddr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smaddr(bar))
      : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smaddr(b)), "r"(bytes) : "memory");
}

// BATCH: one pair of tensor maps per matrix in global memory (gmaps[2 b], gmaps[2 b + 1], b = the
// task's pad_), operand offsets relative to the matrix (a_off - b * a_stride = row * lda + first column,
// b_off - b * b_stride = row * ldb), and the running maximum of the written |C|^2 (kGemmTrackMax) -- the
// batched trailing updates of the subdomain panel BK (bk_panel.cu).
// TA / TB (BATCH only): the operand is stored K x M (K x N), as the subdomain solves read the factor and
// the right-hand sides.  Its slice is staged as 8-column boxes of the stored rows: box q of a slice holds
// k = 0..7 as 128-byte rows of the eight tile rows 8q..8q+7 (SWIZZLE_128B: row element e of k at chunk
// e ^ k), so the fragment of tile row 8q + pr at k reads chunk pr ^ k of row k of box q -- the chunk index
// of the row-major form, and as conflict-free (a quarter warp's rows {q, q + 4} x four k cover the
// eight chunks once).  The k range of such a task must end on a 16-k boundary or at the operand's last
// stored row (rows past the task's K inside the matrix are data, not zeros): the callers check.
template <bool BATCH, bool TA = false, bool TB = false>
__global__ void __launch_bounds__(HNT, 3)
zgemm3m_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, cplx* Cbase,
                   const GemmTask* __restrict__ tasks, int ntasks, int64_t b_base, const CUtensorMap* gmaps,
                   int64_t a_stride, int64_t b_stride, unsigned long long* tmax) {
  extern __shared__ unsigned char smem_dyn[];
  __shared__ __align__(8) uint64_t full[TSTAGES];
  TStage* st = reinterpret_cast<TStage*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) {
#pragma unroll
    for (int s = 0; s < TSTAGES; ++s) mb_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const int tile = blockIdx.x >> 1, half = blockIdx.x & 1;
  const GemmTask tk = tasks[find_task(tasks, ntasks, tile)];      // (its barrier publishes the mbarrier inits)
  int local = tile - tk.tile_start, tm, tn;
  const bool sym = (tk.flags & kGemmSym) != 0;
  if (sym) {
    tm = (int)((sqrt(8.0 * local + 1.0) - 1.0) * 0.5);
    while ((tm + 1) * (tm + 2) / 2 <= local) ++tm;
    while (tm * (tm + 1) / 2 > local) --tm;
    tn = local - tm * (tm + 1) / 2;
  } else {
    tm = local / tk.tiles_n;
    tn = local - tm * tk.tiles_n;
  }
  const int M = tk.m, N = tk.n, K = tk.k;
  const int m0 = tm * BM, n0 = tn * BN + half * HN;
  if (m0 >= M || n0 >= N) return;
  cplx* C = Cbase + tk.c_off;
  int arow, brow, acol = 0;                                     // panel rows of the tile's first A / B row
  const CUtensorMap *pmA = &mapA, *pmB = &mapB;
  int bcol = 0;
  if constexpr (BATCH) {
    const int arel = (int)(tk.a_off - tk.pad_ * a_stride);
    const int brel = (int)(tk.b_off - tk.pad_ * b_stride);
    if constexpr (TA) {            // stored K x M: arow = first stored (k) row, acol = the tile's first column
      arow = arel / tk.lda;
      acol = arel % tk.lda + m0;
    } else {
      arow = arel / tk.lda + m0;
      acol = arel % tk.lda;
    }
    if constexpr (TB) {
      brow = brel / tk.ldb;
      bcol = brel % tk.ldb + n0;
    } else {
      brow = brel / tk.ldb + n0;
      bcol = brel % tk.ldb;
    }
    pmA = gmaps + 2 * tk.pad_;
    pmB = pmA + 1;
  } else {
    arow = (int)(tk.a_off / tk.lda) + m0;
    brow = (int)((tk.b_off - b_base) / tk.ldb) + n0;
  }
  const int ktiles = (K + TKS * BKC - 1) / (TKS * BKC);
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 16;
  const int fr = lane >> 2, fc = lane & 3;
  const int pr = (fr >> 1) | ((fr & 1) << 2);
  constexpr unsigned kStageBytes = (unsigned)sizeof(TStage);
  auto issue = [&](int slot, int kt) {
    // lane 0 of every warp (with k-major operands the stage is up to 24 copies: each warp issues a
    // quarter of the boxes); warp 0 arms the barrier and issues the row-major operands
    if (warp == 0) mb_expect_tx(&full[slot], kStageBytes);
#pragma unroll
    for (int h = 0; h < TKS; ++h) {
      const int k0 = (kt * TKS + h) * BKC;
      if constexpr (TA) {
#pragma unroll
        for (int q = 0; q < BM / 8 / 4; ++q)
          tma_load_2d(&st[slot].a[h][(4 * q + warp) * 8][0], pmA, 2 * (acol + (4 * q + warp) * 8), arow + k0,
                      &full[slot]);
      } else {
        if (warp == 0) tma_load_2d(&st[slot].a[h][0][0], pmA, 2 * (acol + k0), arow, &full[slot]);
      }
      if constexpr (TB) {
        tma_load_2d(&st[slot].b[h][warp * 8][0], pmB, 2 * (bcol + warp * 8), brow + k0, &full[slot]);
      } else {
        if (warp == 0) tma_load_2d(&st[slot].b[h][0][0], pmB, 2 * (bcol + k0), brow, &full[slot]);
      }
    }
  };
  static_assert(HN / 8 == HNT / 32 && (BM / 8) % (HNT / 32) == 0, "k-major boxes split evenly over the warps");
  const bool issuer = (TA || TB) ? lane == 0 : t == 0;
  double P3[4][2][2], Q3[4][2][2], R3[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) P3[i][j][0] = P3[i][j][1] = Q3[i][j][0] = Q3[i][j][1] = R3[i][j][0] = R3[i][j][1] = 0.0;
  const int mode = tk.flags & kGemmModeMask;
  const bool cpre = (!sym || (tk.flags & kGemmLowerOnly)) && mode != kGemmStore && ktiles >= TSTAGES;
  if (issuer) {
#pragma unroll
    for (int s = 0; s < TSTAGES - 1; ++s)
      if (s < ktiles) issue(s, s);
  }
  const int ca0 = fc ^ pr, ca1 = (4 + fc) ^ pr;          // swizzled chunk of k = kk*4 + fc in this lane's rows
  for (int kt = 0; kt < ktiles; ++kt) {
    __syncthreads();                       // every warp is done with slot (kt - 1) % TSTAGES
    const int nk = kt + TSTAGES - 1;
    if (nk < ktiles) {
      if (issuer) issue(nk % TSTAGES, nk);
    } else if (cpre && nk - ktiles < 2) {  // C rows [32c, 32c+32) into the freed stage
      const int ch = nk - ktiles;
      cplx* dst = reinterpret_cast<cplx*>(&st[nk % TSTAGES]);
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int e = p * HNT + t, r = e >> 5, c = e & 31;
        const int gr = m0 + ch * 32 + r;
        const bool ok = gr < M && n0 + c < N;
        cp_async16(dst + r * HCP_PITCH + c, ok ? C + (int64_t)gr * tk.ldc + n0 + c : C, ok);
      }
      cp_commit();
    }
    mb_wait(&full[kt % TSTAGES], (unsigned)(kt / TSTAGES) & 1u);
    const TStage& S = st[kt % TSTAGES];
#pragma unroll
    for (int kq = 0; kq < TKS * BKC / 4; ++kq) {
      const int ca = (kq & 1) ? ca1 : ca0, ks = kq >> 1;
      const int k8 = (kq & 1) * 4 + fc;               // k within the slice (row of a k-major box)
      double bre[2], bim[2], bsum[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const cplx b = S.b[ks][TB ? wn + j * 8 + k8 : wn + j * 8 + pr][ca];
        bre[j] = b.x;
        bim[j] = b.y;
        bsum[j] = b.x + b.y;
      }
      cplx a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = S.a[ks][TA ? wm + i * 8 + k8 : wm + i * 8 + pr][ca];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double asum = a[i].x + a[i].y;
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(P3[i][j][0], P3[i][j][1], a[i].x, bre[j]);
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(Q3[i][j][0], Q3[i][j][1], a[i].y, bim[j]);
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(R3[i][j][0], R3[i][j][1], asum, bsum[j]);
      }
    }
  }
  cp_wait<0>();
  const bool mirror = sym && !(tk.flags & kGemmLowerOnly);
  const int ldc = tk.ldc;
  double tm2 = 0.0;
  if (cpre) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rl = wm + i * 8 + pr, r = m0 + rl, ch = rl >> 5;
      const cplx* crow = reinterpret_cast<const cplx*>(&st[(ktiles + ch) % TSTAGES]) + (rl & 31) * HCP_PITCH;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cl = wn + j * 8 + fc + 4 * h, c = n0 + cl;
          if (r >= M || c >= N || (sym && c > r)) continue;
          const double p = P3[i][j][h], q = Q3[i][j][h];
          const cplx u = mk(p - q, (R3[i][j][h] - p) - q);
          const cplx w = mode == kGemmSub ? c_sub(crow[cl], u) : c_add(crow[cl], u);
          C[(int64_t)r * ldc + c] = w;
          if constexpr (BATCH) tm2 = fmax(tm2, w.x * w.x + w.y * w.y);
        }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = m0 + wm + i * 8 + pr;
      cplx cv[2][2], cq[2][2];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = n0 + wn + j * 8 + fc + 4 * h;
          const bool ok = r < M && c < N && (!sym || c <= r);
          cv[j][h] = mk(0.0, 0.0);
          cq[j][h] = mk(0.0, 0.0);
          if (ok && mode != kGemmStore) cv[j][h] = C[(int64_t)r * ldc + c];
          if (ok && mirror && c < r) cq[j][h] = C[(int64_t)c * ldc + r];
        }
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = n0 + wn + j * 8 + fc + 4 * h;
          if (r >= M || c >= N) continue;
          const double p = P3[i][j][h], q = Q3[i][j][h];
          const cplx u = mk(p - q, (R3[i][j][h] - p) - q);
          if (sym) {
            if (c > r) continue;
            const cplx w = c_sub(cv[j][h], u);
            C[(int64_t)r * ldc + c] = w;
            if constexpr (BATCH) tm2 = fmax(tm2, w.x * w.x + w.y * w.y);
            if (mirror && c < r) C[(int64_t)c * ldc + r] = c_sub(cq[j][h], u);
          } else {
            cplx* pc = C + (int64_t)r * ldc + c;
            if (mode == kGemmSub) *pc = c_sub(cv[j][h], u);
            else if (mode == kGemmStore) *pc = u;
            else *pc = c_add(cv[j][h], u);
          }
        }
    }
  }
  if constexpr (BATCH) {
    if ((tk.flags & kGemmTrackMax) != 0 && tmax != nullptr) {   // non-negative doubles order like their bit patterns
      tm2 = warp_max(tm2);
      if (lane == 0) atomicMax(tmax + tk.pad_, (unsigned long long)__double_as_longlong(tm2));
    }
  }
}

using TmapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmapEncodeFn tmap_encoder() {
  static const TmapEncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<TmapEncodeFn>(p);
  }();
  return fn;
}

// 2-D map over `rows` rows of `cols` doubles (row pitch `pitch_bytes`), box box_cols x box_rows
static int tmap_2d(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t pitch_bytes, int box_cols,
                   int box_rows, CUtensorMapSwizzle sw) {
  const TmapEncodeFn enc = tmap_encoder();
  if (!enc) return -38;
  const cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t gstr[1] = {(cuuint64_t)pitch_bytes};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t est[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), gdim, gstr, box, est,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -22;
}

template <bool TA, bool TB>
static int launch_t(const cplx* A, const cplx* B, cplx* C, const GemmTask* tasks, int ntasks, int ntiles,
                    const LaunchExtra& x, cudaStream_t s) {
  // D3M_GEMM_HALF=0: the 64 x 64 3M kernel for every launch (A/B measurements)
  static const int hk = [] { const char* e = getenv("D3M_GEMM_HALF"); return e ? atoi(e) : 1; }();
  if (!use_3m()) return launch_g<TA, TB, false>(A, B, C, tasks, ntasks, ntiles, x, s);
  // non-transposed operands only, and not for the batched panel updates
  // (max-tracking, device-built tasks with a padded tile budget): there the
  // doubled grid of mostly empty CTAs cost more than the faster tiles gained
  // (config 3: 96 -> 119 ms); the transposed launches of the subdomain solves
  // ran 9% slower on half tiles (config 5 GEMM class 6.40 -> 6.96 s)
  if constexpr (!TA && !TB) {
    if (hk && x.tmax == nullptr) return launch_half<TA, TB>(A, B, C, tasks, ntasks, ntiles, x, s);
  }
  return launch_g<TA, TB, true, true>(A, B, C, tasks, ntasks, ntiles, x, s);   // mbarrier ring
}

}  // namespace d3m

// Host helper: fill tile counts/prefix sums of a task array (host memory).
extern "C" int d3m_gemm_prepare_tasks(d3m::GemmTask* tasks, int ntasks) {
  int total = 0;
  for (int t = 0; t < ntasks; ++t) {
    d3m::GemmTask& k = tasks[t];
    const int tm = (k.m + d3m::BM - 1) / d3m::BM, tn = (k.n + d3m::BN - 1) / d3m::BN;
    k.tiles_n = tn;
    k.tile_start = total;
    if (k.flags & d3m::kGemmSym) total += tm * (tm + 1) / 2;
    else total += tm * tn;
  }
  return total;
}

namespace {
int gemm_launch_x(int ta, int tb, const void* A, const void* B, void* C, const void* dtasks, int ntasks, int ntiles,
                  const d3m::LaunchExtra& x, void* stream) {
  using namespace d3m;
  if (ntiles <= 0 || ntasks <= 0) return 0;
  auto a = static_cast<const cplx*>(A);
  auto b = static_cast<const cplx*>(B);
  auto c = static_cast<cplx*>(C);
  auto t = static_cast<const GemmTask*>(dtasks);
  auto s = reinterpret_cast<cudaStream_t>(stream);
  if (!ta && !tb) return launch_t<false, false>(a, b, c, t, ntasks, ntiles, x, s);
  if (!ta && tb) return launch_t<false, true>(a, b, c, t, ntasks, ntiles, x, s);
  if (ta && !tb) return launch_t<true, false>(a, b, c, t, ntasks, ntiles, x, s);
  return launch_t<true, true>(a, b, c, t, ntasks, ntiles, x, s);
}
}  // namespace

// Select the complex product form of the grouped GEMM: 3 (Gauss 3M) or 4 (4M).
// Returns the form in effect before the call; 0 only queries.
extern "C" int d3m_gemm_set_form(int form) {
  const int prev = d3m::use_3m() ? 3 : 4;
  if (form == 3 || form == 4) d3m::g_form.store(form);
  return prev;
}

extern "C" int d3m_gemm_launch(int ta, int tb, const void* A, const void* B, void* C, const void* dtasks,
                               int ntasks, int ntiles, void* stream) {
  return gemm_launch_x(ta, tb, A, B, C, dtasks, ntasks, ntiles, d3m::LaunchExtra{nullptr, nullptr}, stream);
}

// ---- TMA-staged trailing updates (zgemm3m_tma_kernel) -------------------------
// d3m_gemm_tma_prepare: encode the tensor maps of the panels X (rows_x x n,
// contiguous rows) and L (rows_l x n) into maps_out (host memory, 2 x
// sizeof(CUtensorMap) = 256 bytes).  Returns -38 when the driver has no
// cuTensorMapEncodeTiled (the caller then uses the cp.async kernel).
extern "C" int d3m_gemm_tma_prepare(const void* X, int64_t rows_x, const void* L, int64_t rows_l, int n,
                                    void* maps_out) {
  using namespace d3m;
  if (rows_x <= 0 || rows_l <= 0 || n <= 0) return -22;
  auto* m = static_cast<CUtensorMap*>(maps_out);
  int rc = tmap_2d(&m[0], X, rows_x, 2 * (int64_t)n, (int64_t)n * 16, 2 * BKC, BM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = tmap_2d(&m[1], L, rows_l, 2 * (int64_t)n, (int64_t)n * 16, 2 * BKC, HN, CU_TENSOR_MAP_SWIZZLE_128B);
  return rc;
}

// Launch the tasks (kGemmSub / kGemmSym targets, a_off relative to X, b_off
// relative to Bbase with the L panel at b_base; lda = ldb = k = n of the
// prepared panels) on the TMA kernel.
extern "C" int d3m_gemm_tma_launch(const void* maps, void* C, const void* dtasks, int ntasks, int ntiles,
                                   int64_t b_base, void* stream) {
  using namespace d3m;
  if (ntiles <= 0 || ntasks <= 0) return 0;
  auto* m = static_cast<const CUtensorMap*>(maps);
  static PerDeviceOnce configured;
  if (configured.first())
    cudaFuncSetAttribute(zgemm3m_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTSmem);
  zgemm3m_tma_kernel<false><<<2 * ntiles, HNT, kTSmem, reinterpret_cast<cudaStream_t>(stream)>>>(
      m[0], m[1], static_cast<cplx*>(C), static_cast<const GemmTask*>(dtasks), ntasks, b_base, nullptr, 0, 0, nullptr);
  return (int)cudaGetLastError();
}

// Batched form: per matrix b a map pair over its A matrix (rows x cols complex, leading dimension lda)
// and its B matrix, encoded into h_maps (2 * batch CUtensorMap, host) by d3m_gemm_tma_prepare_batched and
// copied by the caller into d_maps (device, 64-byte aligned).  Tasks carry the matrix index in pad_.
extern "C" int d3m_gemm_tma_prepare_batched(const void* A, int64_t a_stride, int64_t a_rows, int a_cols, int lda,
                                            const void* B, int64_t b_stride, int64_t b_rows, int b_cols, int ldb,
                                            int batch, void* h_maps) {
  using namespace d3m;
  auto* m = static_cast<CUtensorMap*>(h_maps);
  for (int b = 0; b < batch; ++b) {
    int rc = tmap_2d(&m[2 * b], static_cast<const cplx*>(A) + b * a_stride, a_rows, 2 * (int64_t)a_cols,
                     (int64_t)lda * 16, 2 * BKC, BM, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!rc)
      rc = tmap_2d(&m[2 * b + 1], static_cast<const cplx*>(B) + b * b_stride, b_rows, 2 * (int64_t)b_cols,
                   (int64_t)ldb * 16, 2 * BKC, HN, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  return 0;
}

// Map pairs of the blocked subdomain solves (ldlt_solve_blocked_impl): per matrix b
//   forward  h_maps[2 b]                = F_b (n x n) row boxes (A = L[rows, block], not transposed),
//            h_maps[2 b + 1]            = Z_b (n x m) k-major boxes (B = Z[block, :], stored K x N);
//   backward h_maps[2 batch + 2 b]      = F_b k-major boxes (A = L[block, cols]^T, stored K x M),
//            h_maps[2 batch + 2 b + 1]  = Z_b k-major boxes.
extern "C" int d3m_gemm_tma_prepare_solve(const void* F, int64_t stride_f, int n, const void* Z, int64_t stride_z,
                                          int m, int batch, void* h_maps) {
  using namespace d3m;
  auto* mp = static_cast<CUtensorMap*>(h_maps);
  for (int b = 0; b < batch; ++b) {
    const cplx* f = static_cast<const cplx*>(F) + b * stride_f;
    const cplx* z = static_cast<const cplx*>(Z) + b * stride_z;
    int rc = tmap_2d(&mp[2 * b], f, n, 2 * (int64_t)n, (int64_t)n * 16, 2 * BKC, BM, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!rc) rc = tmap_2d(&mp[2 * b + 1], z, n, 2 * (int64_t)m, (int64_t)m * 16, 16, 8, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!rc)
      rc = tmap_2d(&mp[2 * batch + 2 * b], f, n, 2 * (int64_t)n, (int64_t)n * 16, 16, 8, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    mp[2 * batch + 2 * b + 1] = mp[2 * b + 1];
  }
  return 0;
}

// ta = 0: A not transposed, B stored K x N (forward updates); ta = 1: both stored k-major (backward)
extern "C" int d3m_gemm_tma_launch_batched_t(int ta, const void* d_maps, void* C, const void* dtasks, int ntasks,
                                             int ntiles, int64_t a_stride, int64_t b_stride, void* stream) {
  using namespace d3m;
  if (ntiles <= 0 || ntasks <= 0) return 0;
  static PerDeviceOnce configured;
  if (configured.first()) {
    cudaFuncSetAttribute(zgemm3m_tma_kernel<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kTSmem);
    cudaFuncSetAttribute(zgemm3m_tma_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kTSmem);
  }
  CUtensorMap dummy{};
  auto s = reinterpret_cast<cudaStream_t>(stream);
  if (ta)
    zgemm3m_tma_kernel<true, true, true><<<2 * ntiles, HNT, kTSmem, s>>>(
        dummy, dummy, static_cast<cplx*>(C), static_cast<const GemmTask*>(dtasks), ntasks, 0,
        static_cast<const CUtensorMap*>(d_maps), a_stride, b_stride, nullptr);
  else
    zgemm3m_tma_kernel<true, false, true><<<2 * ntiles, HNT, kTSmem, s>>>(
        dummy, dummy, static_cast<cplx*>(C), static_cast<const GemmTask*>(dtasks), ntasks, 0,
        static_cast<const CUtensorMap*>(d_maps), a_stride, b_stride, nullptr);
  return (int)cudaGetLastError();
}

extern "C" int d3m_gemm_tma_launch_batched(const void* d_maps, void* C, const void* dtasks, int ntasks, int ntiles,
                                           int64_t a_stride, int64_t b_stride, void* tmax, void* stream) {
  using namespace d3m;
  if (ntiles <= 0 || ntasks <= 0) return 0;
  static PerDeviceOnce configured;
  if (configured.first())
    cudaFuncSetAttribute(zgemm3m_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTSmem);
  CUtensorMap dummy{};
  zgemm3m_tma_kernel<true><<<2 * ntiles, HNT, kTSmem, reinterpret_cast<cudaStream_t>(stream)>>>(
      dummy, dummy, static_cast<cplx*>(C), static_cast<const GemmTask*>(dtasks), ntasks, 0,
      static_cast<const CUtensorMap*>(d_maps), a_stride, b_stride, static_cast<unsigned long long*>(tmax));
  return (int)cudaGetLastError();
}

// Launch with a column-gather permutation for kGemmTriGather tasks (A not transposed).
extern "C" int d3m_gemm_launch_perm(const void* A, const void* B, void* C, const void* dtasks, int ntasks, int ntiles,
                                    const void* gperm, void* stream) {
  return gemm_launch_x(0, 0, A, B, C, dtasks, ntasks, ntiles,
                       d3m::LaunchExtra{nullptr, static_cast<const int64_t*>(gperm)}, stream);
}

extern "C" int d3m_gemm_launch_tm(int ta, int tb, const void* A, const void* B, void* C, const void* dtasks,
                                  int ntasks, int ntiles, void* tmax, void* stream) {
  return gemm_launch_x(ta, tb, A, B, C, dtasks, ntasks, ntiles,
                       d3m::LaunchExtra{static_cast<unsigned long long*>(tmax), nullptr}, stream);
}
