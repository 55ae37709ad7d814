// solve_gemv.cu -- block substitution kernels (factor.py:243-310), HBM-bound.
//
// A block solve with nrhs <= a few dozen columns reads every stored factor
// entry once per sweep and does nrhs complex FMAs with it: a tall-skinny
// product that the 64x64-tile DMMA GEMM runs at <25% utilisation with long
// serial K loops.  These kernels stage the factor rows and the small RHS
// block in shared memory and compute each output with a fixed summation
// order that does not depend on the number of RHS columns, so a k-RHS solve
// equals k single-RHS solves bit for bit (factor.py:271-279).
//
//  rows_gemv : C[cmap(r)][c] (-)= sum_k A[r][k] B[k][c]          (z = Binv b,
//              b_i -= L_ij z_j with the panel's global row map)
//  cols_gemv : P[chunk][m][c]  = sum_{r in chunk} A[r][m] B[bmap(r)][c]
//              (L_ij^T x_i and Binv^T w, split over row chunks)
//  chunk_reduce : out = base + sign * sum_chunk P[chunk]     (ordered)
#include "d3m_common.cuh"
#include "d3m_kernels.h"

namespace d3m {

constexpr int SG_THREADS = 256;
constexpr int SG_NC = 16;      // RHS columns per pass
constexpr int SG_TR = 16;      // rows per CTA (rows_gemv)
constexpr int SG_KC = 64;      // K chunk staged in shared memory (static smem <= 48 KB)
constexpr int SG_RC = 16;      // rows per chunk (cols_gemv)

__global__ void __launch_bounds__(SG_THREADS)
rows_gemv_kernel(const cplx* __restrict__ A, int lda, int M, int K, const cplx* __restrict__ B, int ldb, int N,
                 cplx* C, int ldc, const int64_t* __restrict__ cmap, int sub) {
  __shared__ __align__(16) cplx As[SG_TR][SG_KC + 1];
  __shared__ __align__(16) cplx Bs[SG_KC][SG_NC];
  const int r0 = blockIdx.x * SG_TR;
  const int row = threadIdx.x / SG_NC, col = threadIdx.x % SG_NC;
  for (int c0 = 0; c0 < N; c0 += SG_NC) {
    cplx acc = mk(0.0, 0.0);
    for (int k0 = 0; k0 < K; k0 += SG_KC) {
      const int kc = min(SG_KC, K - k0);
      {  // all staging loads issued before any shared-memory store
        constexpr int NA = SG_TR * SG_KC / SG_THREADS, NBL = SG_KC * SG_NC / SG_THREADS;
        cplx ra[NA], rb[NBL];
#pragma unroll
        for (int q = 0; q < NA; ++q) {
          const int e = threadIdx.x + q * SG_THREADS, rr = e / SG_KC, kk = e % SG_KC;
          ra[q] = (r0 + rr < M && kk < kc) ? A[(int64_t)(r0 + rr) * lda + k0 + kk] : mk(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < NBL; ++q) {
          const int e = threadIdx.x + q * SG_THREADS, kk = e / SG_NC, cc = e % SG_NC;
          rb[q] = (kk < kc && c0 + cc < N) ? B[(int64_t)(k0 + kk) * ldb + c0 + cc] : mk(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < NA; ++q) {
          const int e = threadIdx.x + q * SG_THREADS;
          As[e / SG_KC][e % SG_KC] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < NBL; ++q) {
          const int e = threadIdx.x + q * SG_THREADS;
          Bs[e / SG_NC][e % SG_NC] = rb[q];
        }
      }
      __syncthreads();
#pragma unroll 4
      for (int kk = 0; kk < kc; ++kk) c_fma(acc, As[row][kk], Bs[kk][col]);
      __syncthreads();
    }
    const int r = r0 + row, c = c0 + col;
    if (r < M && c < N) {
      cplx* p = C + (cmap ? cmap[r] : (int64_t)r) * ldc + c;
      *p = sub ? c_sub(*p, acc) : acc;
    }
  }
}

// one CTA per (row chunk, 256-column block of A); thread = one column m of A,
// all RHS columns of the pass in registers
__global__ void __launch_bounds__(SG_THREADS)
cols_gemv_kernel(const cplx* __restrict__ A, int lda, int R, int Mcols, const cplx* __restrict__ B, int ldb,
                 const int64_t* __restrict__ bmap, int N, cplx* partial) {
  __shared__ __align__(16) cplx Bs[SG_RC][SG_NC];
  const int chunk = blockIdx.x;
  const int m = blockIdx.y * SG_THREADS + threadIdx.x;
  const int r0 = chunk * SG_RC;
  const int rc = min(SG_RC, R - r0);
  for (int c0 = 0; c0 < N; c0 += SG_NC) {
    for (int e = threadIdx.x; e < SG_RC * SG_NC; e += SG_THREADS) {
      const int rr = e / SG_NC, cc = e % SG_NC;
      Bs[rr][cc] = (rr < rc && c0 + cc < N) ? B[(bmap ? bmap[r0 + rr] : (int64_t)(r0 + rr)) * ldb + c0 + cc]
                                            : mk(0.0, 0.0);
    }
    __syncthreads();
    if (m < Mcols) {
      cplx acc[SG_NC];
#pragma unroll
      for (int cc = 0; cc < SG_NC; ++cc) acc[cc] = mk(0.0, 0.0);
      for (int rb0 = 0; rb0 < rc; rb0 += 8) {     // 8 rows of A in flight
        cplx a[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          a[q] = (rb0 + q < rc) ? A[(int64_t)(r0 + rb0 + q) * lda + m] : mk(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int cc = 0; cc < SG_NC; ++cc) c_fma(acc[cc], a[q], Bs[rb0 + q][cc]);
      }
      cplx* out = partial + ((int64_t)chunk * Mcols + m) * N + c0;
#pragma unroll
      for (int cc = 0; cc < SG_NC; ++cc)
        if (c0 + cc < N) out[cc] = acc[cc];
    }
    __syncthreads();
  }
}

// out[e] = (base ? base[e] : 0) + sign * sum_{ch < nch} partial[ch * len + e]
__global__ void chunk_reduce_kernel(const cplx* base, const cplx* partial, int nch, int64_t len, double sign,
                                    cplx* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
    cplx acc = mk(0.0, 0.0);
    for (int ch = 0; ch < nch; ++ch) acc = c_add(acc, partial[ch * len + e]);
    const cplx b = base ? base[e] : mk(0.0, 0.0);
    out[e] = mk(b.x + sign * acc.x, b.y + sign * acc.y);
  }
}

}  // namespace d3m

extern "C" int d3m_rows_gemv_launch(const void* A, int lda, int M, int K, const void* B, int ldb, int N, void* C,
                                    int ldc, const void* cmap, int sub, void* stream) {
  using namespace d3m;
  if (M <= 0 || N <= 0) return 0;
  rows_gemv_kernel<<<(M + SG_TR - 1) / SG_TR, SG_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const cplx*>(A), lda, M, K, static_cast<const cplx*>(B), ldb, N, static_cast<cplx*>(C), ldc,
      static_cast<const int64_t*>(cmap), sub);
  return (int)cudaGetLastError();
}

// returns the number of row chunks written to `partial` (nch x Mcols x N)
extern "C" int d3m_cols_gemv_launch(const void* A, int lda, int R, int Mcols, const void* B, int ldb,
                                    const void* bmap, int N, void* partial, void* stream) {
  using namespace d3m;
  if (R <= 0 || Mcols <= 0 || N <= 0) return 0;
  const dim3 grid((R + SG_RC - 1) / SG_RC, (Mcols + SG_THREADS - 1) / SG_THREADS);
  cols_gemv_kernel<<<grid, SG_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const cplx*>(A), lda, R, Mcols, static_cast<const cplx*>(B), ldb,
      static_cast<const int64_t*>(bmap), N, static_cast<cplx*>(partial));
  return (int)cudaGetLastError();
}

extern "C" int d3m_chunk_reduce_launch(const void* base, const void* partial, int nch, int64_t len, double sign,
                                       void* out, void* stream) {
  using namespace d3m;
  if (len <= 0) return 0;
  const int blocks = (int)std::min<int64_t>((len + 255) / 256, 2048);
  chunk_reduce_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const cplx*>(base), static_cast<const cplx*>(partial), nch, len, sign, static_cast<cplx*>(out));
  return (int)cudaGetLastError();
}

int d3m_solve_rows_per_chunk() { return d3m::SG_RC; }
