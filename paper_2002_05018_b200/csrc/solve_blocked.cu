// solve_blocked.cu -- blocked multi-RHS solves against large packed factors
// (DenseFactor.solve, factor.py:52-66, for reduce_domain's n x (m+1) RHS).
//
// Z = L^-1 Z and Z = L^-T Z are split into 64-row blocks: a diagonal-block
// kernel solves each 64 x 64 unit triangle in shared memory, and the
// off-diagonal coupling is a right-looking DMMA GEMM (d3m_gemm_launch,
// batched over all subdomains).  The GEMM reads the packed factor as L, so
// the e entry of a 2x2 pivot that straddles a block boundary (packed at
// W[k+1][k], L entry zero) is wrongly applied once; the next diagonal kernel
// adds that term back (forward: row r0 += e z[r0-1]; backward: row r1-1 +=
// e z[r1]).
#include "d3m_common.cuh"
#include "d3m_kernels.h"

namespace d3m {

constexpr int DB = 64;           // diagonal block
constexpr int DB_NC = 32;        // RHS columns per CTA
constexpr int DB_THREADS = 256;
constexpr int DB_CW = DB_NC / (DB_THREADS / 32);     // RHS columns per warp
static_assert(DB == 64 && DB_CW * (DB_THREADS / 32) == DB_NC, "two rows per lane, whole columns per warp");

// forward: Z[r0:r0+64] = L_bb^-1 Z[r0:r0+64]   (after the straddle fix)
__global__ void __launch_bounds__(DB_THREADS)
diag_fwd_kernel(const cplx* Fbase, int64_t stride_f, const int8_t* tagsbase, int64_t stride_t, cplx* Zbase,
                int64_t stride_z, int n, int m, int r0) {
  extern __shared__ __align__(16) unsigned char db_smem[];
  cplx(*Ls)[DB + 1] = reinterpret_cast<cplx(*)[DB + 1]>(db_smem);
  cplx(*Zs)[DB_NC] = reinterpret_cast<cplx(*)[DB_NC]>(db_smem + sizeof(cplx) * DB * (DB + 1));
  const int b = blockIdx.y;
  const cplx* F = Fbase + b * stride_f;
  const int8_t* tags = tagsbase + b * stride_t;
  cplx* Z = Zbase + b * stride_z;
  const int c0 = blockIdx.x * DB_NC;
  const int nb = min(DB, n - r0);
  for (int e = threadIdx.x; e < DB * DB; e += DB_THREADS) {
    const int r = e / DB, c = e % DB;
    cplx v = mk(0.0, 0.0);
    if (r < nb && c < r && !(r == c + 1 && tags[r0 + c] == 2)) v = F[(int64_t)(r0 + r) * n + r0 + c];
    Ls[r][c] = v;
  }
  for (int e = threadIdx.x; e < DB * DB_NC; e += DB_THREADS) {
    const int r = e / DB_NC, c = e % DB_NC;
    Zs[r][c] = (r < nb && c0 + c < m) ? Z[(int64_t)(r0 + r) * m + c0 + c] : mk(0.0, 0.0);
  }
  __syncthreads();
  if (r0 > 0 && tags[r0 - 1] == 2 && threadIdx.x < DB_NC && c0 + threadIdx.x < m) {
    const cplx e = F[(int64_t)r0 * n + r0 - 1];
    c_fma(Zs[0][threadIdx.x], e, Z[(int64_t)(r0 - 1) * m + c0 + threadIdx.x]);
  }
  __syncthreads();
  // substitution in registers: warp w owns the RHS columns 4w..4w+3, lane l their rows l and l + 32;
  // the pivot row's values travel by shuffle (no CTA barrier per step).  Every element takes the updates
  // z_r -= L_rc z_c in ascending c with the fused form of c_fms, as the barrier version did.
  {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    cplx z0[DB_CW], z1[DB_CW];
#pragma unroll
    for (int q = 0; q < DB_CW; ++q) {
      z0[q] = Zs[lane][w * DB_CW + q];
      z1[q] = Zs[lane + 32][w * DB_CW + q];
    }
    for (int c = 0; c < nb - 1; ++c) {
      const cplx l0 = Ls[lane][c], l1 = Ls[lane + 32][c];
      const bool hi = c >= 32;
#pragma unroll
      for (int q = 0; q < DB_CW; ++q) {
        const cplx src = hi ? z1[q] : z0[q];
        cplx zc;
        zc.x = __shfl_sync(0xffffffffu, src.x, c & 31);
        zc.y = __shfl_sync(0xffffffffu, src.y, c & 31);
        if (lane > c) c_fms(z0[q], l0, zc);
        if (lane + 32 > c) c_fms(z1[q], l1, zc);
      }
    }
#pragma unroll
    for (int q = 0; q < DB_CW; ++q) {
      Zs[lane][w * DB_CW + q] = z0[q];
      Zs[lane + 32][w * DB_CW + q] = z1[q];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nb * DB_NC; e += DB_THREADS) {
    const int r = e / DB_NC, c = e % DB_NC;
    if (c0 + c < m) Z[(int64_t)(r0 + r) * m + c0 + c] = Zs[r][c];
  }
}

// backward: Z[r0:r0+64] = L_bb^-T Z[r0:r0+64]   (after the straddle fix)
__global__ void __launch_bounds__(DB_THREADS)
diag_bwd_kernel(const cplx* Fbase, int64_t stride_f, const int8_t* tagsbase, int64_t stride_t, cplx* Zbase,
                int64_t stride_z, int n, int m, int r0) {
  extern __shared__ __align__(16) unsigned char db_smem[];
  cplx(*Ls)[DB + 1] = reinterpret_cast<cplx(*)[DB + 1]>(db_smem);
  cplx(*Zs)[DB_NC] = reinterpret_cast<cplx(*)[DB_NC]>(db_smem + sizeof(cplx) * DB * (DB + 1));
  const int b = blockIdx.y;
  const cplx* F = Fbase + b * stride_f;
  const int8_t* tags = tagsbase + b * stride_t;
  cplx* Z = Zbase + b * stride_z;
  const int c0 = blockIdx.x * DB_NC;
  const int nb = min(DB, n - r0);
  for (int e = threadIdx.x; e < DB * DB; e += DB_THREADS) {
    const int r = e / DB, c = e % DB;
    cplx v = mk(0.0, 0.0);
    if (r < nb && c < r && !(r == c + 1 && tags[r0 + c] == 2)) v = F[(int64_t)(r0 + r) * n + r0 + c];
    Ls[r][c] = v;
  }
  for (int e = threadIdx.x; e < DB * DB_NC; e += DB_THREADS) {
    const int r = e / DB_NC, c = e % DB_NC;
    Zs[r][c] = (r < nb && c0 + c < m) ? Z[(int64_t)(r0 + r) * m + c0 + c] : mk(0.0, 0.0);
  }
  __syncthreads();
  const int r1 = r0 + nb;
  if (r1 < n && tags[r1 - 1] == 2 && threadIdx.x < DB_NC && c0 + threadIdx.x < m) {
    const cplx e = F[(int64_t)r1 * n + r1 - 1];
    c_fma(Zs[nb - 1][threadIdx.x], e, Z[(int64_t)r1 * m + c0 + threadIdx.x]);
  }
  __syncthreads();
  // (as the forward kernel: rows r < c take z_r -= L_cr z_c in descending c)
  {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    cplx z0[DB_CW], z1[DB_CW];
#pragma unroll
    for (int q = 0; q < DB_CW; ++q) {
      z0[q] = Zs[lane][w * DB_CW + q];
      z1[q] = Zs[lane + 32][w * DB_CW + q];
    }
    for (int c = nb - 1; c > 0; --c) {
      const cplx l0 = Ls[c][lane], l1 = Ls[c][lane + 32];
      const bool hi = c >= 32;
#pragma unroll
      for (int q = 0; q < DB_CW; ++q) {
        const cplx src = hi ? z1[q] : z0[q];
        cplx zc;
        zc.x = __shfl_sync(0xffffffffu, src.x, c & 31);
        zc.y = __shfl_sync(0xffffffffu, src.y, c & 31);
        if (lane < c) c_fms(z0[q], l0, zc);
        if (lane + 32 < c) c_fms(z1[q], l1, zc);
      }
    }
#pragma unroll
    for (int q = 0; q < DB_CW; ++q) {
      Zs[lane][w * DB_CW + q] = z0[q];
      Zs[lane + 32][w * DB_CW + q] = z1[q];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nb * DB_NC; e += DB_THREADS) {
    const int r = e / DB_NC, c = e % DB_NC;
    if (c0 + c < m) Z[(int64_t)(r0 + r) * m + c0 + c] = Zs[r][c];
  }
}

}  // namespace d3m

extern "C" int d3m_diag_block_launch(int fwd, const void* F, int64_t stride_f, const void* tags, int64_t stride_t,
                                     void* Z, int64_t stride_z, int n, int m, int r0, int batch, void* stream) {
  using namespace d3m;
  if (batch <= 0 || m <= 0 || r0 >= n) return 0;
  const dim3 grid((m + DB_NC - 1) / DB_NC, batch);
  auto s = reinterpret_cast<cudaStream_t>(stream);
  constexpr size_t smem = sizeof(cplx) * (DB * (DB + 1) + DB * DB_NC);
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(diag_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(diag_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cfg = true;
  }
  if (fwd)
    diag_fwd_kernel<<<grid, DB_THREADS, smem, s>>>(static_cast<const cplx*>(F), stride_f,
                                                static_cast<const int8_t*>(tags), stride_t, static_cast<cplx*>(Z),
                                                stride_z, n, m, r0);
  else
    diag_bwd_kernel<<<grid, DB_THREADS, smem, s>>>(static_cast<const cplx*>(F), stride_f,
                                                static_cast<const int8_t*>(tags), stride_t, static_cast<cplx*>(Z),
                                                stride_z, n, m, r0);
  return (int)cudaGetLastError();
}

int d3m_diag_block_rows() { return d3m::DB; }
