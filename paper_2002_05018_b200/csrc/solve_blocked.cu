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
  for (int c = 0; c < nb - 1; ++c) {
    for (int e = threadIdx.x; e < (nb - 1 - c) * DB_NC; e += DB_THREADS) {
      const int r = c + 1 + e / DB_NC, cc = e % DB_NC;
      c_fms(Zs[r][cc], Ls[r][c], Zs[c][cc]);
    }
    __syncthreads();
  }
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
  for (int c = nb - 1; c > 0; --c) {
    for (int e = threadIdx.x; e < c * DB_NC; e += DB_THREADS) {
      const int r = e / DB_NC, cc = e % DB_NC;   // rows r < c
      c_fms(Zs[r][cc], Ls[c][r], Zs[c][cc]);
    }
    __syncthreads();
  }
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
