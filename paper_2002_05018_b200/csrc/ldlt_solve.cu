// ldlt_solve.cu -- triangular solves against a packed Bunch-Kaufman factor.
//
// Packed factor (kernels.py:7-22): strict lower triangle = unit L, except
// W[k+1, k] of a 2x2 pivot (tags[k] == 2) which holds the off-diagonal e[k]
// of D (the L entry there is zero); diagonal = d.  perm[i] = original index
// at position i.
//
// Kernels
//  * lsolve_fwd_kernel   Z = L^-1 Z (optionally U = D^-1 Z)   (kernels.py:149)
//  * lsolve_bwd_kernel   Z = L^-T Z                           (kernels.py:155)
//  * dinv_left_kernel    Z = D^-1 Z                           (kernels.py:161)
//  * gather/scatter rows by perm                              (factor.py:60-65)
//
// Reductions are split over a fixed 16-lane group per right-hand side with a
// fixed order, so each RHS column is computed identically whatever the
// number of columns in the call (block_solve's k-RHS == k x 1-RHS property,
// factor.py:271-279).  D^-1 uses the exact helpers (reference rounding).
#include <algorithm>
#include <cstdlib>
#include "d3m_common.cuh"
#include "d3m_kernels.h"

namespace d3m {

__device__ __forceinline__ cplx lfac(const cplx* F, int ld, const int8_t* tags, int r, int c) {
  // L[r][c] for c < r from the packed factor
  if (r == c + 1 && tags[c] == 2) return mk(0.0, 0.0);
  return F[(int64_t)r * ld + c];
}

// -------------------------------------------------------------------------
// Multi-RHS solves.  Z is a batch of n x m row-major arrays (ld = m); CTA =
// (RHS chunk of 16, batch index); 16 lanes per RHS column.
// -------------------------------------------------------------------------
constexpr int LS_THREADS = 256;
constexpr int LS_RHS = LS_THREADS / 16;


__global__ void __launch_bounds__(LS_THREADS) gather_rows_kernel(SolveBatch a) {
  // Z[i][c] = B[perm[i]][c]
  const int b = blockIdx.y;
  const int64_t total = (int64_t)a.n * a.m;
  const int64_t* perm = a.perm + b * a.stride_p;
  for (int64_t t = blockIdx.x * (int64_t)LS_THREADS + threadIdx.x; t < total; t += (int64_t)gridDim.x * LS_THREADS) {
    const int i = (int)(t / a.m), c = (int)(t % a.m);
    a.Z[b * a.stride_z + (int64_t)i * a.ldz + c] = a.B[b * a.stride_b + perm[i] * a.ldb + c];
  }
}

__global__ void __launch_bounds__(LS_THREADS) scatter_rows_kernel(SolveBatch a) {
  // B[perm[i]][c] = Z[i][c]
  const int b = blockIdx.y;
  const int64_t total = (int64_t)a.n * a.m;
  const int64_t* perm = a.perm + b * a.stride_p;
  for (int64_t t = blockIdx.x * (int64_t)LS_THREADS + threadIdx.x; t < total; t += (int64_t)gridDim.x * LS_THREADS) {
    const int i = (int)(t / a.m), c = (int)(t % a.m);
    cplx* dst = const_cast<cplx*>(a.B) + b * a.stride_b + perm[i] * a.ldb + c;
    *dst = a.Z[b * a.stride_z + (int64_t)i * a.ldz + c];
  }
}

__global__ void __launch_bounds__(LS_THREADS) lsolve_fwd_kernel(SolveBatch a) {
  const int b = blockIdx.y;
  const int g = threadIdx.x >> 4, s = threadIdx.x & 15;
  const int col = blockIdx.x * LS_RHS + g;
  const bool live = col < a.m;
  const int n = a.n;
  const cplx* F = a.F + b * a.stride_f;
  const int8_t* tags = a.tags + b * a.stride_t;
  cplx* Z = a.Z + b * a.stride_z + col;
  const int ldz = a.ldz;
  for (int c = 1; c < n; ++c) {
    cplx acc = mk(0.0, 0.0);
    if (live) {
      const cplx* Lr = F + (int64_t)c * n;
      for (int cp = s; cp < c; cp += 16) {
        const cplx l = (cp == c - 1 && tags[cp] == 2) ? mk(0.0, 0.0) : __ldg(Lr + cp);
        c_fma(acc, l, Z[(int64_t)cp * ldz]);
      }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o, 16);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o, 16);
    }
    if (live && s == 0) Z[(int64_t)c * ldz] = c_sub(Z[(int64_t)c * ldz], acc);
    __syncwarp();
  }
  if (!live || a.U == nullptr) return;
  cplx* U = a.U + b * a.stride_u + col;
  for (int c = s; c < n; c += 16) {
    const int8_t t = tags[c];
    if (t == 1) {
      U[(int64_t)c * ldz] = x_div_np(Z[(int64_t)c * ldz], F[(int64_t)c * n + c]);
    } else if (t == 2) {
      cplx x0 = Z[(int64_t)c * ldz], x1 = Z[(int64_t)(c + 1) * ldz];
      dinv_pair(F[(int64_t)c * n + c], F[(int64_t)(c + 1) * n + c], F[(int64_t)(c + 1) * n + c + 1], x0, x1);
      U[(int64_t)c * ldz] = x0;
      U[(int64_t)(c + 1) * ldz] = x1;
    }
  }
}

__global__ void __launch_bounds__(LS_THREADS) lsolve_bwd_kernel(SolveBatch a) {
  const int b = blockIdx.y;
  const int g = threadIdx.x >> 4, s = threadIdx.x & 15;
  const int col = blockIdx.x * LS_RHS + g;
  const bool live = col < a.m;
  const int n = a.n;
  const cplx* F = a.F + b * a.stride_f;
  const int8_t* tags = a.tags + b * a.stride_t;
  cplx* Z = a.Z + b * a.stride_z + col;
  const int ldz = a.ldz;
  for (int c = n - 2; c >= 0; --c) {
    cplx acc = mk(0.0, 0.0);
    if (live) {
      for (int i = c + 1 + s; i < n; i += 16) {
        const cplx l = (i == c + 1 && tags[c] == 2) ? mk(0.0, 0.0) : __ldg(F + (int64_t)i * n + c);
        c_fma(acc, l, Z[(int64_t)i * ldz]);
      }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o, 16);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o, 16);
    }
    if (live && s == 0) Z[(int64_t)c * ldz] = c_sub(Z[(int64_t)c * ldz], acc);
    __syncwarp();
  }
}

__global__ void __launch_bounds__(LS_THREADS) dinv_left_kernel(SolveBatch a) {
  // Z = D^-1 Z in place; one thread per (row, column), 2x2 pairs handled by
  // the thread of the first row.
  const int b = blockIdx.y;
  const int64_t total = (int64_t)a.n * a.m;
  const cplx* F = a.F + b * a.stride_f;
  const int8_t* tags = a.tags + b * a.stride_t;
  const int n = a.n;
  for (int64_t t = blockIdx.x * (int64_t)LS_THREADS + threadIdx.x; t < total; t += (int64_t)gridDim.x * LS_THREADS) {
    const int c = (int)(t / a.m), col = (int)(t % a.m);
    cplx* Z = a.Z + b * a.stride_z + col;
    const int8_t tg = tags[c];
    if (tg == 1) {
      Z[(int64_t)c * a.ldz] = x_div_np(Z[(int64_t)c * a.ldz], F[(int64_t)c * n + c]);
    } else if (tg == 2) {
      cplx x0 = Z[(int64_t)c * a.ldz], x1 = Z[(int64_t)(c + 1) * a.ldz];
      dinv_pair(F[(int64_t)c * n + c], F[(int64_t)(c + 1) * n + c], F[(int64_t)(c + 1) * n + c + 1], x0, x1);
      Z[(int64_t)c * a.ldz] = x0;
      Z[(int64_t)(c + 1) * a.ldz] = x1;
    }
  }
}

}  // namespace d3m


// phase: 0 gather, 1 forward (+U), 2 dinv, 3 backward, 4 scatter
extern "C" int d3m_solve_phase_launch(int phase, d3m::SolveBatch* a, int batch, void* stream) {
  using namespace d3m;
  if (batch <= 0 || a->n <= 0 || a->m <= 0) return 0;
  auto s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t total = (int64_t)a->n * a->m;
  const int flat_blocks = (int)std::min<int64_t>((total + LS_THREADS - 1) / LS_THREADS, 4096);
  const dim3 gflat(flat_blocks, batch);
  const dim3 grhs((a->m + LS_RHS - 1) / LS_RHS, batch);
  switch (phase) {
    case 0: gather_rows_kernel<<<gflat, LS_THREADS, 0, s>>>(*a); break;
    case 1: lsolve_fwd_kernel<<<grhs, LS_THREADS, 0, s>>>(*a); break;
    case 2: dinv_left_kernel<<<gflat, LS_THREADS, 0, s>>>(*a); break;
    case 3: lsolve_bwd_kernel<<<grhs, LS_THREADS, 0, s>>>(*a); break;
    case 4: scatter_rows_kernel<<<gflat, LS_THREADS, 0, s>>>(*a); break;
    default: return -22;
  }
  return (int)cudaGetLastError();
}

namespace d3m {

// -------------------------------------------------------------------------
// Binv = L^-1 P of a packed factor (n <= 1024), written row-major n x n:
// column q of L^-1 (forward substitution of e_q) lands in column perm[q].
// With it the panel TRSM is one DMMA GEMM,  X_ij = K_ij P^T L^-T =
// K_ij Binv^T, and the block substitutions are GEMMs:  z = Binv b,
// x = Binv^T w.  CTA = 16 columns (one 16-lane group each); the 16 columns
// of L^-1 live in shared memory (column-major per group), rows of L are
// streamed through a double-buffered cp.async ring of INV_ROWS rows.
// -------------------------------------------------------------------------
constexpr int INV_THREADS = 256;
constexpr int INV_COLS = INV_THREADS / 16;
constexpr int INV_ROWS = 4;   // (16 + 2*4) n complex of smem: fits beside one GEMM CTA at n = 256

__device__ __forceinline__ void cp_async16_pred(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(pred ? 16 : 0));
}

__global__ void __launch_bounds__(INV_THREADS)
tri_inv_kernel(const cplx* Fbase, int64_t stride_f, const int64_t* permbase, int64_t stride_p,
               const int8_t* tagsbase, int64_t stride_t, cplx* Binv_base, int64_t stride_b, int n) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = blockIdx.y;
  const cplx* F = Fbase + b * stride_f;
  const int64_t* perm = permbase + b * stride_p;
  const int8_t* tags = tagsbase + b * stride_t;
  cplx* Binv = Binv_base + b * stride_b;
  const int q0 = blockIdx.x * INV_COLS;
  const int g = threadIdx.x >> 4, s = threadIdx.x & 15;
  const int q = q0 + g;
  const int w = n - q0;                          // rows/cols touched by this CTA
  cplx* Y = reinterpret_cast<cplx*>(smem_raw);   // [INV_COLS][w]
  cplx* Lr = Y + (size_t)INV_COLS * w;           // [2][INV_ROWS][w]
  cplx* y = Y + (size_t)g * w;                   // this group's column, index c - q0
  for (int c = s; c < w; c += 16) y[c] = mk(q0 + c == q ? 1.0 : 0.0, 0.0);

  auto load_chunk = [&](int chunk, int buf) {
    // rows q0 + chunk*INV_ROWS + r, columns q0 .. q0 + w - 1 (strict lower part)
    cplx* dst = Lr + (size_t)buf * INV_ROWS * w;
    for (int e = threadIdx.x; e < INV_ROWS * w; e += INV_THREADS) {
      const int r = e / w, c = e - r * w;
      const int row = q0 + chunk * INV_ROWS + r, col = q0 + c;
      const bool ok = row < n && col < row;
      cp_async16_pred(dst + e, ok ? F + (int64_t)row * n + col : F, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  const int nchunks = (w + INV_ROWS - 1) / INV_ROWS;
  load_chunk(0, 0);
  for (int ch = 0; ch < nchunks; ++ch) {
    if (ch + 1 < nchunks) load_chunk(ch + 1, (ch + 1) & 1);
    else asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();
    const cplx* L = Lr + (size_t)(ch & 1) * INV_ROWS * w;
    for (int r = 0; r < INV_ROWS; ++r) {
      const int c = ch * INV_ROWS + r;           // local row index
      if (c >= w) break;
      const cplx* Lc = L + (size_t)r * w;
      cplx acc = mk(0.0, 0.0);
      const int lo = q - q0;                     // y[c'] = 0 below q
      for (int cp = lo + s; cp < c; cp += 16) {
        cplx l = Lc[cp];
        if (cp == c - 1 && tags[q0 + cp] == 2) l = mk(0.0, 0.0);
        c_fma(acc, l, y[cp]);
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o, 16);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o, 16);
      }
      if (s == 0 && c > lo && q < n) y[c] = mk(-acc.x, -acc.y);
      __syncwarp();
    }
    __syncthreads();
  }
  if (q >= n) return;
  const int64_t pc = perm[q];
  for (int row = s; row < n; row += 16)
    Binv[(int64_t)row * n + pc] = row < q0 ? mk(0.0, 0.0) : y[row - q0];
}

// L_panel rows = X rows * D^-1 (apply_dinv_right, kernels.py:184-202);
// one thread per (row, pivot block).
__global__ void dinv_rows_kernel(const cplx* X, cplx* P, int64_t R, int n, const cplx* F, const int8_t* tags) {
  const int64_t total = R * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n;
    const int c = (int)(e - r * n);
    const int8_t t = tags[c];
    if (t == 1) {
      P[r * n + c] = x_div_np(X[r * n + c], F[(int64_t)c * n + c]);
    } else if (t == 2) {
      cplx x0 = X[r * n + c], x1 = X[r * n + c + 1];
      dinv_pair(F[(int64_t)c * n + c], F[(int64_t)(c + 1) * n + c], F[(int64_t)(c + 1) * n + c + 1], x0, x1);
      P[r * n + c] = x0;
      P[r * n + c + 1] = x1;
    }
  }
}

// U = D^-1 Z (apply_dinv_left, kernels.py:161-181), Z and U n x m (ld m)
__global__ void dinv_left_copy_kernel(const cplx* Z, cplx* U, int n, int m, const cplx* F, const int8_t* tags) {
  const int64_t total = (int64_t)n * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / m), col = (int)(e % m);
    const int8_t t = tags[c];
    if (t == 1) {
      U[e] = x_div_np(Z[e], F[(int64_t)c * n + c]);
    } else if (t == 2) {
      cplx x0 = Z[e], x1 = Z[e + m];
      dinv_pair(F[(int64_t)c * n + c], F[(int64_t)(c + 1) * n + c], F[(int64_t)(c + 1) * n + c + 1], x0, x1);
      U[e] = x0;
      U[e + m] = x1;
    }
    (void)col;
  }
}

// out = u - sum_{p < np} partial[p]  (fixed order), each of length len
}  // namespace d3m

extern "C" int d3m_tri_inv_launch(const void* F, int64_t stride_f, const void* perm, int64_t stride_p,
                                  const void* tags, int64_t stride_t, void* Binv, int64_t stride_b, int n, int batch,
                                  void* stream) {
  using namespace d3m;
  if (n <= 0 || batch <= 0) return 0;
  const size_t smem = (size_t)(INV_COLS + 2 * INV_ROWS) * n * sizeof(cplx);
  if (smem > 227 * 1024) return -22;
  static int configured = 0;
  if (!configured) {
    cudaFuncSetAttribute(tri_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = 1;
  }
  const dim3 grid((n + INV_COLS - 1) / INV_COLS, batch);
  tri_inv_kernel<<<grid, INV_THREADS, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const cplx*>(F), stride_f, static_cast<const int64_t*>(perm), stride_p,
      static_cast<const int8_t*>(tags), stride_t, static_cast<cplx*>(Binv), stride_b, n);
  return (int)cudaGetLastError();
}

extern "C" int d3m_dinv_rows_launch(const void* X, void* P, int64_t R, int n, const void* F, const void* tags,
                                    void* stream) {
  using namespace d3m;
  if (R <= 0 || n <= 0) return 0;
  const int64_t total = R * n;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8192);
  dinv_rows_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const cplx*>(X), static_cast<cplx*>(P), R, n, static_cast<const cplx*>(F),
      static_cast<const int8_t*>(tags));
  return (int)cudaGetLastError();
}

extern "C" int d3m_dinv_left_copy_launch(const void* Z, void* U, int n, int m, const void* F, const void* tags,
                                         void* stream) {
  using namespace d3m;
  if (n <= 0 || m <= 0) return 0;
  const int64_t total = (int64_t)n * m;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
  dinv_left_copy_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const cplx*>(Z), static_cast<cplx*>(U), n, m, static_cast<const cplx*>(F),
      static_cast<const int8_t*>(tags));
  return (int)cudaGetLastError();
}

namespace d3m {

// -------------------------------------------------------------------------
// Warp-per-column L^-1 P (n <= 32*NPER): lane l keeps y[l + 32t] and the
// current L row's L[c][l + 32t] in registers, the next row is prefetched
// while the current step reduces, one warp reduction per elimination step.
// Lane 0 of the warp owning column q also writes the D^-1 coefficients of
// pivot column q used by the panel's L = X D^-1 pass:
//   1x1: coef[q] = (1/d, 0, 0);   2x2 starting at q: coef[q] = (p, s, r) with
//   [[a, b], [b, c]]^-1 = [[p, s], [s, r]];   second column of a 2x2: unused.
// -------------------------------------------------------------------------
template <int NPER>
__global__ void __launch_bounds__(256)
tri_inv_warp_kernel(const cplx* __restrict__ F, const int64_t* __restrict__ perm, const int8_t* __restrict__ tags,
                    cplx* Binv, cplx* coef, int n, cplx* Linv) {
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (q >= n) return;
  cplx y[NPER], lr[NPER], nx[NPER];
#pragma unroll
  for (int t = 0; t < NPER; ++t) y[t] = mk(lane + 32 * t == q ? 1.0 : 0.0, 0.0);
  auto load_row = [&](int c, cplx* dst) {
#pragma unroll
    for (int t = 0; t < NPER; ++t) {
      const int cp = lane + 32 * t;
      dst[t] = (c < n && cp >= q && cp < c) ? __ldg(F + (int64_t)c * n + cp) : mk(0.0, 0.0);
    }
  };
  if (q + 1 < n) load_row(q + 1, lr);
  for (int c = q + 1; c < n; ++c) {
    load_row(c + 1, nx);                          // prefetch the next row
    if (tags[c - 1] == 2) {                       // L[c][c-1] of a 2x2 pivot is zero
#pragma unroll
      for (int t = 0; t < NPER; ++t)
        if (lane + 32 * t == c - 1) lr[t] = mk(0.0, 0.0);
    }
    cplx acc = mk(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < NPER; ++t) c_fma(acc, lr[t], y[t]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
#pragma unroll
    for (int t = 0; t < NPER; ++t)
      if (lane + 32 * t == c) y[t] = mk(-acc.x, -acc.y);
#pragma unroll
    for (int t = 0; t < NPER; ++t) lr[t] = nx[t];
  }
  const int64_t pc = perm[q];
#pragma unroll
  for (int t = 0; t < NPER; ++t) {
    const int row = lane + 32 * t;
    if (row < n) {
      Binv[(int64_t)row * n + pc] = row < q ? mk(0.0, 0.0) : y[t];
      if (Linv) Linv[(int64_t)row * n + q] = row < q ? mk(0.0, 0.0) : y[t];
    }
  }
  if (lane == 0 && coef != nullptr) {
    const int8_t tg = tags[q];
    if (tg == 1) {
      coef[3 * q] = x_div_np(mk(1.0, 0.0), F[(int64_t)q * n + q]);
    } else if (tg == 2) {
      const cplx a = F[(int64_t)q * n + q], b = F[(int64_t)(q + 1) * n + q], c = F[(int64_t)(q + 1) * n + q + 1];
      const cplx det = c_sub(c_mul(a, c), c_mul(b, b));
      const cplx inv = x_div_np(mk(1.0, 0.0), det);
      coef[3 * q] = c_mul(c, inv);                              // p
      coef[3 * q + 1] = c_mul(mk(-b.x, -b.y), inv);             // s
      coef[3 * q + 2] = c_mul(a, inv);                          // r
    }
  }
}

// L rows = X rows D^-1 with the precomputed coefficients (row-vectorised)
__global__ void dinv_rows_coef_kernel(const cplx* __restrict__ X, cplx* P, int64_t R, int n,
                                      const int8_t* __restrict__ tags, const cplx* __restrict__ coef) {
  const int64_t total = R * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n;
    const int c = (int)(e - r * n);
    const int8_t t = tags[c];
    if (t == 1) {
      P[e] = c_mul(X[e], coef[3 * c]);
    } else if (t == 2) {
      const cplx x0 = X[e], x1 = X[e + 1];
      const cplx p = coef[3 * c], s = coef[3 * c + 1], q = coef[3 * c + 2];
      P[e] = c_add(c_mul(x0, p), c_mul(x1, s));
      P[e + 1] = c_add(c_mul(x0, s), c_mul(x1, q));
    }
    (void)r;
  }
}

}  // namespace d3m

namespace d3m {

// -------------------------------------------------------------------------
// Blocked L^-1 P for n <= 256 (the diagonal blocks of block_ldlt, on the
// critical chain of every block column).  The warp-per-column kernel walks
// n dependent rows per column with one L2 round trip and one warp reduction
// each (~150 us at n = 256); here the chain is n/16 block steps:
//   tri_inv_diag16:  Dinv_i = L_ii^-1 of every 16 x 16 diagonal block (+ the
//                    D^-1 coefficients, as the warp kernel)
//   tri_inv_colq:    one CTA per column q of X = L^-1:
//                    X_kk = Dinv_k;  X_ik = -Dinv_i (sum_{k<=m<i} L_im X_mk)
//                    (a per-block-column CTA version, 2x slower on the
//                    critical chain, was removed)
// L(i, j) is the packed factor's strict lower part with the sub-diagonal of
// every 2 x 2 pivot read as zero (kernels.py:123-125 stores e there).
// -------------------------------------------------------------------------
constexpr int TI_B = 16;

__device__ __forceinline__ cplx ti_L(const cplx* F, const int8_t* tags, int n, int r, int c) {
  if (r == c + 1 && tags[c] == 2) return mk(0.0, 0.0);
  return F[(int64_t)r * n + c];
}

__global__ void __launch_bounds__(64) tri_inv_diag16(const cplx* __restrict__ F, const int8_t* __restrict__ tags,
                                                     cplx* Dinv, cplx* coef, int n) {
  __shared__ cplx Ls[TI_B][TI_B];
  const int i = blockIdx.x, r0 = i * TI_B, nb = min(TI_B, n - r0);
  for (int e = threadIdx.x; e < TI_B * TI_B; e += 64) {
    const int r = e / TI_B, c = e % TI_B;
    Ls[r][c] = (r < nb && c < r) ? ti_L(F, tags, n, r0 + r, r0 + c) : mk(0.0, 0.0);
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < TI_B) {                     // column t of L_ii^-1 by substitution
    cplx x[TI_B];
#pragma unroll
    for (int r = 0; r < TI_B; ++r) {
      cplx acc = mk(r == t ? 1.0 : 0.0, 0.0);
#pragma unroll
      for (int c = 0; c < r; ++c) {
        const cplx l = Ls[r][c];
        acc = mk(acc.x - (l.x * x[c].x - l.y * x[c].y), acc.y - (l.x * x[c].y + l.y * x[c].x));
      }
      x[r] = acc;
    }
#pragma unroll
    for (int r = 0; r < TI_B; ++r) Dinv[((int64_t)i * TI_B + r) * TI_B + t] = x[r];
  } else if (t < 2 * TI_B && coef != nullptr) {
    const int q = r0 + t - TI_B;
    if (q < n) {
      const int8_t tg = tags[q];
      if (tg == 1) {
        coef[3 * q] = x_div_np(mk(1.0, 0.0), F[(int64_t)q * n + q]);
      } else if (tg == 2) {
        const cplx a = F[(int64_t)q * n + q], b = F[(int64_t)(q + 1) * n + q], c = F[(int64_t)(q + 1) * n + q + 1];
        const cplx det = c_sub(c_mul(a, c), c_mul(b, b));
        const cplx inv = x_div_np(mk(1.0, 0.0), det);
        coef[3 * q] = c_mul(c, inv);
        coef[3 * q + 1] = c_mul(mk(-b.x, -b.y), inv);
        coef[3 * q + 2] = c_mul(a, inv);
      }
    }
  }
}

constexpr int TI_NMAX = 256;
// One CTA per column q of X = L^-1 (n CTAs): the column's 16-row blocks
// below the diagonal block are the dependent chain (at most 15 steps at
// n = 256), each step a 16-row dot over the rows already solved (16 lanes per
// row, butterfly) and the 16 x 16 product with Dinv_i.  Spreads the block
// columns' work over n SMs instead of n/16.
__global__ void __launch_bounds__(256) tri_inv_colq(const cplx* __restrict__ F, const int64_t* __restrict__ perm,
                                                    const int8_t* __restrict__ tags, const cplx* __restrict__ Dinv,
                                                    cplx* Binv, cplx* Linv, int n) {
  __shared__ cplx xs[TI_NMAX];
  __shared__ cplx sv[TI_B];
  const int q = blockIdx.x, k = q / TI_B, c0 = k * TI_B, tid = threadIdx.x;
  const int nbk = (n + TI_B - 1) / TI_B;
  const int r = tid >> 4, l16 = tid & 15;
  for (int i = tid; i < n; i += 256) xs[i] = mk(0.0, 0.0);
  __syncthreads();
  if (tid < TI_B && c0 + tid < n) xs[c0 + tid] = Dinv[((int64_t)k * TI_B + tid) * TI_B + (q - c0)];
  __syncthreads();
  for (int i = k + 1; i < nbk; ++i) {
    const int row = i * TI_B + r, w = TI_B * (i - k);
    cplx a = mk(0.0, 0.0);
    if (row < n) {
      const cplx* Lr = F + (int64_t)row * n + c0;
      const bool zr = r == 0 && tags[i * TI_B - 1] == 2;     // L[16i, 16i-1] of a 2x2 pivot
      // all of this lane's L loads first (one memory round trip per step), then the sum
      cplx lv[TI_NMAX / TI_B];
#pragma unroll
      for (int j = 0; j < TI_NMAX / TI_B; ++j) {
        const int m = l16 + TI_B * j;
        lv[j] = m < w ? Lr[m] : mk(0.0, 0.0);
      }
#pragma unroll
      for (int j = 0; j < TI_NMAX / TI_B; ++j) {
        const int m = l16 + TI_B * j;
        if (m >= w) break;
        cplx l = lv[j];
        if (zr && m == w - 1) l = mk(0.0, 0.0);
        const cplx x = xs[c0 + m];
        a = mk(a.x + (l.x * x.x - l.y * x.y), a.y + (l.x * x.y + l.y * x.x));
      }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
      a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
    }
    if (l16 == 0) sv[r] = a;
    __syncthreads();
    if (tid < TI_B) {
      const cplx* Di = Dinv + ((int64_t)i * TI_B + tid) * TI_B;
      cplx acc = mk(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < TI_B; ++c) {
        const cplx d = Di[c], t = sv[c];
        acc = mk(acc.x + (d.x * t.x - d.y * t.y), acc.y + (d.x * t.y + d.y * t.x));
      }
      if (i * TI_B + tid < n) xs[i * TI_B + tid] = mk(-acc.x, -acc.y);
    }
    __syncthreads();
  }
  const int64_t pc = perm[q];
  for (int row = tid; row < n; row += 256) {
    const cplx v = xs[row];
    Binv[(int64_t)row * n + pc] = v;
    if (Linv) Linv[(int64_t)row * n + q] = v;
  }
}

}  // namespace d3m

// blocked L^-1 P + D^-1 coefficients for n <= 256 (-22 above); dinv: scratch
// of 256 x 16 complex (the 16 x 16 diagonal-block inverses), owned by the
// caller's per-device context
extern "C" int d3m_tri_inv_blocked_launch(const void* F, const void* perm, const void* tags, void* Binv, void* coef,
                                          int n, void* Linv, void* dinv, void* stream) {
  using namespace d3m;
  if (n <= 0) return 0;
  if (n > TI_NMAX || dinv == nullptr) return -22;
  auto s = reinterpret_cast<cudaStream_t>(stream);
  const int nbk = (n + TI_B - 1) / TI_B;
  auto Fp = static_cast<const cplx*>(F);
  auto tp = static_cast<const int8_t*>(tags);
  auto Dp = static_cast<cplx*>(dinv);
  tri_inv_diag16<<<nbk, 64, 0, s>>>(Fp, tp, Dp, static_cast<cplx*>(coef), n);
  tri_inv_colq<<<n, 256, 0, s>>>(Fp, static_cast<const int64_t*>(perm), tp, Dp, static_cast<cplx*>(Binv),
                                 static_cast<cplx*>(Linv), n);
  return (int)cudaGetLastError();
}

// warp-per-column inverse for n <= 512 (returns -22 above: use d3m_tri_inv_launch)
extern "C" int d3m_tri_inv_warp_launch(const void* F, const void* perm, const void* tags, void* Binv, void* coef,
                                       int n, void* stream, void* Linv) {
  using namespace d3m;
  if (n <= 0) return 0;
  const dim3 grid((n + 7) / 8);
  auto s = reinterpret_cast<cudaStream_t>(stream);
  auto Fp = static_cast<const cplx*>(F);
  auto pp = static_cast<const int64_t*>(perm);
  auto tp = static_cast<const int8_t*>(tags);
  if (n <= 256) tri_inv_warp_kernel<8><<<grid, 256, 0, s>>>(Fp, pp, tp, static_cast<cplx*>(Binv), static_cast<cplx*>(coef), n,
                                                static_cast<cplx*>(Linv));
  else if (n <= 512) tri_inv_warp_kernel<16><<<grid, 256, 0, s>>>(Fp, pp, tp, static_cast<cplx*>(Binv), static_cast<cplx*>(coef), n,
                                                 static_cast<cplx*>(Linv));
  else return -22;
  return (int)cudaGetLastError();
}

extern "C" int d3m_dinv_rows_coef_launch(const void* X, void* P, int64_t R, int n, const void* tags, const void* coef,
                                         void* stream) {
  using namespace d3m;
  if (R <= 0 || n <= 0) return 0;
  const int64_t total = R * n;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 16384);
  dinv_rows_coef_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const cplx*>(X), static_cast<cplx*>(P), R, n, static_cast<const int8_t*>(tags),
      static_cast<const cplx*>(coef));
  return (int)cudaGetLastError();
}
