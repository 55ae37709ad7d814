// d3m_capi.cu -- the extern "C" boundary of libd3m (declared in include/d3m.h).
//
// All array arguments are DEVICE pointers unless named h_*; complex arrays are
// interleaved complex128.  Every entry point is asynchronous on the given
// stream and returns 0, a negative errno-like code for invalid arguments, or
// a positive cudaError_t.  Pivot outcomes (info) are written to device
// arrays; the caller raises the reference's exceptions from them.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "d3m_common.cuh"
#include "d3m_gemm.h"
#include "d3m_misc.h"
#include "d3m_kernels.h"
#include "../../include/d3m.h"


namespace {
thread_local std::string g_err;
int fail(int code, const char* what) {
  g_err = what;
  return code;
}
#define D3M_TRY(expr)                                                        \
  do {                                                                       \
    int _rc = (expr);                                                        \
    if (_rc != 0) {                                                          \
      char _b[256];                                                          \
      snprintf(_b, sizeof(_b), "%s failed with %d (%s)", #expr, _rc,        \
               _rc > 0 ? cudaGetErrorString((cudaError_t)_rc) : "invalid"); \
      g_err = _b;                                                            \
      return _rc;                                                            \
    }                                                                        \
  } while (0)

using d3m::cplx;
inline cplx* C(void* p) { return static_cast<cplx*>(p); }
inline const cplx* CC(const void* p) { return static_cast<const cplx*>(p); }

}  // namespace

extern "C" {

int d3m_abi_version(void) { return D3M_ABI_VERSION; }

const char* d3m_last_error(void) { return g_err.c_str(); }

int d3m_bk_factor_batched(int batch, int n, void* W, int64_t stride_w, int lda, double pivot_tol, int check_sym,
                          void* perm, void* tags, void* n2x2, void* growth, void* info, void* scale, void* asym,
                          void* scratch, void* stream) {
  if (batch < 0 || n < 0 || lda < n) return fail(-22, "d3m_bk_factor_batched: bad shape");
  d3m::BkArgs a{C(W), stride_w, n, lda, pivot_tol, check_sym, static_cast<int64_t*>(perm), static_cast<int8_t*>(tags),
                static_cast<int32_t*>(n2x2), static_cast<double*>(growth), static_cast<int32_t*>(info),
                static_cast<double*>(scale), static_cast<double*>(asym), C(scratch)};
  D3M_TRY(d3m_bk_launch(&a, batch, stream));
  return 0;
}

int d3m_ldlt_solve_batched(int batch, int n, const void* F, int64_t stride_f, const void* perm, int64_t stride_p,
                           const void* tags, int64_t stride_t, void* B, int64_t stride_b, int ldb, int m, void* work,
                           void* stream) {
  if (batch < 0 || n < 0 || m < 0 || ldb < m) return fail(-22, "d3m_ldlt_solve_batched: bad shape");
  if (batch == 0 || n == 0 || m == 0) return 0;
  d3m::SolveBatch s{CC(F), stride_f, static_cast<const int8_t*>(tags), stride_t, static_cast<const int64_t*>(perm),
                    stride_p, C(work), (int64_t)n * m, nullptr, 0, CC(B), stride_b, n, m, m, ldb};
  D3M_TRY(d3m_solve_phase_launch(0, &s, batch, stream));   // Z = B[perm]
  D3M_TRY(d3m_solve_phase_launch(1, &s, batch, stream));   // Z = L^-1 Z
  D3M_TRY(d3m_solve_phase_launch(2, &s, batch, stream));   // Z = D^-1 Z
  D3M_TRY(d3m_solve_phase_launch(3, &s, batch, stream));   // Z = L^-T Z
  D3M_TRY(d3m_solve_phase_launch(4, &s, batch, stream));   // B[perm] = Z
  return 0;
}

int d3m_zgemm_grouped(int ta, int tb, const void* A, const void* B, void* Cm, void* h_tasks, int ntasks,
                      void* d_tasks, void* stream) {
  if (ntasks <= 0) return 0;
  auto* t = static_cast<d3m::GemmTask*>(h_tasks);
  const int tiles = d3m_gemm_prepare_tasks(t, ntasks);
  cudaError_t e = cudaMemcpyAsync(d_tasks, t, sizeof(d3m::GemmTask) * ntasks, cudaMemcpyHostToDevice,
                                  reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail((int)e, "d3m_zgemm_grouped: task upload");
  D3M_TRY(d3m_gemm_launch(ta, tb, A, B, Cm, d_tasks, ntasks, tiles, stream));
  return 0;
}

int d3m_schur_reduce_batched(int batch, int n, int m, void* A, const void* D, const void* f, double pivot_tol,
                             void* perm, void* tags, void* n2x2, void* growth, void* info, void* scale, void* asym,
                             void* K_out, void* g_out, void* work_z, void* work_x, void* work_c, void* bk_scratch,
                             void* d_tasks, void* stream) {
  // A: batch x n x n (factored in place -> packed factor); D: batch x n x m;
  // f: batch x n; work_z, work_x: batch x n x (m+1); work_c: batch x m x (m+1)
  if (batch < 0 || n < 0 || m < 0) return fail(-22, "d3m_schur_reduce_batched: bad shape");
  if (batch == 0) return 0;
  const int64_t nn = (int64_t)n * n, nm1 = (int64_t)n * (m + 1);
  D3M_TRY(d3m_bk_factor_batched(batch, n, A, nn, n, pivot_tol, 1, perm, tags, n2x2, growth, info, scale, asym,
                                bk_scratch, stream));
  if (n == 0) return 0;
  // RHS = [D | f]  (subdomain.py:177-179), X = A^-1 RHS (factor.py:52-66)
  D3M_TRY(d3m_pack_rhs_launch(D, f, work_x, n, m, batch, (int64_t)n * m, n, nm1, stream));
  D3M_TRY(d3m_ldlt_solve_batched(batch, n, A, nn, perm, n, tags, n, work_x, nm1, m + 1, m + 1, work_z, stream));
  if (m == 0) return 0;
  // C = D^T [X | x_f]  (subdomain.py:181,183) on DMMA, one task per domain
  std::vector<d3m::GemmTask> t(batch);
  for (int b = 0; b < batch; ++b) {
    d3m::GemmTask& k = t[b];
    std::memset(&k, 0, sizeof(k));
    k.a_off = (int64_t)b * n * m;          // D stored n x m = K x M  (TA)
    k.b_off = (int64_t)b * nm1;            // X stored n x (m+1) = K x N (TB)
    k.c_off = (int64_t)b * m * (m + 1);
    k.m = m;
    k.n = m + 1;
    k.k = n;
    k.lda = m;
    k.ldb = m + 1;
    k.ldc = m + 1;
    k.flags = d3m::kGemmStore;
  }
  D3M_TRY(d3m_zgemm_grouped(1, 1, D, work_x, work_c, t.data(), batch, d_tasks, stream));
  // K_D = 0.5 (K_D + K_D^T), g_d
  D3M_TRY(d3m_schur_finalize_launch(work_c, K_out, g_out, m, batch, (int64_t)m * (m + 1), (int64_t)m * m, m, stream));
  return 0;
}

int d3m_block_copy(const void* src, void* dst, const void* d_tasks, int ntasks, int64_t max_elems, void* stream) {
  D3M_TRY(d3m_block_copy_launch(src, dst, d_tasks, ntasks, max_elems, stream));
  return 0;
}

int d3m_gather_rows(const void* src, const void* idx, void* out, int64_t nrows, int cols, void* stream) {
  D3M_TRY(d3m_gather_index_launch(src, idx, out, nrows, cols, stream));
  return 0;
}

int d3m_ordered_average(const void* E, const void* ptr, const void* src, void* out, int64_t ng, void* stream) {
  D3M_TRY(d3m_ordered_average_launch(E, ptr, src, out, ng, stream));
  return 0;
}

int d3m_zero(void* p, int64_t n, void* stream) {
  D3M_TRY(d3m_zero_launch(p, n, stream));
  return 0;
}

// ---------------------------------------------------------------------------
// block_ldlt executor (factor.py:154-240).
//
// Device pool layout (built by the host planner): per block column j a
// diagonal slot (n_j x n_j, packed BK factor after the call) and a panel
// (R_j x n_j) stacking the pattern blocks i in ascending order; the panel
// holds W_ij on entry and L_ij on exit.  GEMM tasks of column j are split in
// "next" (targets in column j+1) and "rest"; the next column's BK + TRSM run
// on the caller's stream while the rest of column j's trailing update runs on
// a helper stream (lookahead depth 1).
// ---------------------------------------------------------------------------
int d3m_block_ldlt_exec(int nb, const int64_t* h_sizes, const int64_t* h_diag_off, const int64_t* h_panel_off,
                        const int64_t* h_panel_rows, const int64_t* h_piv_off, const int64_t* h_task_ptr,
                        const int64_t* h_task_next, const int64_t* h_tiles_next, const int64_t* h_tiles_rest,
                        const void* d_tasks, void* d_pool, void* d_xbuf, int64_t xbuf_elems, void* d_perm,
                        void* d_tags, void* d_info, void* d_n2x2, void* d_growth, void* d_scale, void* d_asym,
                        void* d_bk_scratch, double pivot_tol, int check_sym, int lookahead, void* stream) {
  static cudaStream_t side = nullptr;
  static cudaEvent_t ev_next = nullptr, ev_rest = nullptr;
  if (!side) {
    if (cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_next, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_rest, cudaEventDisableTiming) != cudaSuccess)
      return fail(-12, "d3m_block_ldlt_exec: stream/event creation");
  }
  cudaStream_t s0 = reinterpret_cast<cudaStream_t>(stream);
  auto* tasks = static_cast<const d3m::GemmTask*>(d_tasks);
  cplx* pool = C(d_pool);
  bool rest_pending = false;
  for (int j = 0; j < nb; ++j) {
    const int nj = (int)h_sizes[j];
    const int64_t R = h_panel_rows[j];
    cplx* xbuf = C(d_xbuf) + (lookahead ? (j & 1) * (xbuf_elems / 2) : 0);
    if (R * nj > (lookahead ? xbuf_elems / 2 : xbuf_elems)) return fail(-22, "d3m_block_ldlt_exec: xbuf too small");
    d3m::BkArgs a{pool + h_diag_off[j], 0, nj, nj, pivot_tol, check_sym,
                  static_cast<int64_t*>(d_perm) + h_piv_off[j], static_cast<int8_t*>(d_tags) + h_piv_off[j],
                  static_cast<int32_t*>(d_n2x2) + j, static_cast<double*>(d_growth) + j,
                  static_cast<int32_t*>(d_info) + j, static_cast<double*>(d_scale) + j,
                  static_cast<double*>(d_asym) + j, C(d_bk_scratch)};
    if (nj > 0) D3M_TRY(d3m_bk_launch(&a, 1, s0));
    if (R > 0)
      D3M_TRY(d3m_panel_trsm_launch(pool + h_panel_off[j], xbuf, (int)R, nj, pool + h_diag_off[j],
                                    static_cast<int64_t*>(d_perm) + h_piv_off[j],
                                    static_cast<int8_t*>(d_tags) + h_piv_off[j], s0));
    const int64_t t0 = h_task_ptr[j], tn = h_task_next[j], t1 = h_task_ptr[j + 1];
    if (rest_pending) {
      cudaStreamWaitEvent(s0, ev_rest, 0);
      rest_pending = false;
    }
    if (tn > t0)
      D3M_TRY(d3m_gemm_launch(0, 0, xbuf, pool, pool, tasks + t0, (int)(tn - t0), (int)h_tiles_next[j], s0));
    if (t1 > tn) {
      if (lookahead) {
        cudaEventRecord(ev_next, s0);
        cudaStreamWaitEvent(side, ev_next, 0);
        D3M_TRY(d3m_gemm_launch(0, 0, xbuf, pool, pool, tasks + tn, (int)(t1 - tn), (int)h_tiles_rest[j], side));
        cudaEventRecord(ev_rest, side);
        rest_pending = true;
      } else {
        D3M_TRY(d3m_gemm_launch(0, 0, xbuf, pool, pool, tasks + tn, (int)(t1 - tn), (int)h_tiles_rest[j], s0));
      }
    }
  }
  if (rest_pending) cudaStreamWaitEvent(s0, ev_rest, 0);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail((int)e, "d3m_block_ldlt_exec: launch");
  return 0;
}

// ---------------------------------------------------------------------------
// block_solve executor (factor.py:243-310), all RHS in one pass.
//   b   : N x nrhs, plan order, overwritten by the forward sweep
//   u   : N x nrhs, receives D^-1 z, then w, then the permuted solution
//   x   : N x nrhs, solution in plan order
//   tmp : max_j n_j x nrhs;  gbuf : max_j R_j x nrhs
//   d_gidx: concatenated global row indices of every panel (per column j the
//           rows of its pattern blocks), h_gptr its CSR pointer.
// ---------------------------------------------------------------------------
int d3m_block_solve_exec(int nb, const int64_t* h_sizes, const int64_t* h_row_off, const int64_t* h_diag_off,
                         const int64_t* h_panel_off, const int64_t* h_panel_rows, const int64_t* h_piv_off,
                         const int64_t* h_pat_ptr, const int64_t* h_pat_idx, const int64_t* h_gptr,
                         const void* d_gidx, const void* d_pool, const void* d_perm, const void* d_tags, void* d_b,
                         void* d_u, void* d_x, void* d_tmp, void* d_gbuf, int nrhs, void* d_tasks, int64_t task_cap,
                         void* stream) {
  if (nb <= 0 || nrhs <= 0) return 0;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const cplx* pool = CC(d_pool);
  // forward-update tasks: one per pattern block (i, j); backward: one per j
  const int64_t npat = h_pat_ptr[nb];
  if (npat + nb > task_cap) return fail(-22, "d3m_block_solve_exec: task buffer too small");
  std::vector<d3m::GemmTask> t(npat + nb);
  std::vector<int> tiles_f(nb), tiles_b(nb);
  for (int j = 0; j < nb; ++j) {
    const int nj = (int)h_sizes[j];
    int64_t prow = 0;
    for (int64_t p = h_pat_ptr[j]; p < h_pat_ptr[j + 1]; ++p) {
      const int64_t i = h_pat_idx[p];
      d3m::GemmTask& k = t[p];
      std::memset(&k, 0, sizeof(k));
      k.a_off = h_panel_off[j] + prow * nj;    // L_ij: n_i x n_j row-major (A, normal)
      k.b_off = 0;                             // z_j in tmp: n_j x nrhs = K x N (TB)
      k.c_off = h_row_off[i] * nrhs;           // b_i
      k.m = (int)h_sizes[i];
      k.n = nrhs;
      k.k = nj;
      k.lda = nj;
      k.ldb = nrhs;
      k.ldc = nrhs;
      k.flags = d3m::kGemmSub;
      prow += h_sizes[i];
    }
    tiles_f[j] = d3m_gemm_prepare_tasks(t.data() + h_pat_ptr[j], (int)(h_pat_ptr[j + 1] - h_pat_ptr[j]));
    d3m::GemmTask& k = t[npat + j];
    std::memset(&k, 0, sizeof(k));
    k.a_off = h_panel_off[j];                  // panel stored R_j x n_j = K x M (TA)
    k.b_off = 0;                               // gbuf R_j x nrhs = K x N (TB)
    k.c_off = h_row_off[j] * nrhs;             // u_j
    k.m = nj;
    k.n = nrhs;
    k.k = (int)h_panel_rows[j];
    k.lda = nj;
    k.ldb = nrhs;
    k.ldc = nrhs;
    k.flags = d3m::kGemmSub;
    tiles_b[j] = d3m_gemm_prepare_tasks(&k, 1);
  }
  cudaError_t e = cudaMemcpyAsync(d_tasks, t.data(), sizeof(d3m::GemmTask) * t.size(), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return fail((int)e, "d3m_block_solve_exec: task upload");
  auto* dt = static_cast<const d3m::GemmTask*>(d_tasks);
  cplx* b = C(d_b);
  cplx* u = C(d_u);
  cplx* x = C(d_x);
  cplx* tmp = C(d_tmp);
  for (int j = 0; j < nb; ++j) {
    const int nj = (int)h_sizes[j];
    if (nj == 0) continue;
    d3m::SolveBatch sb{pool + h_diag_off[j], 0, static_cast<const int8_t*>(d_tags) + h_piv_off[j], 0,
                       static_cast<const int64_t*>(d_perm) + h_piv_off[j], 0, tmp, 0, u + h_row_off[j] * nrhs, 0,
                       b + h_row_off[j] * nrhs, 0, nj, nrhs, nrhs, nrhs};
    D3M_TRY(d3m_solve_phase_launch(0, &sb, 1, s));   // z_j = b_j[perm]
    D3M_TRY(d3m_solve_phase_launch(1, &sb, 1, s));   // z_j = L_jj^-1 z_j, u_j = D^-1 z_j
    const int64_t p0 = h_pat_ptr[j], p1 = h_pat_ptr[j + 1];
    if (p1 > p0) D3M_TRY(d3m_gemm_launch(0, 1, pool, tmp, b, dt + p0, (int)(p1 - p0), tiles_f[j], s));
  }
  for (int j = nb - 1; j >= 0; --j) {
    const int nj = (int)h_sizes[j];
    if (nj == 0) continue;
    const int64_t R = h_panel_rows[j];
    if (R > 0) {
      D3M_TRY(d3m_gather_index_launch(x, static_cast<const int64_t*>(d_gidx) + h_gptr[j], d_gbuf, R, nrhs, s));
      D3M_TRY(d3m_gemm_launch(1, 1, pool, d_gbuf, u, dt + npat + j, 1, tiles_b[j], s));
    }
    d3m::SolveBatch sb{pool + h_diag_off[j], 0, static_cast<const int8_t*>(d_tags) + h_piv_off[j], 0,
                       static_cast<const int64_t*>(d_perm) + h_piv_off[j], 0, u + h_row_off[j] * nrhs, 0, nullptr, 0,
                       x + h_row_off[j] * nrhs, 0, nj, nrhs, nrhs, nrhs};
    D3M_TRY(d3m_solve_phase_launch(3, &sb, 1, s));   // w = L_jj^-T w
    D3M_TRY(d3m_solve_phase_launch(4, &sb, 1, s));   // x_j[perm] = w
  }
  return 0;
}

// recover_primal (subdomain.py:217-237): rhs_d = f_d - D_d lam_d on DMMA,
// E_d = A_d^-1 rhs_d with the cached factors, ordered average into the
// global vector.
int d3m_recover_batched(int batch, int n, int m, const void* F, const void* perm, const void* tags, const void* D,
                        const void* lam, void* rhs, void* work, const void* avg_ptr, const void* avg_src, void* out,
                        int64_t nglob, void* d_tasks, void* stream) {
  // F: batch x n x n packed; D: batch x n x m; lam: batch x m; rhs: batch x n (holds f on entry)
  if (batch <= 0) return 0;
  if (m > 0) {
    std::vector<d3m::GemmTask> t(batch);
    for (int b = 0; b < batch; ++b) {
      d3m::GemmTask& k = t[b];
      std::memset(&k, 0, sizeof(k));
      k.a_off = (int64_t)b * n * m;   // D: n x m (A normal)
      k.b_off = (int64_t)b * m;       // lam: m x 1 = K x N (TB)
      k.c_off = (int64_t)b * n;
      k.m = n;
      k.n = 1;
      k.k = m;
      k.lda = m;
      k.ldb = 1;
      k.ldc = 1;
      k.flags = d3m::kGemmSub;
    }
    D3M_TRY(d3m_zgemm_grouped(0, 1, D, lam, rhs, t.data(), batch, d_tasks, stream));
  }
  D3M_TRY(d3m_ldlt_solve_batched(batch, n, F, (int64_t)n * n, perm, n, tags, n, rhs, n, 1, 1, work, stream));
  D3M_TRY(d3m_ordered_average_launch(rhs, avg_ptr, avg_src, out, nglob, stream));
  return 0;
}

}  // extern "C"
