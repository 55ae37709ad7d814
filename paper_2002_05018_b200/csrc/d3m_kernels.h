// d3m_kernels.h -- internal launch interfaces shared by the .cu files.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace d3m {

using cplx = double2;

// Batched exact Bunch-Kaufman (bk_exact.cu).
struct BkArgs {
  cplx* W;            // batch of n x n row-major matrices
  int64_t stride_w;   // elements between matrices
  int n, lda;
  double pivot_tol;
  int check_sym;
  int64_t* perm;      // batch x n
  int8_t* tags;       // batch x n
  int32_t* n2x2;      // batch
  double* growth;     // batch
  int32_t* info;      // batch: -1 ok, k singular step, -2 asymmetric
  double* scale;      // batch: np.abs(W).max()
  double* asym;       // batch: np.abs(W - W.T).max()
  cplx* scratch;      // batch x 4n, used when the staging does not fit smem
  const int* check_sym_dev = nullptr;   // optional device copy of check_sym (read by the kernel, batch 1)
  // optional pivot-decision diagnostic, batch x 2 doubles: [0] the minimum
  // decision_margin over all steps, [1] the minimum argmax_gap of the colmax
  // searches (d3m_common.cuh); nullptr = not tracked
  double* margin = nullptr;
  bool abs_tol = false;               // pivot_tol is the absolute threshold (d3m_bk_factor_batched check_sym bit 2)
  // panel BK only (d3m_bk_panel_batched check_sym bit 3): the scale is the
  // maximum over the lower triangle and the upper triangle is never read --
  // the split upload, where the upper half is still in flight and the
  // symmetry check / full scale run separately (d3m_sym_scan_batched)
  bool lower_only = false;
};

// Device-resident plan of the persistent block solve (skinny_dmma.cu)
struct SolvePlanDev {
  const int64_t *sizes, *row_off, *diag_off, *panel_off, *panel_rows, *piv_off, *binv_off, *gptr;
  const int64_t* gidx;
  const cplx *pool, *binv;
  const int8_t* tags;
  cplx *b, *u, *x, *tmp, *part;
  int nb, N;                       // N: RHS columns of this pass (<= 16), leading dimension ldn
  int ldn, c0;                     // row stride of b / u / x and the pass's first column
};


// Multi-RHS solve phases against packed factors (ldlt_solve.cu).
struct SolveBatch {
  const cplx* F;  int64_t stride_f;   // packed factors (ld n)
  const int8_t* tags; int64_t stride_t;
  const int64_t* perm; int64_t stride_p;
  cplx* Z; int64_t stride_z;          // working arrays n x m (ld ldz)
  cplx* U; int64_t stride_u;          // optional D^-1 Z output of the forward phase
  const cplx* B; int64_t stride_b;    // gather source / scatter destination (ld ldb)
  int n, m, ldz, ldb;
};

}  // namespace d3m

extern "C" {
int d3m_bk_launch(d3m::BkArgs* a, int batch, void* stream);
int d3m_bk_cluster_launch(d3m::BkArgs* a, int batch, void* stream);
int d3m_bk_cluster_launch_cs(d3m::BkArgs* a, int batch, int cs, void* stream);
int d3m_bk_cluster_max_n(int cs);
int d3m_skinny_launch(int ta, const void* A, int lda, int M, int K, const void* B, int ldb, const void* bmap, int N,
                      void* C, int ldc, const void* cmap, int mode, int kchunk, void* stream);
int d3m_block_solve_persistent_launch(void* plan, void* stream);
int d3m_block_solve_flow_launch(void* plan, const void* items, int nitems, int nchain, const void* deps, const void* part_off,
                                void* cnt, int ncounters, void* stream);
int d3m_skinny_reduce_launch(const void* base, int ldb, const void* part, int nch, int M, int np, double sign,
                             void* out, int ldo, void* stream);
// phase: 0 gather Z=B[perm], 1 forward (+U=D^-1 Z), 2 D^-1, 3 backward, 4 scatter B[perm]=Z
int d3m_solve_phase_launch(int phase, d3m::SolveBatch* a, int batch, void* stream);
int d3m_gemm_launch(int ta, int tb, const void* A, const void* B, void* C, const void* dtasks, int ntasks, int ntiles,
                    void* stream);
int d3m_schur_finalize_launch(const void* C, void* K, void* g, int m, int nrhs, int batch, int64_t stride_c,
                              int64_t stride_k, int64_t stride_g, void* stream);
int d3m_gather_rows_batched_launch(const void* src, int64_t stride_src, int ld_src, const void* idx, int nr, int cols,
                                   void* out, int64_t stride_out, int batch, void* stream);
int d3m_pack_rhs_launch(const void* D, const void* f, void* Z, int n, int m, int nrhs, int batch, int64_t stride_d,
                        int64_t stride_f, int64_t stride_z, void* stream);
int d3m_ordered_average_launch(const void* E, const void* ptr, const void* src, void* out, int64_t ng, void* stream);
int d3m_gather_index_launch(const void* src, const void* idx, void* out, int64_t nrows, int cols, void* stream);
int d3m_block_copy_launch(const void* src, void* dst, const void* dtasks, int ntasks, int64_t max_elems, void* stream);
int d3m_zero_launch(void* p, int64_t n, void* stream);
int d3m_sym_exact_launch(const void* pool, const void* off, const void* n, int nb, void* flag, void* stream);
int d3m_tri_inv_launch(const void* F, int64_t stride_f, const void* perm, int64_t stride_p, const void* tags,
                       int64_t stride_t, void* Binv, int64_t stride_b, int n, int batch, void* stream);
int d3m_dinv_rows_launch(const void* X, void* P, int64_t R, int n, const void* F, const void* tags, void* stream);
int d3m_dinv_left_copy_launch(const void* Z, void* U, int n, int m, const void* F, const void* tags, void* stream);
int d3m_sym_flags_launch(const void* pool, const void* off, const void* n, const void* idx, int count, void* flags,
                         void* stream);
int d3m_nonzero_rows_launch(int B, int n, int m, const void* D, void* flag, void* idx, void* count, void* stream);
int d3m_wait_flag_launch(const int* flag, int value, void* stream);
int d3m_tri_inv_blocked_launch(const void* F, const void* perm, const void* tags, void* Binv, void* coef, int n,
                               void* Linv, void* dinv, void* stream);
int d3m_gemm_launch_perm(const void* A, const void* B, void* C, const void* dtasks, int ntasks, int ntiles,
                         const void* gperm, void* stream);
int d3m_tri_inv_warp_launch(const void* F, const void* perm, const void* tags, void* Binv, void* coef, int n,
                            void* stream, void* Linv = nullptr);
int d3m_dinv_rows_coef_launch(const void* X, void* P, int64_t R, int n, const void* tags, const void* coef,
                              void* stream);
int d3m_diag_block_launch(int fwd, const void* F, int64_t stride_f, const void* tags, int64_t stride_t, void* Z,
                          int64_t stride_z, int n, int m, int r0, int batch, void* stream);
int d3m_diag_block_rows();
int d3m_bk_panel_batched_launch(d3m::BkArgs* a, int batch, void* workspace, void* stream);
size_t d3m_bk_panel_workspace_bytes(int n, int batch);
int d3m_sym_scan_batched_launch(d3m::BkArgs* a, int batch, void* red_ws, void* stream);
int d3m_gemm_tma_prepare(const void* X, int64_t rows_x, const void* L, int64_t rows_l, int n, void* maps_out);
int d3m_gemm_tma_launch(const void* maps, void* C, const void* dtasks, int ntasks, int ntiles, int64_t b_base,
                        void* stream);
int d3m_gemm_tma_prepare_batched(const void* A, int64_t a_stride, int64_t a_rows, int a_cols, int lda, const void* B,
                                 int64_t b_stride, int64_t b_rows, int b_cols, int ldb, int batch, void* h_maps);
int d3m_gemm_tma_launch_batched(const void* d_maps, void* C, const void* dtasks, int ntasks, int ntiles,
                                int64_t a_stride, int64_t b_stride, void* tmax, void* stream);
int d3m_gemm_tma_prepare_solve(const void* F, int64_t stride_f, int n, const void* Z, int64_t stride_z, int m,
                               int batch, void* h_maps);
int d3m_gemm_tma_launch_batched_t(int ta, const void* d_maps, void* C, const void* dtasks, int ntasks, int ntiles,
                                  int64_t a_stride, int64_t b_stride, void* stream);
}

#include "d3m_gemm.h"
extern "C" int d3m_gemm_prepare_tasks(d3m::GemmTask* tasks, int ntasks);
extern "C" int d3m_gemm_set_form(int form);
extern "C" int d3m_gemm_launch_tm(int ta, int tb, const void* A, const void* B, void* C, const void* dtasks,
                                  int ntasks, int ntiles, void* tmax, void* stream);
