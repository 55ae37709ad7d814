/*
 * d3m.h -- C ABI of libd3m, the sm_100a implementation of the D3M
 * factorisation hot path (reference: /root/reference/pkg/src/ddsolve).
 *
 * Conventions
 *   - complex arrays are interleaved complex128 (numpy layout), row-major;
 *   - every pointer is a DEVICE pointer unless its name starts with h_;
 *   - every call is asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and returns 0, a negative errno-like code for invalid
 *     arguments, or a positive cudaError_t; d3m_last_error() describes it;
 *   - pivot outcomes are written to device arrays (info: -1 ok, k = singular
 *     elimination step, -2 = symmetry check failed); the Python host layer
 *     turns them into the reference's exceptions with the same messages.
 *
 * Each entry point names the reference interface it replaces.  The
 * reference's own operator API is the five kernels of kernels.py swapped by
 * accel.maybe_jit (accel.py:36-40); they are per-block host calls, so the
 * GPU boundary sits one level up, at the batched functions below.
 */
#ifndef D3M_H_
#define D3M_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define D3M_ABI_VERSION 13

int d3m_abi_version(void);
const char* d3m_last_error(void);

/* Batched complex-symmetric Bunch-Kaufman LDL^T, in place, bit-exact with the
 * reference.  Replaces kernels.bk_factor (kernels.py:36-146) as called by
 * factor.dense_ldlt_bk (factor.py:83-116), including its scale
 * (np.abs(W).max()) and symmetry check (factor.py:94-98) when check_sym.
 * W: batch x (n x lda) with stride_w elements between matrices.
 * Outputs per matrix: perm[n] int64, tags[n] int8, n2x2 int32, growth f64,
 * info int32, scale f64, asym f64.  scratch: batch*4*n complex, needed only
 * when 64*n bytes exceed the shared-memory staging (n > 3200).
 * check_sym bit 2 (value 4, ABI v9): pivot_tol is the absolute threshold
 * itself (kernels.bk_factor(W, tol_abs) semantics); otherwise the threshold
 * is pivot_tol * scale.  Bits 0-1: 0 no symmetry check, 1 numpy-style check.
 * margin (ABI v9; NULL = not tracked): batch x 2 f64 pivot-decision
 * diagnostics -- [0] the minimum over all steps of the relative distance of
 * every evaluated BK test (kernels.py:59-77: singularity, alpha colmax,
 * alpha colmax^2 / rowmax, alpha rowmax) to its threshold, [1] the minimum
 * relative gap between the colmax argmax winner and the runner-up.  A kernel
 * whose arithmetic differs from the reference's by rounding takes the
 * reference's decisions whenever both stay well above ~1e-14.  The same
 * argument on d3m_bk_panel_batched, d3m_schur_reduce_batched and
 * (per block column) d3m_block_ldlt_exec. */
int d3m_bk_factor_batched(int batch, int n, void* W, int64_t stride_w, int lda, double pivot_tol, int check_sym,
                          void* perm, void* tags, void* n2x2, void* growth, void* info, void* scale, void* asym,
                          void* scratch, void* margin, void* stream);

/* Largest block order the bit-exact cluster BK (bk_cluster.cu) holds in the
 * shared memory of a cs-CTA cluster (cs = 2, 4, 8, 16; 0 = any size).
 * block_ldlt factors supernodes wider than 128 and up to this order on the
 * cluster kernel, wider ones on the single-CTA exact kernel; both are
 * bit-identical to kernels.py:36-146.  Host-only query (no device call). */
int d3m_bk_cluster_max_n(int cs);

/* Multi-RHS solve M X = B with packed factors: gather by perm, unit-L forward,
 * D^-1, unit-L^T backward, scatter.  Replaces DenseFactor.solve
 * (factor.py:52-66) with kernels.solve_unit_lower / apply_dinv_left /
 * solve_unit_lower_t (kernels.py:149-181).  B (batch x n x ldb) is
 * overwritten by X; work: batch x n x m complex. */
int d3m_ldlt_solve_batched(int batch, int n, const void* F, int64_t stride_f, const void* perm, int64_t stride_p,
                           const void* tags, int64_t stride_t, void* B, int64_t stride_b, int ldb, int m, void* work,
                           void* stream);

/* Batched blocked Bunch-Kaufman for large dense matrices (zlasyf form): per
 * panel of 63-64 columns (127-128 from n = 8192) a thread-block cluster of
 * 1-16 CTAs per matrix (contiguous row slices, pivot searches merged through
 * distributed shared memory) + one grouped DMMA GEMM for all matrices'
 * trailing updates.  Same outputs as d3m_bk_factor_batched;
 * identical pivot decisions whenever no test sits within rounding of its
 * threshold, values to rounding.  workspace: d3m_bk_panel_workspace(n, batch)
 * bytes.  Used by d3m_schur_reduce_batched for n > 512. */
int d3m_bk_panel_batched(int batch, int n, void* W, int64_t stride_w, int lda, double pivot_tol, int check_sym,
                         void* perm, void* tags, void* n2x2, void* growth, void* info, void* scale, void* asym,
                         void* workspace, void* margin, void* stream);
size_t d3m_bk_panel_workspace(int n, int batch);
/* check_sym bit 3 (value 8, ABI v11) on d3m_bk_panel_batched: the scale is
 * np.abs(tril(W)).max() and the upper triangle is never read (no symmetry
 * check) -- the split upload of host matrices, where the upper halves are
 * still in flight when the factorisation starts; the caller checks symmetry
 * and the full scale with d3m_sym_scan_batched on an intact copy and
 * refactors when the full scale differs (an inexactly symmetric input). */

/* scale[b] = np.abs(W_b).max(), asym[b] = np.abs(W_b - W_b.T).max()
 * (factor.py:94-98) exactly as the factorisation kernels compute them.
 * workspace: >= 64 * batch bytes.  (ABI v11) */
int d3m_sym_scan_batched(int batch, int n, const void* W, int64_t stride_w, int lda, void* scale, void* asym,
                         void* workspace, void* stream);

/* Row-block pieces of row-major n x n complex128 matrices src[b] (leading
 * dimension src_ld) into dst + b * dst_stride (leading dimension dst_ld):
 * part 0 = rows [r0, r0+128) x columns [0, r0+128) of every 128-row block
 * (the lower triangle and the diagonal blocks), part 1 = the remainder
 * (strict upper triangle outside the diagonal blocks).  kind is a
 * cudaMemcpyKind (1 host->device, 3 device->device).  (ABI v11) */
int d3m_copy_triangle(int batch, const void* const* src, int64_t src_ld, void* dst, int64_t dst_stride,
                      int64_t dst_ld, int n, int part, int kind, void* stream);

/* Blocked multi-RHS solve (64-row diagonal blocks in shared memory +
 * right-looking DMMA GEMM updates), same contract as d3m_ldlt_solve_batched;
 * d_tasks: 2 * ceil(n/64) * batch GEMM records (64 B each). */
int d3m_ldlt_solve_blocked_batched(int batch, int n, const void* F, int64_t stride_f, const void* perm,
                                   int64_t stride_p, const void* tags, int64_t stride_t, void* B, int64_t stride_b,
                                   int ldb, int m, void* work, void* d_tasks, void* stream);

/* Grouped complex GEMM on DMMA: for each task C (op)= A_eff B_eff^T.
 * h_tasks: host array of 64-byte task records (see d3m_gemm.h; tile fields
 * are filled in place), d_tasks: device buffer of the same size.
 * ta: A stored K x M; tb: B stored K x N.  Replaces the numpy '@' calls of
 * factor.py:215, subdomain.py:181,183,233. */
int d3m_zgemm_grouped(int ta, int tb, const void* A, const void* B, void* C, void* h_tasks, int ntasks,
                      void* d_tasks, void* stream);

/* The TMA-staged update GEMM of d3m_block_ldlt_exec on one panel pair (ABI
 * v12): X (rows_x x n) and L (rows_l x n) are contiguous row-major panels,
 * every task has lda = ldb = k = n, a_off relative to X, b_off relative to L,
 * and the flags of a trailing update (C -= A B^T, optionally the symmetric
 * diagonal target).  Tile operands are staged by cp.async.bulk.tensor from
 * tensor maps over the panels.  Results are bitwise those of
 * d3m_zgemm_grouped(0, 0, ...).  h_tasks / d_tasks as d3m_zgemm_grouped.
 * Replaces factor.py:215. */
int d3m_zgemm_tma_panels(const void* X, int64_t rows_x, const void* L, int64_t rows_l, int n, void* C, void* h_tasks,
                         int ntasks, void* d_tasks, void* stream);

/* Complex product form of every grouped GEMM launched afterwards in this
 * process: 3 = Gauss 3M (three real DMMA products per complex product, the
 * default), 4 = 4M (four).  0 only queries.  Returns the previous form.
 * The environment variable D3M_ZGEMM=3m|4m sets the initial form. */
int d3m_gemm_set_form(int form);

/* Batched Schur reduction of equal-sized subdomains: factor A_d in place,
 * X = A_d^-1 [D_d | F_d], K_D = 0.5 (D^T X_D + (D^T X_D)^T), G_d = D^T X_F.
 * Replaces subdomain.reduce_domain (subdomain.py:166-184) for a batch; F_d
 * holds nrhs load columns (n x nrhs row-major; the reference's single f is
 * nrhs = 1), G_d is m x nrhs.  work_z / work_x: batch x n x (m+nrhs),
 * work_c: batch x m x (m+nrhs); work_x holds X on return.  Optional (ABI v3)
 * rows: batch x nrows ascending row indices where D_d has nonzeros (-1
 * padded): D^T X then runs over those rows only (work_d: batch x nrows x m;
 * work_z is reused for the gathered X rows).  rows = NULL: dense product.
 * flags (ABI v4): bit 0 = Schur only -- forward sweep Z = L^-1 P [D | F]
 * and K = Z_D^T D^-1 Z (no backward sweep; work_x does not hold X then).
 * Bit 1 (ABI v11): A already holds the packed factor and perm/tags/... are
 * filled (the caller ran d3m_bk_panel_batched itself); the BK is skipped.
 * n <= 512: exact BK + chain solves (bk_scratch: batch*4n complex if n>3200);
 * n > 512: panel BK + blocked solves (bk_scratch: d3m_bk_panel_workspace
 * bytes, d_tasks: max(batch, 4 ceil(n/64) batch) records).
 * h_mcols (ABI v13, HOST int32[batch] or NULL): the coupling columns each
 * domain really has when its D_d is zero-padded to m; the blocked solves'
 * GEMM updates then skip the padded columns [h_mcols[b], m) (their solution
 * is exactly zero, so every result is unchanged bit for bit). */
int d3m_schur_reduce_batched(int batch, int n, int m, int nrhs, void* A, const void* D, const void* f,
                             double pivot_tol,
                             void* perm, void* tags, void* n2x2, void* growth, void* info, void* scale, void* asym,
                             void* K_out, void* g_out, void* work_z, void* work_x, void* work_c, void* bk_scratch,
                             void* d_tasks, const void* rows, int nrows, void* work_d, int flags, void* margin,
                             const int32_t* h_mcols, void* stream);

/* Grouped block copy / ordered accumulate (40-byte CopyTask records, see
 * d3m_misc.h).  Used for factor._permute_blocks (factor.py:139-151) and the
 * scatter-add of assemble_reduced (subdomain.py:206-213 via
 * blockmat.add_block, blockmat.py:69-81). */
int d3m_block_copy(const void* src, void* dst, const void* d_tasks, int ntasks, int64_t max_elems, void* stream);

/* out[i, :] = src[idx[i], :] (cols complex per row). */
int d3m_gather_rows(const void* src, const void* idx, void* out, int64_t nrows, int cols, void* stream);

/* out[g] = (sum of E[src[p]] for p in [ptr[g], ptr[g+1]), ascending domain
 * order) / count -- the acc/cnt averaging of recover_primal
 * (subdomain.py:222-237). */
int d3m_ordered_average(const void* E, const void* ptr, const void* src, void* out, int64_t ng, void* stream);

int d3m_zero(void* p, int64_t n, void* stream);

/* flag[0] is cleared when any of the nb diagonal slots (pool + off[b], order
 * n[b], device int64 arrays) is not bitwise symmetric.  block_ldlt uses it to
 * pass check_sym = 2 (lower-triangle-only scale, asym = 0) to the diagonal
 * BK: updates of diagonal targets are mirrored exactly, so symmetric K
 * blocks stay exactly symmetric through the factorisation. */
int d3m_diag_sym_exact(const void* pool, const void* off, const void* n, int nb, void* flag, void* stream);

/* Per-block version (ABI v8): CTA b checks diagonal block idx[b] (int64
 * device list of count blocks) and writes flags[idx[b]] = 2 (bitwise
 * symmetric) or 1 (int32 device array, one per block).  With the chunked
 * upload every chunk flags the diagonal blocks it carries, and
 * d3m_block_ldlt_exec's d_check_sym makes each column's BK read its own flag
 * on the device (no host sync on the whole of K's diagonal). */
int d3m_diag_sym_flags(const void* pool, const void* off, const void* n, const void* idx, int count, void* flags,
                       void* stream);

/* Test hook: hyp[i] = glibc-hypot modulus (numba abs, kernels.py:50-77) and
 * npabs[i] = numpy np.abs modulus (factor.py:94-96) of z[i], as computed by
 * the device code that makes the pivot decisions. */
int d3m_modulus_probe(const void* z, void* hyp, void* npabs, int64_t n, void* stream);

/* Right-looking block LDL^T over an elimination plan with restricted
 * Bunch-Kaufman pivoting.  Replaces factor.block_ldlt (factor.py:154-240).
 * The device pool holds, per block column j, a diagonal slot (offset
 * h_diag_off[j], n_j x n_j) and a panel (h_panel_off[j], h_panel_rows[j] x
 * n_j) stacking the pattern blocks in ascending row order; on entry they hold
 * the permuted K (W of factor.py:168), on exit the packed factors and L_ij.
 * Per column: BK of the diagonal block, Binv_j = L_jj^-1 P_j into d_binv at
 * h_binv_off[j] (kept for the solve), X = panel Binv_j^T on DMMA (task
 * d_trsm_tasks[j], h_tiles_trsm[j] tiles), L = X D^-1 into the panel, then
 * the trailing-update GEMM tasks d_tasks[h_task_ptr[j] .. h_task_ptr[j+1]),
 * the first (h_task_next[j] - h_task_ptr[j]) of which target column j+1 and
 * run on the high-priority critical stream (lookahead), the rest on a
 * low-priority stream.  Per-column pivots go to d_perm/d_tags at
 * h_piv_off[j]; info/n2x2/growth/scale/asym are nb-long device arrays.
 * check_sym: 1 = full numpy-style symmetry check per diagonal block,
 * 2 = blocks known exactly symmetric (d3m_diag_sym_exact).
 * xbuf: X scratch (4 x max R_j n_j with lookahead: a ring of X panels of
 * the columns in flight).  bk_scratch (only for supernodes > 3200): 4 x 4 x
 * max n_j complex, one per critical stream.
 * lookahead 0: every launch in column order on `stream`.  lookahead 1
 * (etree-parallel, ABI v9): each column's critical chain (BK -> L^-1 ->
 * panel TRSM -> D^-1 -> update of column j+1) runs on one of 4 high-priority
 * streams, h_sched[3j] (independent subtrees of the elimination tree
 * overlap); the bulk trailing updates run in column order on one
 * low-priority stream, so every block receives its updates in ascending
 * source-column order and the factor is bitwise that of lookahead 0.
 * h_sched[3j+1] / [3j+2]: the last column k < j whose bulk update writes
 * column j / column j+1 (-1: none), the events column j's BK / its update
 * of column j+1 wait for (planner.etree_schedule).
 * nwait / h_wait_col / h_wait_ev (ABI v6; 0 / NULL / NULL = none): cudaEvent_t
 * handles, h_wait_col ascending; a stream about to run a column >=
 * h_wait_col[w] first waits on h_wait_ev[w] (blocks of K still being
 * uploaded on a copy stream).
 * d_check_sym (ABI v8; NULL = use check_sym): nb int32 device flags, column
 * j's BK reads d_check_sym[j] (d3m_diag_sym_flags) instead of check_sym. */
int d3m_block_ldlt_exec(int nb, const int64_t* h_sizes, const int64_t* h_diag_off, const int64_t* h_panel_off,
                        const int64_t* h_panel_rows, const int64_t* h_piv_off, const int64_t* h_binv_off,
                        const int64_t* h_task_ptr, const int64_t* h_task_next, const int64_t* h_tiles_next,
                        const int64_t* h_tiles_rest, const int64_t* h_tiles_trsm, const void* d_tasks,
                        const void* d_trsm_tasks, void* d_pool, void* d_binv, void* d_xbuf, int64_t xbuf_elems,
                        void* d_perm, void* d_tags, void* d_info, void* d_n2x2, void* d_growth, void* d_scale,
                        void* d_asym, void* d_bk_scratch, double pivot_tol, int check_sym, int lookahead,
                        int nwait, const int64_t* h_wait_col, void* const* h_wait_ev, const void* d_check_sym,
                        void* d_margin, const int32_t* h_sched, void* stream);

/* ---- Native planner (host functions: no device, callable on a CPU box) ----
 * Trailing-update GEMM task table of block_ldlt (factor.py:209-219): for each
 * column j and pattern pair (i, k), k <= i, one GemmTask (64-byte records,
 * csrc/d3m_gemm.h), "next" (k == j+1) before "rest" per column.  Two-pass:
 * tasks = NULL counts.  Returns the record count, -1 for an update outside
 * the pattern (FactorConsistencyError), -2 when cap is too small.  Fills
 * task_ptr[nb+1], task_next/tiles_next/tiles_rest[nb], flops[0]. */
int64_t d3m_plan_gemm_tasks(int nb, const int64_t* sizes, const int64_t* pat_ptr, const int64_t* pat_idx,
                            const int64_t* diag_off, const int64_t* panel_off, void* tasks, int64_t cap,
                            int64_t* task_ptr, int64_t* task_next, int64_t* tiles_next, int64_t* tiles_rest,
                            int64_t* flops);
/* Work items (int32 x 8) and dependency pairs (int32 x 2) of
 * d3m_block_solve_dataflow (factor.py:243-310 as tiles), a topological order
 * with each column's critical items first.  Two-pass (items = NULL
 * counts); out[0..3] = items, deps, counters, partial elements;
 * part_off[nb].  0, or -2 on overflow. */
int d3m_plan_flow_items(int nb, const int64_t* sizes, const int64_t* pat_ptr, const int64_t* pat_idx,
                        const int64_t* panel_rows, int32_t* items, int64_t cap_items, int32_t* deps,
                        int64_t cap_deps, int64_t* part_off, int64_t* out);

/* Host-staged upload of pageable inputs (ABI v9): a native host thread copies
 * chunk c's blocks (blocks [chunk_ptr[c], chunk_ptr[c+1]) of the n copies
 * src[i] -> dst + dst_off[i], nbytes[i] bytes; dst is pinned host memory)
 * with up to nthreads threads, then stores c + 1 into the pinned int *flag.
 * The sources must stay alive until d3m_host_stage_join.  Returns a handle,
 * NULL on failure.  Used by block_ldlt for numpy K blocks (the reference
 * API's inputs) so the H2D transfer of later chunks overlaps the first
 * columns' factorisation. */
void* d3m_host_stage_start(int nchunks, const int64_t* chunk_ptr, int n, const void* const* src,
                           const int64_t* dst_off, const int64_t* nbytes, void* dst, void* flag, int nthreads);
/* Join the host thread of d3m_host_stage_start and free its handle. */
int d3m_host_stage_join(void* handle);
/* Make `stream` wait until the pinned host int *flag >= value. */
int d3m_stream_wait_flag(const void* flag, int value, void* stream);

/* n asynchronous copies dst + dst_off[i] <- src + src_off[i] (bytes, kind a
 * cudaMemcpyKind) on `stream`: the chunked upload of K's blocks from pinned
 * host memory. */
int d3m_memcpy_batch(void* dst, const void* src, const int64_t* dst_off, const int64_t* src_off,
                     const int64_t* nbytes, int n, int kind, void* stream);

/* Scheduler scratch the dataflow solve keeps after the planner's counters
 * (ABI v10): d_counters holds (planner count + D3M_FLOW_EXTRA_COUNTERS) ints. */
#define D3M_FLOW_EXTRA_COUNTERS 2052

/* Block substitution as a dataflow of work items (ABI v7): the products of
 * d3m_block_solve_exec (same tiles and summation order, so bitwise equal to
 * it), taken from an atomic queue by one resident grid per pass of <= 16 RHS
 * and ordered only by their true dependencies (per-item counter waits)
 * instead of ~5 grid-wide barriers per block column.  d_items: nitems
 * records of 8 int32 {type, column, p0, p1, dep_off, dep_cnt, inc0, inc1};
 * d_deps: int32 pairs {counter, target}; d_part_off: per-column int64 offset
 * of its split-K partials in d_part (sum over columns of
 * ceil(R_j/256) * n_j * 16 complex); d_counters: ncounters int32 scratch
 * (zeroed here before every pass; the last D3M_FLOW_EXTRA_COUNTERS are the
 * queues').  ABI v10: the first nchain items are the critical chain (each
 * column's z_j, parent update, parent-chunk partials, reduce and x_j), run
 * by CTAs that own their SM; the others by the rest of the grid; each part
 * keeps the planner's (topological) order.  The item list is built by the
 * host (factor.py _solve_flow).  Replaces the substitutions of
 * factor.py:271-310 like d3m_block_solve_exec. */
int d3m_block_solve_dataflow(int nb, const void* d_plan, const void* d_items, int nitems, int nchain, const void* d_deps,
                             const void* d_part_off, void* d_counters, int ncounters, const void* d_gidx,
                             const void* d_pool, const void* d_binv, const void* d_tags, void* d_b, void* d_u,
                             void* d_x, void* d_part, int nrhs, void* stream);

/* Rows where each coupling block has entries (ABI v7): D is B x n x m
 * complex128 (device); flag: B*n int8 scratch; idx: B*n int64, block b's
 * nonzero rows ascending in idx[b*n ...], -1 after count[b] (int32 x B).
 * Feeds the row list of d3m_schur_reduce_batched (D^T X over those rows,
 * subdomain.py:181). */
int d3m_nonzero_rows(int B, int n, int m, const void* D, void* flag, void* idx, void* count, void* stream);

/* Block residual r -= K x for iterative refinement of block_solve (ABI v7).
 * K's stored blocks (original numbering) stay in device buffers h_abase[l];
 * x and r are N x cols in plan-order rows.  Launch l is a grouped GEMM
 * (transposed A iff h_ta[l]; B_eff = x^T, so tb = 1) over h_ntasks[l]
 * prepared task records at d_tasks + h_task_off[l] (h_ntiles[l] tiles), every
 * target block at most once per launch; the launch order fixes the summation
 * order, so the result is deterministic.  No reference counterpart: the
 * reference's block_solve (factor.py:243-310) does not refine. */
int d3m_block_residual(int nlaunch, const int32_t* h_ta, const int32_t* h_ntasks, const int32_t* h_ntiles,
                       const int64_t* h_task_off, const void* const* h_abase, const void* x, void* r,
                       const void* d_tasks, void* stream);

/* Forward / D^-1 / backward block substitution for nrhs right-hand sides in
 * one pass: z = Binv b, u = D^-1 z, b_i -= L_ij z (forward), w = u - sum_i
 * L_ij^T x_i, x = Binv^T w (backward), with HBM-streaming tall-skinny kernels;
 * each RHS column is computed with a fixed summation order independent of
 * nrhs (k-RHS == k x 1-RHS bitwise).  Replaces factor.block_solve /
 * _solve_one (factor.py:243-310).  b: plan-ordered RHS (N x nrhs, consumed);
 * x: solution in plan order; tmp: max n_j x nrhs; part: partial-sum buffer of
 * part_elems complex (>= max_j ceil(max(R_j, n_j)/16) n_j nrhs);
 * d_gidx/h_gptr: global plan-order row of every panel row.  d_plan (ABI v5,
 * optional): the same plan arrays on the device, int64 [sizes | row_off |
 * diag_off | panel_off | panel_rows | piv_off | binv_off] (nb each) then
 * gptr (nb + 1); when given, both sweeps run as one persistent cooperative
 * kernel per pass of 16 RHS (bitwise the same results), else one launch per
 * product. */
int d3m_block_solve_exec(int nb, const int64_t* h_sizes, const int64_t* h_row_off, const int64_t* h_diag_off,
                         const int64_t* h_panel_off, const int64_t* h_panel_rows, const int64_t* h_piv_off,
                         const int64_t* h_binv_off, const int64_t* h_gptr, const void* d_gidx, const void* d_pool,
                         const void* d_binv, const void* d_tags, void* d_b, void* d_u, void* d_x, void* d_tmp,
                         void* d_part, int64_t part_elems, int nrhs, const void* d_plan, void* stream);

/* Primal recovery of equal-sized subdomains: rhs = f - D lam (rhs holds f on
 * entry), E = A^-1 rhs with the cached packed factors, then the ordered
 * average into out[nglob].  Replaces subdomain.recover_primal
 * (subdomain.py:217-237). */
int d3m_recover_batched(int batch, int n, int m, const void* F, const void* perm, const void* tags, const void* D,
                        const void* lam, void* rhs, void* work, const void* avg_ptr, const void* avg_src, void* out,
                        int64_t nglob, void* d_tasks, void* stream);

/* Instrumentation used by bench.py: launch counter and optional per-class
 * CUDA-event timing of every kernel launched through this library (classes:
 * 0 diagonal BK, 1 panel TRSM, 2 trailing-update / reduction GEMM,
 * 3 substitution kernels, 4 data movement).  Events are recorded on the
 * launching stream around each launch; d3m_counters_read synchronises them.
 * ms[0..4]: summed per-launch event time per class; ms[5..9]: measure of the
 * union of the launch intervals per class (concurrent launches of one class
 * on the critical and bulk streams counted once).  n[0..4]: launch counts. */
void d3m_set_timing(int on);
/* (class, start_ms, end_ms) triplets of the launches timed before the last
 * d3m_counters_read; returns their number (diagnostics). */
int64_t d3m_timing_intervals(double* out, int64_t max_triplets);
void d3m_counters_reset(void);
int d3m_counters_read(int64_t* launches, double* ms, int64_t* n);

#ifdef __cplusplus
}
#endif

#endif /* D3M_H_ */
