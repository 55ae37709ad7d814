// d3m_capi.cu -- the extern "C" boundary of libd3m (declared in include/d3m.h).
//
// All array arguments are DEVICE pointers unless named h_*; complex arrays are
// interleaved complex128.  Every entry point is asynchronous on the given
// stream and returns 0, a negative errno-like code for invalid arguments, or
// a positive cudaError_t.  Pivot outcomes (info) are written to device
// arrays; the caller raises the reference's exceptions from them.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
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
      char _b[1024];                                                          \
      snprintf(_b, sizeof(_b), "%s failed with %d (%s)", #expr, _rc,        \
               _rc > 0 ? cudaGetErrorString((cudaError_t)_rc) : "invalid"); \
      g_err = _b;                                                            \
      return _rc;                                                            \
    }                                                                        \
  } while (0)

// ---- launch accounting / per-class CUDA-event timing (bench.py roofline) ----
// Every kernel launched through this file increments g_launches.  When timing
// is on, each launch is bracketed by a pair of events on its own stream and
// the elapsed times are summed per class at d3m_counters_read().
enum { kClsBk = 0, kClsTrsm = 1, kClsGemm = 2, kClsSolve = 3, kClsMisc = 4, kNumCls = 5 };
// supernodes up to this order get the unpermuted L^-1 from the triangular-inverse kernels and the
// gathered / triangular panel TRSM (factor.py sets kGemmTriGather on exactly these TRSM tasks)
constexpr int kTrsmTriMax = 512;
// The counters are process-wide (a measurement facility of bench.py and the
// tools); the timing records are guarded by g_tmu.
std::atomic<long long> g_launches{0};
std::atomic<bool> g_timing{false};
std::mutex g_tmu;
struct TimedRec { int cls; cudaEvent_t a, b; };
std::vector<TimedRec> g_pending;
std::vector<cudaEvent_t> g_free_ev;
double g_ms[kNumCls] = {0, 0, 0, 0, 0};
double g_union[kNumCls] = {0, 0, 0, 0, 0};
std::atomic<long long> g_cnt[kNumCls];
cudaEvent_t g_ref = nullptr;          // common origin for interval unions
std::vector<double> g_iv;             // (class, start ms, end ms) of the last d3m_counters_read

cudaEvent_t take_event() {
  if (!g_free_ev.empty()) {
    cudaEvent_t e = g_free_ev.back();
    g_free_ev.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

template <typename Fn>
int launch(int cls, void* stream, Fn fn) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  g_cnt[cls].fetch_add(1, std::memory_order_relaxed);
  if (!g_timing.load(std::memory_order_relaxed)) return fn();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  TimedRec r{cls, nullptr, nullptr};
  {
    std::lock_guard<std::mutex> g(g_tmu);
    r.a = take_event();
    r.b = take_event();
  }
  cudaEventRecord(r.a, s);
  const int rc = fn();
  cudaEventRecord(r.b, s);
  std::lock_guard<std::mutex> g(g_tmu);
  g_pending.push_back(r);
  return rc;
}

using d3m::cplx;
constexpr int kExactBkMax = 128;    // supernodes up to this use the bit-exact BK kernel
constexpr int kPanelBkMin = 512;    // subdomains above this use the batched panel BK + blocked solves
inline cplx* C(void* p) { return static_cast<cplx*>(p); }
inline const cplx* CC(const void* p) { return static_cast<const cplx*>(p); }

// Per-device state of the block LDL^T executor: the critical / bulk streams
// and their events, the D^-1 coefficient buffer, the unpermuted L^-1 of every
// column and the diagonal-inverse scratch.  One context per device, created
// on first use on that device; calls on a device serialise on its mutex.
constexpr int kCritStreams = 4;       // critical streams of the etree-parallel executor
constexpr int kXSlots = 4;            // X-panel / D^-1-coefficient ring slots (columns in flight)
struct ExecCtx {
  std::mutex mu;
  cudaStream_t crit[kCritStreams] = {}, side = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::vector<cudaEvent_t> ev_col, ev_rest;   // per block column: critical work done / bulk update done
  void* coef_buf = nullptr;
  size_t coef_cap = 0;
  cplx* linv = nullptr;
  int64_t linv_cap = 0;
  cplx* dinv[kCritStreams] = {};      // 256 x 16 complex each: tri_inv_diag16 output, one per stream
  bool grow_events(size_t nb) {
    while (ev_col.size() < nb) {
      cudaEvent_t a, b;
      if (cudaEventCreateWithFlags(&a, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&b, cudaEventDisableTiming) != cudaSuccess)
        return false;
      ev_col.push_back(a);
      ev_rest.push_back(b);
    }
    return true;
  }
};

ExecCtx* exec_ctx() {
  static std::mutex m;
  static std::map<int, std::unique_ptr<ExecCtx>> ctxs;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> g(m);
  std::unique_ptr<ExecCtx>& p = ctxs[dev];
  if (!p) {
    auto c = std::make_unique<ExecCtx>();
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    for (int q = 0; q < kCritStreams; ++q)
      if (cudaStreamCreateWithPriority(&c->crit[q], cudaStreamNonBlocking, hi) != cudaSuccess ||
          cudaMalloc(&c->dinv[q], sizeof(cplx) * 256 * 16) != cudaSuccess)
        return nullptr;
    if (cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, lo) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming) != cudaSuccess)
      return nullptr;
    p = std::move(c);
  }
  return p.get();
}

}  // namespace

extern "C" {

int d3m_abi_version(void) { return D3M_ABI_VERSION; }
int d3m_bk_panel_batched(int batch, int n, void* W, int64_t stride_w, int lda, double pivot_tol, int check_sym,
                         void* perm, void* tags, void* n2x2, void* growth, void* info, void* scale, void* asym,
                         void* workspace, void* margin, void* stream);
int d3m_ldlt_solve_blocked_batched(int batch, int n, const void* F, int64_t stride_f, const void* perm,
                                   int64_t stride_p, const void* tags, int64_t stride_t, void* B, int64_t stride_b,
                                   int ldb, int m, void* work, void* d_tasks, void* stream);

const char* d3m_last_error(void) { return g_err.c_str(); }

int d3m_bk_factor_batched(int batch, int n, void* W, int64_t stride_w, int lda, double pivot_tol, int check_sym,
                          void* perm, void* tags, void* n2x2, void* growth, void* info, void* scale, void* asym,
                          void* scratch, void* margin, void* stream) {
  if (batch < 0 || n < 0 || lda < n) return fail(-22, "d3m_bk_factor_batched: bad shape");
  const bool abs_tol = (check_sym & 4) != 0;
  check_sym &= 3;
  d3m::BkArgs a{C(W), stride_w, n, lda, pivot_tol, check_sym, static_cast<int64_t*>(perm), static_cast<int8_t*>(tags),
                static_cast<int32_t*>(n2x2), static_cast<double*>(growth), static_cast<int32_t*>(info),
                static_cast<double*>(scale), static_cast<double*>(asym), C(scratch)};
  a.margin = static_cast<double*>(margin);
  a.abs_tol = abs_tol;
  D3M_TRY(launch(kClsBk, stream, [&] { return d3m_bk_launch(&a, batch, stream); }));
  return 0;
}

int d3m_ldlt_solve_batched(int batch, int n, const void* F, int64_t stride_f, const void* perm, int64_t stride_p,
                           const void* tags, int64_t stride_t, void* B, int64_t stride_b, int ldb, int m, void* work,
                           void* stream) {
  if (batch < 0 || n < 0 || m < 0 || ldb < m) return fail(-22, "d3m_ldlt_solve_batched: bad shape");
  if (batch == 0 || n == 0 || m == 0) return 0;
  d3m::SolveBatch s{CC(F), stride_f, static_cast<const int8_t*>(tags), stride_t, static_cast<const int64_t*>(perm),
                    stride_p, C(work), (int64_t)n * m, nullptr, 0, CC(B), stride_b, n, m, m, ldb};
  // Z = B[perm]; Z = L^-1 Z; Z = D^-1 Z; Z = L^-T Z; B[perm] = Z
  for (int phase = 0; phase < 5; ++phase)
    D3M_TRY(launch(kClsSolve, stream, [&] { return d3m_solve_phase_launch(phase, &s, batch, stream); }));
  return 0;
}

// Blocked multi-RHS solve for large factors (n > kBlockedSolveMin): gather,
// 64-row diagonal solves + right-looking DMMA GEMM updates (forward, then
// backward with L^T), D^-1, scatter.  Two-level blocking: inside a 256-row
// outer block each 64-row block updates only the rest of its outer block
// (K = 64, <= 192 rows); the last 64-row block of an outer block applies the
// whole outer block to every remaining row with one K = 256 GEMM, which runs
// near the DMMA roofline where K = 64 tiles do not.  Each 64-row block still
// owns exactly one GEMM, so every straddling 2x2 e-entry is applied once and
// corrected once by the next diagonal kernel.  d_tasks: >= 2 * ceil(n/64) *
// batch GEMM records.
static int ldlt_solve_blocked_impl(int batch, int n, const void* F, int64_t stride_f, const void* perm,
                                   int64_t stride_p, const void* tags, int64_t stride_t, void* B, int64_t stride_b,
                                   int ldb, int m, void* work, void* d_tasks, void* stream, bool fwd_only,
                                   const int32_t* h_mcols = nullptr, int tail = 0);

int d3m_ldlt_solve_blocked_batched(int batch, int n, const void* F, int64_t stride_f, const void* perm,
                                   int64_t stride_p, const void* tags, int64_t stride_t, void* B, int64_t stride_b,
                                   int ldb, int m, void* work, void* d_tasks, void* stream) {
  return ldlt_solve_blocked_impl(batch, n, F, stride_f, perm, stride_p, tags, stride_t, B, stride_b, ldb, m, work,
                                 d_tasks, stream, false);
}

// fwd_only: stop after Z = L^-1 P B (left in `work`, pivot order): the Schur
// reduction K = Z^T D^-1 Z needs no backward sweep.
// h_mcols / tail: matrix b's columns [h_mcols[b], m - tail) are zero right-hand sides (padding of the
// coupling block): the GEMM updates run on [0, h_mcols[b]) and [m - tail, m) only -- up to two tasks per
// matrix and block step (d_tasks: 4 * ceil(n/64) * batch records then).
static int ldlt_solve_blocked_impl(int batch, int n, const void* F, int64_t stride_f, const void* perm,
                                   int64_t stride_p, const void* tags, int64_t stride_t, void* B, int64_t stride_b,
                                   int ldb, int m, void* work, void* d_tasks, void* stream, bool fwd_only,
                                   const int32_t* h_mcols, int tail) {
  if (batch < 0 || n < 0 || m < 0 || ldb < m) return fail(-22, "d3m_ldlt_solve_blocked_batched: bad shape");
  if (batch == 0 || n == 0 || m == 0) return 0;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int DBR = d3m_diag_block_rows();
  const int OBR = 4 * DBR;                       // outer block rows
  const int nblk = (n + DBR - 1) / DBR;
  const int64_t sz = (int64_t)n * m;
  d3m::SolveBatch sb{CC(F), stride_f, static_cast<const int8_t*>(tags), stride_t, static_cast<const int64_t*>(perm),
                     stride_p, C(work), sz, nullptr, 0, CC(B), stride_b, n, m, m, ldb};
  // column ranges with nonzero right-hand sides: (matrix, first column, count)
  struct Range { int b, c0, nc; };
  std::vector<Range> rg;
  for (int b = 0; b < batch; ++b) {
    const int mc = h_mcols ? std::max(0, std::min((int)h_mcols[b], m - tail)) : m - tail;
    if (h_mcols && mc < m - tail) {
      if (mc > 0) rg.push_back({b, 0, mc});
      if (tail > 0) rg.push_back({b, m - tail, tail});
    } else {
      rg.push_back({b, 0, m});
    }
  }
  const int T = (int)rg.size();          // tasks per block step and sweep
  // GEMM task table: [fwd ib][q] then [bwd ib][q]
  std::vector<d3m::GemmTask> t((size_t)2 * nblk * T);
  std::memset(t.data(), 0, sizeof(d3m::GemmTask) * t.size());
  std::vector<int> tiles(2 * nblk, 0);
  for (int ib = 0; ib < nblk; ++ib) {
    const int r0 = ib * DBR, r1 = std::min(n, r0 + DBR);
    const int R0 = (r0 / OBR) * OBR, R1 = std::min(n, R0 + OBR);
    for (int q = 0; q < T; ++q) {
      const int b = rg[q].b, c0 = rg[q].c0, nc = rg[q].nc;
      d3m::GemmTask& f = t[(size_t)ib * T + q];
      if (r1 < R1) {          // Z[r1:R1] -= L[r1:R1, r0:r1] Z[r0:r1]
        f.a_off = b * stride_f + (int64_t)r1 * n + r0;
        f.b_off = b * sz + (int64_t)r0 * m + c0;
        f.c_off = b * sz + (int64_t)r1 * m + c0;
        f.m = R1 - r1; f.k = r1 - r0;
      } else {                // Z[R1:] -= L[R1:, R0:R1] Z[R0:R1]
        f.a_off = b * stride_f + (int64_t)R1 * n + R0;
        f.b_off = b * sz + (int64_t)R0 * m + c0;
        f.c_off = b * sz + (int64_t)R1 * m + c0;
        f.m = n - R1; f.k = R1 - R0;
      }
      f.n = nc; f.lda = n; f.ldb = m; f.ldc = m; f.flags = d3m::kGemmSub;
      f.pad_ = b;             // matrix index (the TMA kernel's per-matrix tensor maps)
      d3m::GemmTask& g = t[(size_t)(nblk + ib) * T + q];
      if (r0 > R0) {          // Z[R0:r0] -= L[r0:r1, R0:r0]^T Z[r0:r1]
        g.a_off = b * stride_f + (int64_t)r0 * n + R0;
        g.b_off = b * sz + (int64_t)r0 * m + c0;
        g.c_off = b * sz + (int64_t)R0 * m + c0;
        g.m = r0 - R0; g.k = r1 - r0;
      } else {                // Z[:R0] -= L[R0:R1, :R0]^T Z[R0:R1]
        g.a_off = b * stride_f + (int64_t)R0 * n;
        g.b_off = b * sz + (int64_t)R0 * m + c0;
        g.c_off = b * sz + c0;
        g.m = R0; g.k = R1 - R0;
      }
      g.n = nc; g.lda = n; g.ldb = m; g.ldc = m; g.flags = d3m::kGemmSub;
      g.pad_ = b;
    }
    tiles[ib] = d3m_gemm_prepare_tasks(&t[(size_t)ib * T], T);
    tiles[nblk + ib] = d3m_gemm_prepare_tasks(&t[(size_t)(nblk + ib) * T], T);
  }
  // The task table and the tensor maps go up from a pinned, event-guarded staging buffer kept per
  // (device, stream): a copy from pageable memory of this size would synchronise the stream first, i.e.
  // hold the host until the factorisation before this solve has finished, and the solve's launches would
  // then be enqueued with the GPU idle.
  // TMA-staged updates (3M form; D3M_SOLVE_TMA=0: the cp.async grouped kernel): per matrix tensor maps over
  // the factor and the work array.  A launch qualifies when its k range is a multiple of 16 (all but a
  // ragged last block): rows past K inside the matrices are data, not zeros.
  const size_t task_bytes = sizeof(d3m::GemmTask) * t.size();
  const size_t map_bytes = (size_t)batch * 4 * 128;
  const char* tma_str = getenv("D3M_SOLVE_TMA");
  const bool want_tma = !(tma_str && atoi(tma_str) == 0) && d3m_gemm_set_form(0) == 3;
  const void* d_maps = nullptr;
  {
    struct Stage {
      void* host = nullptr;      // pinned: [tasks | maps]
      size_t host_cap = 0;
      void* dev_maps = nullptr;
      size_t dev_cap = 0;
      cudaEvent_t done = nullptr;
    };
    static std::mutex mu;
    static std::map<std::pair<int, void*>, Stage> stages;      // grow-only
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    Stage& st = stages[{dev, stream}];
    if (!st.done && cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming) != cudaSuccess)
      return fail(-12, "d3m_ldlt_solve_blocked_batched: event");
    cudaEventSynchronize(st.done);                             // the previous call's copies have left the buffer
    const size_t need = task_bytes + map_bytes;
    if (st.host_cap < need) {
      if (st.host) cudaFreeHost(st.host);
      st.host = nullptr;
      st.host_cap = 0;
      if (cudaMallocHost(&st.host, need) != cudaSuccess) return fail(-12, "d3m_ldlt_solve_blocked_batched: pinned staging");
      st.host_cap = need;
    }
    std::memcpy(st.host, t.data(), task_bytes);
    unsigned char* hm = static_cast<unsigned char*>(st.host) + task_bytes;
    bool maps_ok = false;
    if (want_tma) {
      const int rc = d3m_gemm_tma_prepare_solve(F, stride_f, n, work, sz, m, batch, hm);
      if (rc == 0) {
        if (st.dev_cap < map_bytes) {
          if (st.dev_maps) { cudaStreamSynchronize(s); cudaFree(st.dev_maps); }
          st.dev_maps = nullptr;
          st.dev_cap = 0;
          if (cudaMalloc(&st.dev_maps, map_bytes) == cudaSuccess) st.dev_cap = map_bytes;
          else cudaGetLastError();
        }
        maps_ok = st.dev_maps != nullptr;
      } else if (rc != -38) {
        return fail(rc, "d3m_ldlt_solve_blocked_batched: tensor map");
      }
    }
    cudaError_t e = cudaMemcpyAsync(d_tasks, st.host, task_bytes, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && maps_ok) {
      e = cudaMemcpyAsync(st.dev_maps, hm, map_bytes, cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) d_maps = st.dev_maps;
    }
    cudaEventRecord(st.done, s);
    if (e != cudaSuccess) return fail((int)e, "d3m_ldlt_solve_blocked_batched: task upload");
  }
  auto* dt = static_cast<const d3m::GemmTask*>(d_tasks);
  const char* d_fwd_maps = static_cast<const char*>(d_maps);
  const char* d_bwd_maps = d_fwd_maps ? d_fwd_maps + (size_t)batch * 2 * 128 : nullptr;
  auto tma_ok = [&](int task_row) { return d_maps && (t[(size_t)task_row * T].k % 16) == 0; };
  D3M_TRY(launch(kClsSolve, stream, [&] { return d3m_solve_phase_launch(0, &sb, batch, stream); }));   // Z = B[perm]
  for (int ib = 0; ib < nblk; ++ib) {
    const int r0 = ib * DBR;
    D3M_TRY(launch(kClsSolve, stream, [&] {
      return d3m_diag_block_launch(1, F, stride_f, tags, stride_t, work, sz, n, m, r0, batch, stream);
    }));
    if (tiles[ib] > 0)
      D3M_TRY(launch(kClsGemm, stream, [&] {
        if (tma_ok(ib))
          return d3m_gemm_tma_launch_batched_t(0, d_fwd_maps, work, dt + (size_t)ib * T, T, tiles[ib], stride_f, sz,
                                               stream);
        return d3m_gemm_launch(0, 1, F, work, work, dt + (size_t)ib * T, T, tiles[ib], stream);
      }));
  }
  if (fwd_only) return 0;
  D3M_TRY(launch(kClsSolve, stream, [&] { return d3m_solve_phase_launch(2, &sb, batch, stream); }));   // D^-1
  for (int ib = nblk - 1; ib >= 0; --ib) {
    const int r0 = ib * DBR;
    D3M_TRY(launch(kClsSolve, stream, [&] {
      return d3m_diag_block_launch(0, F, stride_f, tags, stride_t, work, sz, n, m, r0, batch, stream);
    }));
    if (tiles[nblk + ib] > 0)
      D3M_TRY(launch(kClsGemm, stream, [&] {
        if (tma_ok(nblk + ib))
          return d3m_gemm_tma_launch_batched_t(1, d_bwd_maps, work, dt + (size_t)(nblk + ib) * T, T, tiles[nblk + ib],
                                               stride_f, sz, stream);
        return d3m_gemm_launch(1, 1, F, work, work, dt + (size_t)(nblk + ib) * T, T, tiles[nblk + ib], stream);
      }));
  }
  D3M_TRY(launch(kClsSolve, stream, [&] { return d3m_solve_phase_launch(4, &sb, batch, stream); }));   // B[perm] = Z
  return 0;
}

int d3m_bk_panel_batched(int batch, int n, void* W, int64_t stride_w, int lda, double pivot_tol, int check_sym,
                         void* perm, void* tags, void* n2x2, void* growth, void* info, void* scale, void* asym,
                         void* workspace, void* margin, void* stream) {
  if (batch < 0 || n < 0 || lda < n) return fail(-22, "d3m_bk_panel_batched: bad shape");
  const bool lower_only = (check_sym & 8) != 0;      // ABI v11: scale from the lower triangle only
  check_sym = lower_only ? 0 : (check_sym & 3);
  d3m::BkArgs a{C(W), stride_w, n, lda, pivot_tol, check_sym, static_cast<int64_t*>(perm), static_cast<int8_t*>(tags),
                static_cast<int32_t*>(n2x2), static_cast<double*>(growth), static_cast<int32_t*>(info),
                static_cast<double*>(scale), static_cast<double*>(asym), nullptr};
  a.margin = static_cast<double*>(margin);
  a.lower_only = lower_only;
  D3M_TRY(launch(kClsBk, stream, [&] { return d3m_bk_panel_batched_launch(&a, batch, workspace, stream); }));
  return 0;
}

size_t d3m_bk_panel_workspace(int n, int batch) { return d3m_bk_panel_workspace_bytes(n, batch); }

int d3m_sym_scan_batched(int batch, int n, const void* W, int64_t stride_w, int lda, void* scale, void* asym,
                         void* workspace, void* stream) {
  if (batch < 0 || n < 0 || lda < n) return fail(-22, "d3m_sym_scan_batched: bad shape");
  d3m::BkArgs a{C(const_cast<void*>(W)), stride_w, n, lda, 0.0, 1, nullptr, nullptr, nullptr, nullptr, nullptr,
                static_cast<double*>(scale), static_cast<double*>(asym), nullptr};
  D3M_TRY(launch(kClsMisc, stream, [&] { return d3m_sym_scan_batched_launch(&a, batch, workspace, stream); }));
  return 0;
}

// Row-block pieces of square row-major n x n matrices (16-byte elements):
// part 0 copies rows [r0, r1) x columns [0, r1) of each 128-row block -- the
// lower triangle plus the upper triangles inside the diagonal blocks (53% of
// the bytes at n = 2048) -- and part 1 the rest, rows [r0, r1) x [r1, n).
// One cudaMemcpy2DAsync per piece; kind is a cudaMemcpyKind.
int d3m_copy_triangle(int batch, const void* const* src, int64_t src_ld, void* dst, int64_t dst_stride,
                      int64_t dst_ld, int n, int part, int kind, void* stream) {
  if (batch < 0 || n < 0 || src_ld < n || dst_ld < n || (part != 0 && part != 1))
    return fail(-22, "d3m_copy_triangle: bad arguments");
  constexpr int kRb = 128;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  for (int b = 0; b < batch; ++b) {
    const char* sb = static_cast<const char*>(src[b]);
    char* db = static_cast<char*>(dst) + (size_t)b * dst_stride * 16;
    for (int r0 = 0; r0 < n; r0 += kRb) {
      const int r1 = std::min(n, r0 + kRb);
      const int c0 = part == 0 ? 0 : r1, c1 = part == 0 ? r1 : n;
      if (c1 <= c0) continue;
      cudaError_t e = cudaMemcpy2DAsync(db + ((size_t)r0 * dst_ld + c0) * 16, (size_t)dst_ld * 16,
                                        sb + ((size_t)r0 * src_ld + c0) * 16, (size_t)src_ld * 16,
                                        (size_t)(c1 - c0) * 16, (size_t)(r1 - r0), (cudaMemcpyKind)kind, s);
      if (e != cudaSuccess) return fail((int)e, "d3m_copy_triangle: cudaMemcpy2DAsync");
    }
  }
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
  D3M_TRY(launch(kClsGemm, stream, [&] { return d3m_gemm_launch(ta, tb, A, B, Cm, d_tasks, ntasks, tiles, stream); }));
  return 0;
}

int d3m_zgemm_tma_panels(const void* X, int64_t rows_x, const void* L, int64_t rows_l, int n, void* Cm,
                         void* h_tasks, int ntasks, void* d_tasks, void* stream) {
  if (ntasks <= 0) return 0;
  if (rows_x <= 0 || rows_l <= 0 || n <= 0) return fail(-22, "d3m_zgemm_tma_panels: bad shape");
  auto* t = static_cast<d3m::GemmTask*>(h_tasks);
  for (int i = 0; i < ntasks; ++i)
    if (t[i].lda != n || t[i].ldb != n || t[i].k != n || t[i].a_off % n || t[i].b_off % n ||
        (t[i].flags & ~(d3m::kGemmModeMask | d3m::kGemmSym | d3m::kGemmLowerOnly)))
      return fail(-22, "d3m_zgemm_tma_panels: task does not fit the panel form");
  const int tiles = d3m_gemm_prepare_tasks(t, ntasks);
  cudaError_t e = cudaMemcpyAsync(d_tasks, t, sizeof(d3m::GemmTask) * ntasks, cudaMemcpyHostToDevice,
                                  reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail((int)e, "d3m_zgemm_tma_panels: task upload");
  alignas(64) unsigned char maps[256];
  const int prc = d3m_gemm_tma_prepare(X, rows_x, L, rows_l, n, maps);
  if (prc) return fail(prc, "d3m_zgemm_tma_panels: tensor map encoding");
  D3M_TRY(launch(kClsGemm, stream,
                 [&] { return d3m_gemm_tma_launch(maps, Cm, d_tasks, ntasks, tiles, 0, stream); }));
  return 0;
}

int d3m_schur_reduce_batched(int batch, int n, int m, int nrhs, void* A, const void* D, const void* f,
                             double pivot_tol, void* perm, void* tags, void* n2x2, void* growth, void* info,
                             void* scale, void* asym, void* K_out, void* g_out, void* work_z, void* work_x,
                             void* work_c, void* bk_scratch, void* d_tasks, const void* rows, int nrows,
                             void* work_d, int flags, void* margin, const int32_t* h_mcols, void* stream) {
  // A: batch x n x n (factored in place -> packed factor); D: batch x n x m;
  // F: batch x n x nrhs; work_z, work_x: batch x n x (m+nrhs); work_c: batch x m x (m+nrhs)
  if (batch < 0 || n < 0 || m < 0 || nrhs < 0) return fail(-22, "d3m_schur_reduce_batched: bad shape");
  if (batch == 0) return 0;
  const int w = m + nrhs;
  const int64_t nn = (int64_t)n * n, nw = (int64_t)n * w;
  const bool big = n > kPanelBkMin;
  // large subdomains: batched blocked BK (panel kernel + grouped DMMA trailing
  // updates, bk_scratch >= d3m_bk_panel_workspace(n, batch) bytes); small:
  // the unblocked bit-exact kernel.  flags bit 1: A already holds the factor
  // (the caller ran the BK itself, e.g. on a split upload)
  const bool factored = (flags & 2) != 0;
  if (big && !factored)
    D3M_TRY(d3m_bk_panel_batched(batch, n, A, nn, n, pivot_tol, 1, perm, tags, n2x2, growth, info, scale, asym,
                                 bk_scratch, margin, stream));
  else if (!factored)
    D3M_TRY(d3m_bk_factor_batched(batch, n, A, nn, n, pivot_tol, 1, perm, tags, n2x2, growth, info, scale, asym,
                                  bk_scratch, margin, stream));
  if (n == 0 || w == 0) return 0;
  // RHS = [D | F]  (subdomain.py:177-179)
  D3M_TRY(launch(kClsMisc, stream, [&] {
    return d3m_pack_rhs_launch(D, f, work_x, n, m, nrhs, batch, (int64_t)n * m, (int64_t)n * nrhs, nw, stream);
  }));
  if ((flags & 1) && m > 0) {
    // Schur only: A^-1 = P^T L^-T D^-1 L^-1 P, so with Z = L^-1 P [D | F]
    // (forward sweep only) C = Z_D^T D^-1 Z = D^T A^-1 [D | F]
    if (big)
      D3M_TRY(ldlt_solve_blocked_impl(batch, n, A, nn, perm, n, tags, n, work_x, nw, w, w, work_z, d_tasks, stream,
                                      true, h_mcols, nrhs));
    else {
      d3m::SolveBatch sf{CC(A), nn, static_cast<const int8_t*>(tags), n, static_cast<const int64_t*>(perm), n,
                         C(work_z), nw, nullptr, 0, CC(work_x), nw, n, w, w, w};
      for (int phase = 0; phase < 2; ++phase)
        D3M_TRY(launch(kClsSolve, stream, [&] { return d3m_solve_phase_launch(phase, &sf, batch, stream); }));
    }
    // U = D^-1 Z (work_x), Z stays in work_z
    cudaError_t ce = cudaMemcpyAsync(work_x, work_z, sizeof(cplx) * (size_t)batch * nw, cudaMemcpyDeviceToDevice,
                                     reinterpret_cast<cudaStream_t>(stream));
    if (ce != cudaSuccess) return fail((int)ce, "d3m_schur_reduce_batched: copy");
    d3m::SolveBatch su{CC(A), nn, static_cast<const int8_t*>(tags), n, static_cast<const int64_t*>(perm), n,
                       C(work_x), nw, nullptr, 0, CC(work_x), nw, n, w, w, w};
    D3M_TRY(launch(kClsSolve, stream, [&] { return d3m_solve_phase_launch(2, &su, batch, stream); }));
    std::vector<d3m::GemmTask> t(batch);
    for (int b = 0; b < batch; ++b) {
      d3m::GemmTask& k = t[b];
      std::memset(&k, 0, sizeof(k));
      k.a_off = (int64_t)b * nw;           // Z_D: n x (m + nrhs), first m columns = K x M (TA)
      k.b_off = (int64_t)b * nw;           // U: n x (m + nrhs) = K x N (TB)
      k.c_off = (int64_t)b * m * w;
      k.m = m;
      k.n = w;
      k.k = n;
      k.lda = w;
      k.ldb = w;
      k.ldc = w;
      k.flags = d3m::kGemmStore;
    }
    D3M_TRY(d3m_zgemm_grouped(1, 1, work_z, work_x, work_c, t.data(), batch, d_tasks, stream));
    D3M_TRY(launch(kClsMisc, stream, [&] {
      return d3m_schur_finalize_launch(work_c, K_out, g_out, m, nrhs, batch, (int64_t)m * w, (int64_t)m * m,
                                       (int64_t)m * nrhs, stream);
    }));
    return 0;
  }
  // X = A^-1 RHS (factor.py:52-66)
  if (big)
    D3M_TRY(ldlt_solve_blocked_impl(batch, n, A, nn, perm, n, tags, n, work_x, nw, w, w, work_z, d_tasks, stream,
                                    false, h_mcols, nrhs));
  else
    D3M_TRY(d3m_ldlt_solve_batched(batch, n, A, nn, perm, n, tags, n, work_x, nw, w, w, work_z, stream));
  if (m == 0) return 0;
  // C = D^T [X_D | X_F]  (subdomain.py:181,183) on DMMA, one task per domain.
  // With a row list (the rows where D has nonzeros, ascending, -1 padded) the
  // product runs over those rows only: D and X rows are gathered into
  // compact buffers first (work_d: batch x nrows x m; work_z reused for X).
  const bool sparse = rows != nullptr && nrows > 0 && nrows < n;
  if (sparse) {
    D3M_TRY(launch(kClsMisc, stream, [&] {
      return d3m_gather_rows_batched_launch(D, (int64_t)n * m, m, rows, nrows, m, work_d, (int64_t)nrows * m, batch,
                                            stream);
    }));
    D3M_TRY(launch(kClsMisc, stream, [&] {
      return d3m_gather_rows_batched_launch(work_x, nw, w, rows, nrows, w, work_z, (int64_t)nrows * w, batch, stream);
    }));
  }
  const int kdim = sparse ? nrows : n;
  std::vector<d3m::GemmTask> t(batch);
  for (int b = 0; b < batch; ++b) {
    d3m::GemmTask& k = t[b];
    std::memset(&k, 0, sizeof(k));
    k.a_off = (int64_t)b * kdim * m;       // D stored kdim x m = K x M  (TA)
    k.b_off = (int64_t)b * (sparse ? (int64_t)nrows * w : nw);   // X stored kdim x (m+nrhs) = K x N (TB)
    k.c_off = (int64_t)b * m * w;
    k.m = m;
    k.n = w;
    k.k = kdim;
    k.lda = m;
    k.ldb = w;
    k.ldc = w;
    k.flags = d3m::kGemmStore;
  }
  D3M_TRY(d3m_zgemm_grouped(1, 1, sparse ? work_d : D, sparse ? work_z : work_x, work_c, t.data(), batch, d_tasks,
                            stream));
  // K_D = 0.5 (K_D + K_D^T), G_d
  D3M_TRY(launch(kClsMisc, stream, [&] {
    return d3m_schur_finalize_launch(work_c, K_out, g_out, m, nrhs, batch, (int64_t)m * w, (int64_t)m * m,
                                     (int64_t)m * nrhs, stream);
  }));
  return 0;
}

int d3m_block_copy(const void* src, void* dst, const void* d_tasks, int ntasks, int64_t max_elems, void* stream) {
  D3M_TRY(launch(kClsMisc, stream, [&] { return d3m_block_copy_launch(src, dst, d_tasks, ntasks, max_elems, stream); }));
  return 0;
}

int d3m_block_residual(int nlaunch, const int32_t* h_ta, const int32_t* h_ntasks, const int32_t* h_ntiles,
                       const int64_t* h_task_off, const void* const* h_abase, const void* x, void* r,
                       const void* d_tasks, void* stream) {
  if (nlaunch < 0) return fail(-22, "d3m_block_residual: bad launch count");
  const auto* tasks = static_cast<const d3m::GemmTask*>(d_tasks);
  for (int l = 0; l < nlaunch; ++l) {
    D3M_TRY(launch(kClsSolve, stream, [&] {
      return d3m_gemm_launch(h_ta[l], 1, h_abase[l], x, r, tasks + h_task_off[l], h_ntasks[l], h_ntiles[l], stream);
    }));
  }
  return 0;
}

int d3m_nonzero_rows(int B, int n, int m, const void* D, void* flag, void* idx, void* count, void* stream) {
  if (B < 0 || n < 0 || m < 0) return fail(-22, "d3m_nonzero_rows: bad shape");
  D3M_TRY(launch(kClsMisc, stream, [&] { return d3m_nonzero_rows_launch(B, n, m, D, flag, idx, count, stream); }));
  return 0;
}

int d3m_gather_rows(const void* src, const void* idx, void* out, int64_t nrows, int cols, void* stream) {
  D3M_TRY(launch(kClsMisc, stream, [&] { return d3m_gather_index_launch(src, idx, out, nrows, cols, stream); }));
  return 0;
}

int d3m_ordered_average(const void* E, const void* ptr, const void* src, void* out, int64_t ng, void* stream) {
  D3M_TRY(launch(kClsMisc, stream, [&] { return d3m_ordered_average_launch(E, ptr, src, out, ng, stream); }));
  return 0;
}

int d3m_diag_sym_flags(const void* pool, const void* off, const void* n, const void* idx, int count, void* flags,
                       void* stream) {
  D3M_TRY(launch(kClsMisc, stream, [&] { return d3m_sym_flags_launch(pool, off, n, idx, count, flags, stream); }));
  return 0;
}

int d3m_diag_sym_exact(const void* pool, const void* off, const void* n, int nb, void* flag, void* stream) {
  D3M_TRY(launch(kClsMisc, stream, [&] { return d3m_sym_exact_launch(pool, off, n, nb, flag, stream); }));
  return 0;
}

int d3m_zero(void* p, int64_t n, void* stream) {
  D3M_TRY(launch(kClsMisc, stream, [&] { return d3m_zero_launch(p, n, stream); }));
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
                        const int64_t* h_panel_rows, const int64_t* h_piv_off, const int64_t* h_binv_off,
                        const int64_t* h_task_ptr, const int64_t* h_task_next, const int64_t* h_tiles_next,
                        const int64_t* h_tiles_rest, const int64_t* h_tiles_trsm, const void* d_tasks,
                        const void* d_trsm_tasks, void* d_pool, void* d_binv, void* d_xbuf, int64_t xbuf_elems,
                        void* d_perm, void* d_tags, void* d_info, void* d_n2x2, void* d_growth, void* d_scale,
                        void* d_asym, void* d_bk_scratch, double pivot_tol, int check_sym, int lookahead,
                        int nwait, const int64_t* h_wait_col, void* const* h_wait_ev, const void* d_check_sym,
                        void* d_margin, const int32_t* h_sched, void* stream) {
  // rest-update tiles above which a column's diagonal BK runs on a 4-CTA cluster (D3M_BKC4_TILES)
  static const int64_t bkc4_tiles = [] {
    const char* e = getenv("D3M_BKC4_TILES");
    return e ? (int64_t)atoll(e) : (int64_t)5000;
  }();
  static const bool trsm_tri = [] { const char* e = getenv("D3M_TRSM_TRI"); return !(e && e[0] == '0'); }();
  // update GEMM staging: 1 = TMA tensor copies (default), 0 = the cp.async kernel (D3M_GEMM_TMA, A/B runs)
  static const int gemm_tma = [] { const char* e = getenv("D3M_GEMM_TMA"); return e ? atoi(e) : 1; }();
  // every column's X panel must fit its xbuf slot: checked before anything is launched
  const int nslots = lookahead ? kXSlots : 1;
  const int64_t slot_elems = xbuf_elems / nslots;
  for (int j = 0; j < nb; ++j)
    if (h_panel_rows[j] * h_sizes[j] > slot_elems) return fail(-22, "d3m_block_ldlt_exec: xbuf too small");
  if (lookahead && !h_sched) return fail(-22, "d3m_block_ldlt_exec: etree schedule missing");
  ExecCtx* ctx = exec_ctx();
  if (!ctx) return fail(-12, "d3m_block_ldlt_exec: stream/event/scratch creation");
  // calls on one device share its streams and buffers: they enqueue one at a
  // time (stream order then keeps their kernels apart)
  std::lock_guard<std::mutex> guard(ctx->mu);
  if (!ctx->grow_events((size_t)nb)) return fail(-12, "d3m_block_ldlt_exec: event creation");
  int64_t nmax = 0;
  for (int j = 0; j < nb; ++j) nmax = std::max<int64_t>(nmax, h_sizes[j]);
  // D^-1 coefficients of the columns in flight (3 complex per pivot column), one ring slot per column
  const size_t coef_bytes = (size_t)nslots * 3 * std::max<int64_t>(nmax, 1) * sizeof(cplx);
  if (coef_bytes > ctx->coef_cap) {
    if (ctx->coef_buf) cudaFree(ctx->coef_buf);      // synchronising: no earlier call still reads it
    ctx->coef_buf = nullptr;
    ctx->coef_cap = 0;
    if (cudaMalloc(&ctx->coef_buf, coef_bytes) != cudaSuccess) return fail(-12, "d3m_block_ldlt_exec: coef alloc");
    ctx->coef_cap = coef_bytes;
  }
  // unpermuted L_jj^-1 of every column (same layout as binv), for the triangular panel TRSM
  cplx* linv_use = nullptr;
  if (trsm_tri) {
    const int64_t need = h_binv_off[nb];
    if (need > ctx->linv_cap) {
      if (ctx->linv) cudaFree(ctx->linv);
      ctx->linv = nullptr;
      ctx->linv_cap = 0;
      if (cudaMalloc(&ctx->linv, sizeof(cplx) * (size_t)std::max<int64_t>(need, 1)) != cudaSuccess)
        return fail(-12, "d3m_block_ldlt_exec: linv alloc");
      ctx->linv_cap = need;
    }
    linv_use = ctx->linv;
  }
  int tma_mode = d3m_gemm_set_form(0) == 3 ? gemm_tma : 0;     // the TMA kernel is a 3M kernel
  // Streams.  lookahead = 0: everything in order on the caller's stream.
  // lookahead = 1 (etree-parallel): the critical chain of column j (BK ->
  // L^-1 -> panel TRSM -> D^-1 -> the "next" update into column j+1) runs on
  // one of kCritStreams high-priority streams, h_sched[3j] (the stream of
  // its last child, so a chain stays on one stream and independent subtrees
  // of the elimination tree overlap); the bulk ("rest") updates of every
  // column run on ONE low-priority stream in column order, so every target
  // block receives its updates in ascending source-column order and the
  // factor is bitwise that of the sequential executor.  Cross-stream
  // dependencies are events:
  //   BK(j)        after the bulk update of h_sched[3j+1] = the last column
  //                k < j-1 whose bulk update writes column j (the side stream
  //                is ordered, so all earlier ones are done too), and after
  //                column j-1's critical work when it updates column j;
  //   next(j)      after the bulk update of h_sched[3j+2] = the last k < j
  //                whose bulk update writes column j+1 (ascending order);
  //   TRSM(j)      after the readers of its X ring slot, column j - kXSlots
  //                (its next and bulk updates);
  //   rest(j)      after column j's critical work.
  // Waits a stream already implies (an earlier wait on a later bulk event, or
  // its own earlier work) are skipped, so a chain-shaped plan (natural order)
  // enqueues exactly the lookahead-1 pipeline.
  cudaStream_t user = reinterpret_cast<cudaStream_t>(stream);
  cudaStream_t side = ctx->side;
  int rest_waited[kCritStreams];                      // largest bulk-event column each stream has waited on
  int chunk_waited[kCritStreams] = {};                // upload chunks each stream has waited on
  bool used[kCritStreams] = {};
  for (int q = 0; q < kCritStreams; ++q) rest_waited[q] = -1;
  if (lookahead) {
    cudaEventRecord(ctx->ev_in, user);
    for (int q = 0; q < kCritStreams; ++q) cudaStreamWaitEvent(ctx->crit[q], ctx->ev_in, 0);
    cudaStreamWaitEvent(side, ctx->ev_in, 0);
  }
  std::vector<int> col_stream(nb, 0);
  std::vector<char> has_rest(nb, 0);
  auto* tasks = static_cast<const d3m::GemmTask*>(d_tasks);
  auto* ttasks = static_cast<const d3m::GemmTask*>(d_trsm_tasks);
  cplx* pool = C(d_pool);
  cplx* binv = C(d_binv);
  auto wait_rest = [&](int q, cudaStream_t st, int k) {     // stream q waits for the bulk update of column k
    if (k < 0 || k <= rest_waited[q]) return;
    // the latest bulk update at or before k that exists (columns without one recorded nothing)
    while (k >= 0 && !has_rest[k]) --k;
    if (k < 0 || k <= rest_waited[q]) return;
    cudaStreamWaitEvent(st, ctx->ev_rest[k], 0);
    rest_waited[q] = k;
  };
  // all columns; an early return (a failed launch) still reaches the join below
  auto columns = [&]() -> int {
    for (int j = 0; j < nb; ++j) {
      const int q = lookahead ? std::min(std::max(h_sched[3 * j], 0), kCritStreams - 1) : 0;
      cudaStream_t s0 = lookahead ? ctx->crit[q] : user;
      col_stream[j] = q;
      used[q] = true;
      // blocks of K still being uploaded: before column j its stream waits
      // for every chunk first touched at or before column j that it has not
      // waited for yet (the chunks' columns ascend)
      while (chunk_waited[q] < nwait && h_wait_col[chunk_waited[q]] <= j)
        cudaStreamWaitEvent(s0, static_cast<cudaEvent_t>(h_wait_ev[chunk_waited[q]++]), 0);
      if (lookahead) {
        wait_rest(q, s0, h_sched[3 * j + 1]);
        // column j-1's next update writes column j (j = parent(j-1)): on another stream, wait for it
        if (j > 0 && h_task_next[j - 1] > h_task_ptr[j - 1] && col_stream[j - 1] != q)
          cudaStreamWaitEvent(s0, ctx->ev_col[j - 1], 0);
        // the X / coefficient ring slot of column j was last used by column j - nslots
        const int o = j - nslots;
        if (o >= 0) {
          if (col_stream[o] != q) cudaStreamWaitEvent(s0, ctx->ev_col[o], 0);
          wait_rest(q, s0, has_rest[o] ? o : -1);
        }
      }
      const int nj = (int)h_sizes[j];
      const int64_t R = h_panel_rows[j];
      const int slot = j % nslots;
      cplx* xbuf = C(d_xbuf) + slot * slot_elems;
      int64_t* perm = static_cast<int64_t*>(d_perm) + h_piv_off[j];
      int8_t* tags = static_cast<int8_t*>(d_tags) + h_piv_off[j];
      cplx* diag = pool + h_diag_off[j];
      cplx* coef = static_cast<cplx*>(ctx->coef_buf) + (size_t)slot * 3 * nmax;
      d3m::BkArgs a{diag, 0, nj, nj, pivot_tol, check_sym, perm, tags,
                    static_cast<int32_t*>(d_n2x2) + j, static_cast<double*>(d_growth) + j,
                    static_cast<int32_t*>(d_info) + j, static_cast<double*>(d_scale) + j,
                    static_cast<double*>(d_asym) + j,
                    d_bk_scratch ? C(d_bk_scratch) + (size_t)q * 4 * nmax : nullptr};
      if (d_check_sym) a.check_sym_dev = static_cast<const int*>(d_check_sym) + j;   // per-block flag (ABI v8)
      if (d_margin) a.margin = static_cast<double*>(d_margin) + 2 * j;               // decision margins (ABI v9)
      if (nj > 0) {
        // supernodes up to kExactBkMax use the bit-exact unblocked kernel (so a
        // one-block K factors exactly like dense_ldlt_bk, test_block_factor.py:
        // 24-32); wider ones the bit-exact cluster kernel (lower triangle in the
        // cluster's shared memory, 8- or 16-CTA clusters), else the exact one
        D3M_TRY(launch(kClsBk, s0, [&] {
          if (nj <= kExactBkMax) return d3m_bk_launch(&a, 1, s0);
          // 4-CTA clusters while the column's bulk update is long enough to hide the slower BK
          // (frees 4 SMs for the update GEMMs), 8-CTA clusters on the exposed chain at the ends;
          // a block too wide for the requested size moves to a larger cluster
          const int cs = (lookahead && h_tiles_rest[j] >= bkc4_tiles) ? 4 : 0;
          const int rc = d3m_bk_cluster_launch_cs(&a, 1, cs, s0);
          return rc == -22 ? d3m_bk_launch(&a, 1, s0) : rc;
        }));
        // Binv_j = L_jj^-1 P_j (also used by block_solve) + D_jj^-1 coefficients
        D3M_TRY(launch(kClsTrsm, s0, [&] {
          // blocked 16 x 16 inverse (n <= 256), else warp per column (n <= 512), else the generic kernel
          cplx* lj = linv_use ? linv_use + h_binv_off[j] : nullptr;   // unpermuted L^-1 for the panel TRSM
          int rc = d3m_tri_inv_blocked_launch(diag, perm, tags, binv + h_binv_off[j], coef, nj, lj, ctx->dinv[q], s0);
          if (rc == -22) rc = d3m_tri_inv_warp_launch(diag, perm, tags, binv + h_binv_off[j], coef, nj, s0, lj);
          return rc == -22 ? d3m_tri_inv_launch(diag, 0, perm, 0, tags, 0, binv + h_binv_off[j], 0, nj, 1, s0) : rc;
        }));
      }
      if (R > 0) {
        // X_ij = K_ij P^T L_jj^-T = panel * Binv^T on DMMA, then L_ij = X_ij D_jj^-1
        D3M_TRY(launch(kClsTrsm, s0, [&] {
          // nj <= kTrsmTriMax: X = (K P^T) L^-T with the column gather and the triangular K cut
          // (the task carries kGemmTriGather, factor.py); else X = K Binv^T
          if (linv_use && nj <= kTrsmTriMax)
            return d3m_gemm_launch_perm(pool, linv_use, xbuf, ttasks + j, 1, (int)h_tiles_trsm[j], d_perm, s0);
          return d3m_gemm_launch(0, 0, pool, binv, xbuf, ttasks + j, 1, (int)h_tiles_trsm[j], s0);
        }));
        D3M_TRY(launch(kClsTrsm, s0, [&] {
          return nj <= 512 ? d3m_dinv_rows_coef_launch(xbuf, pool + h_panel_off[j], R, nj, tags, coef, s0)
                           : d3m_dinv_rows_launch(xbuf, pool + h_panel_off[j], R, nj, diag, tags, s0);
        }));
      }
      const int64_t t0 = h_task_ptr[j], tn = h_task_next[j], t1 = h_task_ptr[j + 1];
      // the update launches of this column stage X_j / L_j tiles by TMA from tensor maps over the two panels
      alignas(64) unsigned char maps[256];
      bool col_tma = false;
      if (tma_mode && R > 0 && t1 > t0) {
        const int prc = d3m_gemm_tma_prepare(xbuf, R, pool + h_panel_off[j], R, nj, maps);
        if (prc == -38) tma_mode = 0;                    // driver without tensor-map encoding: cp.async kernel
        else if (prc) return fail(prc, "d3m_block_ldlt_exec: tensor map");
        else col_tma = true;
      }
      // next update (targets in column j+1): after every earlier bulk update into column j+1
      if (tn > t0) {
        if (lookahead) wait_rest(q, s0, h_sched[3 * j + 2]);
        D3M_TRY(launch(kClsGemm, s0, [&] {
          if (col_tma)
            return d3m_gemm_tma_launch(maps, pool, tasks + t0, (int)(tn - t0), (int)h_tiles_next[j], h_panel_off[j],
                                       s0);
          return d3m_gemm_launch(0, 0, xbuf, pool, pool, tasks + t0, (int)(tn - t0), (int)h_tiles_next[j], s0);
        }));
      }
      if (lookahead) cudaEventRecord(ctx->ev_col[j], s0);
      // the bulk ("rest") update of column j targets columns >= j+2 and only
      // reads X_j / L_j: it starts once column j's critical work (including
      // the next update, which then has the SMs to itself) is done
      if (t1 > tn) {
        cudaStream_t sb = lookahead ? side : s0;
        if (lookahead) cudaStreamWaitEvent(side, ctx->ev_col[j], 0);
        D3M_TRY(launch(kClsGemm, sb, [&] {
          if (col_tma)
            return d3m_gemm_tma_launch(maps, pool, tasks + tn, (int)(t1 - tn), (int)h_tiles_rest[j], h_panel_off[j],
                                       sb);
          return d3m_gemm_launch(0, 0, xbuf, pool, pool, tasks + tn, (int)(t1 - tn), (int)h_tiles_rest[j], sb);
        }));
        if (lookahead) {
          cudaEventRecord(ctx->ev_rest[j], side);
          has_rest[j] = 1;
        }
      }
    }
    return 0;
  };
  const int rc = columns();
  // join, on success and on failure alike: the caller's stream waits for
  // everything enqueued on the critical and bulk streams, so buffers it frees
  // after a raised error are not still in use
  if (lookahead) {
    cudaEventRecord(ctx->ev_out, side);
    cudaStreamWaitEvent(user, ctx->ev_out, 0);
    for (int q = 0; q < kCritStreams; ++q)
      if (used[q]) {
        cudaEventRecord(ctx->ev_out, ctx->crit[q]);
        cudaStreamWaitEvent(user, ctx->ev_out, 0);
      }
  }
  if (rc != 0) return rc;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail((int)e, "d3m_block_ldlt_exec: launch");
  return 0;
}

// ---------------------------------------------------------------------------
// block_solve executor (factor.py:243-310), all RHS in one pass, tall-skinny
// DMMA products against the stored factor (skinny_dmma.cu):
//   forward  z_j = Binv_j b_j,  u_j = D_j^-1 z_j,  b_i -= L_ij z_j
//   backward w_j = u_j - sum_i L_ij^T x_i  (split-K partials, ordered sum),
//            x_j = Binv_j^T w_j
//   b, u, x : N x nrhs plan order (b consumed);  tmp: max n_j x nrhs;
//   part    : partial sums, part_elems complex
// ---------------------------------------------------------------------------
int d3m_block_solve_dataflow(int nb, const void* d_plan, const void* d_items, int nitems, int nchain, const void* d_deps,
                             const void* d_part_off, void* d_counters, int ncounters, const void* d_gidx,
                             const void* d_pool, const void* d_binv, const void* d_tags, void* d_b, void* d_u,
                             void* d_x, void* d_part, int nrhs, void* stream) {
  if (nb <= 0 || nrhs <= 0) return 0;
  if (!d_plan || !d_items || nitems <= 0 || ncounters <= D3M_FLOW_EXTRA_COUNTERS || nchain < 0 || nchain > nitems)
    return fail(-22, "d3m_block_solve_dataflow: empty plan or counters without the scheduler scratch");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t* d_arr = static_cast<const int64_t*>(d_plan);
  d3m::SolvePlanDev pl{};
  pl.sizes = d_arr; pl.row_off = d_arr + nb; pl.diag_off = d_arr + 2 * nb; pl.panel_off = d_arr + 3 * nb;
  pl.panel_rows = d_arr + 4 * nb; pl.piv_off = d_arr + 5 * nb; pl.binv_off = d_arr + 6 * nb;
  pl.gptr = d_arr + 7 * nb;
  pl.gidx = static_cast<const int64_t*>(d_gidx); pl.pool = CC(d_pool); pl.binv = CC(d_binv);
  pl.tags = static_cast<const int8_t*>(d_tags);
  pl.b = C(d_b); pl.u = C(d_u); pl.x = C(d_x); pl.tmp = nullptr; pl.part = C(d_part);
  pl.nb = nb; pl.ldn = nrhs;
  for (int c0 = 0; c0 < nrhs; c0 += 16) {
    pl.c0 = c0;
    pl.N = std::min(16, nrhs - c0);
    const int rc = launch(kClsSolve, s, [&] {
      return d3m_block_solve_flow_launch(&pl, d_items, nitems, nchain, d_deps, d_part_off, d_counters, ncounters, s);
    });
    if (rc != 0) return fail(rc, "d3m_block_solve_dataflow: launch");
  }
  return 0;
}

int d3m_block_solve_exec(int nb, const int64_t* h_sizes, const int64_t* h_row_off, const int64_t* h_diag_off,
                         const int64_t* h_panel_off, const int64_t* h_panel_rows, const int64_t* h_piv_off,
                         const int64_t* h_binv_off, const int64_t* h_gptr, const void* d_gidx, const void* d_pool,
                         const void* d_binv, const void* d_tags, void* d_b, void* d_u, void* d_x, void* d_tmp,
                         void* d_part, int64_t part_elems, int nrhs, const void* d_plan, void* stream) {
  // Forward (per column j, plan order):  z = Binv_j b_j;  u_j = D_j^-1 z;  b_i -= L_ij z
  // Backward (reverse):  w = u_j - sum_i L_ij^T x_i (split-K partials, ordered
  // reduce);  x_j = Binv_j^T w.  All products on DMMA (skinny_dmma.cu), in
  // passes of 16 RHS.  d_part: >= ceil(R_j / 256) * n_j * 16 complex.
  if (nb <= 0 || nrhs <= 0) return 0;
  constexpr int KCH = 256, NP = 16;
  for (int j = 0; j < nb; ++j) {
    const int64_t nj = h_sizes[j], R = h_panel_rows[j];
    const int64_t need = ((R + KCH - 1) / KCH) * nj * NP;
    if (need > part_elems) return fail(-22, "d3m_block_solve_exec: partial buffer too small");
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const cplx* pool = CC(d_pool);
  const cplx* binv = CC(d_binv);
  const int64_t* gidx = static_cast<const int64_t*>(d_gidx);
  cplx* b = C(d_b);
  cplx* u = C(d_u);
  cplx* x = C(d_x);
  cplx* tmp = C(d_tmp);
  const int N = nrhs;
  static const char* solve_env = getenv("D3M_SOLVE");      // dev switch: 'l' = one launch per product
  if (d_plan && !(solve_env && solve_env[0] == 'l')) {
    // persistent cooperative kernel (skinny_dmma.cu) over the device plan arrays
    const int64_t* d_arr = static_cast<const int64_t*>(d_plan);
    d3m::SolvePlanDev pl{};
    pl.sizes = d_arr; pl.row_off = d_arr + nb; pl.diag_off = d_arr + 2 * nb; pl.panel_off = d_arr + 3 * nb;
    pl.panel_rows = d_arr + 4 * nb; pl.piv_off = d_arr + 5 * nb; pl.binv_off = d_arr + 6 * nb;
    pl.gptr = d_arr + 7 * nb;
    pl.gidx = gidx; pl.pool = pool; pl.binv = binv; pl.tags = static_cast<const int8_t*>(d_tags);
    pl.b = b; pl.u = u; pl.x = x; pl.tmp = tmp; pl.part = C(d_part);
    pl.nb = nb; pl.ldn = N;
    int rc = 0;
    for (int c0 = 0; c0 < N && rc == 0; c0 += 16) {
      pl.c0 = c0;
      pl.N = std::min(16, N - c0);
      rc = launch(kClsSolve, s, [&] { return d3m_block_solve_persistent_launch(&pl, s); });
    }
    if (rc == 0) return 0;
    if (rc != -22) return fail(rc, "d3m_block_solve_exec: persistent solve");
    cudaGetLastError();
  }
  auto sk = [&](int ta, const cplx* A, int lda, int M, int K, const cplx* Bp, const int64_t* bmap, cplx* Cp,
                const int64_t* cmap, int mode, int kchunk, int c0) -> int {
    const int np = std::min(NP, N - c0);
    const int rc = d3m_skinny_launch(ta, A, lda, M, K, Bp + c0, N, bmap, np, mode == 2 ? Cp : Cp + c0, N, cmap,
                                     mode, kchunk, s);
    return rc < 0 ? -rc : 0;
  };
  for (int j = 0; j < nb; ++j) {
    const int nj = (int)h_sizes[j];
    const int R = (int)h_panel_rows[j];
    if (nj == 0) continue;
    const int8_t* tags = static_cast<const int8_t*>(d_tags) + h_piv_off[j];
    for (int c0 = 0; c0 < N; c0 += NP)
      D3M_TRY(launch(kClsSolve, s, [&] {
        return sk(0, binv + h_binv_off[j], nj, nj, nj, b + h_row_off[j] * N, nullptr, tmp, nullptr, 0, 0, c0);
      }));
    D3M_TRY(launch(kClsSolve, s, [&] {
      return d3m_dinv_left_copy_launch(tmp, u + h_row_off[j] * N, nj, N, pool + h_diag_off[j], tags, s);
    }));
    if (R > 0)
      for (int c0 = 0; c0 < N; c0 += NP)
        D3M_TRY(launch(kClsSolve, s, [&] {
          return sk(0, pool + h_panel_off[j], nj, R, nj, tmp, nullptr, b, gidx + h_gptr[j], 1, 0, c0);
        }));
  }
  for (int j = nb - 1; j >= 0; --j) {
    const int nj = (int)h_sizes[j];
    const int R = (int)h_panel_rows[j];
    if (nj == 0) continue;
    cplx* uj = u + h_row_off[j] * N;
    for (int c0 = 0; c0 < N; c0 += NP) {
      const int np = std::min(NP, N - c0);
      if (R > 0) {
        D3M_TRY(launch(kClsSolve, s, [&] {
          return sk(1, pool + h_panel_off[j], nj, nj, R, x, gidx + h_gptr[j], C(d_part), nullptr, 2, KCH, c0);
        }));
        const int nch = (R + KCH - 1) / KCH;
        D3M_TRY(launch(kClsSolve, s, [&] {
          return d3m_skinny_reduce_launch(uj + c0, N, d_part, nch, nj, np, -1.0, tmp + c0, N, s);
        }));
      } else {
        D3M_TRY(launch(kClsSolve, s, [&] {
          return d3m_skinny_reduce_launch(uj + c0, N, d_part, 0, nj, np, -1.0, tmp + c0, N, s);
        }));
      }
    }
    for (int c0 = 0; c0 < N; c0 += NP)
      D3M_TRY(launch(kClsSolve, s, [&] {
        return sk(1, binv + h_binv_off[j], nj, nj, nj, tmp, nullptr, x + h_row_off[j] * N, nullptr, 0, 0, c0);
      }));
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
  D3M_TRY(launch(kClsMisc, stream, [&] { return d3m_ordered_average_launch(rhs, avg_ptr, avg_src, out, nglob, stream); }));
  return 0;
}

void d3m_set_timing(int on) {
  std::lock_guard<std::mutex> g(g_tmu);
  g_timing = on != 0;
  if (on) {
    if (!g_ref) cudaEventCreate(&g_ref);
    cudaDeviceSynchronize();
    cudaEventRecord(g_ref, 0);
  }
}

void d3m_counters_reset(void) {
  std::lock_guard<std::mutex> g(g_tmu);
  for (auto& r : g_pending) {
    cudaEventSynchronize(r.b);
    g_free_ev.push_back(r.a);
    g_free_ev.push_back(r.b);
  }
  g_pending.clear();
  g_launches.store(0);
  for (int c = 0; c < kNumCls; ++c) { g_ms[c] = 0; g_cnt[c] = 0; g_union[c] = 0; }
}

// launches: total kernel launches since reset; ms[5] / n[5]: summed event
// time and launch count per class (bk, trsm, gemm-update, solve, misc).
int d3m_counters_read(int64_t* launches, double* ms, int64_t* n) {
  std::lock_guard<std::mutex> g(g_tmu);
  std::vector<std::pair<double, double>> iv[kNumCls];
  g_iv.clear();
  for (auto& r : g_pending) {
    cudaEventSynchronize(r.b);
    float t = 0.f, t0 = 0.f, t1 = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    g_ms[r.cls] += t;
    if (g_ref && cudaEventElapsedTime(&t0, g_ref, r.a) == cudaSuccess &&
        cudaEventElapsedTime(&t1, g_ref, r.b) == cudaSuccess) {
      iv[r.cls].emplace_back(t0, t1);
      g_iv.insert(g_iv.end(), {(double)r.cls, (double)t0, (double)t1});
    }
    g_free_ev.push_back(r.a);
    g_free_ev.push_back(r.b);
  }
  g_pending.clear();
  for (int c = 0; c < kNumCls; ++c) {       // measure of the union of intervals
    auto& v = iv[c];
    std::sort(v.begin(), v.end());
    double lo = -1, hi = -1;
    for (auto& x : v) {
      if (x.first > hi) {
        if (hi > lo) g_union[c] += hi - lo;
        lo = x.first;
        hi = x.second;
      } else if (x.second > hi) {
        hi = x.second;
      }
    }
    if (hi > lo) g_union[c] += hi - lo;
  }
  if (launches) *launches = g_launches.load();
  for (int c = 0; c < kNumCls; ++c) {
    if (ms) { ms[c] = g_ms[c]; ms[kNumCls + c] = g_union[c]; }
    if (n) n[c] = g_cnt[c];
  }
  return 0;
}

// Diagnostics: the timed launch intervals collected by the last
// d3m_counters_read, as (class, start_ms, end_ms) triplets; returns the count.
int64_t d3m_timing_intervals(double* out, int64_t max_triplets) {
  std::lock_guard<std::mutex> g(g_tmu);
  const int64_t n = (int64_t)g_iv.size() / 3;
  if (out) std::memcpy(out, g_iv.data(), sizeof(double) * 3 * (size_t)std::min(n, max_triplets));
  return n;
}

}  // extern "C"

// n asynchronous copies dst + dst_off[i] <- src + src_off[i] (bytes) on one
// stream (kind: cudaMemcpyKind); lets the host enqueue a chunk of K's blocks
// without one Python call per block.
int d3m_memcpy_batch(void* dst, const void* src, const int64_t* dst_off, const int64_t* src_off,
                     const int64_t* nbytes, int n, int kind, void* stream) {
  auto s = reinterpret_cast<cudaStream_t>(stream);
  for (int i = 0; i < n; ++i) {
    const cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + dst_off[i], static_cast<const char*>(src) + src_off[i],
                                          (size_t)nbytes[i], static_cast<cudaMemcpyKind>(kind), s);
    if (e != cudaSuccess) return fail((int)e, "d3m_memcpy_batch");
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Host-staged upload of pageable inputs (block_ldlt with numpy K blocks).
//
// A host thread copies the blocks of chunk c into a pinned staging buffer
// (nthreads-way parallel memcpy) and then publishes the chunk by storing
// c + 1 into a pinned flag; on the copy stream, d3m_stream_wait_flag holds
// chunk c's H2D copy until the flag reaches c + 1.  The factorisation's
// first columns start as soon as their chunk is staged, while the host is
// still copying the later ones.
// ---------------------------------------------------------------------------
namespace {
struct HostStage {
  std::thread th;
  std::atomic<int> err{0};
};

void host_stage_run(HostStage* h, int nchunks, std::vector<int64_t> chunk_ptr, std::vector<const char*> src,
                    std::vector<int64_t> dst_off, std::vector<int64_t> nbytes, char* dst, int* flag, int nthreads) {
  std::vector<std::thread> pool;
  for (int c = 0; c < nchunks; ++c) {
    const int64_t b0 = chunk_ptr[c], b1 = chunk_ptr[c + 1];
    int64_t tot = 0;
    for (int64_t b = b0; b < b1; ++b) tot += nbytes[b];
    // split the chunk's bytes evenly over the threads (each copies a
    // contiguous byte range of the concatenated blocks)
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(nthreads, tot >> 22));   // >= 4 MB per thread
    auto copy_range = [&](int64_t lo, int64_t hi) {
      int64_t pos = 0;
      for (int64_t b = b0; b < b1 && pos < hi; ++b) {
        const int64_t s0 = std::max(lo, pos), s1 = std::min(hi, pos + nbytes[b]);
        if (s1 > s0) std::memcpy(dst + dst_off[b] + (s0 - pos), src[b] + (s0 - pos), (size_t)(s1 - s0));
        pos += nbytes[b];
      }
    };
    pool.clear();
    for (int t = 1; t < nt; ++t) pool.emplace_back(copy_range, tot * t / nt, tot * (t + 1) / nt);
    copy_range(0, tot / nt);
    for (auto& th : pool) th.join();
    __atomic_store_n(flag, c + 1, __ATOMIC_RELEASE);
  }
}
}  // namespace

extern "C" {

// Start the host thread: nchunks chunks, chunk c = blocks [chunk_ptr[c],
// chunk_ptr[c+1]) of the n block copies src[i] -> dst + dst_off[i] (nbytes[i]
// bytes; dst a pinned buffer, flag a pinned int).  The source arrays must stay
// alive until d3m_host_stage_join.  Returns a handle (NULL on failure).
void* d3m_host_stage_start(int nchunks, const int64_t* chunk_ptr, int n, const void* const* src,
                           const int64_t* dst_off, const int64_t* nbytes, void* dst, void* flag, int nthreads) {
  try {
    auto* h = new HostStage;
    std::vector<int64_t> cp(chunk_ptr, chunk_ptr + nchunks + 1);
    std::vector<const char*> sv(n);
    for (int i = 0; i < n; ++i) sv[i] = static_cast<const char*>(src[i]);
    std::vector<int64_t> doff(dst_off, dst_off + n), nb(nbytes, nbytes + n);
    h->th = std::thread(host_stage_run, h, nchunks, std::move(cp), std::move(sv), std::move(doff), std::move(nb),
                        static_cast<char*>(dst), static_cast<int*>(flag), std::max(1, nthreads));
    return h;
  } catch (...) {
    return nullptr;
  }
}

// Wait for the host thread and release the handle; 0 on success.
int d3m_host_stage_join(void* handle) {
  if (!handle) return fail(-22, "d3m_host_stage_join: null handle");
  auto* h = static_cast<HostStage*>(handle);
  h->th.join();
  const int e = h->err.load();
  delete h;
  return e;
}

// The stream waits until the pinned host int *flag >= value (a one-thread
// kernel polling the mapped host memory; traps after ~60 s instead of
// hanging the stream when the host side never publishes).
int d3m_stream_wait_flag(const void* flag, int value, void* stream) {
  return launch(kClsMisc, stream, [&] {
    return d3m_wait_flag_launch(static_cast<const int*>(flag), value, stream);
  });
}

}  // extern "C"
