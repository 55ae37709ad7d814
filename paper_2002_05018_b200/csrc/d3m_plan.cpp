// d3m_plan.cpp -- host-side planning of the block LDL^T executor and the
// dataflow block solve (no device code).
//
// Both tables depend only on the elimination plan (supernode sizes and the
// block pattern of every column, symbolic.py:36-64), so they are built once
// per plan.  They used to be Python loops (0.9 s for a config-5-shaped plan);
// here they take milliseconds.
//
//   d3m_plan_gemm_tasks  the trailing-update GEMM task table of block_ldlt
//                        (factor.py:209-219: K_ik -= X_ij L_kj^T for every
//                        pattern pair i >= k of column j), grouped per column
//                        as "next" (targets in column j+1) then "rest"
//   d3m_plan_flow_items  the work items and dependency counters of
//                        d3m_block_solve_dataflow (factor.py:243-310's
//                        forward and backward substitutions as tiles)
#include <algorithm>
#include <cstdint>
#include <deque>
#include <vector>

#include "d3m_gemm.h"
#include "../../include/d3m.h"

namespace {

constexpr int kBM = 64;                   // GEMM output tile (zgemm_dmma.cu)
constexpr int kKCH = 256;                 // backward split-K chunk (panel rows), skinny_dmma.cu
constexpr int kFdRows = 32, kBrRows = 16;  // rows per D^-1 / reduce work item
enum { FA = 0, FD = 1, FB = 2, BC = 3, BR = 4, BE = 5 };   // skinny_dmma.cu FlowItem types

struct Pattern {
  int nb;
  const int64_t* sizes;
  const int64_t* ptr;
  const int64_t* idx;
  int64_t size(int j) const { return sizes[j]; }
  int len(int j) const { return (int)(ptr[j + 1] - ptr[j]); }
  int at(int j, int a) const { return (int)idx[ptr[j] + a]; }
  // panel row offset of block i in panel j, -1 when i is not in pattern(j)
  int64_t rowpos(int j, int i, const std::vector<int64_t>& prow) const {
    for (int64_t p = ptr[j]; p < ptr[j + 1]; ++p)
      if (idx[p] == i) return prow[p];
    return -1;
  }
};

std::vector<int64_t> panel_row_offsets(const Pattern& P) {
  std::vector<int64_t> prow(P.ptr[P.nb]);
  for (int j = 0; j < P.nb; ++j) {
    int64_t r = 0;
    for (int a = 0; a < P.len(j); ++a) {
      prow[P.ptr[j] + a] = r;
      r += P.size(P.at(j, a));
    }
  }
  return prow;
}

}  // namespace

extern "C" {

// Trailing-update GEMM tasks of block_ldlt.  For column j (plan order) and
// every pattern pair (i = pattern[a], k = pattern[b]), b <= a:
//   A = X_j rows of block i (xbuf, offset prow[a] * n_j), B = L_kj (pool,
//   panel_off[j] + prow[b] * n_j), C = the diagonal slot of i (k == i:
//   symmetric target, lower tiles, kGemmSym) or block (i, k) in panel k.
// Records of column j come "next" (k == j + 1) first, then "rest"; tile_start
// counts output tiles within each group.  tasks: capacity cap records
// (NULL: count only).  Returns the record count, -1 when an update targets a
// block outside the pattern (factor.py:224-226 FactorConsistencyError), -2
// when cap is too small.  Per column: task_ptr[nb+1], task_next[nb] (end of
// the "next" group), tiles_next[nb], tiles_rest[nb].  flops[0] = the
// algorithmic update flops (8 n_i n_k n_j, 4 n_i^2 n_j for diagonal targets).
int64_t d3m_plan_gemm_tasks(int nb, const int64_t* sizes, const int64_t* pat_ptr, const int64_t* pat_idx,
                            const int64_t* diag_off, const int64_t* panel_off, void* tasks_v, int64_t cap,
                            int64_t* task_ptr, int64_t* task_next, int64_t* tiles_next, int64_t* tiles_rest,
                            int64_t* flops) {
  auto* tasks = static_cast<d3m::GemmTask*>(tasks_v);
  const Pattern P{nb, sizes, pat_ptr, pat_idx};
  const std::vector<int64_t> prow = panel_row_offsets(P);
  int64_t count = 0, fl = 0;
  if (task_ptr) task_ptr[0] = 0;
  std::vector<d3m::GemmTask> nxt, rest;
  for (int j = 0; j < nb; ++j) {
    const int64_t nj = P.size(j);
    nxt.clear();
    rest.clear();
    const int L = P.len(j);
    for (int a = 0; a < L; ++a) {
      const int i = P.at(j, a);
      const int64_t ni = P.size(i);
      for (int b = 0; b <= a; ++b) {
        const int k = P.at(j, b);
        const int64_t nk = P.size(k);
        d3m::GemmTask t{};
        t.a_off = prow[P.ptr[j] + a] * nj;
        t.b_off = panel_off[j] + prow[P.ptr[j] + b] * nj;
        int64_t tiles;
        if (i == k) {
          t.c_off = diag_off[i];
          t.ldc = (int32_t)ni;
          t.flags = d3m::kGemmSub | d3m::kGemmSym;
          const int64_t tm = (ni + kBM - 1) / kBM;
          tiles = tm * (tm + 1) / 2;
          fl += 4 * ni * ni * nj;
        } else {
          const int64_t rp = P.rowpos(k, i, prow);
          if (rp < 0) return -1;
          t.c_off = panel_off[k] + rp * nk;
          t.ldc = (int32_t)nk;
          t.flags = d3m::kGemmSub;
          tiles = ((ni + kBM - 1) / kBM) * ((nk + kBM - 1) / kBM);
          fl += 8 * ni * nk * nj;
        }
        t.m = (int32_t)ni;
        t.n = (int32_t)nk;
        t.k = t.lda = t.ldb = (int32_t)nj;
        t.tiles_n = (int32_t)((nk + kBM - 1) / kBM);
        t.tile_start = (int32_t)tiles;           // tile count; turned into the group prefix below
        t.pad_ = 0;
        (k == j + 1 ? nxt : rest).push_back(t);
      }
    }
    int64_t tn = 0, tr = 0;
    for (auto* g : {&nxt, &rest}) {
      int64_t start = 0;
      for (auto& t : *g) {
        const int64_t c = t.tile_start;
        t.tile_start = (int32_t)start;
        start += c;
        if (tasks) {
          if (count >= cap) return -2;
          tasks[count] = t;
        }
        ++count;
      }
      (g == &nxt ? tn : tr) = start;
    }
    if (task_next) task_next[j] = count - (int64_t)rest.size();
    if (task_ptr) task_ptr[j + 1] = count;
    if (tiles_next) tiles_next[j] = tn;
    if (tiles_rest) tiles_rest[j] = tr;
  }
  if (flops) flops[0] = fl;
  return count;
}

// Work items of the dataflow block solve (include/d3m.h
// d3m_block_solve_dataflow): int32 records (type, column, p0, p1, dep_start,
// dep_count, counter, counter2) and int32 dependency pairs (counter, target).
// The order is a topological order that puts each column's critical items
// first (forward: z_j, then the parent block's update, then the previous
// column's farther updates; backward: the parent chunk's partials, the
// reduce and the Binv^T tiles, then the next column's farther chunks).
// Updates of one 16-row tile keep ascending column order through per-tile
// sequence counters.  items / deps: capacities cap_items / cap_deps (NULL:
// count only).  out[0..3] = item count, dependency count, counter count
// (+1 for the queue head), partial-sum elements; part_off[nb] (>= 1 entry).
// Returns 0, or -2 when a capacity is too small.
int d3m_plan_flow_items(int nb, const int64_t* sizes, const int64_t* pat_ptr, const int64_t* pat_idx,
                        const int64_t* panel_rows, int32_t* items, int64_t cap_items, int32_t* deps,
                        int64_t cap_deps, int64_t* part_off, int64_t* out) {
  const Pattern P{nb, sizes, pat_ptr, pat_idx};
  const std::vector<int64_t> prow = panel_row_offsets(P);
  std::vector<int64_t> T(nb);
  for (int j = 0; j < nb; ++j) T[j] = (P.size(j) + 15) / 16;
  const int64_t ZC = 0, BLK = nb, UC = 2 * (int64_t)nb, CC = 3 * (int64_t)nb, RC = 4 * (int64_t)nb,
                XC = 5 * (int64_t)nb;
  std::vector<int64_t> seq_base(nb + 1);
  seq_base[0] = 6 * (int64_t)nb;
  for (int j = 0; j < nb; ++j) seq_base[j + 1] = seq_base[j] + T[j];
  const int64_t ncnt = seq_base[nb] + 1;            // + queue head
  int64_t ni = 0, nd = 0;
  bool overflow = false;
  auto add = [&](int typ, int j, int64_t p0, int64_t p1, std::initializer_list<std::pair<int64_t, int64_t>> dl,
                 int64_t inc0, int64_t inc1) {
    if (items) {
      if (ni >= cap_items) { overflow = true; return; }
      int32_t* r = items + 8 * ni;
      r[0] = typ; r[1] = j; r[2] = (int32_t)p0; r[3] = (int32_t)p1;
      r[4] = (int32_t)nd; r[5] = (int32_t)dl.size(); r[6] = (int32_t)inc0; r[7] = (int32_t)inc1;
    }
    ++ni;
    for (const auto& d : dl) {
      if (deps) {
        if (nd >= cap_deps) { overflow = true; return; }
        deps[2 * nd] = (int32_t)d.first;
        deps[2 * nd + 1] = (int32_t)d.second;
      }
      ++nd;
    }
  };
  std::vector<std::pair<int64_t, int64_t>> dyn;       // dependency list of variable length (BC)
  auto add_dyn = [&](int typ, int j, int64_t p0, int64_t p1, int64_t inc0) {
    if (items) {
      if (ni >= cap_items) { overflow = true; return; }
      int32_t* r = items + 8 * ni;
      r[0] = typ; r[1] = j; r[2] = (int32_t)p0; r[3] = (int32_t)p1;
      r[4] = (int32_t)nd; r[5] = (int32_t)dyn.size(); r[6] = (int32_t)inc0; r[7] = -1;
    }
    ++ni;
    for (const auto& d : dyn) {
      if (deps) {
        if (nd >= cap_deps) { overflow = true; return; }
        deps[2 * nd] = (int32_t)d.first;
        deps[2 * nd + 1] = (int32_t)d.second;
      }
      ++nd;
    }
  };

  // ---- forward -------------------------------------------------------------
  std::vector<int64_t> n_into(nb, 0);                   // FB tile items into each block
  for (int j = 0; j < nb; ++j)
    for (int a = 0; a < P.len(j); ++a) n_into[P.at(j, a)] += T[P.at(j, a)];
  std::vector<int64_t> seq_k(seq_base[nb] - seq_base[0], 0);
  auto update = [&](int j, int i) {
    const int64_t rp = P.rowpos(j, i, prow);
    for (int64_t t = 0; t < T[i]; ++t) {
      const int64_t rows = std::min<int64_t>(16, P.size(i) - 16 * t);
      int64_t& sk = seq_k[seq_base[i] - seq_base[0] + t];
      add(FB, j, rp + 16 * t, rows, {{ZC + j, T[j]}, {seq_base[i] + t, sk}}, seq_base[i] + t, BLK + i);
      ++sk;
    }
  };
  std::vector<std::deque<int>> pending(nb);             // deferred updates (column j) per target block, FIFO
  auto flush = [&](int i, int upto) {                   // upto < 0: all
    while (!pending[i].empty() && (upto < 0 || pending[i].front() <= upto)) {
      const int j = pending[i].front();
      pending[i].pop_front();
      update(j, i);
    }
  };
  for (int j = 0; j < nb; ++j) {
    if (P.size(j)) {
      for (int64_t t = 0; t < T[j]; ++t) {
        if (n_into[j]) add(FA, j, t, 0, {{BLK + j, n_into[j]}}, ZC + j, -1);
        else add(FA, j, t, 0, {}, ZC + j, -1);
      }
      for (int64_t r0 = 0; r0 < P.size(j); r0 += kFdRows)
        add(FD, j, r0, std::min<int64_t>(P.size(j), r0 + kFdRows), {{ZC + j, T[j]}}, UC + j, -1);
    }
    if (P.len(j)) {
      const int par = P.at(j, 0);
      flush(par, -1);
      update(j, par);
    }
    if (j >= 1)
      for (int a = 1; a < P.len(j - 1); ++a) flush(P.at(j - 1, a), j - 1);
    for (int a = 1; a < P.len(j); ++a) pending[P.at(j, a)].push_back(j);
  }
  for (int i = 0; i < nb; ++i) flush(i, -1);

  // ---- backward ------------------------------------------------------------
  std::vector<int64_t> nch(nb);
  for (int j = 0; j < nb; ++j) nch[j] = (panel_rows[j] + kKCH - 1) / kKCH;
  // blocks of pattern(j) overlapping panel rows of chunk ch (non-empty blocks)
  auto chunk_blocks = [&](int j, int64_t ch, std::vector<int>& out_blocks) {
    out_blocks.clear();
    const int64_t lo = ch * kKCH, hi = std::min<int64_t>(panel_rows[j], ch * kKCH + kKCH);
    for (int a = 0; a < P.len(j); ++a) {
      const int i = P.at(j, a);
      const int64_t r = prow[P.ptr[j] + a];
      if (r < hi && r + P.size(i) > lo && P.size(i)) out_blocks.push_back(i);
    }
  };
  std::vector<int> cb;
  auto parent_chunk = [&](int j, int64_t ch) {
    if (!P.len(j)) return false;
    chunk_blocks(j, ch, cb);
    return std::find(cb.begin(), cb.end(), P.at(j, 0)) != cb.end();
  };
  std::vector<char> done_far(nb, 0);
  auto chunks = [&](int j, bool far) {
    for (int64_t ch = 0; ch < nch[j]; ++ch) {
      if (parent_chunk(j, ch) != far) {
        chunk_blocks(j, ch, cb);
        dyn.clear();
        for (int i : cb) dyn.emplace_back(XC + i, T[i]);
        for (int64_t mt = 0; mt < T[j]; ++mt) add_dyn(BC, j, ch, mt, CC + j);
      }
    }
  };
  for (int j = nb - 1; j >= 0; --j) {
    if (!P.size(j)) continue;
    if (!done_far[j]) {
      chunks(j, true);
      done_far[j] = 1;
    }
    chunks(j, false);
    const int64_t npc = (P.size(j) + kBrRows - 1) / kBrRows;
    const int64_t nfd = (P.size(j) + kFdRows - 1) / kFdRows;
    for (int64_t pc = 0; pc < npc; ++pc)
      add(BR, j, kBrRows * pc, std::min<int64_t>(P.size(j), kBrRows * pc + kBrRows),
          {{CC + j, nch[j] * T[j]}, {UC + j, nfd}}, RC + j, -1);
    for (int64_t t = 0; t < T[j]; ++t) add(BE, j, t, 0, {{RC + j, npc}}, XC + j, -1);
    if (j >= 1 && P.size(j - 1) && !done_far[j - 1]) {
      chunks(j - 1, true);
      done_far[j - 1] = 1;
    }
  }
  if (overflow) return -2;
  int64_t acc = 0;
  for (int j = 0; j < nb; ++j) {
    if (part_off) part_off[j] = acc;
    acc += nch[j] * P.size(j) * 16;
  }
  if (part_off && nb == 0) part_off[0] = 0;
  if (out) {
    out[0] = ni;
    out[1] = nd;
    out[2] = ncnt;
    out[3] = std::max<int64_t>(acc, 1);
  }
  return 0;
}

}  // extern "C"
