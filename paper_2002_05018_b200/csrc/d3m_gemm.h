// d3m_gemm.h -- task descriptor of the grouped complex DMMA GEMM.
#pragma once
#include <cstdint>

namespace d3m {

enum : int32_t {
  kGemmSub = 0,        // C -= A B^T
  kGemmStore = 1,      // C  = A B^T
  kGemmAdd = 2,        // C += A B^T
  kGemmModeMask = 3,
  kGemmSym = 4,        // symmetric diagonal target: lower tiles, mirrored write
  kGemmLowerOnly = 8,  // with kGemmSym: write the lower triangle only (no mirror)
  kGemmTrackMax = 16,  // atomically max |C|^2 of written entries into tmax[pad_]
  kGemmTriGather = 32, // A(r, k) = A[r*lda + gperm[pad_ + k]] (column gather) and B lower
                       // triangular (B_eff[c][k] = 0 for k > c): output column tile tn
                       // needs k < (tn + 1) * 64 only (the panel TRSM X = K P^T L^-T)
};

// One GEMM of a grouped launch.  Offsets are in complex elements relative to
// the A/B/C base pointers of the launch.  tile_start / tiles_n are filled by
// d3m_gemm_prepare_tasks.
struct GemmTask {
  int64_t a_off, b_off, c_off;
  int32_t m, n, k;
  int32_t lda, ldb, ldc;
  int32_t flags;
  int32_t tile_start;
  int32_t tiles_n;
  int32_t pad_;
};
static_assert(sizeof(GemmTask) == 64, "GemmTask layout is shared with Python (numpy dtype)");

}  // namespace d3m
