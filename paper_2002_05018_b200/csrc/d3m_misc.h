// d3m_misc.h -- task descriptor of the grouped block copy kernel.
#pragma once
#include <cstdint>

namespace d3m {

enum : int32_t { kCopyStore = 0, kCopyAdd = 1, kCopyZeroAdd = 2 };

// dst[dst_off + r*ld_dst + c] (op)= src(r, c), r < rows, c < cols, where
// src(r, c) = src[src_off + r*ld_src + c], or src[src_off + c*ld_src + r]
// when transpose != 0.
struct CopyTask {
  int64_t src_off, dst_off;
  int32_t rows, cols;
  int32_t ld_src, ld_dst;
  int32_t transpose, mode;
};
static_assert(sizeof(CopyTask) == 40, "CopyTask layout is shared with Python (numpy dtype)");

}  // namespace d3m
