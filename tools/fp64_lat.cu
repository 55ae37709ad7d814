// Dependent-chain latencies (cycles per op) of the FP64 operations on the
// cluster BK's pivot chain (dev aid): nvcc -arch=sm_100a -O3 -I paper_2002_05018_b200/csrc
#include <cstdio>
#include "d3m_common.cuh"
using namespace d3m;
template <int OP>
__global__ void lat(double* out, long long* cyc, double seed, int iters) {
  double x = seed + threadIdx.x * 1e-20, y = 0.7 + seed * 1e-3;
  cplx a = mk(x, y), b = mk(1.3, -0.4);
  __shared__ double sm[64];
  sm[threadIdx.x & 63] = x;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) x = __dadd_rn(x, 1e-300);
    if (OP == 1) x = __dmul_rn(x, 1.0000000001);
    if (OP == 2) x = __ddiv_rn(x, 1.0000000001);
    if (OP == 3) x = __dsqrt_rn(x + 1.0);
    if (OP == 4) { a = x_div_py(a, b); }
    if (OP == 5) { x = glibc_hypot(x, y) * 0.5; }
    if (OP == 6) { a = x_div_np(a, b); }
    if (OP == 7) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-300;
    if (OP == 8) x = sm[(__double_as_longlong(x) & 1) + (threadIdx.x & 31)] ;
    if (OP == 9) x = fma(x, 1.0000000001, 1e-300);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x + a.x + a.y;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; long long h;
  cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
  const char* nm[] = {"dadd", "dmul", "ddiv_rn", "dsqrt_rn(+dadd)", "x_div_py", "glibc_hypot(+dmul)", "x_div_np",
                      "shfl.f64(+dadd)", "lds.f64", "dfma"};
  const int it = 4096;
#define RUN(K) lat<K><<<1, 32>>>(o, c, 1.1, it); cudaDeviceSynchronize(); lat<K><<<1, 32>>>(o, c, 1.1, it); \
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("%-20s %7.1f cycles/op\n", nm[K], (double)h / it);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9)
  return 0;
}
