// DMMA issue-mix microbenchmark for B200 (sm_100a) (dev aid).
// How much DMMA.8x8x4 throughput is lost when the 3M operand sums (DADD) and
// the fragment loads (LDS.128) share the SM with the DMMAs?  One "k4 step" of
// the 3M half-tile kernel is 24 DMMAs + 6 DADDs + 6 LDS.128 per warp; the
// variants below keep the 24 DMMAs and vary the rest.  12 warps per SM
// (3 CTAs of 4 warps), as the kernel runs.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// MODE 0: DMMAs only, register operands
// MODE 1: + 6 DADDs per step feeding the R products (operands from registers)
// MODE 2: + 6 LDS.128 per step (operands from shared memory), no DADD
// MODE 3: LDS + DADD (the kernel's mix)
// MODE 4: LDS + sums read from shared memory as a third plane (6 more LDS.64), no DADD
template <int MODE>
__global__ void __launch_bounds__(128, 3) mix(double* out, int iters) {
  __shared__ double2 sa[64][12], sb[32][12];
  __shared__ double ssa[64][12], ssb[32][12];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int e = t; e < 64 * 12; e += 128) { sa[e / 12][e % 12] = make_double2(1.0 + e * 1e-9, 1.0 - e * 1e-9); ssa[e / 12][e % 12] = 2.0; }
  for (int e = t; e < 32 * 12; e += 128) { sb[e / 12][e % 12] = make_double2(1.0 - e * 1e-9, 1.0 + e * 1e-9); ssb[e / 12][e % 12] = 2.0; }
  __syncthreads();
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 16, fr = lane >> 2, fc = lane & 3;
  double P[4][2][2] = {}, Q[4][2][2] = {}, R[4][2][2] = {};
  double2 ar[4], br[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) ar[i] = sa[wm + i * 8 + fr][fc];
#pragma unroll
  for (int j = 0; j < 2; ++j) br[j] = sb[wn + j * 8 + fr][fc];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      double2 a[4], b[2];
      double as[4], bs[2];
      if (MODE >= 2) {
        const int ko = (kk * 4 + fc + it) & 7;
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j] = sb[wn + j * 8 + fr][ko];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = sa[wm + i * 8 + fr][ko];
        if (MODE == 4) {
#pragma unroll
          for (int j = 0; j < 2; ++j) bs[j] = ssb[wn + j * 8 + fr][ko];
#pragma unroll
          for (int i = 0; i < 4; ++i) as[i] = ssa[wm + i * 8 + fr][ko];
        }
      } else {
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j] = br[j];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = ar[i];
      }
      if (MODE == 1 || MODE == 3) {
#pragma unroll
        for (int j = 0; j < 2; ++j) bs[j] = b[j].x + b[j].y;
      } else if (MODE != 4) {
#pragma unroll
        for (int j = 0; j < 2; ++j) bs[j] = b[j].x;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double asum;
        if (MODE == 1 || MODE == 3) asum = a[i].x + a[i].y;
        else if (MODE == 4) asum = as[i];
        else asum = a[i].y;
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(P[i][j][0], P[i][j][1], a[i].x, b[j].x);
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(Q[i][j][0], Q[i][j][1], a[i].y, b[j].y);
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(R[i][j][0], R[i][j][1], asum, bs[j]);
      }
      if (MODE == 1) {   // keep the register operands changing so the sums are not hoisted
#pragma unroll
        for (int i = 0; i < 4; ++i) ar[i].x = -ar[i].x;
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) s += P[i][j][0] + P[i][j][1] + Q[i][j][0] + Q[i][j][1] + R[i][j][0] + R[i][j][1];
  if (s == 12345.0) out[0] = s;
}


// Issue-order variants of the kernel's mix (LDS + DADD + DMMA), DMMAs in volatile asm so their order is the source's:
// ORDER 0: per fragment row i: sum, P, Q, R (the kernel's order)
// ORDER 1: all six sums at the top of the step, then all P, all Q, all R (R products >= 16 DMMAs behind their sums)
// ORDER 2: the sums of step s+1 are formed at the end of step s from prefetched fragments (one step ahead)
template <int ORDER>
__global__ void __launch_bounds__(128, 3) mixo(double* out, int iters) {
  __shared__ double2 sa[64][12], sb[32][12];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int e = t; e < 64 * 12; e += 128) sa[e / 12][e % 12] = make_double2(1.0 + e * 1e-9, 1.0 - e * 1e-9);
  for (int e = t; e < 32 * 12; e += 128) sb[e / 12][e % 12] = make_double2(1.0 - e * 1e-9, 1.0 + e * 1e-9);
  __syncthreads();
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 16, fr = lane >> 2, fc = lane & 3;
  double P[4][2][2] = {}, Q[4][2][2] = {}, R[4][2][2] = {};
  double2 a[4], b[2];
  double as[4], bs[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) { b[j] = sb[wn + j * 8 + fr][fc]; bs[j] = b[j].x + b[j].y; }
#pragma unroll
  for (int i = 0; i < 4; ++i) { a[i] = sa[wm + i * 8 + fr][fc]; as[i] = a[i].x + a[i].y; }
  for (int it = 0; it < 2 * iters; ++it) {
    const int ko = (fc + 4 * it + (it >> 1)) & 7;
    double2 an[4], bn[2];
    if (ORDER == 2) {                       // prefetch the next step's fragments
#pragma unroll
      for (int j = 0; j < 2; ++j) bn[j] = sb[wn + j * 8 + fr][ko];
#pragma unroll
      for (int i = 0; i < 4; ++i) an[i] = sa[wm + i * 8 + fr][ko];
    } else {
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = sb[wn + j * 8 + fr][ko];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sa[wm + i * 8 + fr][ko];
    }
    if (ORDER == 0) {
#pragma unroll
      for (int j = 0; j < 2; ++j) bs[j] = b[j].x + b[j].y;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double asum = a[i].x + a[i].y;
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(P[i][j][0], P[i][j][1], a[i].x, b[j].x);
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(Q[i][j][0], Q[i][j][1], a[i].y, b[j].y);
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(R[i][j][0], R[i][j][1], asum, bs[j]);
      }
    } else {
      if (ORDER == 1) {
#pragma unroll
        for (int j = 0; j < 2; ++j) bs[j] = b[j].x + b[j].y;
#pragma unroll
        for (int i = 0; i < 4; ++i) as[i] = a[i].x + a[i].y;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(P[i][j][0], P[i][j][1], a[i].x, b[j].x);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(Q[i][j][0], Q[i][j][1], a[i].y, b[j].y);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(R[i][j][0], R[i][j][1], as[i], bs[j]);
      if (ORDER == 2) {
#pragma unroll
        for (int j = 0; j < 2; ++j) { b[j] = bn[j]; bs[j] = bn[j].x + bn[j].y; }
#pragma unroll
        for (int i = 0; i < 4; ++i) { a[i] = an[i]; as[i] = an[i].x + an[i].y; }
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) s += P[i][j][0] + P[i][j][1] + Q[i][j][0] + Q[i][j][1] + R[i][j][0] + R[i][j][1];
  if (s == 12345.0) out[0] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  const int iters = 4000;
  const int blocks = sms * 3;
  const double flops = 2.0 * 256 * 48.0 * iters * (double)blocks * 4;
  float ms;
  ms = timeit([&] { mix<0><<<blocks, 128>>>(out, iters); }); printf("DMMA only (regs)          : %6.2f TFLOP/s\n", flops / ms / 1e9);
  ms = timeit([&] { mix<1><<<blocks, 128>>>(out, iters); }); printf("DMMA + DADD (regs)        : %6.2f TFLOP/s\n", flops / ms / 1e9);
  ms = timeit([&] { mix<2><<<blocks, 128>>>(out, iters); }); printf("DMMA + LDS                : %6.2f TFLOP/s\n", flops / ms / 1e9);
  ms = timeit([&] { mix<3><<<blocks, 128>>>(out, iters); }); printf("DMMA + LDS + DADD (kernel): %6.2f TFLOP/s\n", flops / ms / 1e9);
  ms = timeit([&] { mix<4><<<blocks, 128>>>(out, iters); }); printf("DMMA + LDS + sum plane    : %6.2f TFLOP/s\n", flops / ms / 1e9);
  ms = timeit([&] { mixo<0><<<blocks, 128>>>(out, iters); }); printf("order 0 (kernel: sum,P,Q,R per row)   : %6.2f TFLOP/s\n", flops / ms / 1e9);
  ms = timeit([&] { mixo<1><<<blocks, 128>>>(out, iters); }); printf("order 1 (sums first, P*,Q*,R*)        : %6.2f TFLOP/s\n", flops / ms / 1e9);
  ms = timeit([&] { mixo<2><<<blocks, 128>>>(out, iters); }); printf("order 2 (sums one step ahead)         : %6.2f TFLOP/s\n", flops / ms / 1e9);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
