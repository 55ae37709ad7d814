// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA.
// Measures burst throughput with CUDA events; each warp runs independent
// accumulator chains so the pipe, not latency, is the bound.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void dfma_chain(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
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
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  double* out; cudaMalloc(&out, 8);
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps, threads = 32 * wpb;
      float ms = timeit([&] { dmma_m8n8k4<8><<<blocks, threads>>>(out, iters); });
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)blocks * wpb;
      printf("DMMA m8n8k4   wpb=%2d bps=%d : %7.2f TFLOP/s\n", wpb, bps, flops / ms / 1e9);
      ms = timeit([&] { dmma_m16n8k16<4><<<blocks, threads>>>(out, iters / 4); });
      flops = 2.0 * 16 * 8 * 16 * 4.0 * (iters / 4) * (double)blocks * wpb;
      printf("DMMA m16n8k16 wpb=%2d bps=%d : %7.2f TFLOP/s\n", wpb, bps, flops / ms / 1e9);
      ms = timeit([&] { dfma_chain<8><<<blocks, threads>>>(out, iters); });
      flops = 2.0 * 8 * (double)iters * blocks * threads;
      printf("DFMA          wpb=%2d bps=%d : %7.2f TFLOP/s\n", wpb, bps, flops / ms / 1e9);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(e));
  return 0;
}
