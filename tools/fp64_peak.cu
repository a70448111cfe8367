// FP64 pipe micro-benchmark for B200 (sm_100a).
// Measures the FP64 ceilings that bound the FMM kernels (the driver's
// MEASURED_PEAKS.json carries HBM and bf16 numbers only):
//   dfma  : vector DFMA throughput (independent chains)
//   dadd  : vector DADD throughput
//   dmma  : FP64 tensor-core mma.sync m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16
//   mixed : DFMA warps and DMMA warps co-resident (do the pipes add?)
//   rcp   : MUFU.RCP64H + 2 Newton steps (the P2P reciprocal)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3,
         x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_dadd(double* out, double a) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3,
         x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    x0 += a; x1 += a; x2 += a; x3 += a; x4 += a; x5 += a; x6 += a; x7 += a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_rcp(double* out, double a) {
  double x0 = threadIdx.x + 1.5, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double s = 0;
#pragma unroll 4
  for (int i = 0; i < ITERS / 4; ++i) {
    double r0 = 1.0 / x0, r1 = 1.0 / x1, r2 = 1.0 / x2, r3 = 1.0 / x3;
    s += r0 + r1 + r2 + r3;
    x0 += a; x1 += a; x2 += a; x3 += a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__global__ void k_rcp_nr(double* out, double a) {
  double x0 = threadIdx.x + 1.5, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double s = 0;
#pragma unroll 4
  for (int i = 0; i < ITERS / 4; ++i) {
    double r0 = rcp_nr(x0), r1 = rcp_nr(x1), r2 = rcp_nr(x2), r3 = rcp_nr(x3);
    s += r0 + r1 + r2 + r3;
    x0 += a; x1 += a; x2 += a; x3 += a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// m8n8k4: A 8x4 (1 elem/thread), B 4x8 (1 elem/thread), C 8x8 (2 elem/thread)
__global__ void k_dmma884(double* out, double a) {
  double A = a + threadIdx.x, B = a - threadIdx.x;
  double c[4][2] = {};
#pragma unroll 4
  for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(A), "d"(B));
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// m16n8k4: A 16x4 (2/thread), B 4x8 (1/thread), C 16x8 (4/thread)
__global__ void k_dmma1684(double* out, double a) {
  double A0 = a + threadIdx.x, A1 = A0 + 1, B = a - threadIdx.x;
  double c[4][4] = {};
#pragma unroll 4
  for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(A0), "d"(A1), "d"(B));
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// m16n8k16: A 16x16 (8/thread), B 16x8 (4/thread), C 16x8 (4/thread)
__global__ void k_dmma16816(double* out, double a) {
  double A[8], B[4];
  for (int i = 0; i < 8; ++i) A[i] = a + threadIdx.x + i;
  for (int i = 0; i < 4; ++i) B[i] = a - threadIdx.x - i;
  double c[2][4] = {};
#pragma unroll 2
  for (int i = 0; i < ITERS / 8; ++i) {
#pragma unroll
    for (int t = 0; t < 2; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(A[0]), "d"(A[1]), "d"(A[2]), "d"(A[3]), "d"(A[4]), "d"(A[5]), "d"(A[6]), "d"(A[7]),
                     "d"(B[0]), "d"(B[1]), "d"(B[2]), "d"(B[3]));
  }
  double s = 0;
  for (int t = 0; t < 2; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// half the warps DFMA, half DMMA m8n8k4
__global__ void k_mixed(double* out, double a, double b) {
  int w = threadIdx.x >> 5;
  double s = 0;
  if (w & 1) {
    double A = a + threadIdx.x, B = a - threadIdx.x;
    double c[4][2] = {};
#pragma unroll 4
    for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(A), "d"(B));
    }
    for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  } else {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3,
           x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
    for (int i = 0; i < ITERS; ++i) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
float timeit(F f, int reps = 5) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  int sms = pr.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", pr.name, sms);
  double* out; CK(cudaMalloc(&out, sizeof(double) * 4096 * 1024));
  const int blocks = sms * 8, threads = 256;
  const double nthr = double(blocks) * threads;
  float ms;
  ms = timeit([&] { k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7); });
  printf(", \"dfma_tflops\": %.2f", nthr * ITERS * 8 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_dadd<<<blocks, threads>>>(out, 1e-7); });
  printf(", \"dadd_tops\": %.2f", nthr * ITERS * 8 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_rcp<<<blocks, threads>>>(out, 1e-7); });
  printf(", \"ieee_div_gops\": %.1f", nthr * ITERS / (ms * 1e-3) / 1e9);
  ms = timeit([&] { k_rcp_nr<<<blocks, threads>>>(out, 1e-7); });
  printf(", \"rcp_nr_gops\": %.1f", nthr * ITERS / (ms * 1e-3) / 1e9);
  const double warps = nthr / 32;
  ms = timeit([&] { k_dmma884<<<blocks, threads>>>(out, 0.5); });
  printf(", \"dmma_m8n8k4_tflops\": %.2f", warps * ITERS * 8 * 8 * 4 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_dmma1684<<<blocks, threads>>>(out, 0.5); });
  printf(", \"dmma_m16n8k4_tflops\": %.2f", warps * ITERS * 16 * 8 * 4 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_dmma16816<<<blocks, threads>>>(out, 0.5); });
  printf(", \"dmma_m16n8k16_tflops\": %.2f", warps * (ITERS / 8) * 2 * 16 * 8 * 16 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_mixed<<<blocks, threads>>>(out, 0.999999, 1e-7); });
  // half warps: ITERS*8 fma each; other half: ITERS dmma each (256 fma)
  double fl = (warps / 2) * 32 * ITERS * 8 * 2 + (warps / 2) * ITERS * 256 * 2;
  printf(", \"mixed_tflops\": %.2f, \"mixed_ms\": %.3f", fl / (ms * 1e-3) / 1e12, ms);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf(", \"clock_khz_attr\": %d}\n", clk);
  return 0;
}
