// Throughput probe for the near-field interaction's instruction mix on one
// B200: is MUFU.RCP64H (one per interaction) a limiter next to the 10 FP64
// instructions, and what would a MUFU-free seed (FP32 Newton on the
// mantissa, integer exponent fix-up) cost?  Each kernel runs the P2P term on
// synthetic register-resident sources (4 independent chains per thread) and
// reports G interactions/s; the FP64-only kernel is the roof for the mix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_mix tools/p2p_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ double seed_mufu(double r2) {
  double y;
  asm("{\n\t.reg .b32 h, q, h2, q2;\n\t.reg .b64 s, t;\n\t"
      "mov.b64 {q, h}, %1;\n\tmax.s32 h, h, 0x2d000000;\n\tmov.b64 s, {q, h};\n\t"
      "rcp.approx.ftz.f64 t, s;\n\tmov.b64 {q2, h2}, t;\n\tmov.b64 %0, {h, h2};\n\t}"
      : "=d"(y) : "d"(r2));
  return y;
}

// 1/r2 to ~2^-22 without the MUFU: m = mantissa of r2 in [1, 2) as a float,
// a minimax line + two FP32 Newton steps give 1/m, and the exponent is
// re-biased in the integer pipe (y in (0.5, 1], double hi word from the
// float bits)
__device__ __forceinline__ double seed_soft(double r2) {
  int hi = max(__double2hiint(r2), 0x2d000000);
  const float m = __int_as_float(0x3f800000 | ((hi << 3) & 0x7fffff));
  float y = fmaf(-0.47058824f, m, 1.4117647f);   // 24/17 - 8/17 m
  float e = fmaf(-m, y, 1.0f);
  y = fmaf(y, e, y);
  e = fmaf(-m, y, 1.0f);
  y = fmaf(y, e, y);
  const int yb = __float_as_int(y);
  const int dhi = (yb >> 3) + ((1023 - 127 + 1023) << 20) - (hi & 0x7ff00000);
  return __hiloint2double(dhi, yb << 29);
}

template <int MODE>  // 0: MUFU seed, 1: soft seed, 2: no seed (FP64 only: y = r2)
__global__ void k_mix(double* out, double a) {
  const double yx = threadIdx.x * 1e-3, yy = blockIdx.x * 1e-3;
  double zx[4], zy[4], bx[4] = {}, by[4] = {};
#pragma unroll
  for (int u = 0; u < 4; ++u) { zx[u] = 0.5 + u * 0.01; zy[u] = 0.25 - u * 0.02; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double dx = zx[u] - yx, dy = zy[u] - yy;
      const double r2 = fma(dx, dx, dy * dy);
      const double y = MODE == 0 ? seed_mufu(r2) : MODE == 1 ? seed_soft(r2) : r2;
      const double e = fma(-r2, y, 1.0);
      const double gs = a * fma(fma(e, e, e), y, y);
      bx[u] = fma(gs, dx, bx[u]);
      by[u] = fma(gs, dy, by[u]);
      zx[u] += 1e-9;   // keep the sources moving (one extra DADD per term)
    }
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) s += bx[u] + by[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
__global__ void k_seed_err(const double* x, int n, double* err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double r2 = x[i];
  const double y = MODE == 0 ? seed_mufu(r2) : seed_soft(r2);
  const double e = fma(-r2, y, 1.0);
  const double s = fma(fma(e, e, e), y, y);
  err[i] = fabs(s * r2 - 1.0);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * 8;
  double* out;
  cudaMalloc(&out, sizeof(double) * threads * blocks);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto kern, const char* name) {
    kern<<<blocks, threads>>>(out, 1.0);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out, 1.0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double inter = 5.0 * blocks * threads * ITERS * 4.0;
    printf("\"%s_ginter_s\": %.1f, ", name, inter / (ms * 1e-3) / 1e9);
  };
  printf("{");
  run(k_mix<0>, "mufu_seed");
  run(k_mix<1>, "soft_seed");
  run(k_mix<2>, "fp64_only");
  // accuracy of the two seeds after the cubic step on r2 over 2^-300 .. 2^300
  const int n = 1 << 20;
  double *x, *err;
  cudaMallocManaged(&x, sizeof(double) * n);
  cudaMallocManaged(&err, sizeof(double) * n);
  unsigned long long s = 12345;
  for (int i = 0; i < n; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    const double u = (double)(s >> 11) / 9007199254740992.0;
    x[i] = ldexp(1.0 + u, (int)((s >> 3) % 600) - 300);
  }
  for (int mode = 0; mode < 2; ++mode) {
    if (mode == 0) k_seed_err<0><<<(n + 255) / 256, 256>>>(x, n, err);
    else k_seed_err<1><<<(n + 255) / 256, 256>>>(x, n, err);
    cudaDeviceSynchronize();
    double mx = 0;
    for (int i = 0; i < n; ++i) mx = err[i] > mx ? err[i] : mx;
    printf("\"%s_max_rel_err\": %.3e%s", mode ? "soft" : "mufu", mx, mode ? "" : ", ");
  }
  printf("}\n");
  return 0;
}
