// FP32 FMA issue rate on B200 (the narrow engine's roofline denominator).
// Each thread runs an 8 x 8 outer-product update from register operands (the shape of the
// narrow engine's GEMM inner loops, 3-register FFMA form, operands refreshed every iteration so
// nothing folds to immediates), at full occupancy and at 8 warps per SM (the narrow engine's
// residency: one 256-thread CTA per SM).  Prints FLOP/s and the fraction of the nominal
// 148 SMs x 128 lanes x 2 x clock.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ffma_rate ffma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int M, int N>
__global__ void k_outer(float* out, int iters, float s) {
  float acc[M][N];
  float a[M], b[N];
#pragma unroll
  for (int m = 0; m < M; ++m) a[m] = threadIdx.x * 1e-3f + m;
#pragma unroll
  for (int n = 0; n < N; ++n) b[n] = blockIdx.x * 1e-3f + n;
#pragma unroll
  for (int m = 0; m < M; ++m)
#pragma unroll
    for (int n = 0; n < N; ++n) acc[m][n] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
      for (int n = 0; n < N; ++n) acc[m][n] = fmaf(a[m], b[n], acc[m][n]);
#pragma unroll
    for (int m = 0; m < M; ++m) a[m] = a[m] * s;  // (FMUL: keeps operands live, 1/N of the work)
  }
  float t = 0.f;
#pragma unroll
  for (int m = 0; m < M; ++m)
#pragma unroll
    for (int n = 0; n < N; ++n) t += acc[m][n];
  if (t == 1234.5f) out[threadIdx.x] = t;
}

template <int M, int N>
void run(const char* name, int blocks, int threads, double clk_mhz) {
  float* out;
  cudaMalloc(&out, 4096);
  const int iters = 4096;
  k_outer<M, N><<<blocks, threads>>>(out, 16, 0.999f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k_outer<M, N><<<blocks, threads>>>(out, iters, 0.999f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = 5.0 * blocks * threads * (double)iters * M * N * 2.0;
  const double tf = flop / (ms * 1e-3) / 1e12;
  const double nominal = 148.0 * 128 * 2 * clk_mhz * 1e6 / 1e12;
  printf("%-28s blocks %5d x %4d thr: %7.2f TFLOP/s  = %.3f of nominal %.1f TF @ %.0f MHz\n", name, blocks, threads, tf,
         tf / nominal, nominal, clk_mhz);
  cudaFree(out);
}

int main() {
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double mhz = clk_khz / 1000.0;
  run<8, 8>("8x8 full occupancy", 148 * 8, 256, mhz);
  run<8, 8>("8x8 8 warps/SM", 148, 256, mhz);
  run<4, 4>("4x4 full occupancy", 148 * 8, 256, mhz);
  run<4, 4>("4x4 8 warps/SM", 148, 256, mhz);
  run<4, 8>("4x8 8 warps/SM", 148, 256, mhz);
  return 0;
}
