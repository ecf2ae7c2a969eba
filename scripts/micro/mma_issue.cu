// Microbenchmark (dev tool): tcgen05.mma kind::tf32 (M=128, N=128, A from TMEM) issue loop with
// the per-K-block bookkeeping of the GEMM engine: MODE bit0 = 3 commits per 12 MMAs,
// bit1 = tcgen05.fence::after_thread_sync x2, bit2 = elect.sync + __syncwarp (whole warp),
// bit3 = mbarrier try_wait on a completed barrier x2.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .pred %%px;\nelect.sync _|%%px, %1;\n@%%px mov.s32 %0, 1;\n}\n" : "+r"(pred) : "r"(0xffffffffu));
  return pred != 0;
}
template <int MODE>
__global__ void k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar[4];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) ((float*)base)[i] = 0.f;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = holder;
  const uint32_t ID = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint64_t bd = sdesc(su32(base));
  if (threadIdx.x < 32 && ((MODE & 4) || threadIdx.x == 0)) {
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (MODE & 8) {
        // try_wait on bar[3] phase parity 1 (the "previous" phase: completes immediately)
        asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 1; @!P1 bra W;}" ::"r"(su32(&bar[3])) : "memory");
        asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 1; @!P1 bra W;}" ::"r"(su32(&bar[3])) : "memory");
      }
      if (MODE & 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      const uint32_t d = tm + (it % 3) * 128;
      const uint32_t a = tm + 384 + (it & 1) * 64;
      bool go = (MODE & 4) ? elect_one() : true;
      if (go) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}" ::"r"(d), "r"(a + 32 + 8 * kk), "l"(bd + 2 * kk), "r"(ID), "r"(kk));
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}" ::"r"(d), "r"(a + 8 * kk), "l"(bd + 1024 + 2 * kk), "r"(ID), "r"(1));
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}" ::"r"(d), "r"(a + 8 * kk), "l"(bd + 2 * kk), "r"(ID), "r"(1));
        if (MODE & 1) {
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[0])) : "memory");
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[1])) : "memory");
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[2])) : "memory");
        }
      }
      if (MODE & 4) __syncwarp();
    }
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[3])) : "memory");
      asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @!P1 bra W;}" ::"r"(su32(&bar[3])) : "memory");
      out[blockIdx.x] = clock64() - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
template <int MODE>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  const int iters = 20000;
  k<MODE><<<148, 128, 40000>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double macs = (double)iters * 12 * 128 * 128 * 8;
  printf("mode %2d: %.1f%% of 2048 MAC/clk/SM, %.0f clk per 12-MMA block  %s\n", MODE, 100.0 * macs / h[0] / 2048,
         (double)h[0] / iters, cudaGetErrorString(e));
  cudaFree(d);
}
int main() {
  run<0>(); run<1>(); run<2>(); run<3>(); run<4>(); run<5>(); run<8>(); run<15>();
  return 0;
}
