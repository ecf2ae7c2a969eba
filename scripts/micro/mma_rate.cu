// Microbenchmark (dev tool): tcgen05.mma kind::tf32 issue rate, M=128, N in {128,256},
// A from TMEM ("ts") or SMEM ("ss"), B from SMEM (K-major 128B swizzle, data = zeros).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
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
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ volatile int g_stop;
__device__ float g_src[148 * 16384];
template <int N, bool TS, int NOISE>
__global__ void k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u ^ (blockIdx.x * 40503u);
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    ((float*)base)[i] = NOISE == 7 ? ((float)(h & 0xffffff) / 16777216.0f - 0.5f) : 0.f;
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = holder;
  if (NOISE == 7 && threadIdx.x < 128) {  // random A hi/lo columns 384..447 in TMEM
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = __float_as_uint((float)((threadIdx.x * 37 + i * 11) % 97) / 97.0f - 0.5f);
    const uint32_t ta = tm + ((uint32_t)(32 * (threadIdx.x >> 5)) << 16) + 384;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      :: "r"(ta), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),"r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]) : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      :: "r"(ta + 32), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),"r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if ((NOISE == 5 || NOISE == 6) && threadIdx.x >= 32) {
    // bulk async copies global -> shared (the TMA engine) into a separate 16 KB region, 2 in flight
    constexpr int NB = NOISE == 6 ? 6 : 2;
    __shared__ __align__(8) uint64_t cb[6];
    if (threadIdx.x == 32) {
      for (int i = 0; i < NB; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cb[i])));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      unsigned long long n = 0;
      uint32_t ph[6] = {0, 0, 0, 0, 0, 0};
      const char* src = (const char*)g_src + (size_t)blockIdx.x * 65536;
      for (int i = 0; i < NB; ++i) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&cb[i])), "r"(8192) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(base + 65536 + i * 8192)), "l"(src + i * 8192), "r"(8192), "r"(su32(&cb[i])) : "memory");
      }
      while (!stop) {
        for (int i = 0; i < NB; ++i) {
          asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra W;}" ::"r"(su32(&cb[i])), "r"(ph[i]) : "memory");
          ph[i] ^= 1;
          ++n;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&cb[i])), "r"(8192) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(base + 65536 + i * 8192)), "l"(src + ((n & 7) * 8192)), "r"(8192), "r"(su32(&cb[i])) : "memory");
        }
      }
      for (int i = 0; i < NB; ++i)
        asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra W;}" ::"r"(su32(&cb[i])), "r"(ph[i]) : "memory");
      out[148 + blockIdx.x] = n;
    }
  } else if (NOISE >= 3 && threadIdx.x >= 32) {
    // TMEM traffic from the other warps (3: tcgen05.ld, 4: tcgen05.st) on columns 256..383
    const int w = threadIdx.x >> 5;
    const uint32_t ta = tm + ((uint32_t)(32 * (w & 3)) << 16) + 256 + ((w >> 2) & 1) * 64;
    unsigned long long n = 0;
    float accf = 0.f;
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = i;
    while (!stop) {
      if (NOISE == 3) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31])
          : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        accf += __uint_as_float(r[0]) + __uint_as_float(r[31]);
      } else {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
          :: "r"(ta), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),"r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      ++n;
    }
    if (accf == 12345.f) out[0] = n;
    if (threadIdx.x == 32) out[148 + blockIdx.x] = n;
  } else if (NOISE > 0 && NOISE < 3 && threadIdx.x >= 32) {
    // shared-memory traffic from the other warps: v4 loads + stores on a separate 16 KB region
    float4* reg = (float4*)(base + 49152);
    const int t = threadIdx.x - 32;
    float4 acc = make_float4(0, 0, 0, 0);
    unsigned long long n = 0;
    while (!stop) {
#pragma unroll 8
      for (int i = 0; i < 8; ++i) {
        float4 v = reg[(t + i * 96) & 1023];
        acc.x += v.x;
        if (NOISE > 1) reg[(t + i * 96 + 512) & 1023] = acc;
      }
      n += 8;
    }
    if (acc.x == 12345.f) out[0] = n;
    if (t == 0) out[148 + blockIdx.x] = n;
  }
  if (threadIdx.x == 0) {
    const uint32_t ID = idesc(128, N);
    const uint64_t bd = sdesc(su32(base));
    const uint64_t ad = sdesc(su32(base + 32768));
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (TS)
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}" ::"r"(tm),
                       "r"(tm + 384 + 8 * kk), "l"(bd + 2 * kk), "r"(ID), "r"(1));
        else
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}" ::"r"(tm),
                       "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(ID), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @!P1 bra W;}" ::"r"(su32(&bar)) : "memory");
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
template <int N, bool TS, int NOISE>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 2 * 148 * 8);
  cudaFuncSetAttribute(k<N, TS, NOISE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  const int iters = 20000;
  k<N, TS, NOISE><<<148, (NOISE >= 3 && NOISE != 7) ? 288 : 128, 140000>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2 * 148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double macs = (double)iters * 4 * 128 * N * 8;
  const double lsu = (NOISE == 5 || NOISE == 6) ? (double)h[148] * 8192 / h[0] : NOISE >= 3 ? (double)h[148] * 8 * 4096 / h[0]
                                 : (NOISE ? (double)h[148] * 96 * 16 * (NOISE > 1 ? 2 : 1) / h[0] : 0.0);
  printf("%s N=%d noise=%d: %.0f MAC/clk/SM (%.1f%% of 2048), LSU smem %.1f B/clk  %s\n", name, N, NOISE, macs / h[0],
         100.0 * macs / h[0] / 2048, lsu, cudaGetErrorString(e));
  cudaFree(d);
}
int main() {
  run<128, true, 7>("ts-rand");
  run<128, false, 7>("ss-rand");
  run<256, false, 7>("ss-rand");
  run<128, true, 6>("ts");
  run<128, false, 6>("ss");
  run<128, true, 5>("ts");
  run<128, false, 5>("ss");
  run<256, false, 5>("ss");
  run<128, true, 3>("ts");
  run<128, true, 4>("ts");
  run<128, false, 3>("ss");
  run<128, true, 0>("ts");
  run<128, false, 0>("ss");
  run<256, false, 0>("ss");
  run<128, true, 1>("ts");
  run<128, true, 2>("ts");
  run<128, false, 1>("ss");
  run<128, false, 2>("ss");
  run<256, false, 2>("ss");
  run<256, true, 2>("ts");
  return 0;
}
