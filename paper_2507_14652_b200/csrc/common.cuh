// Shared device helpers for libhmc (sm_100a).  Product code only: nothing here is shared
// with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hmc {

enum Act : int { ACT_ID = 0, ACT_TANH = 1, ACT_SIN = 2 };

// Philox4x32-10 (counter-based RNG; DESIGN.md §3 "RNG").  Round function as in the
// Random123 construction: two 32x32->64 multiplies, xor with the key, key bumped by the
// Weyl constants between rounds.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    if (r < 9) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
  }
  return c;
}

// u = (x + 0.5) 2^-32 in fp64, strictly inside (0, 1).
__device__ __forceinline__ double u01(uint32_t x) { return ((double)x + 0.5) * 2.3283064365386963e-10; }

// Four standard normals from one Philox block by Box-Muller on (u0,u1) and (u2,u3), fp64.
__device__ __forceinline__ void box_muller4(uint4 w, double z[4]) {
  const double r01 = sqrt(-2.0 * log(u01(w.x)));
  const double r23 = sqrt(-2.0 * log(u01(w.z)));
  double s, c;
  sincospi(2.0 * u01(w.y), &s, &c);
  z[0] = r01 * c;
  z[1] = r01 * s;
  sincospi(2.0 * u01(w.w), &s, &c);
  z[2] = r23 * c;
  z[3] = r23 * s;
}

// TF32 hi part, round-to-nearest-away (cvt.rna), as a float bit pattern with 13 zero low bits
__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// tanh in fp32 without branches (tensor-core epilogue): |x| < 0.6: x p(x^2), p a degree-5
// least-squares-minimax fit of tanh(x)/x (max relative error 1.03e-7 in fp32 Horner); else
// sign(x) (1 - 2 / (2^(2|x| log2 e) + 1)) (max relative error ~2.5e-7 with ex2/rcp.approx).
__device__ __forceinline__ float tanh_acc(float x) {
  const float ax = fabsf(x);
  const float x2 = x * x;
  float p = -0.005852516740560532f;
  p = fmaf(p, x2, 0.020753972232341766f);
  p = fmaf(p, x2, -0.0537688285112381f);
  p = fmaf(p, x2, 0.13331690430641174f);
  p = fmaf(p, x2, -0.3333328366279602f);
  p = fmaf(p, x2, 1.0f);
  const float small = p * x;
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(ax * 2.8853900817779268f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.0f));
  const float big = copysignf(fmaf(-2.0f, r, 1.0f), x);
  return ax < 0.6f ? small : big;
}

// the same function on two values with packed fp32x2 arithmetic (FFMA2 / FMUL2 / FADD2; the
// ex2 / rcp steps stay scalar), bitwise equal to tanh_acc on each lane
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ void tanh_acc2(float& x0, float& x1) {
  const uint64_t x = pk2(x0, x1);
  const uint64_t x2 = fmul2(x, x);
  uint64_t p = ffma2(pk2(-0.005852516740560532f, -0.005852516740560532f), x2,
                     pk2(0.020753972232341766f, 0.020753972232341766f));
  p = ffma2(p, x2, pk2(-0.0537688285112381f, -0.0537688285112381f));
  p = ffma2(p, x2, pk2(0.13331690430641174f, 0.13331690430641174f));
  p = ffma2(p, x2, pk2(-0.3333328366279602f, -0.3333328366279602f));
  p = ffma2(p, x2, pk2(1.0f, 1.0f));
  float s0, s1;
  upk2(fmul2(p, x), s0, s1);
  const float a0 = fabsf(x0), a1 = fabsf(x1);
  float t0, t1;
  upk2(fmul2(pk2(a0, a1), pk2(2.8853900817779268f, 2.8853900817779268f)), t0, t1);
  float e0, e1, r0, r1;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(t0));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(t1));
  float d0, d1;
  upk2(fadd2(pk2(e0, e1), pk2(1.0f, 1.0f)), d0, d1);
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(d0));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(d1));
  float b0, b1;
  upk2(ffma2(pk2(-2.0f, -2.0f), pk2(r0, r1), pk2(1.0f, 1.0f)), b0, b1);
  x0 = a0 < 0.6f ? s0 : copysignf(b0, x0);
  x1 = a1 < 0.6f ? s1 : copysignf(b1, x1);
}

// tanh of a pair with 3 MUFU ops instead of 4 (MUFU / FMA pipes balanced): x0 as tanh_acc,
// x1 for |x| >= 0.6 as (1 - e) / (1 + e) = Q(e), e = 2^(-2|x| log2 e) in (0, 0.3012], Q a degree-7
// minimax polynomial (max relative error 1.8e-7 over the range, scripts/micro/tanh_rate.cu)
__device__ __forceinline__ void tanh_mix2(float& x0, float& x1) {
  const uint64_t x = pk2(x0, x1);
  const uint64_t x2 = fmul2(x, x);
  uint64_t p = ffma2(pk2(-0.005852516740560532f, -0.005852516740560532f), x2,
                     pk2(0.020753972232341766f, 0.020753972232341766f));
  p = ffma2(p, x2, pk2(-0.0537688285112381f, -0.0537688285112381f));
  p = ffma2(p, x2, pk2(0.13331690430641174f, 0.13331690430641174f));
  p = ffma2(p, x2, pk2(-0.3333328366279602f, -0.3333328366279602f));
  p = ffma2(p, x2, pk2(1.0f, 1.0f));
  float s0, s1;
  upk2(fmul2(p, x), s0, s1);
  const float a0 = fabsf(x0), a1 = fabsf(x1);
  float t0, t1;
  upk2(fmul2(pk2(a0, a1), pk2(2.8853900817779268f, -2.8853900817779268f)), t0, t1);
  float e0, e1, r0;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(t0));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(t1));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(e0 + 1.0f));
  const float b0 = fmaf(-2.0f, r0, 1.0f);
  float q = fmaf(-0.6660300493240356f, e1, 1.4774857759475708f);
  q = fmaf(q, e1, -1.8797743320465088f);
  q = fmaf(q, e1, 1.9838345050811768f);
  q = fmaf(q, e1, -1.998784065246582f);
  q = fmaf(q, e1, 1.999954104423523f);
  q = fmaf(q, e1, -1.9999992847442627f);
  q = fmaf(q, e1, 1.0f);
  x0 = a0 < 0.6f ? s0 : copysignf(b0, x0);
  x1 = a1 < 0.6f ? s1 : copysignf(q, x1);
}

__device__ __forceinline__ float act_fwd(int act, float z) {
  if (act == ACT_TANH) return tanhf(z);
  if (act == ACT_SIN) return sinf(z);
  return z;
}

// Deterministic block reduction of a double (fixed tree; every call site uses the same
// blockDim so the summation order is a function of the data layout only).
template <int NT>
__device__ __forceinline__ double block_sum_d(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (threadIdx.x < NT / 32) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;  // valid in thread 0
}

}  // namespace hmc
