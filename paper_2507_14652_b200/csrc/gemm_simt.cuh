// Chain-batched FP32 SIMT GEMM with the hot path's fused epilogues (libhmc, sm_100a).
//
// C[b] (M x N) = A[b] (M x K) . B[b] (K x N), fp32 FMA accumulate, one CTA per BMxBN tile and
// batch b (= chain).  Used for narrow layers (widths <= 64, the "warp-level FP32 FMA" engine
// of the north star) and as the generic engine for any shape the tcgen05 engine does not take.
// Operand layouts (template):
//   A_KMAJOR: A(m,k) = A[m*lda + k]   else   A(m,k) = A[k*lda + m]
//   B_KMAJOR: B(k,n) = B[n*ldb + k]   else   B(k,n) = B[k*ldb + n]
// The layer GEMMs of a gradient evaluation ("forward pass and gradient computation"):
//   forward      Z_l = A_{l-1} W_l^T          (A K-major, B K-major)  epilogue EPI_FWD
//   input grad   G_{l-1} = (G_l W_l) o act'   (A K-major, B N-major)  epilogue EPI_DACT
//   weight grad  dW_l = G_l^T [A_{l-1} | 1]   (A M-major, B N-major)  epilogue EPI_WGRAD
//   DeepONet combine O = B T^T + b0           (A K-major, B K-major)  epilogue EPI_RESID
// Every summation order is fixed (k ascending within a thread; fp64 fixed-tree partials).
#pragma once
#include "common.cuh"

namespace hmc {

enum Epi : int { EPI_STORE = 0, EPI_FWD = 1, EPI_DACT = 2, EPI_WGRAD = 3, EPI_RESID = 4 };

struct GemmArgs {
  int M, N, K, batch;
  const float* A; int64_t lda, sA;
  const float* B; int64_t ldb, sB;
  float* C; int64_t ldc, sC;
  int ones_col;  // >= 0: B(k, n == ones_col) = 1 (bias column of the weight gradient)
  int epi;
  int max_pairs;  // tcgen05 engine: > 0 caps the launch's CTA pairs (several tiles per pair); 0 = one round of the SMs
  int act;       // EPI_FWD: activation of this layer; EPI_DACT: activation of the producer
  // EPI_FWD
  const float* bias; int64_t s_bias;  // per-batch stride (nullptr = no bias)
  float* D; int64_t ldd, sD;          // cos(z) for sin layers (nullptr otherwise)
  // EPI_DACT: act' evaluated from the producer's stored output (tanh: 1 - a^2) or D (sin)
  const float* dsrc; int64_t ld_dsrc, s_dsrc;
  // EPI_WGRAD: slot_w[m*n_in + n] (n < n_in) or slot_b[m] (n == ones_col); -1 = frozen
  const int32_t* slot_w; const int32_t* slot_b; int n_in;
  // optional compact form of slot_w for the tensor-core epilogue: per row m and 32-column group
  // g, gmask[m*n_grp + g] = active columns, gbase[...] = slot of the group's first active entry
  // (slots are ranks of ascending flat indices, so slot(m, 32g + j) = gbase + popc(mask below j))
  const uint32_t* gmask; const int32_t* gbase; int n_grp;
  // tensor-core EPI_WGRAD split over K (ksplit > 1): split s writes its partial k-vector entries
  // to gl_part + s * batch * k (summed in fixed order afterwards)
  int ksplit; float* gl_part;
  // tensor-core EPI_WGRAD: also reduce this layer's bias gradient from the fused column partials
  // (bcs[b * s_bcs + blk * M + o], blk < bcs_nblk, fixed order) into gl[b * k + bcs_slot[o]]
  const float* bcs; int64_t s_bcs; int bcs_nblk; const int32_t* bcs_slot;
  float* gl; int64_t k;
  // EPI_RESID: R = (V - (acc + b0)) * inv_s2; partial sums of r^2 and of R per tile (fp64)
  const float* V; int64_t ldv;
  const float* b0; int64_t s_b0;
  double inv_s2;
  double* part_sq; double* part_r; int n_part;
  // EPI_DACT (tensor-core engine only): column sums of the output per 32-row block,
  // colsum[b * s_colsum + (m / 32) * N + n] (bias gradient of the layer below, fused)
  float* colsum; int64_t s_colsum;
  // sensitivity mode (NEXT-1): EPI_WGRAD multiplies the SQUARED operands (sum_n G^2 X^2) and
  // EPI_DACT's column partials sum the squared outputs
  int sq;
};

template <int BM>
struct SimtCfg {
  static constexpr int BN = BM, BK = 8, NT = 256;
  static constexpr int TM = BM / 16, TN = BM / 16;   // per-thread outputs along M / N
  static constexpr int EA = BM * BK / NT;            // elements each thread loads per operand
};

template <int BM, bool A_KMAJOR, bool B_KMAJOR>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs a) {
  using Cfg = SimtCfg<BM>;
  constexpr int BN = Cfg::BN, BK = Cfg::BK, TM = Cfg::TM, TN = Cfg::TN, EA = Cfg::EA;
  constexpr int HM = TM / 2, HN = TN / 2;
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  __shared__ double red[16];

  const int b = blockIdx.z;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const float* __restrict__ A = a.A + (int64_t)b * a.sA;
  const float* __restrict__ B = a.B + (int64_t)b * a.sB;

  float ra[EA], rb[EA];
  // loader coordinates
  int la_m, la_k, lb_n, lb_k;
  if (A_KMAJOR) { la_m = tid / (BK / EA); la_k = (tid % (BK / EA)) * EA; }
  else          { la_k = tid / (BM / EA); la_m = (tid % (BM / EA)) * EA; }
  if (B_KMAJOR) { lb_n = tid / (BK / EA); lb_k = (tid % (BK / EA)) * EA; }
  else          { lb_k = tid / (BN / EA); lb_n = (tid % (BN / EA)) * EA; }

  auto load = [&](int kt) {
    const int kb = kt * BK;
#pragma unroll
    for (int e = 0; e < EA; ++e) {
      int m = A_KMAJOR ? la_m : la_m + e, kk = A_KMAJOR ? la_k + e : la_k;
      int gm = m0 + m, gk = kb + kk;
      ra[e] = (gm < a.M && gk < a.K) ? (A_KMAJOR ? A[(int64_t)gm * a.lda + gk] : A[(int64_t)gk * a.lda + gm]) : 0.f;
      if (a.sq && a.epi == EPI_WGRAD) ra[e] *= ra[e];
      int n = B_KMAJOR ? lb_n : lb_n + e, kn = B_KMAJOR ? lb_k + e : lb_k;
      int gn = n0 + n, gkn = kb + kn;
      float v = 0.f;
      if (gn < a.N && gkn < a.K) {
        if (gn == a.ones_col) v = 1.f;
        else v = B_KMAJOR ? B[(int64_t)gn * a.ldb + gkn] : B[(int64_t)gkn * a.ldb + gn];
      }
      rb[e] = (a.sq && a.epi == EPI_WGRAD) ? v * v : v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < EA; ++e) {
      if (A_KMAJOR) As[buf][la_k + e][la_m] = ra[e]; else As[buf][la_k][la_m + e] = ra[e];
      if (B_KMAJOR) Bs[buf][lb_k + e][lb_n] = rb[e]; else Bs[buf][lb_k][lb_n + e] = rb[e];
    }
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  const int nk = (a.K + BK - 1) / BK;
  load(0);
  store(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) load(kt + 1);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < HM; ++i) {
        av[i] = As[cur][kk][ty * HM + i];
        av[HM + i] = As[cur][kk][BM / 2 + ty * HM + i];
      }
#pragma unroll
      for (int j = 0; j < HN; ++j) {
        bv[j] = Bs[cur][kk][tx * HN + j];
        bv[HN + j] = Bs[cur][kk][BN / 2 + tx * HN + j];
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) store(cur ^ 1);
    __syncthreads();
  }

  // ---- fused epilogue ----
  double psq = 0.0, pr = 0.0;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + (i < HM ? ty * HM + i : BM / 2 + ty * HM + (i - HM));
    if (m >= a.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + (j < HN ? tx * HN + j : BN / 2 + tx * HN + (j - HN));
      if (n >= a.N) continue;
      float v = acc[i][j];
      switch (a.epi) {
        case EPI_FWD: {
          if (a.bias) v += a.bias[(int64_t)b * a.s_bias + n];
          if (a.D) a.D[(int64_t)b * a.sD + (int64_t)m * a.ldd + n] = cosf(v);
          a.C[(int64_t)b * a.sC + (int64_t)m * a.ldc + n] = act_fwd(a.act, v);
        } break;
        case EPI_DACT: {
          if (a.act == ACT_TANH) {
            const float t = a.dsrc[(int64_t)b * a.s_dsrc + (int64_t)m * a.ld_dsrc + n];
            v *= (1.f - t * t);
          } else if (a.act == ACT_SIN) {
            v *= a.dsrc[(int64_t)b * a.s_dsrc + (int64_t)m * a.ld_dsrc + n];
          }
          a.C[(int64_t)b * a.sC + (int64_t)m * a.ldc + n] = v;
        } break;
        case EPI_WGRAD: {
          const int s = (n == a.ones_col) ? a.slot_b[m] : a.slot_w[(int64_t)m * a.n_in + n];
          if (s >= 0) a.gl[(int64_t)b * a.k + s] = v;
        } break;
        case EPI_RESID: {
          const float o = v + (a.b0 ? a.b0[(int64_t)b * a.s_b0] : 0.f);
          const float r = a.V[(int64_t)m * a.ldv + n] - o;
          const float R = (float)((double)r * a.inv_s2);
          a.C[(int64_t)b * a.sC + (int64_t)m * a.ldc + n] = R;
          psq += (double)r * (double)r;
          pr += (double)R;
        } break;
        default:
          a.C[(int64_t)b * a.sC + (int64_t)m * a.ldc + n] = v;
      }
    }
  }
  if (a.epi == EPI_RESID) {
    const double s1 = block_sum_d<256>(psq, red);
    const double s2 = block_sum_d<256>(pr, red);
    if (tid == 0) {
      const int t = blockIdx.y * gridDim.x + blockIdx.x;
      a.part_sq[(int64_t)b * a.n_part + t] = s1;
      a.part_r[(int64_t)b * a.n_part + t] = s2;
    }
  }
}

}  // namespace hmc
