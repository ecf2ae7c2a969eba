// Non-GEMM kernels of the hot path (libhmc, sm_100a): output layer + likelihood reduction,
// rank-1 input gradient, output-layer weight gradient, partial-sum reduction, and the
// leapfrog / momentum / Metropolis kernels.  Citations: PAPER.md P:n, DESIGN.md §3 readings.
#pragma once
#include "common.cuh"

namespace hmc {

// Device-side record of hmc_sample progress (written by k_mh / k_advance inside the graph).
// |H* - H0| above which a trajectory counts as divergent (SPEC S:445's threshold, kept as a
// diagnostic only: Q5)
constexpr double DIVERGENCE_DH = 1000.0;

struct Rec {
  float* samples;   // [C x S x k] or nullptr
  uint8_t* acc;     // [C x S] or nullptr
  double* dH;       // [C x S] or nullptr
  int64_t S;
  int64_t sidx;     // current sample slot
  int64_t iter;     // Philox iteration counter
  int32_t adapt;    // 1: dual-averaging step-size adaptation after every trajectory (NEXT-2)
  double delta;     // its target acceptance statistic
};

// Everything the per-chain state kernels need.
struct KState {
  int C;
  int64_t k, P;
  const int32_t* idx;
  const float* inv_mass;       // nullptr = identity
  const uint32_t* chain_ids;
  float* Wd;                   // [C x P] dense per-chain parameters (frozen mu + active theta)
  float* Whi; float* Wlo;      // [C x Ptc] the tensor-core layers' weights: one raw plane (Wlo = nullptr)
                               // or tf32 hi / lo planes; 16B-aligned rows for TMA
  const int32_t* tcpos;        // [k] position of active entry j in the planes, -1 if none
  int64_t Ptc;
  float* cur_theta; float* cur_grad; double* cur_logp;   // chain state (the cache)
  float* wrk_theta; float* wrk_grad; double* wrk_logp;   // trajectory working state
  float* p; double* H0;
  const float* gl;             // [C x k] likelihood part of the gradient
  const double* lik;           // [C] sum of squared residuals
  double inv_2s2;              // 1 / (2 sigma^2)
  double inv_sp2;              // 1 / sigma_p^2
  double* eps;                 // [C] per-chain step sizes (device)
  double* da;                  // [C x 4] dual-averaging state: mu, Hbar, log epsbar, m
  uint32_t* div;               // [C] divergent trajectories (non-finite or |dH| > 1000) since reset
  Rec* rec;
  uint32_t key0, key1;
};

constexpr int KT = 256;  // threads of the per-chain state kernels

// theta_j of chain c -> dense parameters and/or the tf32 hi/lo planes of tensor-core layers:
// tcpos[j] = -1: dense only; q >= 0: dense and planes at q; -(q + 2): planes only (layers whose
// every weight-reading GEMM runs on the tensor cores: one scattered write fewer per step)
__device__ __forceinline__ void put_param(const KState& s, int64_t c, int64_t j, float th) {
  int64_t q = s.tcpos ? (int64_t)__ldg(s.tcpos + j) : -1;
  if (q >= -1) s.Wd[c * s.P + __ldg(s.idx + j)] = th;
  if (q < -1) q = -q - 2;
  if (q >= 0) {
    if (s.Wlo) {  // pre-split hi / lo planes
      const float h = tf32_hi(th);
      s.Whi[c * s.Ptc + q] = h;
      s.Wlo[c * s.Ptc + q] = th - h;
    } else {      // one raw plane (split in shared memory by the GEMM's converters)
      s.Whi[c * s.Ptc + q] = th;
    }
  }
}

// ---- scatter theta_s into the dense per-chain parameter vector (Theta_~s = mu_~s) --
__global__ void k_scatter(KState s, const float* __restrict__ theta) {
  const int64_t c = blockIdx.y;  // chain (grid.y), entries j grid-strided over grid.x
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < s.k; j += (int64_t)gridDim.x * blockDim.x)
    put_param(s, c, j, theta[c * s.k + j]);
}

// tf32 hi/lo planes of one layer's weights for every chain, from the dense parameters
__global__ void k_split_layer(const float* __restrict__ Wd, int64_t P, int64_t w_off, int64_t n,
                              float* __restrict__ Whi, float* __restrict__ Wlo, int64_t Ptc, int64_t q_off, int C) {
  const int64_t total = (int64_t)C * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / n, i = t - c * n;
    const float w = Wd[c * P + w_off + i];
    if (Wlo) {
      const float h = tf32_hi(w);
      Whi[c * Ptc + q_off + i] = h;
      Wlo[c * Ptc + q_off + i] = w - h;
    } else {
      Whi[c * Ptc + q_off + i] = w;
    }
  }
}

// ---- MLP output layer (width 1, identity): f = A w + b; r = y - f; R = r / sigma^2;
//      fp64 partial sums of r^2 per 64-row block (likelihood P:564) ----
__global__ void __launch_bounds__(256) k_out_fwd(const float* __restrict__ Ain, int64_t sA, int n_in,
                                                 int64_t rows, const float* __restrict__ Wd, int64_t P,
                                                 int64_t w_off, int64_t b_off, const float* __restrict__ y,
                                                 float* __restrict__ R, double inv_s2,
                                                 double* __restrict__ part_sq, int n_part) {
  extern __shared__ float w_s[];
  __shared__ double red[8];
  const int c = blockIdx.y;
  const float* w = Wd + (int64_t)c * P + w_off;
  for (int j = threadIdx.x; j < n_in; j += blockDim.x) w_s[j] = w[j];
  const float bias = (b_off >= 0) ? Wd[(int64_t)c * P + b_off] : 0.f;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* A = Ain + (int64_t)c * sA;
  double psq = 0.0;
  for (int rr = 0; rr < 8; ++rr) {
    const int64_t n = (int64_t)blockIdx.x * 64 + warp * 8 + rr;
    if (n >= rows) break;
    float s = 0.f;
    for (int j = lane; j < n_in; j += 32) s = fmaf(A[n * n_in + j], w_s[j], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const float f = s + bias;
      if (y) {
        const float r = y[n] - f;
        R[(int64_t)c * rows + n] = (float)((double)r * inv_s2);
        psq += (double)r * (double)r;
      } else {
        R[(int64_t)c * rows + n] = f;  // prediction mode (hmc_predict): the output itself
      }
    }
  }
  const double tot = block_sum_d<256>(psq, red);
  if (threadIdx.x == 0) part_sq[(int64_t)c * n_part + blockIdx.x] = tot;
}

// ---- the MLP output layer in ONE pass over its input A (training mode; tanh / identity below it):
//      f = A w + b, r = y - f, R = r / sigma^2, fp64 sum r^2 per 64-row block, the weight-
//      and bias-gradient partials of the output layer per 256-row chunk (part[c][chunk][j] =
//      sum_n R[n] A[n][j], j = n_in: sum_n R[n]; reduced by k_colred_p2) and, when the backward
//      continues, the input gradient G[n][j] = R[n] w[j] act'(A[n][j]).  Every step is row-local
//      once R[n] is known, so A (the largest activation) is read once instead of three times; the
//      input gradient's column sums per 32-row block (the next layer's bias-gradient partials, in
//      the layout of the tcgen05 input-gradient epilogue's) come with it.
//      CTA = 256 rows (8 warps x 32 rows); lane j-slots j = lane + 32 m (m < MO, n_in <= 32 MO);
//      column partials: each warp over its rows in order, then the warps in order (fixed order).
template <int MO>
__global__ void __launch_bounds__(256) k_out_fused(const float* __restrict__ Ain, int64_t sA, int n_in, int64_t rows,
                                                   const float* __restrict__ Wd, int64_t P, int64_t w_off,
                                                   int64_t b_off, const float* __restrict__ y, float* __restrict__ R,
                                                   double inv_s2, double* __restrict__ part_sq, int n_part,
                                                   float* __restrict__ colpart, int n_chunks, float* __restrict__ G,
                                                   int act, float* __restrict__ cs, int64_t s_cs) {
  __shared__ float wp[8][32 * MO + 1];  // per-warp column partials (j = n_in: sum R)
  __shared__ double red[8];
  const int c = blockIdx.y, ch = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* w = Wd + (int64_t)c * P + w_off;
  float wr[MO];
#pragma unroll
  for (int m = 0; m < MO; ++m) wr[m] = (lane + 32 * m < n_in) ? __ldg(w + lane + 32 * m) : 0.f;
  const float bias = (b_off >= 0) ? __ldg(Wd + (int64_t)c * P + b_off) : 0.f;
  const float* A = Ain + (int64_t)c * sA;
  float cp[MO];
#pragma unroll
  for (int m = 0; m < MO; ++m) cp[m] = 0.f;
  float gsum[MO];  // bias-gradient partials of the layer below: sum of G over this warp's 32-row block
#pragma unroll
  for (int m = 0; m < MO; ++m) gsum[m] = 0.f;
  float rsum = 0.f;
  double psq = 0.0;
  const int64_t n0 = (int64_t)ch * 256 + warp * 32;
  for (int rr = 0; rr < 32; ++rr) {
    const int64_t n = n0 + rr;
    if (n >= rows) break;
    float a[MO];
    float s = 0.f;
#pragma unroll
    for (int m = 0; m < MO; ++m) {
      a[m] = (lane + 32 * m < n_in) ? A[n * n_in + lane + 32 * m] : 0.f;
      s = fmaf(a[m], wr[m], s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float r = y[n] - (s + bias);
    const float Rn = (float)((double)r * inv_s2);
    psq += (double)r * (double)r;
    if (lane == 0) R[(int64_t)c * rows + n] = Rn;
    rsum += Rn;
#pragma unroll
    for (int m = 0; m < MO; ++m) {
      cp[m] = fmaf(Rn, a[m], cp[m]);
      if (G && lane + 32 * m < n_in) {
        float v = Rn * wr[m];
        if (act == ACT_TANH) v *= (1.f - a[m] * a[m]);
        G[((int64_t)c * rows + n) * n_in + lane + 32 * m] = v;
        gsum[m] += v;
      }
    }
  }
  if (G && cs && n0 < rows) {  // (the 32-row block partials the weight-gradient GEMM's bias fusion reads)
    const int64_t blk = n0 / 32;
#pragma unroll
    for (int m = 0; m < MO; ++m)
      if (lane + 32 * m < n_in) cs[(int64_t)c * s_cs + blk * n_in + lane + 32 * m] = gsum[m];
  }
#pragma unroll
  for (int m = 0; m < MO; ++m) wp[warp][lane + 32 * m] = cp[m];
  if (lane == 0) {
    wp[warp][32 * MO] = rsum;
    red[warp] = psq;  // (lane-local: every lane of the warp holds the same sum r^2)
  }
  __syncthreads();
  float* pc = colpart + ((int64_t)c * n_chunks + ch) * (n_in + 1);
  for (int j = threadIdx.x; j <= n_in; j += 256) {
    const int jj = j < n_in ? j : 32 * MO;
    float t = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += wp[q][jj];
    pc[j] = t;
  }
  if (threadIdx.x < 4) {  // sum r^2 of each 64-row block: warps 2 b, 2 b + 1
    const int64_t blk = (int64_t)ch * 4 + threadIdx.x;
    if (blk < n_part) part_sq[(int64_t)c * n_part + blk] = red[2 * threadIdx.x] + red[2 * threadIdx.x + 1];
  }
}

// ---- input gradient of the width-1 output layer: G[n, j] = R[n] w[j] act'(A[n, j]) ----
__global__ void k_rank1_dact(const float* __restrict__ R, const float* __restrict__ Wd, int64_t P,
                             int64_t w_off, const float* __restrict__ Aprev, const float* __restrict__ Dprev,
                             int act, int64_t rows, int n_in, int C, float* __restrict__ G) {
  const int64_t per = rows * n_in, total = per * C;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / per, rem = t - c * per, n = rem / n_in;
    const int j = (int)(rem - n * n_in);
    float v = R[c * rows + n] * Wd[c * P + w_off + j];
    if (act == ACT_TANH) { const float a = Aprev[t]; v *= (1.f - a * a); }
    else if (act == ACT_SIN) v *= Dprev[t];
    G[t] = v;
  }
}

// ---- weight gradient of the width-1 output layer, pass 1: per 256-row chunk,
//      part[c][chunk][j] = sum_n R[n] X[n, j] (j < n_in), and sum_n R[n] at j = n_in ----
constexpr int COLRED_CH = 256;
__global__ void k_colred_p1(const float* __restrict__ R, const float* __restrict__ X, int64_t sX,
                            int64_t rows, int n_in, float* __restrict__ part, int n_chunks, int sq = 0) {
  const int c = blockIdx.y, ch = blockIdx.x;
  const float* Xc = X + (int64_t)c * sX;
  const float* Rc = R ? R + (int64_t)c * rows : nullptr;
  const int64_t n0 = (int64_t)ch * COLRED_CH;
  const int64_t n1 = min(rows, n0 + COLRED_CH);
  for (int j = threadIdx.x; j <= n_in; j += blockDim.x) {
    float s = 0.f;
    if (j < n_in) {
      if (sq) {  // sensitivity mode: sum R^2 X^2 (sum X^2 without R)
        for (int64_t n = n0; n < n1; ++n) {
          const float xv = Xc[n * n_in + j], rv = R ? Rc[n] : 1.f;
          s = fmaf(rv * rv, xv * xv, s);
        }
      } else if (R) for (int64_t n = n0; n < n1; ++n) s = fmaf(Rc[n], Xc[n * n_in + j], s);
      else for (int64_t n = n0; n < n1; ++n) s += Xc[n * n_in + j];
    } else if (R) {
      for (int64_t n = n0; n < n1; ++n) s += sq ? Rc[n] * Rc[n] : Rc[n];
    }
    part[((int64_t)c * n_chunks + ch) * (n_in + 1) + j] = s;
  }
}

// pass 2: fixed-order sum over chunks, compaction into the k-vector through the slot map
__global__ void k_colred_p2(const float* __restrict__ part, int n_chunks, int n_in,
                            const int32_t* __restrict__ slot_w, const int32_t* __restrict__ slot_b,
                            float* __restrict__ gl, int64_t k) {
  const int c = blockIdx.x;
  for (int j = threadIdx.x; j <= n_in; j += blockDim.x) {
    const int s = (j < n_in) ? slot_w[j] : (slot_b ? slot_b[0] : -1);
    if (s < 0) continue;
    float acc = 0.f;
    for (int ch = 0; ch < n_chunks; ++ch) acc += part[((int64_t)c * n_chunks + ch) * (n_in + 1) + j];
    gl[(int64_t)c * k + s] = acc;
  }
}

// ---- narrow-input layers (n_in <= NARROW_MAX, the networks' first layers: 1-8 inputs) ----
// These are HBM-bound (K = n_in is tiny), so they are plain coalesced kernels, not GEMMs.
constexpr int NARROW_MAX = 16;
constexpr int NARROW_ROWS = 64;  // rows per CTA (forward)
constexpr int NARROW_WROWS = 256;  // rows per CTA (weight gradient, pass 1)

// forward Z = X W^T + b, A = act(Z): thread n owns output column n (weights in
// registers), the CTA's NARROW_ROWS input rows are staged in shared memory, stores coalesced.
template <int DIN>
__global__ void __launch_bounds__(256) k_fwd_narrow(const float* __restrict__ X, int64_t sX, int64_t rows, int n_out,
                                                    const float* __restrict__ Wd, int64_t P, int64_t w_off,
                                                    int64_t b_off, int act, float* __restrict__ A,
                                                    float* __restrict__ D) {
  __shared__ __align__(16) float xs[NARROW_ROWS * DIN];
  const int c = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * NARROW_ROWS;
  const int nr = (int)min((int64_t)NARROW_ROWS, rows - r0);
  const float* Xc = X + (int64_t)c * sX + r0 * DIN;
  for (int t = threadIdx.x; t < nr * DIN; t += blockDim.x) xs[t] = Xc[t];
  __syncthreads();
  const float* W = Wd + (int64_t)c * P + w_off;
  for (int n = threadIdx.x; n < n_out; n += blockDim.x) {
    float w[DIN];
#pragma unroll
    for (int i = 0; i < DIN; ++i) w[i] = W[(int64_t)n * DIN + i];
    const float bias = (b_off >= 0) ? Wd[(int64_t)c * P + b_off + n] : 0.f;
    float* out = A + ((int64_t)c * rows + r0) * n_out + n;
    float* dout = D ? D + ((int64_t)c * rows + r0) * n_out + n : nullptr;
    int r = 0;
    // 4 rows at a time: independent tanh chains (packed pairs, bitwise equal to tanh_acc)
    for (; r + 4 <= nr; r += 4) {
      float z[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float xr[DIN];
        if (DIN % 4 == 0) {  // broadcast row of X as float4 loads
#pragma unroll
          for (int i = 0; i < DIN; i += 4) {
            const float4 x4 = *reinterpret_cast<const float4*>(xs + (r + u) * DIN + i);
            xr[i] = x4.x; xr[i + 1] = x4.y; xr[i + 2] = x4.z; xr[i + 3] = x4.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < DIN; ++i) xr[i] = xs[(r + u) * DIN + i];
        }
        z[u] = bias;
#pragma unroll
        for (int i = 0; i < DIN; ++i) z[u] = fmaf(xr[i], w[i], z[u]);
      }
      if (dout) {
#pragma unroll
        for (int u = 0; u < 4; ++u) dout[(int64_t)(r + u) * n_out] = cosf(z[u]);
      }
      if (act == ACT_TANH) {
        tanh_acc2(z[0], z[1]);
        tanh_acc2(z[2], z[3]);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) z[u] = act_fwd(act, z[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) out[(int64_t)(r + u) * n_out] = z[u];
    }
    for (; r < nr; ++r) {
      float z = bias;
#pragma unroll
      for (int i = 0; i < DIN; ++i) z = fmaf(xs[r * DIN + i], w[i], z);
      if (dout) dout[(int64_t)r * n_out] = cosf(z);
      out[(int64_t)r * n_out] = (act == ACT_TANH) ? tanh_acc(z) : act_fwd(act, z);
    }
  }
}

// weight + bias gradient, pass 1: per chunk of wrows <= NARROW_WROWS rows (host: the long chunk when
// it still gives >= 8 CTAs per SM - a quarter of the partials to write and re-read - else the
// forward's 64; 16 loads of G in flight per thread),
//   part[c][chunk][o][i] = sum_r G[r][o] X[r][i] (i < DIN), part[c][chunk][o][DIN] = sum_r G[r][o]
template <int DIN>
__global__ void __launch_bounds__(256) k_wgrad_narrow_p1(const float* __restrict__ G, int64_t sG, const float* __restrict__ X,
                                                         int64_t sX, int64_t rows, int n_out, float* __restrict__ part,
                                                         int n_chunks, int sq, int wrows) {
  __shared__ __align__(16) float xs[NARROW_WROWS * DIN];
  const int c = blockIdx.y, ch = blockIdx.x;
  const int64_t r0 = (int64_t)ch * wrows;
  const int nr = (int)min((int64_t)wrows, rows - r0);
  const float* Xc = X + (int64_t)c * sX + r0 * DIN;
  for (int t = threadIdx.x; t < nr * DIN; t += blockDim.x) {
    const float xv = Xc[t];
    xs[t] = sq ? xv * xv : xv;  // sensitivity mode: sum G^2 X^2 and sum G^2
  }
  __syncthreads();
  for (int o = threadIdx.x; o < n_out; o += blockDim.x) {
    float acc[DIN + 1];
#pragma unroll
    for (int i = 0; i <= DIN; ++i) acc[i] = 0.f;
    const float* g = G + (int64_t)c * sG + r0 * n_out + o;
#pragma unroll 16
    for (int r = 0; r < nr; ++r) {  // (unrolled: 16 loads of G in flight per thread)
      float gv = g[(int64_t)r * n_out];
      if (sq) gv *= gv;
      float xr[DIN];
      if (DIN % 4 == 0) {  // broadcast row of X as float4 loads
#pragma unroll
        for (int i = 0; i < DIN; i += 4) {
          const float4 x4 = *reinterpret_cast<const float4*>(xs + r * DIN + i);
          xr[i] = x4.x; xr[i + 1] = x4.y; xr[i + 2] = x4.z; xr[i + 3] = x4.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < DIN; ++i) xr[i] = xs[r * DIN + i];
      }
#pragma unroll
      for (int i = 0; i < DIN; ++i) acc[i] = fmaf(gv, xr[i], acc[i]);
      acc[DIN] += gv;
    }
    float* pp = part + (((int64_t)c * n_chunks + ch) * n_out + o) * (DIN + 1);
#pragma unroll
    for (int i = 0; i <= DIN; ++i) pp[i] = acc[i];
  }
}

// pass 2: fixed-order sum over chunks, compaction into the k-vector (W[o][i] at o*DIN + i)
// (grid: (entries / 256, chains); one (o, i) entry per thread, chunks summed in order with 8
//  loads in flight)
__global__ void k_wgrad_narrow_p2(const float* __restrict__ part, int n_chunks, int n_out, int din,
                                  const int32_t* __restrict__ slot_w, const int32_t* __restrict__ slot_b,
                                  float* __restrict__ gl, int64_t k) {
  const int c = blockIdx.y;
  const int per = n_out * (din + 1);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < per; t += gridDim.x * blockDim.x) {
    const int o = t / (din + 1), i = t - o * (din + 1);
    const int sl = (i < din) ? slot_w[o * din + i] : (slot_b ? slot_b[o] : -1);
    if (sl < 0) continue;
    float acc = 0.f;
    const float* p = part + (int64_t)c * n_chunks * per + t;
#pragma unroll 8
    for (int ch = 0; ch < n_chunks; ++ch) acc += p[(int64_t)ch * per];
    gl[(int64_t)c * k + sl] = acc;
  }
}

// ---- posterior predictive (NEXT-4): per datum j, sum and sum of squares over samples of
//      F_j = out[c][j] (+ b0 of sample c), chains in fixed order, fp64 ----
__global__ void k_pred_accum(const float* __restrict__ out, int64_t N, int nb, const float* __restrict__ Wd, int64_t P,
                             int64_t b0_off, double* __restrict__ sum, double* __restrict__ sumsq) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    double s = sum[j], q = sumsq[j];
    for (int c = 0; c < nb; ++c) {
      const double v = (double)out[(int64_t)c * N + j] + (b0_off >= 0 ? (double)Wd[(int64_t)c * P + b0_off] : 0.0);
      s += v;
      q += v * v;
    }
    sum[j] = s;
    sumsq[j] = q;
  }
}
__global__ void k_pred_final(const double* __restrict__ sum, const double* __restrict__ sumsq, int64_t N, double S,
                             double* __restrict__ mean, double* __restrict__ var) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    const double m = sum[j] / S;
    mean[j] = m;
    var[j] = fmax(sumsq[j] / S - m * m, 0.0);
  }
}

// ---- convergence diagnostics (NEXT-4, BDA3 §11.4-11.5 on split chains): one block per
//      parameter j; samples[c][s][j]; half-chain h < C is chain h's first n draws, h >= C the
//      last n draws of chain h - C (n = S / 2, m = 2C).  fp64, fixed-order reductions ----
constexpr int DIAG_T = 256;
__device__ __forceinline__ double diag_val(const float* x, int h, int C, int64_t S, int64_t k, int64_t n, int64_t i,
                                           int64_t j) {
  const int c = h < C ? h : h - C;
  const int64_t off = h < C ? 0 : S - n;
  return (double)x[((int64_t)c * S + off + i) * k + j];
}
__global__ void __launch_bounds__(DIAG_T) k_diag(const float* __restrict__ x, int C, int64_t S, int64_t k,
                                                 double* __restrict__ rhat, double* __restrict__ ess) {
  __shared__ double hm[2 * 1024], hv[2 * 1024];  // per half-chain mean / variance (m <= 2048)
  __shared__ double red[DIAG_T / 32];
  __shared__ double sh[4];
  const int m = 2 * C;
  const int64_t n = S / 2;
  for (int64_t j = blockIdx.x; j < k; j += gridDim.x) {
    for (int h = threadIdx.x; h < m; h += DIAG_T) {
      double su = 0.0;
      for (int64_t i = 0; i < n; ++i) su += diag_val(x, h, C, S, k, n, i, j);
      const double mu = su / (double)n;
      double q = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        const double d = diag_val(x, h, C, S, k, n, i, j) - mu;
        q += d * d;
      }
      hm[h] = mu;
      hv[h] = q / (double)(n - 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double W = 0.0, mm = 0.0;
      for (int h = 0; h < m; ++h) { W += hv[h]; mm += hm[h]; }
      W /= m;
      mm /= m;
      double B = 0.0;
      for (int h = 0; h < m; ++h) B += (hm[h] - mm) * (hm[h] - mm);
      B /= (m - 1);
      const double vp = (double)(n - 1) / (double)n * W + B;
      sh[0] = W;
      sh[1] = vp;
      rhat[j] = sqrt(vp / W);
    }
    __syncthreads();
    const double vp = sh[1];
    // rho_t on demand (block reduction of the variogram)
    auto rho = [&](int64_t t) -> double {
      double v = 0.0;
      const int64_t per = n - t, tot = (int64_t)m * per;
      for (int64_t q = threadIdx.x; q < tot; q += DIAG_T) {
        const int h = (int)(q / per);
        const int64_t i = t + (q - (int64_t)h * per);
        const double d = diag_val(x, h, C, S, k, n, i, j) - diag_val(x, h, C, S, k, n, i - t, j);
        v += d * d;
      }
      v = block_sum_d<DIAG_T>(v, red);
      if (threadIdx.x == 0) sh[2] = 1.0 - (v / ((double)m * (double)per)) / (2.0 * vp);
      __syncthreads();
      const double r = sh[2];
      __syncthreads();
      return r;
    };
    // truncation (BDA3 11.8): sum rho_1 .. rho_T, T the first ODD lag with rho_{T+1} + rho_{T+2}
    // < 0 (all available lags when none qualifies); left-to-right like the oracle
    double ssum = 0.0;
    double rt = n > 1 ? rho(1) : 0.0;  // rho_t of the odd candidate t
    for (int64_t t = 1; t < n; t += 2) {
      ssum += rt;
      if (t + 1 >= n) break;
      const double ra = rho(t + 1);
      if (t + 2 < n) {
        const double rb = rho(t + 2);
        if (ra + rb < 0.0) break;  // T = t
        ssum += ra;
        rt = rb;
      } else {
        ssum += ra;
        break;
      }
    }
    if (threadIdx.x == 0) ess[j] = (double)m * (double)n / (1.0 + 2.0 * ssum);
    __syncthreads();
  }
}

// ---- sensitivity step (NEXT-1, eqn:sensitivities P:193-197) ----
__global__ void k_fill(float* __restrict__ p, int64_t n, float v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    p[t] = v;
}

// DeepONet output seeds: G[m][r][k] = seed[m][k] * act'(output_k of row r) (the reverse pass
// of seed . B (or seed . T) through the net's top layer, one seed vector per virtual chain m)
__global__ void k_seed_top(const float* __restrict__ A, const float* __restrict__ D, int act,
                           const float* __restrict__ seed, int64_t rows, int p, int C, float* __restrict__ G) {
  const int64_t per = rows * p, total = per * C;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = t / per, k = t % p;
    float v = seed[m * p + k];
    if (act == ACT_TANH) { const float a = A[t]; v *= (1.f - a * a); }
    else if (act == ACT_SIN) v *= D[t];
    G[t] = v;
  }
}

// S2[j] = sigma_j^2 * (sum_m sumsq[m][j]) / N_d in fp64, chains summed in fixed order
__global__ void k_sens_finalize(const float* __restrict__ sumsq, int C, int64_t P, const float* __restrict__ sigma,
                                double n_d, int64_t b0, double* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P; j += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    if (j == b0) s = n_d;  // dF/db0 = 1 for every pair
    else
      for (int m = 0; m < C; ++m) s += (double)sumsq[(int64_t)m * P + j];
    const double sg = (double)sigma[j];
    out[j] = sg * sg * s / n_d;
  }
}

// ---- bias gradient from the column partials the tensor-core input-gradient epilogue wrote
//      (one per 32-row block): gl[c][slot_b[o]] = sum_blk colsum[c][blk][o], fixed order ----
// bias gradient from the fused column partials: block (32-column group, chain) of 32 warps, warp w
// sums row blocks w, w + 32, ... of its lane's column (coalesced 128 B rows), then the 32 warp sums
// are added in warp order (fixed order: deterministic)
__global__ void __launch_bounds__(1024) k_colsum_reduce(const float* __restrict__ colsum, int64_t s_colsum, int nblk,
                                                       int N, const int32_t* __restrict__ slot_b,
                                                       float* __restrict__ gl, int64_t k) {
  __shared__ float part[32][33];
  const int c = blockIdx.y;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int o = blockIdx.x * 32 + lane;
  float acc = 0.f;
  if (o < N) {
    const float* p = colsum + (int64_t)c * s_colsum + o;
#pragma unroll 4
    for (int blk = w; blk < nblk; blk += 32) acc += p[(int64_t)blk * N];
  }
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0 && o < N) {
    const int sl = slot_b[o];
    if (sl >= 0) {
      float t = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i) t += part[i][lane];
      gl[(int64_t)c * k + sl] = t;
    }
  }
}


// ---- K-split weight gradient: gl[c][j] = sum_s part[s][c][j] in split order, j in this layer's
//      weight-slot range [lo, hi) ----
__global__ void k_ksplit_reduce(const float* __restrict__ part, int ksplit, int64_t Ck, int64_t k, int64_t lo,
                                int64_t hi, float* __restrict__ gl) {
  const int64_t c = blockIdx.y;
  for (int64_t j = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < hi; j += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < ksplit; ++s) acc += part[(int64_t)s * Ck + c * k + j];
    gl[c * k + j] = acc;
  }
}

// ---- per-chain fixed-order reduction of the likelihood partials: lik[c] = sum r^2; the
//      DeepONet output-bias gradient sum_n R_n goes to its k-slot ----
__global__ void __launch_bounds__(KT) k_reduce_partials(const double* __restrict__ part_sq,
                                                        const double* __restrict__ part_r, int n_part,
                                                        double* __restrict__ lik, float* __restrict__ gl,
                                                        int64_t k, int b0_slot) {
  __shared__ double red[KT / 32];
  const int c = blockIdx.x;
  double s = 0.0, r = 0.0;
  for (int t = threadIdx.x; t < n_part; t += KT) {
    s += part_sq[(int64_t)c * n_part + t];
    if (b0_slot >= 0) r += part_r[(int64_t)c * n_part + t];
  }
  s = block_sum_d<KT>(s, red);
  if (b0_slot >= 0) r = block_sum_d<KT>(r, red);
  if (threadIdx.x == 0) {
    lik[c] = s;
    if (b0_slot >= 0) gl[(int64_t)c * k + b0_slot] = (float)r;
  }
}

// ---- finalize a gradient evaluation: g = g_lik - theta / sigma_p^2 (prior P:233, Q8),
//      log pi = -sum r^2 / (2 sigma^2) - sum theta^2 / (2 sigma_p^2) (fp64);
//      mode 0: plain (hmc_grad); 1: + full kick p += eps g, drift theta += eps M^-1 p and
//      scatter (an inner leapfrog step, Q2); 2: + closing half kick p += eps/2 g ----
__global__ void __launch_bounds__(KT) k_finalize(KState s, int mode) {
  __shared__ double red[KT / 32];
  const int c = blockIdx.x;
  const double eps = (mode != 0) ? s.eps[c] : 0.0;
  const float fe = (float)eps, fh = (float)(0.5 * eps);
  double ss = 0.0;
  for (int64_t j = threadIdx.x; j < s.k; j += KT) {
    const int64_t t = (int64_t)c * s.k + j;
    float th = s.wrk_theta[t];
    const float g = s.gl[t] - (float)((double)th * s.inv_sp2);
    s.wrk_grad[t] = g;
    ss += (double)th * (double)th;
    if (mode == 1) {
      const float im = s.inv_mass ? s.inv_mass[j] : 1.f;
      const float p = fmaf(fe, g, s.p[t]);
      s.p[t] = p;
      th = fmaf(fe * im, p, th);
      s.wrk_theta[t] = th;
      put_param(s, c, j, th);
    } else if (mode == 2) {
      s.p[t] = fmaf(fh, g, s.p[t]);
    }
  }
  ss = block_sum_d<KT>(ss, red);
  if (threadIdx.x == 0) s.wrk_logp[c] = -s.lik[c] * s.inv_2s2 - 0.5 * ss * s.inv_sp2;
}

// ---- inner leapfrog step (Q2), all chains at once: g = g_lik - theta / sigma_p^2,
//      full kick p += eps g, drift theta += eps M^-1 p, scatter.  log pi is not needed at the
//      inner points (only at the trajectory end, k_finalize mode 2), so no reduction here ----
__global__ void __launch_bounds__(256) k_leapfrog(KState s) {
  const int64_t c = blockIdx.y;  // chain (grid.y), entries j grid-strided over grid.x
  const float fe = (float)s.eps[c];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < s.k; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = c * s.k + j;
    float th = s.wrk_theta[t];
    const float g = s.gl[t] - (float)((double)th * s.inv_sp2);
    s.wrk_grad[t] = g;
    const float im = s.inv_mass ? __ldg(s.inv_mass + j) : 1.f;
    const float p = fmaf(fe, g, s.p[t]);
    s.p[t] = p;
    th = fmaf(fe * im, p, th);
    s.wrk_theta[t] = th;
    put_param(s, c, j, th);
  }
}

// ---- start of a trajectory (Algorithm 2): p = sqrt(m) z with z from Philox
//      (key = seed, counter = (j>>2, tag 0, iter, chain_id)), K0 = 1/2 sum p^2 / m (fp64),
//      H0 = -log pi(theta) + K0; then the opening half kick and first drift (+ scatter).
//      L0 != 0: identity trajectory (no kick / drift; working state = current state) ----
__global__ void __launch_bounds__(KT) k_traj_begin(KState s, int L0) {
  __shared__ double red[KT / 32];
  const int c = blockIdx.x;
  const uint32_t iter = (uint32_t)s.rec->iter;
  const uint32_t chain = s.chain_ids[c];
  const double eps = s.eps[c];
  const float fe = (float)eps, fh = (float)(0.5 * eps);
  double K0 = 0.0;
  const int64_t nb = (s.k + 3) / 4;
  for (int64_t blk = threadIdx.x; blk < nb; blk += KT) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)blk, 0u, iter, chain), s.key0, s.key1);
    double z[4];
    box_muller4(w, z);
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int64_t j = blk * 4 + l;
      if (j >= s.k) break;
      const int64_t t = (int64_t)c * s.k + j;
      const float im = s.inv_mass ? s.inv_mass[j] : 1.f;
      float p = (float)(sqrt(1.0 / (double)im) * z[l]);
      K0 += 0.5 * (double)p * (double)p * (double)im;
      float th = s.cur_theta[t];
      if (L0) {
        s.wrk_grad[t] = s.cur_grad[t];
      } else {
        p = fmaf(fh, s.cur_grad[t], p);
        th = fmaf(fe * im, p, th);
        put_param(s, c, j, th);
      }
      s.p[t] = p;
      s.wrk_theta[t] = th;
    }
  }
  K0 = block_sum_d<KT>(K0, red);
  if (threadIdx.x == 0) {
    s.H0[c] = -s.cur_logp[c] + K0;
    if (L0) s.wrk_logp[c] = s.cur_logp[c];
  }
}

// ---- Metropolis-Hastings: H* = -log pi(theta*) + K(p*); u from Philox tag 1
//      word 0; accept iff ln u < H0 - H* (strict; NaN rejects, Q4/Q5).  On accept the
//      working state becomes the chain state; the (possibly repeated) state is recorded ----
__global__ void __launch_bounds__(KT) k_mh(KState s) {
  __shared__ double red[KT / 32];
  __shared__ int acc_s;
  const int c = blockIdx.x;
  double K1 = 0.0;
  for (int64_t j = threadIdx.x; j < s.k; j += KT) {
    const float p = s.p[(int64_t)c * s.k + j];
    const float im = s.inv_mass ? s.inv_mass[j] : 1.f;
    K1 += 0.5 * (double)p * (double)p * (double)im;
  }
  K1 = block_sum_d<KT>(K1, red);
  Rec* rec = s.rec;
  const int64_t sidx = rec->sidx;
  if (threadIdx.x == 0) {
    const double H1 = -s.wrk_logp[c] + K1;
    const double H0 = s.H0[c];
    const uint4 w = philox4x32_10(make_uint4(0u, 1u, (uint32_t)rec->iter, s.chain_ids[c]), s.key0, s.key1);
    const double lu = log(u01(w.x));
    const int acc = (isfinite(H1) && (lu < H0 - H1)) ? 1 : 0;
    acc_s = acc;
    if (acc) s.cur_logp[c] = s.wrk_logp[c];
    if (rec->acc) rec->acc[(int64_t)c * rec->S + sidx] = (uint8_t)acc;
    if (rec->dH) rec->dH[(int64_t)c * rec->S + sidx] = H1 - H0;
    // divergence diagnostic ("gradient explosion" P:488; Q5): flagged, never a
    // rejection rule of its own (the exact test above decides)
    if (!isfinite(H1) || fabs(H1 - H0) > DIVERGENCE_DH) s.div[c] += 1u;
    if (rec->adapt) {
      // dual averaging (Hoffman & Gelman Algorithm 5; DESIGN.md NEXT-2): gamma 0.05,
      // t0 10, kappa 0.75; alpha = min(1, exp(H0 - H*)), 0 for a non-finite H*
      double* da = s.da + (int64_t)c * 4;
      const double alpha = isfinite(H1) ? ((H0 - H1 >= 0.0) ? 1.0 : exp(H0 - H1)) : 0.0;
      const double m = da[3] + 1.0;
      const double eta = 1.0 / (m + 10.0);
      const double hbar = (1.0 - eta) * da[1] + eta * (rec->delta - alpha);
      const double log_eps = da[0] - sqrt(m) / 0.05 * hbar;
      const double w = pow(m, -0.75);
      da[1] = hbar;
      da[2] = w * log_eps + (1.0 - w) * da[2];
      da[3] = m;
      s.eps[c] = exp(log_eps);  // the next trajectory's step
    }
  }
  __syncthreads();
  const int acc = acc_s;
  for (int64_t j = threadIdx.x; j < s.k; j += KT) {
    const int64_t t = (int64_t)c * s.k + j;
    float th;
    if (acc) {
      th = s.wrk_theta[t];
      s.cur_theta[t] = th;
      s.cur_grad[t] = s.wrk_grad[t];
    } else {
      th = s.cur_theta[t];
    }
    if (rec->samples) rec->samples[((int64_t)c * rec->S + sidx) * s.k + j] = th;
  }
}

// dual-averaging start (mu = log(10 eps0), Hbar = 0, log epsbar = 0, m = 0; eps = eps0) and
// finish (eps = epsbar, copied out)
__global__ void k_da_init(double* __restrict__ eps, double* __restrict__ da, int C, double eps0) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    eps[c] = eps0;
    da[4 * c + 0] = log(10.0 * eps0);
    da[4 * c + 1] = 0.0;
    da[4 * c + 2] = 0.0;
    da[4 * c + 3] = 0.0;
  }
}
__global__ void k_da_finish(double* __restrict__ eps, const double* __restrict__ da, int C, double* __restrict__ out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) out[c] = exp(da[4 * c + 2]);
}
__global__ void k_fill_d(double* __restrict__ p, int n, double v) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) p[c] = v;
}

__global__ void k_advance(Rec* rec) {
  rec->sidx += 1;
  rec->iter += 1;
}

// ---- diagnostics ----
__global__ void k_philox_words(uint32_t k0, uint32_t k1, uint32_t tag, uint32_t iter, uint32_t chain,
                               int64_t nblocks, uint32_t* __restrict__ out) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblocks;
       b += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)b, tag, iter, chain), k0, k1);
    out[4 * b + 0] = w.x;
    out[4 * b + 1] = w.y;
    out[4 * b + 2] = w.z;
    out[4 * b + 3] = w.w;
  }
}

__global__ void k_momentum(KState s, uint32_t iter, float* __restrict__ out) {
  const int c = blockIdx.x;
  const uint32_t chain = s.chain_ids[c];
  const int64_t nb = (s.k + 3) / 4;
  for (int64_t blk = threadIdx.x; blk < nb; blk += blockDim.x) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)blk, 0u, iter, chain), s.key0, s.key1);
    double z[4];
    box_muller4(w, z);
    for (int l = 0; l < 4; ++l) {
      const int64_t j = blk * 4 + l;
      if (j >= s.k) break;
      const float im = s.inv_mass ? s.inv_mass[j] : 1.f;
      out[(int64_t)c * s.k + j] = (float)(sqrt(1.0 / (double)im) * z[l]);
    }
  }
}


// ================= unaligned DeepONet (per-pair trunk inputs) =================
// Pair (c, x) has its own trunk row r = c * n_x + x: F_cx = sum_k B_ck T_rk + b0.  The
// combine is a row-wise dot (no GEMM: each trunk row meets one branch row), read once from HBM.

// act' of a layer output at element t: tanh -> 1 - a^2 (a = output), sin -> D (cos z, stored by
// the forward), identity -> 1
__device__ __forceinline__ float dact_at(int act, const float* __restrict__ A, const float* __restrict__ D, int64_t t) {
  if (act == ACT_TANH) { const float a = A[t]; return 1.f - a * a; }
  if (act == ACT_SIN) return D[t];
  return 1.f;
}

// ---- K-split dT (DeepONet trunk output gradient): G[c][t] = (sum_s part[c * ks + s][t]) act'(t),
//      the ks row slabs' partial products summed in slab order; t over the M x N tile of chain c ----
__global__ void k_dact_ksplit_reduce(const float* __restrict__ part, int ks, int64_t MN, int act,
                                     const float* __restrict__ A, const float* __restrict__ D,
                                     float* __restrict__ G) {
  const int64_t c = blockIdx.y;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < MN; t += (int64_t)gridDim.x * blockDim.x) {
    const float* p = part + c * ks * MN + t;
    float acc = 0.f;
    for (int s = 0; s < ks; ++s) acc += p[(int64_t)s * MN];
    G[c * MN + t] = acc * dact_at(act, A, D, c * MN + t);
  }
}

// combine + residual: block (c, chain), one warp per pair row x (lanes over k).  V != nullptr:
// R_cx = (V_cx - F_cx) / sigma^2 and the fixed-order fp64 partials sum r^2, sum R of the block go
// to slot c of the chain; V == nullptr (prediction): R_cx = F_cx.
__global__ void __launch_bounds__(256) k_pair_combine(const float* __restrict__ B, const float* __restrict__ T,
                                                      int p, int64_t n_c, int64_t n_x,
                                                      const float* __restrict__ V, const float* __restrict__ b0,
                                                      int64_t s_b0, double inv_s2, float* __restrict__ R,
                                                      double* __restrict__ part_sq, double* __restrict__ part_r,
                                                      int n_part) {
  extern __shared__ float sBrow[];
  __shared__ double red[2][8];
  const int64_t c = blockIdx.x;
  const int ch = blockIdx.y;
  const float* Bc = B + ((int64_t)ch * n_c + c) * p;
  for (int k = threadIdx.x; k < p; k += blockDim.x) sBrow[k] = Bc[k];
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float bb = b0 ? b0[(int64_t)ch * s_b0] : 0.f;
  const float is2 = (float)inv_s2;
  double sq = 0.0, sr = 0.0;
  for (int64_t xi = w; xi < n_x; xi += 8) {
    const float* Tr = T + ((int64_t)ch * n_c * n_x + c * n_x + xi) * p;
    float d = 0.f;
    for (int k = lane; k < p; k += 32) d = fmaf(sBrow[k], Tr[k], d);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    const float F = d + bb;
    const int64_t o_idx = ((int64_t)ch * n_c + c) * n_x + xi;
    if (V) {
      const float r = V[c * n_x + xi] - F;
      const float e = r * is2;
      if (lane == 0) R[o_idx] = e;
      sq += (double)r * (double)r;
      sr += (double)e;
    } else if (lane == 0) {
      R[o_idx] = F;
    }
  }
  if (!V) return;
  if (lane == 0) { red[0][w] = sq; red[1][w] = sr; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < 8; ++i) { a += red[0][i]; b += red[1][i]; }
    part_sq[(int64_t)ch * n_part + c] = a;
    part_r[(int64_t)ch * n_part + c] = b;
  }
}

// branch output gradient: G_ck = act'_B(c, k) * sum_x R_cx T_(c n_x + x) k; block (c, chain),
// threads over k (rows of T read coalesced), fixed-order sum over x
__global__ void __launch_bounds__(256) k_pair_dB(const float* __restrict__ R, const float* __restrict__ T, int p,
                                                 int64_t n_c, int64_t n_x, int act, const float* __restrict__ A,
                                                 const float* __restrict__ D, float* __restrict__ G) {
  const int64_t c = blockIdx.x;
  const int ch = blockIdx.y;
  const float* Rc = R + ((int64_t)ch * n_c + c) * n_x;
  const float* Tc = T + ((int64_t)ch * n_c * n_x + c * n_x) * p;
  for (int k = threadIdx.x; k < p; k += blockDim.x) {
    float s = 0.f;
    for (int64_t xi = 0; xi < n_x; ++xi) s = fmaf(Rc[xi], Tc[xi * p + k], s);
    const int64_t t = ((int64_t)ch * n_c + c) * p + k;
    G[t] = s * dact_at(act, A, D, t);
  }
}

// trunk output gradient: G_(c n_x + x) k = R_cx B_ck act'_T(row, k), element-wise
__global__ void k_pair_dT(const float* __restrict__ R, const float* __restrict__ B, int p, int64_t n_c, int64_t n_x,
                          int C, int act, const float* __restrict__ A, const float* __restrict__ D,
                          float* __restrict__ G) {
  const int64_t rows = n_c * n_x, total = (int64_t)C * rows * p;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t % p, rr = t / p;     // rr = chain * rows + c * n_x + x
    const int64_t ch = rr / rows, row = rr - ch * rows, c = row / n_x;
    G[t] = R[rr] * B[(ch * n_c + c) * p + k] * dact_at(act, A, D, t);
  }
}

// ================= DATA mode POINTS_XB layout: rank r owns condition block r ====
// all-gather result [rank][chain][i][k] -> per-chain rows of all conditions [chain][r*n_loc + i][k]
__global__ void k_xb_gather(const float* __restrict__ recv, float* __restrict__ full, int C, int G, int64_t n_loc,
                            int p) {
  const int64_t per = n_loc * p, total = (int64_t)G * C * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / ((int64_t)C * per), rem = t - r * C * per, c = rem / per, e = rem - c * per;
    full[(c * G + r) * per + e] = recv[t];
  }
}
// per-chain rows of all conditions -> reduce-scatter input [rank][chain][i][k] (block r to rank r)
__global__ void k_xb_scatter(const float* __restrict__ full, float* __restrict__ send, int C, int G, int64_t n_loc,
                             int p) {
  const int64_t per = n_loc * p, total = (int64_t)G * C * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / ((int64_t)C * per), rem = t - r * C * per, c = rem / per, e = rem - c * per;
    send[t] = full[(c * G + r) * per + e];
  }
}

}  // namespace hmc
