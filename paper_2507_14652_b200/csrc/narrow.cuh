// narrow.cuh - the narrow-network engine (BASELINE north_star subsystem (1): "warp-level FP32
// FMA with weights resident in shared memory for the narrow networks").
//
// For MLPs whose hidden widths are small (cfg1 1-20-20-1, cfg2 1-64x4-1) the per-layer GEMMs of
// a gradient evaluation are microseconds of work each, so a launch per layer operation is bound
// by launch latency, not by the FP32 pipes.  Here ONE kernel runs whole leapfrog steps
// (forward pass + gradient computation) for every chain:
//
//   * the data rows are cut into nblk row blocks of rb rows (a function of the per-chain problem
//     only); a thread-block cluster of nc CTAs per chain holds them, bpc consecutive blocks per
//     CTA (nc and bpc are a launch choice that never changes a result);
//   * every CTA keeps ALL the chain's weights and its rows' activations in shared memory;
//   * forward, output residual, input-gradient chain and the weight gradient restricted
//     to the active entries (last sentence) run on the FP32 pipes out of shared memory
//     (4 x 4 register tiles, float4 operand loads; compile-time shapes when every hidden layer
//     has the same width HW);
//   * the weight gradient of each row block goes, compacted through the slot map, straight into
//     the shared memory of the CTA that owns that slice of the k-vector (st.shared::cluster); after
//     a cluster barrier CTA r sums its slice over the nblk blocks in block order, adds
//     the prior, applies the kick / drift of the leapfrog step (Q2), and writes
//     the new theta into every CTA's resident weights (st.shared::cluster) - consecutive steps
//     never leave the chip;
//   * a second cluster barrier publishes the new weights; the next step starts.
//
// Every sum over data rows is a fixed function of (rb, nblk): a chain's results are bitwise the
// same for any cluster size, blocks per CTA, or number of chains in the batch.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace hmc {
namespace nw {

constexpr int NT = 256;     // threads per CTA: a 16 x 16 grid of 4 x 4 output tiles
constexpr int MAXL = 8;     // linear layers (hidden + output)
constexpr int TILE = 64;    // rows / columns covered by one pass of the thread grid
constexpr int NBMAX = 32;   // row blocks per chain
constexpr int NCMAX = 16;   // largest cluster (non-portable size, opted in at setup)

struct NarrowArgs {
  int nl;                     // linear layers; layer nl-1 is the output layer (width 1, identity)
  int width[MAXL + 1];        // width[0] = d_in .. width[nl] = 1
  int act[MAXL];              // ACT_TANH / ACT_ID for hidden layers
  int64_t w_off[MAXL];        // flat offsets of W_l [n_out x n_in] row-major
  int64_t b_off[MAXL];        // flat offset of b_l, -1 if the layer has no bias
  int ldw[MAXL];              // padded row length of W_l in shared memory (>= n_in, multiple of 4)
  int sw[MAXL], sb[MAXL];     // shared-memory float offsets of W_l and b_l
  int lda[MAXL];              // padded row length of A_l (A_0 = the input rows), l < nl
  int sa[MAXL];               // shared-memory float offsets of A_l
  int s_r, s_rr, s_gp;        // offsets of R = r / sigma^2 [rows], the residual r [rows] and the block
                              // partials [bpc x kp]
  int kp;                     // padded k (stride of the block partials)
  int s_recv;                 // receive buffer [nblk x ksp] of the pushed block partials
  int s_sl, ksp;              // this CTA's k-slice of theta and p, resident across steps [2 x ksp]
  int s_y;                    // this CTA's targets y [rows]
  int s_slot;                 // the slot map [P], resident: int16 when k < 32768 (slot16), else int32
  int slot16;
  // grid mode (cooperative launch, every CTA resident; used when a chain's CTAs cannot all be
  // co-resident clusters): the exchanges go through L2 instead of distributed shared memory and
  // the barriers are per-chain counters
  int grid;
  float* xtheta;              // [C][k] the new theta of the step
  float* xpart;               // [C][nc][nblk][ksp] block partials, by owner slice
  double* xsq;                // [C][nblk] sum r^2 per block
  unsigned* xbar;             // [C] barrier counters (zeroed before every launch)
  int dbg;                    // dev experiments (HMC_NW_DBG, -DHMC_DEV only): bit 0 skip weight-gradient
                              // FMAs, 1 skip input-gradient GEMMs, 2 skip forward GEMMs (results wrong)
  int s_red;                  // offset (floats, 8-byte aligned) of the fp64 reduction slots
  int smem_bytes;
  int rb;                     // rows per block (multiple of 4)
  int nblk;                   // row blocks per chain (<= NBMAX)
  int bpc;                    // blocks per CTA
  int nc;                     // CTAs per chain (cluster size), nc * bpc >= nblk
  int l_min;                  // lowest layer with an active entry
  int64_t n;                  // data rows
  const float* x;             // [n x d_in]
  const float* y;             // [n]
  const int32_t* slot;        // [P] k-slot of a flat index or -1
  const int32_t* soff;        // [k] shared-memory float offset of active entry j (its W or b word)
  float inv_s2;               // 1 / sigma^2 (the residual R = (y - f) / sigma^2 in fp32)
};

// ---- cluster / distributed shared memory primitives ----
__device__ __forceinline__ uint32_t rank_in_cluster() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// address of the same shared-memory word in CTA `cta` of the cluster
__device__ __forceinline__ uint32_t map_cta(uint32_t saddr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(cta));
  return r;
}
__device__ __forceinline__ float ld_cluster(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ double ld_cluster_d(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// the resident slot map (int16 entries when every slot fits, else int32); off(f) = the map from
// flat index f on
struct SlotRef {
  const void* p = nullptr;
  int s16 = 0;
  __device__ __forceinline__ int operator[](int i) const {
    return s16 ? (int)static_cast<const int16_t*>(p)[i] : static_cast<const int32_t*>(p)[i];
  }
  __device__ __forceinline__ SlotRef off(int64_t f) const {
    SlotRef r;
    r.p = s16 ? (const void*)(static_cast<const int16_t*>(p) + f) : (const void*)(static_cast<const int32_t*>(p) + f);
    r.s16 = s16;
    return r;
  }
  __device__ __forceinline__ bool valid() const { return p != nullptr; }
};

__device__ __forceinline__ void st_cluster4(uint32_t addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// Block partials: written locally, gp[b][j] (b = this CTA's row block, stride kp = nc ksp), then
// PUSHED to the CTA that owns slice j / ksp of the k-vector: recv[global block][j mod ksp] there
// (st.shared::cluster.v4 - fire-and-forget remote stores, so no CTA waits on a remote load)
struct Push {
  float* gp;      // local partials [bpc x kp]
  int kp;
  int dbg;
  __device__ __forceinline__ void put(int j, int b_local, float v) const { gp[b_local * kp + j] = v; }
};

#ifdef HMC_DEV
// dev build: clock cycles per phase, thread 0 of CTA 0 of chain 0 (hmc_debug_nw_profile)
__device__ unsigned long long g_nwprof[10];
#define NW_T(i)                                                              \
  if (blockIdx.x == 0 && threadIdx.x == 0) {                                 \
    const long long t_ = clock64();                                          \
    g_nwprof[i] += (unsigned long long)(t_ - nw_t0);                         \
    nw_t0 = t_;                                                              \
  }
#else
#define NW_T(i)
#endif

// grid mode: barrier of the nc CTAs of one chain (monotonic counter; target = nc x barrier count)
__device__ __forceinline__ void chain_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

__device__ __forceinline__ float nw_act(int act, float z) { return act == ACT_TANH ? tanh_acc(z) : z; }
__device__ __forceinline__ float nw_dact(int act, float a) { return act == ACT_TANH ? fmaf(-a, a, 1.f) : 1.f; }

// The three shared-memory GEMMs of a layer.  Template arguments: compile-time sizes (0 = the
// runtime argument) and leading dimensions LD (0 = runtime); the operand loads of the next K chunk
// are issued before the FMAs of the current one (one chunk in flight, so the ~30-cycle shared
// memory latency overlaps the 64 FMAs of a chunk even with two warps per scheduler).
#define NW_FMA_4x4_KMAJOR(acc, a, w)                        \
  _Pragma("unroll") for (int j = 0; j < 4; ++j)             \
  _Pragma("unroll") for (int m = 0; m < 4; ++m) {           \
    acc[j][m] = fmaf(a[j].x, w[m].x, acc[j][m]);            \
    acc[j][m] = fmaf(a[j].y, w[m].y, acc[j][m]);            \
    acc[j][m] = fmaf(a[j].z, w[m].z, acc[j][m]);            \
    acc[j][m] = fmaf(a[j].w, w[m].w, acc[j][m]);            \
  }

// A_out[r][o] = act(b[o] + sum_i A_in[r][i] W[o][i]) for r < rows, o < n_out.  Thread (ty, tx):
// rows 4 ty + j, columns tx + 16 m (interleaved, so the 16 W rows a warp reads per instruction
// fall in distinct bank groups); K in chunks of 4 (float4 loads of both operands).
template <int KC, int NC, int LI, int LW, int LO>
__device__ __forceinline__ void fwd_layer(const float* __restrict__ Ain, int lda_in_rt, const float* __restrict__ W,
                                          int ldw_rt, int k_rt, const float* __restrict__ b, float* __restrict__ Aout,
                                          int lda_out_rt, int rows, int nout_rt, int act) {
  const int K = KC ? KC : k_rt;
  const int n_out = NC ? NC : nout_rt;
  const int lda_in = LI ? LI : lda_in_rt, ldw = LW ? LW : ldw_rt, lda_out = LO ? LO : lda_out_rt;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  for (int mb = 0; mb < rows; mb += TILE) {
    const int r0 = mb + 4 * ty;
    if (r0 >= rows) continue;
#pragma unroll
    for (int nb = 0; nb < (NC ? NC : 1 << 30); nb += TILE) {
      if (!NC && nb >= n_out) break;
      float acc[4][4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int m = 0; m < 4; ++m) acc[j][m] = 0.f;
      bool om[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) om[m] = (NC && NC % TILE == 0) ? true : (nb + tx + 16 * m < n_out);
      const float* a0 = Ain + r0 * lda_in;
      const float* w0 = W + (nb + tx) * ldw;
      auto load = [&](float4 (&a)[4], float4 (&w)[4], int k) {
#pragma unroll
        for (int j = 0; j < 4; ++j) a[j] = *reinterpret_cast<const float4*>(a0 + j * lda_in + k);
#pragma unroll
        for (int m = 0; m < 4; ++m)
          w[m] = om[m] ? *reinterpret_cast<const float4*>(w0 + 16 * m * ldw + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      };
      float4 a[4], w[4];
      load(a, w, 0);
#pragma unroll(KC ? (KC / 4 <= 16 ? KC / 4 : 8) : 1)
      for (int k = 0; k < K; k += 4) {
        float4 an[4], wn[4];
        const bool more = k + 4 < K;
        if (more) load(an, wn, k + 4);
        NW_FMA_4x4_KMAJOR(acc, a, w)
        if (more) {
#pragma unroll
          for (int j = 0; j < 4; ++j) { a[j] = an[j]; w[j] = wn[j]; }
        }
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        if (!om[m]) continue;
        const int o = nb + tx + 16 * m;
        const float bo = b ? b[o] : 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) Aout[(r0 + j) * lda_out + o] = nw_act(act, acc[j][m] + bo);
      }
    }
  }
}

// Input gradient, in place: A[r][i] <- (sum_o D[r][o] W[o][i]) * act'(A[r][i]) for i < n_in
// (D = delta of the layer above, n_out columns, a multiple of 4).  Thread (ty, tx): rows 4 ty + j,
// columns 4 tx .. 4 tx + 3 (float4 along i).  The caller separates the preceding readers of A
// (the weight gradient) with a barrier; each thread overwrites only its own tile.
template <int OC, int IC, int LD, int LW, int LA>
__device__ __forceinline__ void dgrad_layer(const float* __restrict__ D, int ldd_rt, int nout_rt, const float* __restrict__ W,
                                            int ldw_rt, float* __restrict__ A, int lda_rt, int rows, int nin_rt, int act) {
  const int n_out = OC ? OC : nout_rt;
  const int n_in = IC ? IC : nin_rt;
  const int ldd = LD ? LD : ldd_rt, ldw = LW ? LW : ldw_rt, lda = LA ? LA : lda_rt;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  for (int mb = 0; mb < rows; mb += TILE) {
    const int r0 = mb + 4 * ty;
    if (r0 >= rows) continue;
#pragma unroll
    for (int nb = 0; nb < (IC ? IC : 1 << 30); nb += TILE) {
      if (!IC && nb >= n_in) break;
      const int i0 = nb + 4 * tx;
      if (i0 >= n_in) continue;
      float acc[4][4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int m = 0; m < 4; ++m) acc[j][m] = 0.f;
      const float* d0 = D + r0 * ldd;
      const float* w0 = W + i0;
      auto load = [&](float4 (&d)[4], float4 (&w)[4], int o) {
#pragma unroll
        for (int j = 0; j < 4; ++j) d[j] = *reinterpret_cast<const float4*>(d0 + j * ldd + o);
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = *reinterpret_cast<const float4*>(w0 + (o + q) * ldw);
      };
      float4 d[4], w[4];
      load(d, w, 0);
#pragma unroll(OC ? (OC / 4 <= 16 ? OC / 4 : 8) : 1)
      for (int o = 0; o < n_out; o += 4) {
        float4 dn[4], wn[4];
        const bool more = o + 4 < n_out;
        if (more) load(dn, wn, o + 4);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float dj[4] = {d[j].x, d[j].y, d[j].z, d[j].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[j][0] = fmaf(dj[q], w[q].x, acc[j][0]);
            acc[j][1] = fmaf(dj[q], w[q].y, acc[j][1]);
            acc[j][2] = fmaf(dj[q], w[q].z, acc[j][2]);
            acc[j][3] = fmaf(dj[q], w[q].w, acc[j][3]);
          }
        }
        if (more) {
#pragma unroll
          for (int j = 0; j < 4; ++j) { d[j] = dn[j]; w[j] = wn[j]; }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float4* p = reinterpret_cast<float4*>(A + (r0 + j) * lda + i0);
        const float4 a = *p;
        *p = make_float4(acc[j][0] * nw_dact(act, a.x), acc[j][1] * nw_dact(act, a.y), acc[j][2] * nw_dact(act, a.z),
                         acc[j][3] * nw_dact(act, a.w));
      }
    }
  }
}

// Masked weight gradient of one layer, per row block: for each of the nb blocks of rb rows
// (block b at D + b rb ldd / A + b rb lda), dW[o][i] = sum_r D[r][o] A[r][i] and db[o] =
// sum_r D[r][o], written to that block's partial (push.put) for active entries only.  Thread
// (ty, tx): outputs o = 4 ty + m, inputs i = 4 tx + q (float4 along both operands, two rows in
// flight); the tile's 16 slots are read once and a tile without an active entry is skipped.
template <int OC, int IC, int LD, int LA>
__device__ __forceinline__ void wgrad_layer(const float* __restrict__ D, int ldd_rt, int nout_rt, const float* __restrict__ A,
                                            int lda_rt, int nin_rt, int rb, int nb, const Push& push, SlotRef slot_w,
                                            SlotRef slot_b) {
  const int n_out = OC ? OC : nout_rt;
  const int n_in = IC ? IC : nin_rt;
  const int ldd = LD ? LD : ldd_rt, lda = LA ? LA : lda_rt;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  if (!IC && n_in <= 4) {
    // a narrow input (the first layer): dW[o][i] for i < n_in the way the bias is reduced below -
    // thread (ty, tx) sums rows r = tx (mod 16) of columns 4 ty .. 4 ty + 3 times A[r][i], then a
    // fixed xor-butterfly over the 16 lanes of its half-warp (the 4 x 4 register tiles would
    // leave all but one thread in 16 idle)
    for (int ob = 0; ob < n_out; ob += TILE) {
      const int o0 = ob + 4 * ty;
      for (int i = 0; i < n_in; ++i) {
        int sl[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) sl[m] = o0 + m < n_out ? slot_w[(o0 + m) * n_in + i] : -1;
        for (int b = 0; b < nb; ++b) {
          float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
          if (o0 < n_out)
            for (int r = tx; r < rb; r += 16) {
              const float4 d = *reinterpret_cast<const float4*>(D + (b * rb + r) * ldd + o0);
              const float av = A[(b * rb + r) * lda + i];
              s.x = fmaf(d.x, av, s.x); s.y = fmaf(d.y, av, s.y); s.z = fmaf(d.z, av, s.z); s.w = fmaf(d.w, av, s.w);
            }
#pragma unroll
          for (int off = 8; off > 0; off >>= 1) {
            s.x += __shfl_xor_sync(0xffffffffu, s.x, off);
            s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
            s.z += __shfl_xor_sync(0xffffffffu, s.z, off);
            s.w += __shfl_xor_sync(0xffffffffu, s.w, off);
          }
          if (tx == 0) {
            const float sv[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
            for (int m = 0; m < 4; ++m)
              if (sl[m] >= 0) push.put(sl[m], b, sv[m]);
          }
        }
      }
    }
  } else
#pragma unroll
  for (int ob = 0; ob < (OC ? OC : 1 << 30); ob += TILE) {
    if (!OC && ob >= n_out) break;
    const int o0 = ob + 4 * ty;
#pragma unroll
    for (int ib = 0; ib < (IC ? IC : 1 << 30); ib += TILE) {
      if (!IC && ib >= n_in) break;
      const int i0 = ib + 4 * tx;
      if (o0 < n_out && i0 < n_in) {
        int sl[4][4];
        bool any = false;
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool in = o0 + m < n_out && i0 + q < n_in;
            sl[m][q] = in ? slot_w[(o0 + m) * n_in + i0 + q] : -1;
            any |= sl[m][q] >= 0;
          }
        if (any) {
          for (int b = 0; b < nb; ++b) {
#ifdef HMC_DEV
            if (push.dbg & 1) break;
#endif
            float acc[4][4];
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[m][q] = 0.f;
            const float* dp = D + b * rb * ldd + o0;
            const float* ap = A + b * rb * lda + i0;
            // two register sets of two rows each: set B loads while set A computes and vice versa
            // (static registers - no predicated moves of prefetched values); rb % 4 == 0
            float4 dA0, aA0, dA1, aA1, dB0, aB0, dB1, aB1;
            auto ld2 = [&](float4& d0, float4& a0, float4& d1, float4& a1, int r) {
              d0 = *reinterpret_cast<const float4*>(dp + r * ldd);
              a0 = *reinterpret_cast<const float4*>(ap + r * lda);
              d1 = *reinterpret_cast<const float4*>(dp + (r + 1) * ldd);
              a1 = *reinterpret_cast<const float4*>(ap + (r + 1) * lda);
            };
            auto fma2 = [&](const float4& d0, const float4& a0, const float4& d1, const float4& a1) {
              const float dm0[4] = {d0.x, d0.y, d0.z, d0.w}, dm1[4] = {d1.x, d1.y, d1.z, d1.w};
#pragma unroll
              for (int m = 0; m < 4; ++m) {
                acc[m][0] = fmaf(dm0[m], a0.x, acc[m][0]);
                acc[m][1] = fmaf(dm0[m], a0.y, acc[m][1]);
                acc[m][2] = fmaf(dm0[m], a0.z, acc[m][2]);
                acc[m][3] = fmaf(dm0[m], a0.w, acc[m][3]);
              }
#pragma unroll
              for (int m = 0; m < 4; ++m) {
                acc[m][0] = fmaf(dm1[m], a1.x, acc[m][0]);
                acc[m][1] = fmaf(dm1[m], a1.y, acc[m][1]);
                acc[m][2] = fmaf(dm1[m], a1.z, acc[m][2]);
                acc[m][3] = fmaf(dm1[m], a1.w, acc[m][3]);
              }
            };
            ld2(dA0, aA0, dA1, aA1, 0);
            for (int r = 0; r < rb; r += 4) {
              ld2(dB0, aB0, dB1, aB1, r + 2);
              fma2(dA0, aA0, dA1, aA1);
              if (r + 4 < rb) ld2(dA0, aA0, dA1, aA1, r + 4);
              fma2(dB0, aB0, dB1, aB1);
            }
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (sl[m][q] >= 0) push.put(sl[m][q], b, acc[m][q]);
          }
        }
      }
    }
  }
  if (!slot_b.valid()) return;
  // bias gradient: thread (ty, tx) sums rows r = tx (mod 16) of the block, columns 4 ty .. 4 ty + 3,
  // then a fixed xor-butterfly over the 16 lanes of its half-warp
#pragma unroll
  for (int ob = 0; ob < (OC ? OC : 1 << 30); ob += TILE) {
    if (!OC && ob >= n_out) break;
    const int o0 = ob + 4 * ty;
    int sb[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) sb[m] = o0 + m < n_out ? slot_b[o0 + m] : -1;
    for (int b = 0; b < nb; ++b) {
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      if (o0 < n_out)
        for (int r = tx; r < rb; r += 16) {
          const float4 d = *reinterpret_cast<const float4*>(D + (b * rb + r) * ldd + o0);
          s.x += d.x; s.y += d.y; s.z += d.z; s.w += d.w;
        }
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, off);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
        s.z += __shfl_xor_sync(0xffffffffu, s.z, off);
        s.w += __shfl_xor_sync(0xffffffffu, s.w, off);
      }
      if (tx == 0) {
        const float sv[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
        for (int m = 0; m < 4; ++m)
          if (sb[m] >= 0) push.put(sb[m], b, sv[m]);
      }
    }
  }
}

// One kernel = `nsteps` leapfrog steps of every chain (cluster = chain).  Step modes as in
// k_finalize: 0 = gradient + log pi only (hmc_grad), 1 = inner step (full kick, drift, new
// weights), 2 = closing half kick + log pi.  Steps 0 .. nsteps-2 are mode 1, the last is
// `last_mode`.  Inputs: the chain's parameters in s.Wd (scattered before the launch), the
// working state s.wrk_theta / s.p.  Outputs: s.wrk_grad, s.wrk_theta, s.p, s.Wd, and (modes 0 / 2)
// s.wrk_logp and s.lik.  HW > 0: every hidden layer has width HW (compile-time shapes).
template <int HW>
__global__ void __launch_bounds__(NT, 1) k_narrow(KState s, NarrowArgs a, int nsteps, int last_mode) {
  // padded row length of a hidden layer's activations / weights (host nw_pad: 4 mod 8 floats)
  constexpr int LDH = HW ? ((HW + 3) / 4 * 4) % 8 == 0 ? (HW + 3) / 4 * 4 + 4 : (HW + 3) / 4 * 4 : 0;
  extern __shared__ __align__(16) float sm[];
  const int nc = a.nc;
  const int c = blockIdx.x / nc;
  const uint32_t rank = a.grid ? (uint32_t)(blockIdx.x % nc) : rank_in_cluster();
  unsigned nbar = 0;  // grid mode: barriers passed
  auto sync_chain = [&]() {
    if (a.grid) chain_barrier(a.xbar + c, (unsigned)nc * ++nbar);
    else cluster_barrier();
  };
  const int tid = threadIdx.x;
  const int rows = a.bpc * a.rb;                       // rows of this CTA (blocks rank*bpc ..)
  const int64_t row0 = (int64_t)rank * rows;
  const int nl = a.nl;
  const int out_l = nl - 1;
  float* R = sm + a.s_r;
  float* Rr = sm + a.s_rr;
  float* gp = sm + a.s_gp;    // this CTA's block partials [bpc x kp]
  double* red = reinterpret_cast<double*>(sm + a.s_red);  // [0..NBMAX) sum r^2 per block, [NBMAX] sum theta^2, then 8 scratch
  double* scr = red + NBMAX + 1;

  // ---- resident state: zero the activation region (padding columns stay zero), weights of the
  //      chain, this CTA's data rows ----
  for (int t = tid; t < a.s_r - a.sa[0]; t += NT) sm[a.sa[0] + t] = 0.f;
  const float* Wc = s.Wd + (int64_t)c * s.P;
  for (int l = 0; l < nl; ++l) {
    const int n_in = a.width[l], n_out = a.width[l + 1], ldw = a.ldw[l];
    for (int t = tid; t < n_out * ldw; t += NT) {
      const int o = t / ldw, i = t - o * ldw;
      sm[a.sw[l] + t] = i < n_in ? __ldcg(Wc + a.w_off[l] + (int64_t)o * n_in + i) : 0.f;
    }
    for (int o = tid; o < n_out; o += NT) sm[a.sb[l] + o] = a.b_off[l] >= 0 ? __ldcg(Wc + a.b_off[l] + o) : 0.f;
  }
  __syncthreads();
  SlotRef slot;  // resident slot map
  slot.p = sm + a.s_slot;
  slot.s16 = a.slot16;
  for (int64_t f = tid; f < s.P; f += NT) {
    const int32_t v = __ldg(a.slot + f);
    if (a.slot16) reinterpret_cast<int16_t*>(sm + a.s_slot)[f] = (int16_t)v;
    else reinterpret_cast<int32_t*>(sm + a.s_slot)[f] = v;
  }
  float* ys = sm + a.s_y;
  for (int r = tid; r < rows; r += NT) ys[r] = row0 + r < a.n ? __ldg(a.y + row0 + r) : 0.f;
  {
    const int d_in = a.width[0];
    for (int t = tid; t < rows * d_in; t += NT) {
      const int r = t / d_in, i = t - r * d_in;
      if (row0 + r < a.n) sm[a.sa[0] + r * a.lda[0] + i] = __ldg(a.x + (row0 + r) * d_in + i);
    }
  }
  __syncthreads();

  float* recv = sm + a.s_recv;  // [nblk x ksp] pushed block partials of this CTA's k-slice
  const Push push{gp, a.kp, a.dbg};
  const uint32_t recv_addr = smem_u32(recv);
  const uint32_t red_addr = smem_u32(red);
  const int64_t k = s.k;
  const int64_t ks = a.ksp;  // k-slice of this CTA in the reduction / update (a multiple of 4)
  const int64_t j_lo = (int64_t)rank * ks, j_hi = j_lo + ks < k ? j_lo + ks : k;
  const double eps = s.eps[c];
  const float fe = (float)eps, fh = (float)(0.5 * eps);
  const int my_blocks = (int)((int64_t)a.nblk - (int64_t)rank * a.bpc < a.bpc ? a.nblk - (int)rank * a.bpc : a.bpc);
  // the slice's theta and momentum stay in shared memory across the steps of this launch
  float* sth = sm + a.s_sl;
  float* spp = sth + a.ksp;
  for (int64_t j = j_lo + tid; j < j_hi; j += NT) {
    sth[j - j_lo] = s.wrk_theta[(int64_t)c * k + j];
    spp[j - j_lo] = s.p[(int64_t)c * k + j];
  }

#ifdef HMC_DEV
  long long nw_t0 = clock64();
#endif
  for (int step = 0; step < nsteps; ++step) {
    const int mode = step == nsteps - 1 ? last_mode : 1;
    // ---- forward (hidden layers) ----
    for (int l = 0; l < out_l; ++l) {
#ifdef HMC_DEV
      if (a.dbg & 4) break;
#endif
      const float* bl = a.b_off[l] >= 0 ? sm + a.sb[l] : nullptr;
      const int kr = (a.width[l] + 3) & ~3;
      if (HW && l > 0)
        fwd_layer<HW, HW, LDH, LDH, LDH>(sm + a.sa[l], a.lda[l], sm + a.sw[l], a.ldw[l], kr, bl, sm + a.sa[l + 1],
                                         a.lda[l + 1], rows, HW, a.act[l]);
      else if (HW)
        fwd_layer<0, HW, 0, 0, LDH>(sm + a.sa[l], a.lda[l], sm + a.sw[l], a.ldw[l], kr, bl, sm + a.sa[l + 1], a.lda[l + 1],
                                    rows, HW, a.act[l]);
      else
        fwd_layer<0, 0, 0, 0, 0>(sm + a.sa[l], a.lda[l], sm + a.sw[l], a.ldw[l], kr, bl, sm + a.sa[l + 1], a.lda[l + 1],
                                 rows, a.width[l + 1], a.act[l]);
      __syncthreads();
    }
    NW_T(0)
    // ---- output layer and residual: f = A w + b, R = (y - f) / sigma^2, sum r^2 per
    //      row block ----
    {
      const float* A = sm + a.sa[out_l];
      const int lda = a.lda[out_l], n_in = a.width[out_l];
      const float* w = sm + a.sw[out_l];
      const float b = sm[a.sb[out_l]];
      const int warp = tid >> 5, lane = tid & 31;
      const int kin = (n_in + 3) & ~3;  // (padding columns of A and w are zero)
      // four threads per row: float4 input chunks q, q + 4, ..., then a fixed xor-butterfly
      for (int t = tid; t < 4 * ((rows + 63) / 64) * 64; t += NT) {
        const int r = t >> 2, q = t & 3;
        float f = 0.f;
        if (r < rows)
          for (int i = 4 * q; i < kin; i += 16) {
            const float4 av = *reinterpret_cast<const float4*>(A + r * lda + i);
            const float4 wv = *reinterpret_cast<const float4*>(w + i);
            f = fmaf(av.x, wv.x, f);
            f = fmaf(av.y, wv.y, f);
            f = fmaf(av.z, wv.z, f);
            f = fmaf(av.w, wv.w, f);
          }
        f += __shfl_xor_sync(0xffffffffu, f, 1);
        f += __shfl_xor_sync(0xffffffffu, f, 2);
        if (q == 0 && r < rows) {
          const float rr = row0 + r < a.n ? ys[r] - (f + b) : 0.f;
          Rr[r] = rr;
          R[r] = rr * a.inv_s2;
        }
      }
      __syncthreads();
      if (mode != 1)  // sum r^2 of each block (fp64): a warp per block, lanes over rows, butterfly
        for (int blk = warp; blk < my_blocks; blk += NT / 32) {
          double sq = 0.0;
          for (int r = blk * a.rb + lane; r < (blk + 1) * a.rb; r += 32) sq += (double)Rr[r] * (double)Rr[r];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
          if (lane == 0) {
            red[blk] = sq;
            if (a.grid) __stcg(a.xsq + (int64_t)c * a.nblk + rank * a.bpc + blk, sq);
          }
        }
      // output-layer weight / bias gradient of each block: dw[i] = sum_r R[r] A[r][i], db = sum_r R[r]
      // (four threads per (block, input): rows q, q + 4, ..., then a fixed xor-butterfly)
      const SlotRef slw = slot.off(a.w_off[out_l]);
      const int ntask = (my_blocks > 0 ? my_blocks : 0) * (n_in + 1);
      for (int t = tid; t < 4 * ((ntask + 63) / 64) * 64; t += NT) {
        const int task = t >> 2, q = t & 3;
        const int blk = task / (n_in + 1), i = task - blk * (n_in + 1);
        int sl = -1;
        if (task < ntask && !(i == n_in && a.b_off[out_l] < 0)) sl = i < n_in ? slw[i] : slot[a.b_off[out_l]];
        float g = 0.f;
        if (sl >= 0) {
          const int r0 = blk * a.rb;
          if (i < n_in)
            for (int r = r0 + q; r < r0 + a.rb; r += 4) g = fmaf(R[r], A[r * lda + i], g);
          else
            for (int r = r0 + q; r < r0 + a.rb; r += 4) g += R[r];
        }
        g += __shfl_xor_sync(0xffffffffu, g, 1);
        g += __shfl_xor_sync(0xffffffffu, g, 2);
        if (q == 0 && sl >= 0) push.put(sl, blk, g);
      }
      __syncthreads();
      // delta of the top hidden layer, in place: D[r][i] = R[r] w[i] act'(A[r][i])
      if (a.l_min < out_l) {
        float* Am = sm + a.sa[out_l];
        const int act = a.act[out_l - 1];
        for (int r = warp; r < rows; r += NT / 32)
          for (int i = lane; i < n_in; i += 32) {
            const float av = Am[r * lda + i];
            Am[r * lda + i] = R[r] * w[i] * nw_dact(act, av);
          }
      }
      __syncthreads();
    }
    NW_T(1)
    // ---- backward through the hidden layers: weight gradient of layer l per row block (delta in
    //      A_{l+1}), then the input gradient into A_l (in place) ----
    for (int l = out_l - 1; l >= a.l_min; --l) {
      const float* D = sm + a.sa[l + 1];
      const float* Ai = sm + a.sa[l];
      const SlotRef slw = slot.off(a.w_off[l]);
      const SlotRef slb = a.b_off[l] >= 0 ? slot.off(a.b_off[l]) : SlotRef();
      const int nbk = my_blocks > 0 ? my_blocks : 0;
      NW_T(7)
      if (HW && l > 0)
        wgrad_layer<HW, HW, LDH, LDH>(D, a.lda[l + 1], HW, Ai, a.lda[l], HW, a.rb, nbk, push, slw, slb);
      else if (HW)
        wgrad_layer<HW, 0, LDH, 0>(D, a.lda[l + 1], HW, Ai, a.lda[l], a.width[l], a.rb, nbk, push, slw, slb);
      else
        wgrad_layer<0, 0, 0, 0>(D, a.lda[l + 1], a.width[l + 1], Ai, a.lda[l], a.width[l], a.rb, nbk, push, slw, slb);
      __syncthreads();
      NW_T(8)
#ifdef HMC_DEV
      if (a.dbg & 2) continue;
#endif
      if (l > a.l_min) {
        if (HW)
          dgrad_layer<HW, HW, LDH, LDH, LDH>(D, a.lda[l + 1], HW, sm + a.sw[l], a.ldw[l], sm + a.sa[l], a.lda[l], rows, HW,
                                             a.act[l - 1]);
        else
          dgrad_layer<0, 0, 0, 0, 0>(D, a.lda[l + 1], a.width[l + 1], sm + a.sw[l], a.ldw[l], sm + a.sa[l], a.lda[l], rows,
                                     a.width[l], a.act[l - 1]);
        __syncthreads();
      }
    }
    // ---- push: slice q of every local block partial to CTA q ----
    {
      const int nv = a.ksp / 4;
      const int nb = my_blocks > 0 ? my_blocks : 0;
      for (int t = tid; t < nb * nc * nv; t += NT) {
        const int b = t / (nc * nv), rem = t - b * nc * nv, q = rem / nv, u = rem - q * nv;
        const float4 v = *reinterpret_cast<const float4*>(gp + b * a.kp + q * a.ksp + 4 * u);
        const int gb = (int)rank * a.bpc + b;
        if (a.grid)
          __stcg(reinterpret_cast<float4*>(a.xpart + (((int64_t)c * nc + q) * a.nblk + gb) * a.ksp + 4 * u), v);
        else
          st_cluster4(map_cta(recv_addr + 4u * (uint32_t)(gb * a.ksp + 4 * u), (uint32_t)q), v);
      }
    }
    NW_T(2)
    // ---- barrier 1: every block's partial gradient and sum r^2 are complete ----
    sync_chain();
    NW_T(3)
    // ---- k-slice reduction over the row blocks (block order), prior, kick / drift ----
    for (int64_t j = j_lo + tid; j < j_hi; j += NT) {
      // the pushed block partials of entry j, summed in block order
      float gs = 0.f;
      if (a.grid) {
        const float* src = a.xpart + ((int64_t)c * nc + rank) * a.nblk * a.ksp + (j - j_lo);
        for (int b = 0; b < a.nblk; ++b) gs += __ldcg(src + (int64_t)b * a.ksp);
      } else {
        for (int b = 0; b < a.nblk; ++b) gs += recv[b * a.ksp + (j - j_lo)];
      }
      const int64_t t = (int64_t)c * k + j, jj = j - j_lo;
      float th = sth[jj];
      const float g = gs - (float)((double)th * s.inv_sp2);
      float p = spp[jj];
      if (mode == 1) {
        const float im = s.inv_mass ? __ldg(s.inv_mass + j) : 1.f;
        p = fmaf(fe, g, p);
        th = fmaf(fe * im, p, th);
        sth[jj] = th;
        if (step + 1 < nsteps) {  // the new weight, into every CTA's resident copy
          if (a.grid) {
            __stcg(a.xtheta + t, th);
          } else {
            const uint32_t wa = smem_u32(sm + __ldg(a.soff + j));
            for (int q = 0; q < nc; ++q) st_cluster(map_cta(wa, q), th);
          }
        } else {                  // (a later launch reloads the weights from HBM)
          s.Wd[(int64_t)c * s.P + __ldg(s.idx + j)] = th;
        }
      } else if (mode == 2) {
        p = fmaf(fh, g, p);
      }
      spp[jj] = p;
      if (step + 1 == nsteps) {  // the working state the Metropolis kernel reads
        s.wrk_theta[t] = th;
        s.p[t] = p;
        s.wrk_grad[t] = g;
      }
    }
    NW_T(4)
    // ---- barrier 2: new weights visible everywhere; partials free for the next step ----
    sync_chain();
    if (a.grid && mode == 1 && step + 1 < nsteps) {  // the chain's new theta into this CTA's weights
      for (int64_t j = tid; j < k; j += NT) sm[__ldg(a.soff + j)] = __ldcg(a.xtheta + (int64_t)c * k + j);
      __syncthreads();
    }
    NW_T(5)
    if (mode != 1 && rank == 0) {  // log pi, constants dropped (Q7): the chain's sum
                                   // theta^2 over the final working state (fixed tree over k, the same
                                   // for any nc), sum r^2 over the row blocks in block order
      double th2 = 0.0;
      for (int64_t j = tid; j < k; j += NT) {
        const double v = (double)__ldcg(s.wrk_theta + (int64_t)c * k + j);
        th2 += v * v;
      }
      th2 = block_sum_d<NT>(th2, scr);
      if (tid == 0) {
        double sq = 0.0;
        if (a.grid) {
          for (int blk = 0; blk < a.nblk; ++blk) sq += __ldcg(a.xsq + (int64_t)c * a.nblk + blk);
        } else {
          for (int blk = 0; blk < a.nblk; ++blk) sq += ld_cluster_d(map_cta(red_addr + 8u * (uint32_t)(blk % a.bpc), blk / a.bpc));
        }
        s.wrk_logp[c] = -sq * s.inv_2s2 - 0.5 * th2 * s.inv_sp2;
        const_cast<double*>(s.lik)[c] = sq;
      }
    }
    if (mode != 1 && !a.grid) cluster_barrier();  // (the leader's remote reads finish before any CTA exits)
    NW_T(6)
  }
}

// the instantiations: HW = 0 (any widths) or the uniform hidden width
inline const void* narrow_kernel(int hw) {
  switch (hw) {
    case 16: return (const void*)k_narrow<16>;
    case 32: return (const void*)k_narrow<32>;
    case 64: return (const void*)k_narrow<64>;
    case 128: return (const void*)k_narrow<128>;
    default: return (const void*)k_narrow<0>;
  }
}

}  // namespace nw
}  // namespace hmc
