// Masked weight gradient as a sampled dense-dense product (libhmc, sm_100a).
//
// P:257 (last sentence): the subset sampler circumvents "gradient computations for the
// non-influential parameters".  For a hidden layer z = x W^T + b the likelihood part of the
// gradient of an ACTIVE weight is
//     dW[o][i] = sum_r G[r][o] X[r][i]        (G = delta of the layer, X = its input)
//     db[o]    = sum_r G[r][o]
// so only the (o, i) entries of the mask are computed: |mask| x rows FMAs instead of the dense
// n_out x n_in x rows of a GEMM (cfg5: 3.8 % of the entries).  The choice against the dense
// tensor-core GEMM is made per layer by the planner in hmc.cu (DESIGN.md §5 "masked weight
// gradient").
//
// Work split.  A CTA (MW_NT threads) owns one (chain, row segment, task block).  A task is up to
// MW_G active entries of ONE output row o (its bias is the input column i = n_in, a column of
// ones); thread t of the block runs task t over every row of the segment, so its accumulators
// live in registers and every sum has a fixed order (rows in order within the segment, segments
// summed in segment order by k_ksplit_reduce): results do not depend on the batch or the grid.
//
// Data movement.  The segment streams through a ring of MW_NS stages of MW_R rows, filled by
// bulk asynchronous copies (cp.async.bulk, completion on an mbarrier): the G rows as one
// contiguous copy (pitch n_out), the X rows one copy per row into a pitch of n_in + 4 whose
// extra columns hold the ones of the bias.  A lane reads G[r][o] once per row and X[r][i_p] for
// each of its entries (LDS.32): one shared-memory word per FMA plus 1/n.  The host orders tasks
// so that the 32 lanes of a warp have distinct o mod 32 and, entry by entry, distinct i mod 32
// (a bipartite matching per warp and entry position), so those loads are conflict-free
// wavefronts.  MW_NS - 1 stages stay in flight, which covers the HBM latency at 2 CTAs per SM.
#pragma once
#include "common.cuh"

namespace hmc {

constexpr int MW_NT = 512;  // threads per CTA = tasks per task block
constexpr int MW_G = 8;     // active entries per task (one output row)
constexpr int MW_R = 16;    // rows per stage
constexpr int MW_NS = 3;    // stages in the ring
constexpr int MW_MAXW = 256;  // widths this kernel takes (n_in, n_out <= 256, multiples of 4)

struct MwTasks {
  const int32_t* info;  // [T] o | (n << 16): n = positions used (0: an idle lane)
  const int16_t* pi;    // [MW_G][T] input column of position p (n_in = the bias's column of ones,
                        //           n_in + 1 .. n_in + 3 = zero columns of unused positions)
  const int32_t* ps;    // [MW_G][T] k-slot of position p (-1: unused)
  int T;
};

__device__ __forceinline__ uint32_t mw_su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mw_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(mw_su32(dst)),
               "l"(src), "r"(bytes), "r"(mw_su32(bar))
               : "memory");
}
__device__ __forceinline__ void mw_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "MW_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra MW_WAIT_%=;\n"
      "}\n" ::"r"(mw_su32(b)),
      "r"(parity)
      : "memory");
}

inline int mw_xpitch(int n_in) { return n_in + 4; }
inline size_t mw_stage_floats(int n_out, int n_in) { return (size_t)MW_R * (n_out + mw_xpitch(n_in)); }

// grid: (n_seg x n_tb, chains); results to out + seg * out_seg_stride + chain * k + slot
// (n_seg == 1: the k-vector itself).  NO / NI: compile-time n_out / n_in (0: run-time values), so
// the row offsets of the unrolled chunk are immediates of the shared-memory loads.
template <int NO, int NI>
__global__ void __launch_bounds__(MW_NT, 2)
k_wgrad_mask(const float* __restrict__ G, int64_t sG, const float* __restrict__ X, int64_t sX, int64_t rows,
             int n_out_rt, int n_in_rt, int n_seg, int64_t seg_rows, MwTasks tk, float* __restrict__ out,
             int64_t out_seg_stride, int64_t k, int sq) {
  extern __shared__ __align__(128) float mw_smem[];
  __shared__ __align__(8) uint64_t full[MW_NS];
  const int n_out = NO ? NO : n_out_rt;
  const int n_in = NI ? NI : n_in_rt;
  const int xp = n_in + 4;
  const int tid = threadIdx.x, lane = tid & 31;
  const int c = blockIdx.y;
  const int seg = blockIdx.x % n_seg, tb = blockIdx.x / n_seg;
  const int r_beg = (int)(seg * seg_rows);  // (rows per chain < 2^31)
  const int r_end = (int)min(rows, (int64_t)r_beg + seg_rows);
  const int stage = MW_R * (n_out + xp);
  const float* Gc = G + (int64_t)c * sG;
  const float* Xc = X + (int64_t)c * sX;
  const int nchunk = (r_end - r_beg + MW_R - 1) / MW_R;

  // X pad columns: n_in = the ones of the bias, n_in + 1 .. n_in + 3 = zeros (positions without
  // an entry); never written by the copies
  for (int j = tid; j < MW_NS * MW_R; j += MW_NT) {
    float* xrow = mw_smem + (j / MW_R) * stage + MW_R * n_out + (j % MW_R) * xp;
    xrow[n_in] = 1.f;
    xrow[n_in + 1] = 0.f;
    xrow[n_in + 2] = 0.f;
    xrow[n_in + 3] = 0.f;
  }
  auto issue = [&](int ch) {  // (one thread) rows of chunk ch into its stage
    const int s = ch % MW_NS;
    const int r0 = r_beg + ch * MW_R;
    const int nr = min(MW_R, r_end - r0);
    float* gs = mw_smem + s * stage;
    float* xs = gs + MW_R * n_out;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mw_su32(&full[s])),
                 "r"((uint32_t)(nr * (n_out + n_in) * 4))
                 : "memory");
    mw_bulk(gs, Gc + (int64_t)r0 * n_out, (uint32_t)(nr * n_out * 4), &full[s]);
    for (int q = 0; q < nr; ++q) mw_bulk(xs + q * xp, Xc + (int64_t)(r0 + q) * n_in, (uint32_t)(n_in * 4), &full[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < MW_NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mw_su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int ch = 0; ch < min(MW_NS, nchunk); ++ch) issue(ch);

  // this thread's task; nw = the warp's largest entry count (lanes with fewer read the zeros)
  const int t = tb * MW_NT + tid;
  int o = 0, n = 0;
  if (t < tk.T) {
    const int32_t inf = tk.info[t];
    o = inf & 0xffff;
    n = inf >> 16;
  }
  const int nw = __reduce_max_sync(0xffffffffu, n);
  int ci[MW_G];  // (positions without an entry hold a zero column)
#pragma unroll
  for (int p = 0; p < MW_G; ++p) ci[p] = (p < nw && t < tk.T) ? (int)tk.pi[p * tk.T + t] : n_in + 1;
  float acc[MW_G];
#pragma unroll
  for (int p = 0; p < MW_G; ++p) acc[p] = 0.f;

  for (int ch = 0; ch < nchunk; ++ch) {
    const int s = ch % MW_NS;
    if (lane == 0) mw_wait(&full[s], (uint32_t)((ch / MW_NS) & 1));
    __syncwarp();
    const float* gs = mw_smem + s * stage + o;
    const float* xs = mw_smem + s * stage + MW_R * n_out;
    const int nr = min(MW_R, r_end - r_beg - ch * MW_R);
    if (nw > 0) {
      if (sq) {  // sensitivity mode (hmc_sensitivity): sums of G^2 X^2 and of G^2
        for (int r = 0; r < nr; ++r) {
          float g = gs[r * n_out];
          g *= g;
#pragma unroll
          for (int p = 0; p < MW_G; ++p)
            if (p < nw) {
              const float xv = xs[r * xp + ci[p]];
              acc[p] = fmaf(g, xv * xv, acc[p]);
            }
        }
      } else if (nr == MW_R) {
        const float* xq[MW_G];
#pragma unroll
        for (int p = 0; p < MW_G; ++p) xq[p] = xs + ci[p];
#pragma unroll
        for (int r = 0; r < MW_R; ++r) {
          const float g = gs[r * n_out];
#pragma unroll
          for (int p = 0; p < MW_G; ++p)
            if (p < nw) acc[p] = fmaf(g, xq[p][r * xp], acc[p]);
        }
      } else {
        for (int r = 0; r < nr; ++r) {
          const float g = gs[r * n_out];
#pragma unroll
          for (int p = 0; p < MW_G; ++p)
            if (p < nw) acc[p] = fmaf(g, xs[r * xp + ci[p]], acc[p]);
        }
      }
    }
    __syncthreads();  // stage s consumed by every lane
    if (tid == 0 && ch + MW_NS < nchunk) issue(ch + MW_NS);
  }
  if (n > 0) {
    float* oc = out + (int64_t)seg * out_seg_stride + (int64_t)c * k;
#pragma unroll
    for (int p = 0; p < MW_G; ++p)
      if (p < n) {
        const int sl = tk.ps[p * tk.T + t];
        if (sl >= 0) oc[sl] = acc[p];
      }
  }
}

// the instantiation for a layer shape (the widths of SURVEY §8 configs compile-time; any other
// shape with the run-time one)
using MwKernel = void (*)(const float*, int64_t, const float*, int64_t, int64_t, int, int, int, int64_t, MwTasks,
                          float*, int64_t, int64_t, int);
inline MwKernel mw_kernel(int n_out, int n_in) {
  if (n_out == 256 && n_in == 256) return k_wgrad_mask<256, 256>;
  if (n_out == 128 && n_in == 128) return k_wgrad_mask<128, 128>;
  if (n_out == 128 && n_in == 100) return k_wgrad_mask<128, 100>;
  if (n_out == 100 && n_in == 128) return k_wgrad_mask<100, 128>;
  if (n_out == 64 && n_in == 64) return k_wgrad_mask<64, 64>;
  return k_wgrad_mask<0, 0>;
}

inline size_t mw_smem_bytes(int n_out, int n_in) { return (size_t)MW_NS * mw_stage_floats(n_out, n_in) * sizeof(float); }

}  // namespace hmc
