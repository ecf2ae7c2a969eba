// tau-partition of the parameters by sensitivity on the GPU (libhmc).
//
// PAPER.md eqn:threshold and §3.2: rank the parameters by S_i^2 (largest
// first), form the cumulative fraction c_N = sum_{rank <= N} S^2 / sum S^2, pick N^ and keep the
// N^ most sensitive parameters stochastic (Theta_s).  Reading ("tau rule"):
//   rule 0 ("ge", the text): N^ = min{N : c_N >= tau}   (tau compared with a 1e-15 relative slack)
//   rule 1 ("le", the equation as printed): N^ = max{N : c_N <= tau}
// Ties in S^2 are ranked by ascending flat index.
//
// Steps (all deterministic):
//   1. (key, index) pairs, key = S^2 (>= 0), sorted by (key desc, index asc) with a bitonic
//      network over the next power of two (padding sorts last) - a total order, no stability
//      needed;
//   2. the ranked running sum in fp64, left to right (one thread: the oracle's cumsum order, so
//      the threshold decision is taken on identical values; P <= a few million, once per run);
//   3. N^ from c_N = prefix / total (atomicMin / atomicMax: order independent);
//   4. the N^ selected indices in ascending order: flags at their flat positions, then a fixed-
//      order compaction (the same chunked scan on the flags).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace hmc {
namespace part {

constexpr int CH = 1024;  // prefix-sum chunk

// pad with key -1 (sorts after every S^2 >= 0) and index INT_MAX
__global__ void k_init(const double* __restrict__ s2, int64_t P, int64_t n2, double* __restrict__ key,
                       int32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = i < P ? fabs(s2[i]) : -1.0;
    idx[i] = i < P ? (int32_t)i : 0x7fffffff;
  }
}

// a before b in the ranking: larger key first, then smaller index
__device__ __forceinline__ bool before(double ka, int32_t ia, double kb, int32_t ib) {
  return ka > kb || (ka == kb && ia < ib);
}

// one compare-exchange stage (j) of the bitonic merge of size k
__global__ void k_bitonic(double* __restrict__ key, int32_t* __restrict__ idx, int64_t n2, int64_t j, int64_t k) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = i ^ j;
    if (l <= i) continue;
    const bool up = (i & k) == 0;  // this subsequence sorted in ranking order
    const double ki = key[i], kl = key[l];
    const int32_t ii = idx[i], il = idx[l];
    const bool swap = up ? before(kl, il, ki, ii) : before(ki, ii, kl, il);
    if (swap) {
      key[i] = kl; key[l] = ki;
      idx[i] = il; idx[l] = ii;
    }
  }
}

// the ranked running sum, left to right in one thread (the oracle's cumsum order: the threshold
// decision is taken on the same fp64 values); prefix[i] = sum of the first i + 1 ranked values
__global__ void k_prefix_seq(const double* __restrict__ key, int64_t P, double* __restrict__ prefix) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double s = 0.0;
  for (int64_t i = 0; i < P; ++i) {
    s += key[i];
    prefix[i] = s;
  }
}
// N^ from the prefix sums: c_N = prefix[N-1] / prefix[P-1]
__global__ void k_nhat_seq(const double* __restrict__ prefix, int64_t P, double tau, int rule,
                           unsigned long long* __restrict__ res) {
  const double tot = prefix[P - 1];
  const double lim = tau * (1.0 - 1e-15);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const double frac = __ddiv_rn(prefix[i], tot);
    if (rule == 0) {
      if (frac >= lim) atomicMin(res, (unsigned long long)(i + 1));
    } else if (frac <= tau) {
      atomicMax(res + 1, (unsigned long long)(i + 1));
    }
  }
}

__global__ void k_flags(const int32_t* __restrict__ idx, int64_t nsel, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nsel; i += (int64_t)gridDim.x * blockDim.x)
    flag[idx[i]] = 1;
}
// fixed-order compaction of the flagged positions (chunk counts -> offsets -> sequential write)
__global__ void k_flag_count(const int32_t* __restrict__ flag, int64_t P, int64_t* __restrict__ cnt, int64_t nch) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nch; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = 0;
    const int64_t e = (c + 1) * CH < P ? (c + 1) * CH : P;
    for (int64_t i = c * CH; i < e; ++i) s += flag[i];
    cnt[c] = s;
  }
}
__global__ void k_count_scan(int64_t* __restrict__ cnt, int64_t nch) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int64_t run = 0;
  for (int64_t c = 0; c < nch; ++c) {
    const int64_t t = cnt[c];
    cnt[c] = run;
    run += t;
  }
  cnt[nch] = run;
}
__global__ void k_compact(const int32_t* __restrict__ flag, int64_t P, const int64_t* __restrict__ cnt, int64_t nch,
                          int32_t* __restrict__ out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nch; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = cnt[c];
    const int64_t e = (c + 1) * CH < P ? (c + 1) * CH : P;
    for (int64_t i = c * CH; i < e; ++i)
      if (flag[i]) out[o++] = (int32_t)i;
  }
}

}  // namespace part
}  // namespace hmc
