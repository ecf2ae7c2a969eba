// libhmc: C-ABI implementation (include/hmc.h) of the VI-informed subset HMC hot path on B200.
//
// A gradient evaluation is a fixed sequence of kernels on the context's stream:
//   scatter theta_s -> dense per-chain parameters
//   forward  : layer GEMMs + fused bias/activation epilogue, output layer + residual^2 reduction
//   backward : input-gradient GEMMs with fused act' epilogue, weight-gradient GEMMs restricted
//              to the mask and compacted into the k-vector (P:257 last sentence)
//   [DATA mode: NCCL all-reduce of the likelihood sums]
//   finalize : prior, log pi in fp64, leapfrog kick/drift
// A trajectory = momentum + L such steps + Metropolis, captured as ONE CUDA graph.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <array>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../../include/hmc.h"
#include "gemm_simt.cuh"
#include "kernels.cuh"
#include "masked_wgrad.cuh"
#include "narrow.cuh"
#include "partition.cuh"
#include "tc_gemm.cuh"

using namespace hmc;

static thread_local std::string g_err;

// NVTX range around every public call (SURVEY §5 tracing; header-only NVTX, a no-op unless a tool
// such as Nsight Systems is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

namespace {

struct LayerInfo {
  int net = 0, l = 0, n_in = 0, n_out = 0, act = 0;
  bool bias = false, any_active = false;
  int64_t w_off = 0, b_off = -1, rows = 0;
  bool tc_w = false;          // weights kept as tf32 hi/lo planes for the tensor-core engine
  bool planes_only = false;   // ... and only there: the leapfrog scatter skips the dense copy
  bool bias_active = false;
  int64_t q_off = 0;           // offset of this layer's weights in the hi/lo planes
  int64_t g_off = -1;          // offset of this layer's [n_out x ceil(n_in/32)] group masks (d_gmask)
  int64_t ws_lo = 0, ws_hi = 0; // k-slot range of this layer's active weights
  int ksplit = 1;               // K split of its tensor-core weight-gradient GEMM
  // masked weight gradient (masked_wgrad.cuh) instead of the dense GEMM: task list, row segments,
  // task blocks, the k-slot range of the layer's active weights and bias
  bool mwg = false;
  int mw_seg = 1, mw_tb = 1;
  MwTasks mw{};
  int64_t mw_lo = 0, mw_hi = 0, mw_pairs = 0;
  float* A = nullptr;  // [C x rows x n_out] layer output (hidden layers)
  float* D = nullptr;  // [C x rows x n_out] cos(z) for sin layers
};

struct NetInfo {
  std::vector<int> layers;  // indices into ctx->layers
  int l_min = -1;           // lowest layer (position in `layers`) with an active parameter
  int64_t rows = 0;
  const float* input = nullptr;
  int max_w = 0;
  // gradient buffers: with overlapped weight gradients, nrot of them rotate (one per layer of the
  // net, >= 3), so no input-gradient GEMM waits for a weight gradient to release its delta
  static constexpr int MAXROT = 8;
  float* G[MAXROT] = {};
  int nrot = 2;
  float* colsum = nullptr;  // [C x ceil(rows/32) x max_w] fused bias-gradient partials (layer top)
  float* cs[MAXROT] = {};   // per-layer rotation of colsum (cs[i % nrot] = layer i)
  // weight gradients on their own captured stream ws, overlapping the input-gradient chain:
  // evA[i] = delta_i (and its bias partials) ready, evW[i] = wgrad(i) done
  cudaStream_t ws = nullptr;
  cudaStream_t ws2 = nullptr;  // second weight-gradient stream: layers alternate between ws / ws2, so
                               // wgrad(i - 1) need not wait for wgrad(i) (their outputs - k-slot
                               // ranges, partial buffers - are disjoint; colred has a copy per stream)
  float* colred2 = nullptr;
  std::vector<cudaEvent_t> evA, evW;
  bool cs_ready = false;    // colsum holds the partials of the current G
  // the chains this net runs for (POINTS_XC: the branch runs only this rank's chain block) and the
  // per-net views of the chain-indexed state: dense / plane weights and the k-vector gradient of
  // the net's first chain; every other net buffer is allocated for nch chains
  int nch = 0;
  float *wd = nullptr, *whi = nullptr, *wlo = nullptr, *gl = nullptr;
  float* colred = nullptr;       // two-pass column-reduction scratch (own per net: the DeepONet
  float* narrow_part = nullptr;  // nets run on two streams), narrow-input weight-gradient partials
  float* gl_part = nullptr;      // K-split weight-gradient partials
  float* mw_part = nullptr;      // row-segment partials of the masked weight gradient
};

struct DevBuf {
  std::vector<void*> ptrs;
  ~DevBuf() {
    for (void* p : ptrs) cudaFree(p);
  }
};

}  // namespace

struct hmc_ctx {
  int dev = 0, kind = 0, C = 0, mode = 0, rank = 0, world = 1;
  int64_t P = 0, k = 0;
  int64_t n = 0, n_c = 0, n_x = 0, n_global = 0, d_in = 0;
  bool unaligned = false;  // DeepONet with per-pair trunk inputs q[n_c x n_x x d_t] (NEXT-4)
  // DATA mode, POINTS_XB layout: condition block (n_c_loc = n_c / world rows of u) and point block
  // (n_x rows of q) per rank; all n_c conditions x this rank's points in v / R
  bool xb = false;
  int64_t n_c_loc = 0;
  float *xb_recv = nullptr, *xb_full = nullptr, *xb_dB = nullptr, *xb_send = nullptr;
  // DATA mode, POINTS_XC layout: point block per rank for the trunk and the combine, chain block per
  // rank for the branch (all conditions); the branch outputs of all chains (all-gathered), the
  // partial dB of all chains (reduce-scattered), the all-reduced k-gradient (out of place: this
  // rank's gl has zeros in the branch entries of the other ranks' chains)
  bool xc = false;
  float *xc_Ball = nullptr, *xc_dB = nullptr, *gl_red = nullptr;
  double sigma = 1, sigma_p = 1;
  uint64_t seed = 0;
  bool has_b0 = false;
  int64_t b0_off = -1;
  int b0_slot = -1;
  std::vector<LayerInfo> layers;
  NetInfo nets[2];
  int n_nets = 1;
  // device memory
  DevBuf mem;
  float *d_x = nullptr, *d_y = nullptr, *d_u = nullptr, *d_q = nullptr, *d_v = nullptr;
  float* Wd = nullptr;
  float *Whi = nullptr, *Wlo = nullptr;
  int32_t* d_tcpos = nullptr;
  int64_t Ptc = 0;
  int colred_cap = 0;
  int32_t *d_idx = nullptr, *d_slot = nullptr;
  uint32_t* d_gmask = nullptr;  // per-layer 32-column group masks of the slot map (tc WGRAD epilogue)
  int32_t* d_gbase = nullptr;
  // DeepONet (aligned, ROWS): branch and trunk enqueued on two streams inside the graph
  bool two_streams = false;
  bool wgrad_ov = false;  // weight gradients on their own stream per net (any layout but xb / unaligned)
  // K split of the DeepONet dT = R^T B GEMM (dt_ksplit): ks row slabs as extra batch entries, partial
  // products [C x ks x n_x x p] summed in slab order by k_dact_ksplit_reduce
  int dt_ks = 1;
  float* dt_part = nullptr;
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_fork[2] = {nullptr, nullptr}, ev_join[2] = {nullptr, nullptr};
  float* d_inv_mass = nullptr;
  uint32_t* d_chain = nullptr;
  float *cur_theta = nullptr, *cur_grad = nullptr, *wrk_theta = nullptr, *wrk_grad = nullptr, *p = nullptr;
  double *cur_logp = nullptr, *wrk_logp = nullptr, *H0 = nullptr;
  float* gl = nullptr;
  double* lik = nullptr;
  double *part_sq = nullptr, *part_r = nullptr;
  int n_part = 0;
  float* R = nullptr;
  int sq = 0;                    // sensitivity mode (hmc_sensitivity): squared weight-gradient sums
  int colred_chunks = 0;
  double* d_eps = nullptr;   // [C] per-chain step sizes the trajectory graph reads
  double* d_epsbar = nullptr;  // [C] per-chain averaged steps of the last hmc_adapt (eps == 0 uses them)
  double* d_da = nullptr;    // [C x 4] dual-averaging state (NEXT-2)
  bool adapted = false;      // d_epsbar holds hmc_adapt's result
  uint32_t* d_div = nullptr;  // [C] divergent-trajectory counters (hmc_divergences)
  // grow-only device staging of host output buffers (hmc_sample / hmc_adapt with host pointers);
  // every call that stages synchronises before returning, so a buffer is free at the next call
  struct Stage {
    void* p = nullptr;
    size_t cap = 0;
  } stage_samples, stage_acc, stage_dH, stage_eps;
  Rec* d_rec = nullptr;
  uint8_t* tmp_acc = nullptr;
  double* tmp_dH = nullptr;
  // pinned staging
  Rec* h_rec = nullptr;
  double* h_eps = nullptr;
  cudaEvent_t ev_stage = nullptr, ev_in = nullptr, ev_out = nullptr;
  cudaStream_t st = nullptr;
  // graphs
  cudaGraphExec_t grad_exec = nullptr;
  cudaGraphExec_t traj_exec = nullptr;
  int traj_L = -1;
  // comm
  ncclComm_t comm = nullptr;
  bool emulated = false;  // DATA mode without a communicator: the caller performs the exchange
                          // (hmc_debug_data_phase; test hook)
  // live profiling (event nodes inside the trajectory graph)
  struct ProfRec {
    cudaEvent_t a = nullptr, b = nullptr;
    std::string name;
    double flops = 0, bytes = 0;
    int step = -1;
  };
  std::vector<ProfRec> prof;
  bool prof_on = false, prof_armed = false;
  int prof_step = -1;
  void prof_clear() {
    for (auto& r : prof) {
      if (r.a) cudaEventDestroy(r.a);
      if (r.b) cudaEventDestroy(r.b);
    }
    prof.clear();
  }
  // bookkeeping
  int64_t launches = 0;
  int64_t per_body = 0;
  double body_flops = 0, flop_acc = 0;
  std::string err;
  std::string engine;
  TcPlanner tc;
  // narrow-network engine (csrc/narrow.cuh): whole leapfrog steps in one cluster kernel per chain
  bool narrow = false;
  nw::NarrowArgs nwa;
  int nw_hw = 0, nw_clusters = 0;  // template instantiation (uniform hidden width), co-resident clusters
  int32_t* d_soff = nullptr;

  KState kstate() const {
    KState s;
    s.C = C; s.k = k; s.P = P; s.idx = d_idx; s.inv_mass = d_inv_mass; s.chain_ids = d_chain;
    s.Wd = Wd; s.Whi = Whi; s.Wlo = Wlo; s.tcpos = d_tcpos; s.Ptc = Ptc; s.cur_theta = cur_theta; s.cur_grad = cur_grad; s.cur_logp = cur_logp;
    s.wrk_theta = wrk_theta; s.wrk_grad = wrk_grad; s.wrk_logp = wrk_logp; s.p = p; s.H0 = H0;
    s.gl = xc ? gl_red : gl; s.lik = lik; s.inv_2s2 = 1.0 / (2.0 * sigma * sigma); s.inv_sp2 = 1.0 / (sigma_p * sigma_p);
    s.eps = d_eps; s.da = d_da; s.div = d_div; s.rec = d_rec; s.key0 = (uint32_t)(seed & 0xffffffffu); s.key1 = (uint32_t)(seed >> 32);
    return s;
  }
  ~hmc_ctx() {
    prof_clear();
    for (Stage* g : {&stage_samples, &stage_acc, &stage_dH, &stage_eps})
      if (g->p) cudaFree(g->p);
    if (grad_exec) cudaGraphExecDestroy(grad_exec);
    if (traj_exec) cudaGraphExecDestroy(traj_exec);
    if (comm) ncclCommDestroy(comm);
    if (h_rec) cudaFreeHost(h_rec);
    if (h_eps) cudaFreeHost(h_eps);
    if (ev_stage) cudaEventDestroy(ev_stage);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    for (int i = 0; i < 2; ++i) {
      if (ev_fork[i]) cudaEventDestroy(ev_fork[i]);
      if (ev_join[i]) cudaEventDestroy(ev_join[i]);
    }
    if (st2) cudaStreamDestroy(st2);
    for (auto& N : nets) {
      for (auto e : N.evA) cudaEventDestroy(e);
      for (auto e : N.evW) cudaEventDestroy(e);
      if (N.ws) cudaStreamDestroy(N.ws);
      if (N.ws2) cudaStreamDestroy(N.ws2);
    }
    if (st) cudaStreamDestroy(st);
  }
};

// ---------------------------------------------------------------------------------------------
namespace {

struct Fail {
  int code;
};

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      err = std::string(#call) + ": " + cudaGetErrorString(e_);                               \
      throw Fail{e_ == cudaErrorMemoryAllocation ? HMC_E_OOM : HMC_E_CUDA};                   \
    }                                                                                         \
  } while (0)

#define CKN(call)                                                                             \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) {                                                                  \
      err = std::string(#call) + ": " + ncclGetErrorString(r_);                               \
      throw Fail{HMC_E_NCCL};                                                                 \
    }                                                                                         \
  } while (0)

#define CFG(cond, msg)                                                                        \
  do {                                                                                        \
    if (!(cond)) {                                                                            \
      err = std::string("config: ") + (msg);                                                  \
      throw Fail{HMC_E_CONFIG};                                                               \
    }                                                                                         \
  } while (0)

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <typename T>
T* dalloc(hmc_ctx* x, size_t count, std::string& err) {
  void* p = nullptr;
  size_t bytes = count * sizeof(T);
  if (bytes == 0) bytes = 16;
  CK(cudaMalloc(&p, bytes));
  x->mem.ptrs.push_back(p);
  CK(cudaMemset(p, 0, bytes));
  return (T*)p;
}

// copy `count` elements of a host-or-device array to host
template <typename T>
std::vector<T> to_host(const T* src, size_t count, std::string& err) {
  std::vector<T> h(count);
  if (count) CK(cudaMemcpy(h.data(), src, count * sizeof(T), cudaMemcpyDefault));
  return h;
}

int pick_bm(int M, int N) { return (M <= 64 || N <= 64) ? 64 : 128; }

void launch_gemm_simt(hmc_ctx* x, const GemmArgs& a, bool akm, bool bkm, cudaStream_t st) {
  const int bm = pick_bm(a.M, a.N);
  dim3 grid((a.N + bm - 1) / bm, (a.M + bm - 1) / bm, a.batch);
#define GL(BM, AK, BK) gemm_simt_kernel<BM, AK, BK><<<grid, 256, 0, st>>>(a)
  if (bm == 128) {
    if (akm && bkm) GL(128, true, true);
    else if (akm && !bkm) GL(128, true, false);
    else if (!akm && !bkm) GL(128, false, false);
    else GL(128, false, true);
  } else {
    if (akm && bkm) GL(64, true, true);
    else if (akm && !bkm) GL(64, true, false);
    else if (!akm && !bkm) GL(64, false, false);
    else GL(64, false, true);
  }
#undef GL
  x->launches++;
}

GemmArgs gemm_base(int M, int N, int K, int batch) {
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = M; a.N = N; a.K = K; a.batch = batch; a.ones_col = -1; a.epi = EPI_STORE;
  return a;
}

// event pair around one launch while a profiled capture is armed (or always, for "body")
int prof_begin(hmc_ctx* x, cudaStream_t st, bool force = false) {
  if (!(x->prof_armed || (force && x->prof_on))) return -1;
  hmc_ctx::ProfRec r;
  r.step = x->prof_step;
  if (cudaEventCreate(&r.a) != cudaSuccess || cudaEventCreate(&r.b) != cudaSuccess) return -1;
  cudaEventRecordWithFlags(r.a, st, cudaEventRecordExternal);
  x->prof.push_back(r);
  return (int)x->prof.size() - 1;
}

void prof_end(hmc_ctx* x, int id, cudaStream_t st, const std::string& name, double flops, double bytes) {
  if (id < 0) return;
  auto& r = x->prof[id];
  cudaEventRecordWithFlags(r.b, st, cudaEventRecordExternal);
  r.name = name;
  r.flops = flops;
  r.bytes = bytes;
}

// a GEMM the tensor-core engine accepted must launch there: a failure is an error (HMC_E_CUDA),
// never a silent re-run on the SIMT engine
void tc_launch_or_throw(hmc_ctx* x, const GemmArgs& a, bool akm, bool bkm, cudaStream_t st, const char* tag,
                        const PreSplit* pre = nullptr) {
  const cudaError_t e = x->tc.launch(a, akm, bkm, st, pre);
  if (e != cudaSuccess) {
    x->err = std::string("tcgen05 '") + tag + "' GEMM launch failed: " + cudaGetErrorString(e);
    throw Fail{HMC_E_CUDA};
  }
}

// returns true if the tensor-core engine ran it
bool launch_gemm(hmc_ctx* x, const GemmArgs& a_in, bool akm, bool bkm, cudaStream_t st, const char* tag,
                 const PreSplit* pre = nullptr) {
  GemmArgs a = a_in;
  a.sq = x->sq;
  // an input-gradient GEMM of one tile per CTA pair that would hold more than half of the SM pairs
  // while the weight-gradient GEMMs of the layers above run beside it (wgrad_ov): half the pairs,
  // two tiles each - the second tile's loads overlap the first's epilogue, and the SMs left over go
  // to the concurrent GEMMs instead of queueing them (cfg4: 88.2k -> 90.5k evals/s)
  if (a.epi == EPI_DACT && x->wgrad_ov && !a.max_pairs) {
    const int half_sms = std::max(1, x->tc.num_sms / 2), pt = TcPlanner::pair_tiles(a);
    static const bool halve = !(dev_env("HMC_DACT_HALVE") && atoi(dev_env("HMC_DACT_HALVE")) == 0);
    if (halve && pt <= half_sms && 2 * pt > half_sms) a.max_pairs = (pt + 1) / 2;
  }
  const int id = prof_begin(x, st);
  const bool tc = x->tc.accepts(a, akm, bkm, pre);
  if (tc) {
    tc_launch_or_throw(x, a, akm, bkm, st, tag, pre);
    x->launches++;
  } else {
    if (pre && pre->only) {  // the SIMT engine would read a stale dense copy of these weights
      x->err = std::string("tensor-core engine refused a '") + tag + "' GEMM of a planes-only layer";
      throw Fail{HMC_E_STATE};
    }
    launch_gemm_simt(x, a, akm, bkm, st);
  }
  const double flops = 2.0 * a.M * a.N * (double)a.K * a.batch;
  const double bytes = 4.0 * a.batch * ((double)a.M * a.K + (double)a.K * a.N + (double)a.M * a.N);
  x->flop_acc += flops;
  prof_end(x, id, st, std::string(tc ? "tc_" : "simt_") + tag, flops, bytes);
  return tc;
}

bool is_narrow(const LayerInfo& L) { return L.n_in <= 8; }

void launch_fwd_narrow(hmc_ctx* x, const LayerInfo& L, const float* in, int64_t s_in, cudaStream_t st) {
  const NetInfo& N = x->nets[L.net];
  dim3 grid((unsigned)((L.rows + NARROW_ROWS - 1) / NARROW_ROWS), N.nch);
  const float* W = N.wd;
#define FN(DIN_) k_fwd_narrow<DIN_><<<grid, 256, 0, st>>>(in, s_in, L.rows, L.n_out, W, x->P, L.w_off, L.bias ? L.b_off : -1, \
                                                    L.act, L.A, L.act == ACT_SIN ? L.D : nullptr)
  switch (L.n_in) {
    case 1: FN(1); break; case 2: FN(2); break; case 3: FN(3); break; case 4: FN(4); break;
    case 5: FN(5); break; case 6: FN(6); break; case 7: FN(7); break; default: FN(8); break;
  }
#undef FN
  x->launches++;
}

// rows per CTA of the narrow-input weight gradient: the long chunk when it leaves >= 8 CTAs per SM
inline int narrow_wrows(int64_t rows, int nch) {
  return ((rows + NARROW_WROWS - 1) / NARROW_WROWS) * nch >= 8 * 148 ? NARROW_WROWS : NARROW_ROWS;
}

void launch_wgrad_narrow(hmc_ctx* x, const LayerInfo& L, const float* G, const float* in, int64_t s_in,
                         cudaStream_t st) {
  const NetInfo& N = x->nets[L.net];
  const int wrows = narrow_wrows(L.rows, N.nch);
  const int nch = (int)((L.rows + wrows - 1) / wrows);
  dim3 grid(nch, N.nch);
#define WN(DIN_) k_wgrad_narrow_p1<DIN_><<<grid, 256, 0, st>>>(G, L.rows * L.n_out, in, s_in, L.rows, L.n_out, x->nets[L.net].narrow_part, nch, x->sq, wrows)
  switch (L.n_in) {
    case 1: WN(1); break; case 2: WN(2); break; case 3: WN(3); break; case 4: WN(4); break;
    case 5: WN(5); break; case 6: WN(6); break; case 7: WN(7); break; default: WN(8); break;
  }
#undef WN
  k_wgrad_narrow_p2<<<dim3((unsigned)((L.n_out * (L.n_in + 1) + 255) / 256), N.nch), 256, 0, st>>>(
      N.narrow_part, nch, L.n_out, L.n_in, x->d_slot + L.w_off, L.bias ? x->d_slot + L.b_off : nullptr, N.gl, x->k);
  x->launches += 2;
}

inline const float* layer_input(hmc_ctx* x, const NetInfo& N, int i, int64_t* stride) {
  if (i == 0) {
    *stride = 0;
    return N.input;
  }
  const LayerInfo& P = x->layers[N.layers[i - 1]];
  *stride = P.rows * P.n_out;
  return P.A;
}

void enqueue_forward_hidden(hmc_ctx* x, NetInfo& N, int i, cudaStream_t st) {
  LayerInfo& L = x->layers[N.layers[i]];
  int64_t s_in;
  const float* in = layer_input(x, N, i, &s_in);
  if (is_narrow(L)) {
    const int id = prof_begin(x, st);
    launch_fwd_narrow(x, L, in, s_in, st);
    const double fl = 2.0 * N.nch * L.rows * L.n_out * (double)L.n_in;
    x->flop_acc += fl;
    prof_end(x, id, st, "narrow_fwd", fl, 4.0 * N.nch * L.rows * L.n_out);
    return;
  }
  GemmArgs a = gemm_base((int)L.rows, L.n_out, L.n_in, N.nch);
  a.A = in; a.lda = L.n_in; a.sA = s_in;
  a.B = N.wd + L.w_off; a.ldb = L.n_in; a.sB = x->P;
  a.C = L.A; a.ldc = L.n_out; a.sC = L.rows * L.n_out;
  a.epi = EPI_FWD; a.act = L.act;
  if (L.bias) { a.bias = N.wd + L.b_off; a.s_bias = x->P; }
  if (L.act == ACT_SIN) { a.D = L.D; a.ldd = L.n_out; a.sD = L.rows * L.n_out; }
  PreSplit pre;
  if (L.tc_w) {
    pre.hi = N.whi + L.q_off; pre.lo = N.wlo ? N.wlo + L.q_off : nullptr; pre.ld = L.n_in; pre.stride = x->Ptc;
    pre.only = L.planes_only;
  }
  launch_gemm(x, a, true, true, st, "fwd", L.tc_w ? &pre : nullptr);
}

// backward through layers i = top .. l_min of a net; G of layer `top` is in N.G[cur]
void enqueue_backward_net(hmc_ctx* x, NetInfo& N, int top, int cur, cudaStream_t ms) {
  // ws: the weight-gradient stream (N.ws, when this net's backward runs with overlap) - wgrad(i)
  // starts when delta_i is ready (evA[i]) and runs beside dgrad(i) and dgrad(i - 1); dgrad(i)
  // writes the gradient / bias-partial buffers last read by wgrad(i + nrot - 1) (never, when nrot covers the net)
  const bool ov = N.ws != nullptr && N.nrot >= 3 && (int)N.evA.size() > top && !x->prof_armed;
  for (int i = top; i >= N.l_min; --i) {
    LayerInfo& L = x->layers[N.layers[i]];
    const float* G = N.G[cur];
    int64_t s_in;
    const float* in = layer_input(x, N, i, &s_in);
    cudaStream_t st = ms;
    const bool alt = ov && N.ws2 && (i & 1);
    float* colred = alt ? N.colred2 : N.colred;
    if (ov) {
      cudaStream_t wsi = alt ? N.ws2 : N.ws;
      cudaEventRecord(N.evA[i], ms);
      cudaStreamWaitEvent(wsi, N.evA[i], 0);
      st = wsi;
    }
    float* cs_i = ov ? N.cs[i % N.nrot] : N.colsum;  // this layer's bias partials
    if (L.any_active && L.mwg) {  // masked weight gradient (entries of the mask only, bias included)
      const int id = prof_begin(x, st);
      const int64_t nchunk = (L.rows + MW_R - 1) / MW_R;
      const int64_t seg_rows = ((nchunk + L.mw_seg - 1) / L.mw_seg) * MW_R;
      float* out = L.mw_seg > 1 ? N.mw_part : N.gl;
      mw_kernel(L.n_out, L.n_in)<<<dim3((unsigned)(L.mw_seg * L.mw_tb), N.nch), MW_NT, mw_smem_bytes(L.n_out, L.n_in), st>>>(
          G, L.rows * L.n_out, in, s_in, L.rows, L.n_out, L.n_in, L.mw_seg, seg_rows, L.mw, out,
          (int64_t)N.nch * x->k, x->k, x->sq);
      x->launches++;
      if (L.mw_seg > 1) {  // fixed-order sum of the row segments' partials
        k_ksplit_reduce<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((L.mw_hi - L.mw_lo + 255) / 256, 256)), N.nch),
                          256, 0, st>>>(N.mw_part, L.mw_seg, (int64_t)N.nch * x->k, x->k, L.mw_lo, L.mw_hi, N.gl);
        x->launches++;
      }
      const double fl = 2.0 * N.nch * L.rows * (double)L.mw_pairs;
      x->flop_acc += fl;
      prof_end(x, id, st, "mask_wgrad", fl, 4.0 * N.nch * L.rows * (double)(L.n_out + L.n_in));
    } else if (L.any_active && is_narrow(L)) {
      const int id = prof_begin(x, st);
      launch_wgrad_narrow(x, L, G, in, s_in, st);
      const double fl = 2.0 * N.nch * L.rows * L.n_out * (double)(L.n_in + 1);
      x->flop_acc += fl;
      prof_end(x, id, st, "narrow_wgrad", fl, 4.0 * N.nch * L.rows * L.n_out);
    } else if (L.any_active) {
      GemmArgs a = gemm_base(L.n_out, L.n_in, (int)L.rows, N.nch);
      a.A = G; a.lda = L.n_out; a.sA = L.rows * L.n_out;
      a.B = in; a.ldb = L.n_in; a.sB = s_in;
      a.epi = EPI_WGRAD;
      a.sq = x->sq;
      a.slot_w = x->d_slot + L.w_off; a.slot_b = L.bias ? x->d_slot + L.b_off : nullptr;
      a.n_in = L.n_in; a.gl = N.gl; a.k = x->k;
      if (L.g_off >= 0) { a.gmask = x->d_gmask + L.g_off; a.gbase = x->d_gbase + L.g_off; a.n_grp = (L.n_in + 31) / 32; }
      if (L.ksplit > 1 && N.gl_part) { a.ksplit = L.ksplit; a.gl_part = N.gl_part; }
      static const bool fuse_bias = !(dev_env("HMC_BIAS_FUSE") && atoi(dev_env("HMC_BIAS_FUSE")) == 0);
      const bool bias_in_gemm = fuse_bias && L.bias_active && N.cs_ready;  // (tcgen05 path only)
      if (bias_in_gemm) {
        a.bcs_nblk = (int)((L.rows + 31) / 32);
        a.bcs = cs_i; a.s_bcs = (int64_t)a.bcs_nblk * L.n_out; a.bcs_slot = x->d_slot + L.b_off;
      }
      const int id = prof_begin(x, st);
      const bool tc = x->tc.accepts(a, false, false);
      if (tc) {
        tc_launch_or_throw(x, a, false, false, st, "wgrad");
        x->launches++;
        if (a.ksplit > 1) {  // fixed-order sum of the splits' partial k-vector entries
          k_ksplit_reduce<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((L.ws_hi - L.ws_lo + 255) / 256, 256)), N.nch),
                            256, 0, st>>>(N.gl_part, a.ksplit, (int64_t)N.nch * x->k, x->k, L.ws_lo, L.ws_hi, N.gl);
          x->launches++;
        }
        x->flop_acc += 2.0 * a.M * a.N * (double)a.K * a.batch;
        prof_end(x, id, st, "tc_wgrad", 2.0 * a.M * a.N * (double)a.K * a.batch,
                 4.0 * a.batch * ((double)a.M * a.K + (double)a.K * a.N));
        if (L.bias_active && !bias_in_gemm) {  // bias gradient = column sums of G (fixed order)
          const int id2 = prof_begin(x, st);
          if (N.cs_ready) {  // partials from the producing GEMM's epilogue
            const int nblk = (int)((L.rows + 31) / 32);
            k_colsum_reduce<<<dim3((unsigned)((L.n_out + 31) / 32), N.nch), 1024, 0, st>>>(
                cs_i, (int64_t)nblk * L.n_out, nblk, L.n_out, x->d_slot + L.b_off, N.gl, x->k);
            x->launches += 1;
          } else {
            const int chunks = (int)((L.rows + COLRED_CH - 1) / COLRED_CH);
            k_colred_p1<<<dim3(chunks, N.nch), 256, 0, st>>>(nullptr, G, L.rows * L.n_out, L.rows, L.n_out,
                                                              colred, chunks, x->sq);
            k_colred_p2<<<N.nch, 256, 0, st>>>(colred, chunks, L.n_out, x->d_slot + L.b_off, nullptr, N.gl, x->k);
            x->launches += 2;
          }
          prof_end(x, id2, st, "bias_grad", 1.0 * N.nch * L.rows * L.n_out, 4.0 * N.nch * L.rows * L.n_out);
        }
      } else {
        if (L.bias) { a.N += 1; a.ones_col = L.n_in; }
        launch_gemm_simt(x, a, false, false, st);
        x->flop_acc += 2.0 * a.M * a.N * (double)a.K * a.batch;
        prof_end(x, id, st, "simt_wgrad", 2.0 * a.M * a.N * (double)a.K * a.batch,
                 4.0 * a.batch * ((double)a.M * a.K + (double)a.K * a.N));
      }
    }
    if (ov) cudaEventRecord(N.evW[i], st);
    if (i > N.l_min) {
      st = ms;
      const int nxt = ov ? (cur + 1) % N.nrot : (cur ^ 1);
      if (ov && i + N.nrot - 1 <= top) cudaStreamWaitEvent(ms, N.evW[i + N.nrot - 1], 0);  // buffers of delta_{i+nrot-1}
      const LayerInfo& Pv = x->layers[N.layers[i - 1]];
      GemmArgs a = gemm_base((int)L.rows, L.n_in, L.n_out, N.nch);
      a.A = G; a.lda = L.n_out; a.sA = L.rows * L.n_out;
      a.B = N.wd + L.w_off; a.ldb = L.n_in; a.sB = x->P;
      a.C = N.G[nxt]; a.ldc = L.n_in; a.sC = L.rows * L.n_in;
      a.epi = EPI_DACT; a.act = Pv.act;
      a.dsrc = (Pv.act == ACT_SIN) ? Pv.D : Pv.A; a.ld_dsrc = Pv.n_out; a.s_dsrc = Pv.rows * Pv.n_out;
      PreSplit pre;
      if (L.tc_w) {
        pre.hi = N.whi + L.q_off; pre.lo = N.wlo ? N.wlo + L.q_off : nullptr; pre.ld = L.n_in; pre.stride = x->Ptc;
        pre.only = L.planes_only;
      }
      float* cs_prev = ov ? N.cs[(i - 1) % N.nrot] : N.colsum;
      if (Pv.bias_active && !Pv.mwg && cs_prev) { a.colsum = cs_prev; a.s_colsum = (int64_t)((Pv.rows + 31) / 32) * Pv.n_out; }
      N.cs_ready = launch_gemm(x, a, true, false, st, "dgrad", L.tc_w ? &pre : nullptr) && a.colsum;
      cur = nxt;
    }
  }
  if (ov) {  // all weight gradients done (stream order on each of ws / ws2)
    cudaStreamWaitEvent(ms, N.evW[N.l_min], 0);
    if (N.ws2 && N.l_min + 1 <= top) cudaStreamWaitEvent(ms, N.evW[N.l_min + 1], 0);
  }
}

// POINTS_XB pieces: the all-gather result xb_recv ([rank][chain][i][k]) ordered
// per chain into xb_full; the combine of all conditions with this rank's points (residual and
// likelihood partials); the partial dB over these points for all conditions, ordered for the
// reduce-scatter (xb_send); dT = R^T B_all (complete locally)
void xb_gather_perm(hmc_ctx* x, cudaStream_t st) {
  const int p = x->layers[x->nets[0].layers.back()].n_out;
  k_xb_gather<<<148 * 4, 256, 0, st>>>(x->xb_recv, x->xb_full, x->C, x->world, x->n_c_loc, p);
  x->launches++;
}

void xb_combine(hmc_ctx* x, cudaStream_t st, const float* Ball = nullptr) {
  const LayerInfo& Tl = x->layers[x->nets[1].layers.back()];
  const int p = Tl.n_out;
  GemmArgs a = gemm_base((int)x->n_c, (int)x->n_x, p, x->C);
  a.A = Ball ? Ball : x->xb_full; a.lda = p; a.sA = x->n_c * p;
  a.B = Tl.A; a.ldb = p; a.sB = x->n_x * p;
  a.C = x->R; a.ldc = x->n_x; a.sC = x->n_c * x->n_x;
  a.epi = EPI_RESID; a.V = x->d_v; a.ldv = x->n_x;
  if (x->has_b0) { a.b0 = x->Wd + x->b0_off; a.s_b0 = x->P; }
  a.inv_s2 = 1.0 / (x->sigma * x->sigma);
  a.part_sq = x->part_sq; a.part_r = x->part_r; a.n_part = x->n_part;
  launch_gemm(x, a, true, true, st, "combine");
}

// K split of dT = R^T B (M = n_x, N = p, K = n_c per chain).  With few query points and many
// conditions (cfg4: 100 x 100 outputs from 1000 rows, 16 chains) the GEMM is one tile per chain
// whose K blocks run serially on 16 of the 74 SM pairs - the longest kernel of the trunk's
// backward chain.  The largest ks <= 8 that divides K, keeps every slab >= 4 K blocks with aligned
// strides and fits all pair tiles x ks in one round of SM pairs; 1 = no split.
int dt_ksplit(const hmc_ctx* x, int M, int N, int K, int batch) {
  if (!x->tc.enabled) return 1;
  GemmArgs a = gemm_base(M, N, K, batch);
  const int half_sms = std::max(1, x->tc.num_sms / 2);
  const int pt = TcPlanner::pair_tiles(a);
  for (int ks = 8; ks >= 2; --ks) {
    if (K % ks || K / ks < 128 || (int64_t)pt * ks > half_sms) continue;
    if (((int64_t)(K / ks) * M) % 4 || ((int64_t)(K / ks) * N) % 4) continue;
    return ks;
  }
  return 1;
}

// dT with the context's K split when the launch is the one it was planned for (operands whose
// chain stride is exactly their K rows); returns whether the bias-gradient column partials of the
// result are in a.colsum (only the unsplit GEMM's epilogue writes them)
bool launch_dT(hmc_ctx* x, const GemmArgs& a, cudaStream_t st) {
  const int ks = x->dt_ks;
  if (ks > 1 && x->dt_part && a.K % ks == 0 && a.sA == (int64_t)a.K * a.lda && a.sB == (int64_t)a.K * a.ldb &&
      a.ldc == a.N && a.sC == (int64_t)a.M * a.N && a.ld_dsrc == a.N && a.s_dsrc == a.sC &&
      a.M == (int)x->n_x && a.K == (int)x->n_c && a.batch == x->C && ks == dt_ksplit(x, a.M, a.N, a.K, a.batch)) {
    GemmArgs b = gemm_base(a.M, a.N, a.K / ks, a.batch * ks);
    b.A = a.A; b.lda = a.lda; b.sA = (int64_t)b.K * a.lda;
    b.B = a.B; b.ldb = a.ldb; b.sB = (int64_t)b.K * a.ldb;
    b.C = x->dt_part; b.ldc = a.N; b.sC = a.sC;
    if (x->tc.accepts(b, false, false)) {
      launch_gemm(x, b, false, false, st, "dT");
      const int64_t MN = (int64_t)a.M * a.N;
      k_dact_ksplit_reduce<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((MN + 255) / 256, 64)), a.batch), 256, 0, st>>>(
          x->dt_part, ks, MN, a.act, a.dsrc, a.dsrc, a.C);
      x->launches++;
      return false;
    }
  }
  return launch_gemm(x, a, false, false, st, "dT") && a.colsum;
}

void xb_dB(hmc_ctx* x, cudaStream_t st, const float* Ball = nullptr, float* out = nullptr) {
  const LayerInfo& Bl = x->layers[x->nets[0].layers.back()];
  const LayerInfo& Tl = x->layers[x->nets[1].layers.back()];
  const int p = Bl.n_out;
  GemmArgs a = gemm_base((int)x->n_c, p, (int)x->n_x, x->C);
  a.A = x->R; a.lda = x->n_x; a.sA = x->n_c * x->n_x;
  a.B = Tl.A; a.ldb = p; a.sB = x->n_x * p;
  a.C = out ? out : x->xb_dB; a.ldc = p; a.sC = x->n_c * p;
  a.epi = EPI_DACT; a.act = Bl.act; a.dsrc = Ball ? Ball : x->xb_full; a.ld_dsrc = p; a.s_dsrc = x->n_c * p;
  launch_gemm(x, a, true, false, st, "dB");
  if (!out) {  // POINTS_XB: the reduce-scatter order
    k_xb_scatter<<<148 * 4, 256, 0, st>>>(x->xb_dB, x->xb_send, x->C, x->world, x->n_c_loc, p);
    x->launches++;
  }
  // bias gradient from the reduce-scattered dB (the partials of this partial dB are not summed)
  x->nets[0].cs_ready = false;
}

void xb_dT(hmc_ctx* x, cudaStream_t st, const float* Ball = nullptr) {
  NetInfo& Nt = x->nets[1];
  const LayerInfo& Tl = x->layers[Nt.layers.back()];
  const int p = Tl.n_out;
  GemmArgs a = gemm_base((int)x->n_x, p, (int)x->n_c, x->C);
  a.A = x->R; a.lda = x->n_x; a.sA = x->n_c * x->n_x;
  a.B = Ball ? Ball : x->xb_full; a.ldb = p; a.sB = x->n_c * p;
  a.C = Nt.G[0]; a.ldc = p; a.sC = x->n_x * p;
  a.epi = EPI_DACT; a.act = Tl.act; a.dsrc = (Tl.act == ACT_SIN) ? Tl.D : Tl.A; a.ld_dsrc = p; a.s_dsrc = x->n_x * p;
  if (Tl.bias_active && Nt.colsum) { a.colsum = Nt.colsum; a.s_colsum = (int64_t)((x->n_x + 31) / 32) * p; }
  Nt.cs_ready = launch_dT(x, a, st);
}

// (single-stream sequences, used by the emulated-exchange phases hmc_debug_data_phase)
void xb_mid(hmc_ctx* x, cudaStream_t st) {
  xb_gather_perm(x, st);
  xb_combine(x, st);
  if (x->nets[0].l_min >= 0) xb_dB(x, st);
}

void xb_back(hmc_ctx* x, cudaStream_t st) {
  NetInfo& Nb = x->nets[0];
  NetInfo& Nt = x->nets[1];
  if (Nt.l_min >= 0) xb_dT(x, st);
  if (Nb.l_min >= 0) enqueue_backward_net(x, Nb, (int)Nb.layers.size() - 1, 0, st);
  if (Nt.l_min >= 0) enqueue_backward_net(x, Nt, (int)Nt.layers.size() - 1, 0, st);
}

// forward + backward of one full-batch gradient evaluation (likelihood part only)
void enqueue_body(hmc_ctx* x, cudaStream_t st) {
  const int C = x->C;
  if (x->kind == HMC_MLP) {
    NetInfo& N = x->nets[0];
    const int nl = (int)N.layers.size();
    for (int i = 0; i < nl - 1; ++i) enqueue_forward_hidden(x, N, i, st);
    LayerInfo& O = x->layers[N.layers[nl - 1]];
    int64_t s_in;
    const float* in = layer_input(x, N, nl - 1, &s_in);
    // one pass over the output layer's input: forward, residual, likelihood partials, output-layer
    // gradient partials and the rank-1 input gradient (k_out_fused), when its conditions hold
    const bool back = nl - 1 > N.l_min;
    const int pv_act = back ? x->layers[N.layers[nl - 2]].act : ACT_ID;
    if (!x->sq && N.l_min >= 0 && O.n_in <= 256 && (pv_act == ACT_TANH || pv_act == ACT_ID) &&
        !(dev_env("HMC_OUT_FUSED") && atoi(dev_env("HMC_OUT_FUSED")) == 0)) {
      const int id = prof_begin(x, st);
      dim3 grid((unsigned)x->colred_chunks, C);
      float* G = back ? N.G[0] : nullptr;
      // bias partials of layer nl - 2 into the buffer enqueue_backward_net hands its weight gradient
      const int top = nl - 2;
      const bool ov = N.ws != nullptr && N.nrot >= 3 && (int)N.evA.size() > top && !x->prof_armed;
      float* cs = back && x->layers[N.layers[top]].bias_active ? (ov ? N.cs[top % N.nrot] : N.colsum) : nullptr;
      const int64_t s_cs = (int64_t)((O.rows + 31) / 32) * O.n_in;
#define OF(MO_) k_out_fused<MO_><<<grid, 256, 0, st>>>(in, s_in, O.n_in, O.rows, x->Wd, x->P, O.w_off, O.b_off, x->d_y, \
                                                      x->R, 1.0 / (x->sigma * x->sigma), x->part_sq, x->n_part,       \
                                                      N.colred, x->colred_chunks, G, pv_act, cs, s_cs)
      if (O.n_in <= 32) OF(1);
      else if (O.n_in <= 64) OF(2);
      else if (O.n_in <= 128) OF(4);
      else OF(8);
#undef OF
      x->launches++;
      const double fl = 2.0 * C * O.rows * O.n_in * (back ? 3.0 : 2.0);
      x->flop_acc += fl;
      prof_end(x, id, st, "out_fused", fl, 4.0 * C * O.rows * O.n_in * (back ? 2.0 : 1.0));
      if (O.any_active) {
        k_colred_p2<<<C, 256, 0, st>>>(N.colred, x->colred_chunks, O.n_in, x->d_slot + O.w_off,
                                       O.bias ? x->d_slot + O.b_off : nullptr, x->gl, x->k);
        x->launches++;
      }
      if (back) {
        N.cs_ready = cs != nullptr;
        enqueue_backward_net(x, N, nl - 2, 0, st);
      }
      return;
    }
    {
      const int id = prof_begin(x, st);
      dim3 grid(x->n_part, C);
      k_out_fwd<<<grid, 256, O.n_in * sizeof(float), st>>>(in, s_in, O.n_in, O.rows, x->Wd, x->P, O.w_off,
                                                           O.b_off, x->d_y, x->R, 1.0 / (x->sigma * x->sigma),
                                                           x->part_sq, x->n_part);
      x->launches++;
      x->flop_acc += 2.0 * C * O.rows * O.n_in;
      prof_end(x, id, st, "out_fwd", 2.0 * C * O.rows * O.n_in, 4.0 * C * O.rows * (O.n_in + 1));
    }
    if (x->sq) {  // sensitivity mode: dF/dF = 1 for every datum (output seed, no residual)
      k_fill<<<148 * 4, 256, 0, st>>>(x->R, (int64_t)C * O.rows, 1.f);
      x->launches++;
    }
    if (N.l_min < 0) return;
    if (O.any_active) {
      dim3 g1(x->colred_chunks, C);
      k_colred_p1<<<g1, 256, 0, st>>>(x->R, in, s_in, O.rows, O.n_in, N.colred, x->colred_chunks, x->sq);
      k_colred_p2<<<C, 256, 0, st>>>(N.colred, x->colred_chunks, O.n_in, x->d_slot + O.w_off,
                                     O.bias ? x->d_slot + O.b_off : nullptr, x->gl, x->k);
      x->launches += 2;
    }
    if (nl - 1 > N.l_min) {
      const LayerInfo& Pv = x->layers[N.layers[nl - 2]];
      const int64_t total = (int64_t)C * Pv.rows * Pv.n_out;
      const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
      N.cs_ready = false;
      k_rank1_dact<<<blocks, 256, 0, st>>>(x->R, x->Wd, x->P, O.w_off, Pv.A, Pv.D, Pv.act, Pv.rows, Pv.n_out,
                                           C, N.G[0]);
      x->launches++;
      enqueue_backward_net(x, N, nl - 2, 0, st);
    }
    return;
  }
  // ---- DeepONet (factored over unique branch / trunk inputs, Q16) ----
  // (two_streams: the branch net's kernels go to a second captured stream, so the short branch
  // GEMMs fill the trunk GEMMs' last waves; fork / join through events)
  // (the profiled step - prof_armed - runs on one stream, so each kernel is timed alone)
  const bool two = x->two_streams && !x->unaligned && !x->prof_armed;
  cudaStream_t sb = two ? x->st2 : st;
  auto fork = [&](int i) {
    if (!two) return;
    cudaEventRecord(x->ev_fork[i], st);
    cudaStreamWaitEvent(sb, x->ev_fork[i], 0);
  };
  auto join = [&](int i) {
    if (!two) return;
    cudaEventRecord(x->ev_join[i], sb);
    cudaStreamWaitEvent(st, x->ev_join[i], 0);
  };
  NetInfo& Nb = x->nets[0];
  NetInfo& Nt = x->nets[1];
  const LayerInfo& Bl = x->layers[Nb.layers.back()];
  const LayerInfo& Tl = x->layers[Nt.layers.back()];
  const int p = Bl.n_out;
  if (x->xc) {  // POINTS_XC: the branch for this rank's chain block on all conditions (full tiles),
                // all-gathered by chains; combine / dB / dT / trunk for all chains on this rank's
                // points; dB reduce-scattered back to the chain owners.  Exchanges on the branch
                // stream, overlapping the trunk
    std::string& err = x->err;
    const size_t bblk = (size_t)Nb.nch * x->n_c * p;
    fork(0);
    for (int i = 0; i < (int)Nb.layers.size(); ++i) enqueue_forward_hidden(x, Nb, i, sb);
    if (x->comm) {
      CKN(ncclAllGather(Bl.A, x->xc_Ball, bblk, ncclFloat32, x->comm, sb));
    } else {  // exchange = 2 (timing stand-in): the same bytes moved locally
      for (int r = 0; r < x->world; ++r)
        CK(cudaMemcpyAsync(x->xc_Ball + r * bblk, Bl.A, bblk * 4, cudaMemcpyDeviceToDevice, sb));
    }
    for (int i = 0; i < (int)Nt.layers.size(); ++i) enqueue_forward_hidden(x, Nt, i, st);
    join(0);
    xb_combine(x, st, x->xc_Ball);
    fork(1);
    if (Nb.l_min >= 0) {
      xb_dB(x, sb, x->xc_Ball, x->xc_dB);
      if (x->comm)
        CKN(ncclReduceScatter(x->xc_dB, Nb.G[0], bblk, ncclFloat32, ncclSum, x->comm, sb));
      else
        CK(cudaMemcpyAsync(Nb.G[0], x->xc_dB + x->rank * bblk, bblk * 4, cudaMemcpyDeviceToDevice, sb));
      enqueue_backward_net(x, Nb, (int)Nb.layers.size() - 1, 0, sb);
    }
    if (Nt.l_min >= 0) {
      xb_dT(x, st, x->xc_Ball);
      enqueue_backward_net(x, Nt, (int)Nt.layers.size() - 1, 0, st);
    }
    join(1);
    return;
  }
  if (x->xb) {  // POINTS_XB: gather the branch outputs of all conditions, combine with this rank's
                // points, reduce-scatter dB back to the condition owners, dT stays local.  The
                // exchanges run on the branch stream: the all-gather overlaps the trunk forward,
                // the reduce-scatter (and the branch backward after it) the dT GEMM and the trunk
                // backward
    std::string& err = x->err;  // (CKN reports through it)
    const int64_t blk = (int64_t)C * x->n_c_loc * p;
    fork(0);
    for (int i = 0; i < (int)Nb.layers.size(); ++i) enqueue_forward_hidden(x, Nb, i, sb);
    if (x->comm) {
      CKN(ncclAllGather(Bl.A, x->xb_recv, (size_t)blk, ncclFloat32, x->comm, sb));
    } else {  // exchange = 2 (timing stand-in): the same bytes moved locally
      for (int r = 0; r < x->world; ++r)
        CK(cudaMemcpyAsync(x->xb_recv + (size_t)r * blk, Bl.A, (size_t)blk * 4, cudaMemcpyDeviceToDevice, sb));
    }
    xb_gather_perm(x, sb);
    for (int i = 0; i < (int)Nt.layers.size(); ++i) enqueue_forward_hidden(x, Nt, i, st);
    join(0);
    xb_combine(x, st);
    fork(1);
    if (Nb.l_min >= 0) {
      xb_dB(x, sb);
      if (x->comm)
        CKN(ncclReduceScatter(x->xb_send, Nb.G[0], (size_t)blk, ncclFloat32, ncclSum, x->comm, sb));
      else
        CK(cudaMemcpyAsync(Nb.G[0], x->xb_send + (size_t)x->rank * blk, (size_t)blk * 4, cudaMemcpyDeviceToDevice, sb));
      enqueue_backward_net(x, Nb, (int)Nb.layers.size() - 1, 0, sb);
    }
    if (Nt.l_min >= 0) {
      xb_dT(x, st);
      enqueue_backward_net(x, Nt, (int)Nt.layers.size() - 1, 0, st);
    }
    join(1);
    return;
  }
  fork(0);
  for (int i = 0; i < (int)x->nets[0].layers.size(); ++i) enqueue_forward_hidden(x, x->nets[0], i, sb);
  for (int i = 0; i < (int)x->nets[1].layers.size(); ++i) enqueue_forward_hidden(x, x->nets[1], i, st);
  join(0);
  if (x->unaligned) {  // per-pair trunk rows: row-wise combine, then the two output gradients
    k_pair_combine<<<dim3((unsigned)x->n_c, C), 256, p * sizeof(float), st>>>(
        Bl.A, Tl.A, p, x->n_c, x->n_x, x->d_v, x->has_b0 ? x->Wd + x->b0_off : nullptr, x->P,
        1.0 / (x->sigma * x->sigma), x->R, x->part_sq, x->part_r, x->n_part);
    x->launches++;
    x->flop_acc += 2.0 * C * x->n_c * x->n_x * p;
    if (Nb.l_min >= 0) {
      k_pair_dB<<<dim3((unsigned)x->n_c, C), 256, 0, st>>>(x->R, Tl.A, p, x->n_c, x->n_x, Bl.act, Bl.A, Bl.D,
                                                           Nb.G[0]);
      x->launches++;
      Nb.cs_ready = false;
    }
    if (Nt.l_min >= 0) {
      const int64_t total = (int64_t)C * x->n_c * x->n_x * p;
      k_pair_dT<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st>>>(
          x->R, Bl.A, p, x->n_c, x->n_x, C, Tl.act, Tl.A, Tl.D, Nt.G[0]);
      x->launches++;
      Nt.cs_ready = false;
    }
    x->flop_acc += 4.0 * C * x->n_c * x->n_x * p;
    if (Nb.l_min >= 0) enqueue_backward_net(x, Nb, (int)Nb.layers.size() - 1, 0, st);
    if (Nt.l_min >= 0) enqueue_backward_net(x, Nt, (int)Nt.layers.size() - 1, 0, st);
    return;
  }
  {  // combine O = B T^T + b0, residual, R = (V - O)/sigma^2, partial sums
    GemmArgs a = gemm_base((int)x->n_c, (int)x->n_x, p, C);
    a.A = Bl.A; a.lda = p; a.sA = x->n_c * p;
    a.B = Tl.A; a.ldb = p; a.sB = x->n_x * p;
    a.C = x->R; a.ldc = x->n_x; a.sC = x->n_c * x->n_x;
    a.epi = EPI_RESID; a.V = x->d_v; a.ldv = x->n_x;
    if (x->has_b0) { a.b0 = x->Wd + x->b0_off; a.s_b0 = x->P; }
    a.inv_s2 = 1.0 / (x->sigma * x->sigma);
    a.part_sq = x->part_sq; a.part_r = x->part_r; a.n_part = x->n_part;
    launch_gemm(x, a, true, true, st, "combine");
  }
  fork(1);
  // the branch backward (the longer chain) continues on the combine's stream: its dB is launched
  // programmatically behind the combine and gets its SMs before the trunk's dT does
  static const bool swap_bt = !(dev_env("HMC_SWAP_BT") && atoi(dev_env("HMC_SWAP_BT")) == 0);
  cudaStream_t s_br = (two && swap_bt) ? st : sb, s_tr = (two && swap_bt) ? sb : st;
  if (Nb.l_min >= 0) {  // dB = R T, times act' of the branch output layer
    GemmArgs a = gemm_base((int)x->n_c, p, (int)x->n_x, C);
    a.A = x->R; a.lda = x->n_x; a.sA = x->n_c * x->n_x;
    a.B = Tl.A; a.ldb = p; a.sB = x->n_x * p;
    a.C = Nb.G[0]; a.ldc = p; a.sC = x->n_c * p;
    a.epi = EPI_DACT; a.act = Bl.act; a.dsrc = (Bl.act == ACT_SIN) ? Bl.D : Bl.A; a.ld_dsrc = p; a.s_dsrc = x->n_c * p;
    if (Bl.bias_active && Nb.colsum) { a.colsum = Nb.colsum; a.s_colsum = (int64_t)((x->n_c + 31) / 32) * p; }
    if (const char* e = dev_env("HMC_DB_HALVE")) { if (atoi(e) == 0) a.max_pairs = 1 << 20; }  // dev A/B: dB keeps its full grid
    Nb.cs_ready = launch_gemm(x, a, true, false, s_br, "dB") && a.colsum;
  }
  if (Nt.l_min >= 0) {  // dT = R^T B, times act' of the trunk output layer
    GemmArgs a = gemm_base((int)x->n_x, p, (int)x->n_c, C);
    a.A = x->R; a.lda = x->n_x; a.sA = x->n_c * x->n_x;
    a.B = Bl.A; a.ldb = p; a.sB = x->n_c * p;
    a.C = Nt.G[0]; a.ldc = p; a.sC = x->n_x * p;
    a.epi = EPI_DACT; a.act = Tl.act; a.dsrc = (Tl.act == ACT_SIN) ? Tl.D : Tl.A; a.ld_dsrc = p; a.s_dsrc = x->n_x * p;
    if (Tl.bias_active && Nt.colsum) { a.colsum = Nt.colsum; a.s_colsum = (int64_t)((x->n_x + 31) / 32) * p; }
    Nt.cs_ready = launch_dT(x, a, s_tr);
  }
  if (Nb.l_min >= 0) enqueue_backward_net(x, Nb, (int)Nb.layers.size() - 1, 0, s_br);
  if (Nt.l_min >= 0) enqueue_backward_net(x, Nt, (int)Nt.layers.size() - 1, 0, s_tr);
  join(1);
}

void enqueue_reduce(hmc_ctx* x, cudaStream_t st, std::string& err) {
  k_reduce_partials<<<x->C, KT, 0, st>>>(x->part_sq, x->part_r, x->n_part, x->lik, x->gl, x->k, x->b0_slot);
  x->launches++;
  if (x->mode == HMC_MODE_DATA && x->comm) {
    CKN(ncclGroupStart());
    CKN(ncclAllReduce(x->gl, x->xc ? x->gl_red : x->gl, (size_t)(x->C * x->k), ncclFloat32, ncclSum, x->comm, st));
    CKN(ncclAllReduce(x->lik, x->lik, (size_t)x->C, ncclFloat64, ncclSum, x->comm, st));
    CKN(ncclGroupEnd());
  } else if (x->xc && !x->emulated) {  // (timing stand-in)
    CK(cudaMemcpyAsync(x->gl_red, x->gl, (size_t)x->C * x->k * 4, cudaMemcpyDeviceToDevice, st));
  }
}

// body + reduce + finalize for one gradient evaluation inside a trajectory
void enqueue_step(hmc_ctx* x, int mode, cudaStream_t st, std::string& err) {
  const int idb = prof_begin(x, st, true);
  const double f0 = x->flop_acc;
  enqueue_body(x, st);
  x->body_flops = x->flop_acc - f0;
  prof_end(x, idb, st, "body", x->body_flops, 0.0);
  const int idr = prof_begin(x, st);
  enqueue_reduce(x, st, err);
  prof_end(x, idr, st, "reduce", 0.0, 0.0);
  const int idf = prof_begin(x, st);
  if (mode == 1) {
    const int64_t total = (int64_t)x->C * x->k;
    (void)total;
    k_leapfrog<<<dim3((unsigned)std::min<int64_t>((x->k + 255) / 256, 1024), x->C), 256, 0, st>>>(x->kstate());
  } else {
    k_finalize<<<x->C, KT, 0, st>>>(x->kstate(), mode);
  }
  x->launches++;
  prof_end(x, idf, st, "finalize", 0.0, 0.0);
}

// ---- sensitivity step (eqn:sensitivities P:193-197) ----
// Symmetric eigen-decomposition by cyclic Jacobi rotations (host, fp64): A (n x n, row-major,
// destroyed) -> eigenvalues w[n], eigenvectors as the columns of V.  Used on the p x p output
// Gram matrices of the DeepONet branch / trunk (p <= 256).
void jacobi_eig(std::vector<double>& A, int n, std::vector<double>& w, std::vector<double>& V) {
  V.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) (i == j ? diag : off) += A[(size_t)i * n + j] * A[(size_t)i * n + j];
    if (off <= 1e-30 * (diag + 1e-300)) break;
    for (int pp = 0; pp < n - 1; ++pp)
      for (int q = pp + 1; q < n; ++q) {
        const double apq = A[(size_t)pp * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        const double app = A[(size_t)pp * n + pp], aqq = A[(size_t)q * n + q];
        const double th = 0.5 * (aqq - app) / apq;
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < n; ++k) {  // rotate columns pp, q
          const double akp = A[(size_t)k * n + pp], akq = A[(size_t)k * n + q];
          A[(size_t)k * n + pp] = c * akp - sn * akq;
          A[(size_t)k * n + q] = sn * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {  // rotate rows pp, q
          const double apk = A[(size_t)pp * n + k], aqk = A[(size_t)q * n + k];
          A[(size_t)pp * n + k] = c * apk - sn * aqk;
          A[(size_t)q * n + k] = sn * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V[(size_t)k * n + pp], vkq = V[(size_t)k * n + q];
          V[(size_t)k * n + pp] = c * vkp - sn * vkq;
          V[(size_t)k * n + q] = sn * vkp + c * vkq;
        }
      }
  }
  w.resize(n);
  for (int i = 0; i < n; ++i) w[i] = A[(size_t)i * n + i];
}

// Seeds s_m = sqrt(lambda_m) v_m of G = X^T X (X: rows x p, chain 0 of a net's output), so
// that sum_m (s_m . g)^2 = g^T G g for any g (negative rounding eigenvalues clipped to 0)
std::vector<float> gram_seeds(const std::vector<float>& X, int64_t rows, int p) {
  std::vector<double> G((size_t)p * p, 0.0);
  for (int64_t r = 0; r < rows; ++r)
    for (int i = 0; i < p; ++i) {
      const double xi = X[(size_t)r * p + i];
      if (xi == 0.0) continue;
      for (int j = 0; j < p; ++j) G[(size_t)i * p + j] += xi * (double)X[(size_t)r * p + j];
    }
  std::vector<double> w, V;
  jacobi_eig(G, p, w, V);
  std::vector<float> seeds((size_t)p * p);
  for (int m = 0; m < p; ++m) {
    const double sl = std::sqrt(std::max(w[m], 0.0));
    for (int k = 0; k < p; ++k) seeds[(size_t)m * p + k] = (float)(sl * V[(size_t)k * p + m]);
  }
  return seeds;
}

// Sum over data of the squared output gradients, for every parameter and virtual chain, into
// x->gl [C x P] (x was set up with k = P, theta = mu).  MLP: one chain, output seed 1 per
// datum.  DeepONet: chain m seeds the branch with sqrt(l_m) v_m of the trunk Gram matrix and
// the trunk with those of the branch Gram matrix, since sum_x (dF(c,x)/dtheta_branch)^2 =
// g_c^T (T^T T) g_c with g_c = dB(c)/dtheta (and symmetrically for the trunk).
void enqueue_sensitivity(hmc_ctx* x, std::string& err) {
  cudaStream_t st = x->st;
  x->sq = 1;
  if (x->kind == HMC_MLP) {
    enqueue_body(x, st);
    return;
  }
  for (int ni = 0; ni < 2; ++ni) {
    NetInfo& N = x->nets[ni];
    for (int i = 0; i < (int)N.layers.size(); ++i) enqueue_forward_hidden(x, N, i, st);
  }
  NetInfo& Nb = x->nets[0];
  NetInfo& Nt = x->nets[1];
  const LayerInfo& Bl = x->layers[Nb.layers.back()];
  const LayerInfo& Tl = x->layers[Nt.layers.back()];
  const int p = Bl.n_out;
  std::vector<float> hB((size_t)x->n_c * p), hT((size_t)x->n_x * p);
  CK(cudaMemcpyAsync(hB.data(), Bl.A, hB.size() * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hT.data(), Tl.A, hT.size() * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const std::vector<float> sT = gram_seeds(hT, x->n_x, p);  // seeds of the branch reverse pass
  const std::vector<float> sB = gram_seeds(hB, x->n_c, p);  // seeds of the trunk reverse pass
  float* dseed = dalloc<float>(x, (size_t)2 * p * p, err);
  CK(cudaMemcpyAsync(dseed, sT.data(), sT.size() * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dseed + (size_t)p * p, sB.data(), sB.size() * 4, cudaMemcpyHostToDevice, st));
  if (Nb.l_min >= 0) {
    k_seed_top<<<148 * 4, 256, 0, st>>>(Bl.A, Bl.D, Bl.act, dseed, x->n_c, p, x->C, Nb.G[0]);
    Nb.cs_ready = false;
    enqueue_backward_net(x, Nb, (int)Nb.layers.size() - 1, 0, st);
  }
  if (Nt.l_min >= 0) {
    k_seed_top<<<148 * 4, 256, 0, st>>>(Tl.A, Tl.D, Tl.act, dseed + (size_t)p * p, x->n_x, p, x->C, Nt.G[0]);
    Nt.cs_ready = false;
    enqueue_backward_net(x, Nt, (int)Nt.layers.size() - 1, 0, st);
  }
  CK(cudaGetLastError());
}

// Narrow-network engine planning (csrc/narrow.cuh): an MLP whose hidden layers are tanh /
// identity with widths that are multiples of 4 (<= 128) runs whole leapfrog steps in one kernel,
// a cluster of nc CTAs per chain with the weights and the rows' activations resident in shared
// memory.  nc and the rows per CTA depend on the per-chain problem and the device only (batch
// invariance).  Returns false (the per-layer engines run) when the network does not qualify.
int nw_pad(int w) {
  int p = (w + 3) / 4 * 4;
  return (p % 8 == 0) ? p + 4 : p;  // row stride = 4 (mod 8) floats: float4 rows spread over the banks
}

bool nw_layout(hmc_ctx* x, int bpc, int nc, nw::NarrowArgs& a) {
  const NetInfo& N = x->nets[0];
  const int rows = bpc * a.rb;
  int off = 0;
  for (int l = 0; l < a.nl; ++l) {
    const LayerInfo& L = x->layers[N.layers[l]];
    a.ldw[l] = nw_pad(L.n_in);
    a.sw[l] = off;
    off += L.n_out * a.ldw[l];
    a.sb[l] = off;
    off += (L.n_out + 3) / 4 * 4;
  }
  for (int l = 0; l < a.nl; ++l) {
    a.lda[l] = nw_pad(a.width[l]);
    a.sa[l] = off;
    off += rows * a.lda[l];
  }
  a.s_r = off;
  off += (rows + 3) / 4 * 4;
  a.s_rr = off;
  off += (rows + 3) / 4 * 4;
  a.ksp = (int)(((x->k + nc - 1) / nc + 3) / 4 * 4);  // k-slice per CTA (multiple of 4)
  a.kp = nc * a.ksp;
  a.s_gp = off;    // this CTA's block partials [bpc x kp]
  off += bpc * a.kp;
  a.s_recv = off;  // receive buffer: the nblk block partials of this CTA's k-slice
  off += a.nblk * a.ksp;
  a.s_sl = off;
  off += 2 * a.ksp;
  a.s_y = off;
  off += (rows + 3) / 4 * 4;
  a.s_slot = off;
  a.slot16 = x->k < 32768 ? 1 : 0;
  off += (int)((x->P * (a.slot16 ? 2 : 4) + 15) / 16 * 4);
  off = (off + 3) / 4 * 4;
  a.s_red = off;
  off += 2 * (nw::NBMAX + 1 + 8);  // doubles: per-block sum r^2, sum theta^2, block_sum_d scratch
  a.bpc = bpc;
  a.smem_bytes = off * 4;
  return true;
}

// Row blocks (the unit of every sum over data rows, so a function of the problem only):
// rb = max(16, ceil(n / NBMAX)) rounded to 4, nblk = ceil(n / rb).  Cluster size nc and blocks per
// CTA bpc (results do not depend on them): the feasible (shared memory, co-resident cluster)
// choice with the fewest block-times per chain batch, ceil(C / active clusters) x bpc.
bool plan_narrow(hmc_ctx* x, std::string& err) {
  if (x->kind != HMC_MLP || x->mode == HMC_MODE_DATA || (engine_override() != 0 && engine_override() != 3)) return false;
  const NetInfo& N = x->nets[0];
  const int nl = (int)N.layers.size();
  if (nl > nw::MAXL || N.l_min < 0) return false;
  nw::NarrowArgs a;
  memset(&a, 0, sizeof(a));
  a.nl = nl;
  int hw = -1;  // uniform hidden width (template instantiation), 0 = mixed
  for (int l = 0; l < nl; ++l) {
    const LayerInfo& L = x->layers[N.layers[l]];
    if (l < nl - 1 && (L.act == ACT_SIN || L.n_out % 4 != 0 || L.n_out > 128)) return false;
    if (l == 0 && L.n_in > 64) return false;
    if (l < nl - 1) hw = (hw == -1 || hw == L.n_out) ? L.n_out : 0;
    a.width[l] = L.n_in;
    a.width[l + 1] = L.n_out;
    a.act[l] = L.act;
    a.w_off[l] = L.w_off;
    a.b_off[l] = L.bias ? L.b_off : -1;
  }
  if (hw != 16 && hw != 32 && hw != 64 && hw != 128) hw = 0;
  a.l_min = N.l_min;
  a.n = x->n;
  if (const char* e = dev_env("HMC_NW_DBG")) a.dbg = atoi(e);
  int dev = 0, optin = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  int nsm = 148;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const void* fn = nw::narrow_kernel(hw);
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  // Cost of one leapfrog step for the batch (cycles, a model): waves x (64-row passes of the thread
  // grid x the pass time at ~30 % of the FP32 rate + ~8k cycles of exchange and barriers when a
  // chain spans several CTAs; measured)
  double fma_row = 0.0;
  for (int l = 0; l < nl; ++l) fma_row += 3.0 * a.width[l] * a.width[l + 1];
  int wmin = 1 << 30;  // narrowest hidden layer
  for (int l = 1; l < nl; ++l) wmin = std::min(wmin, a.width[l]);
  const double pass = std::max(2000.0, fma_row * nw::TILE / (128.0 * 0.3));
  // (narrow hidden layers, < 32 columns: the thread grid is mostly idle and the per-row work of the
  // weight-gradient K loops dominates, so the cost is the rows per CTA - more CTAs win)
  auto step_cost = [&](int waves, int rows, int nc) {
    if (wmin < 32) return (double)waves * rows;
    return waves * (std::ceil(rows / (double)nw::TILE) * pass + (nc > 1 ? 8000.0 : 0.0));
  };
  double best = 1e30;
  // row-block size (the unit of every sum over rows, so a function of the problem only): 64 rows
  // (one pass of the thread grid) or, for longer data, n / 32 - else the 16-row rule; the larger
  // wins ties
  // (64-row blocks only when the hidden layers fill the 64-column thread grid reasonably: below 32
  // columns most threads idle and the per-block K loops of the weight gradient dominate, so more
  // CTAs on 16-row blocks win - measured on cfg1, 20 wide: 10 vs 14 us per step)
  const int64_t per32 = ((x->n + nw::NBMAX - 1) / nw::NBMAX + 3) / 4 * 4;
  std::vector<int> rbs;
  if (wmin >= 32) rbs.push_back((int)std::max<int64_t>(nw::TILE, per32));
  rbs.push_back((int)std::max<int64_t>(16, per32));
  for (int rb : rbs) {
    a.rb = rb;
    a.nblk = (int)((x->n + a.rb - 1) / a.rb);
    for (int nc = std::min(nw::NCMAX, a.nblk); nc >= 1; --nc) {  // cluster mode
      const int bpc = (a.nblk + nc - 1) / nc;
      if ((nc - 1) * bpc >= a.nblk) continue;  // no CTA without a row block
      nw::NarrowArgs t = a;
      nw_layout(x, bpc, nc, t);
      if (t.smem_bytes > optin) continue;
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, t.smem_bytes));
      cudaLaunchConfig_t cfg;
      memset(&cfg, 0, sizeof(cfg));
      cfg.gridDim = dim3(nc);
      cfg.blockDim = dim3(nw::NT);
      cfg.dynamicSmemBytes = t.smem_bytes;
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = nc;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      int clusters = 0;
      if (cudaOccupancyMaxActiveClusters(&clusters, fn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      if (clusters < 1) continue;
      const double cost = step_cost((x->C + clusters - 1) / clusters, bpc * rb, nc);
      if (cost < best - 1e-9) {
        best = cost;
        t.nc = nc;
        x->nwa = t;
        x->nw_hw = hw;
        x->nw_clusters = clusters;
      }
    }
    // grid mode: every CTA of every chain resident at once (cooperative launch), any nc up to nblk,
    // exchanges through L2 - chosen when it costs less than the best cluster shape (clusters of
    // 16 are limited by the GPC layout: 7 co-resident at 1 CTA per SM on B200)
    for (int nc = std::min(a.nblk, nsm); nc >= 2 && engine_override() != 3; --nc) {
      const int bpc = (a.nblk + nc - 1) / nc;
      if ((nc - 1) * bpc >= a.nblk) continue;
      nw::NarrowArgs t = a;
      nw_layout(x, bpc, nc, t);
      if (t.smem_bytes > optin) continue;
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, t.smem_bytes));
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nw::NT, t.smem_bytes));
      if ((int64_t)x->C * nc > (int64_t)per_sm * nsm) continue;
      const double cost = step_cost(1, bpc * rb, nc);
      if (cost < best - 1e-9) {
        best = cost;
        t.nc = nc;
        t.grid = 1;
        x->nwa = t;
        x->nw_hw = hw;
        x->nw_clusters = 0;
      }
      break;  // (the largest feasible nc has the fewest rows per CTA)
    }
  }
  if (best >= 1e30) return false;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, x->nwa.smem_bytes));
  return true;
}

void launch_narrow(hmc_ctx* x, int nsteps, int last_mode, cudaStream_t st, std::string& err) {
  nw::NarrowArgs a = x->nwa;
  a.x = x->d_x;
  a.y = x->d_y;
  a.slot = x->d_slot;
  a.soff = x->d_soff;
  a.inv_s2 = (float)(1.0 / (x->sigma * x->sigma));
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)(x->C * a.nc));
  cfg.blockDim = dim3(nw::NT);
  cfg.dynamicSmemBytes = a.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr;
  if (a.grid) {  // every CTA resident (the per-chain barriers spin on each other)
    attr.id = cudaLaunchAttributeCooperative;
    attr.val.cooperative = 1;
    CK(cudaMemsetAsync(a.xbar, 0, (size_t)x->C * sizeof(unsigned), st));
  } else {
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = a.nc;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
  }
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  KState ks = x->kstate();
  void* args[] = {&ks, &a, &nsteps, &last_mode};
  CK(cudaLaunchKernelExC(&cfg, nw::narrow_kernel(x->nw_hw), args));
  x->launches++;
}

// flops of one narrow-engine gradient evaluation of all chains (forward + input-gradient + dense
// weight-gradient tiles, 2 per multiply-add; the bench's roofline numerator)
double narrow_flops(const hmc_ctx* x) {
  const nw::NarrowArgs& a = x->nwa;
  double f = 0.0;
  for (int l = 0; l < a.nl; ++l) {
    const double mac = (double)a.width[l] * a.width[l + 1] * (double)x->n;
    f += 2.0 * mac;                                  // forward
    if (l >= a.l_min) f += 2.0 * mac;                // weight gradient
    if (l > a.l_min) f += 2.0 * mac;                 // input gradient
  }
  return f * x->C;
}

void capture_begin(hmc_ctx* x, std::string& err) {
  CK(cudaStreamBeginCapture(x->st, cudaStreamCaptureModeThreadLocal));
}

cudaGraphExec_t capture_end(hmc_ctx* x, std::string& err) {
  cudaGraph_t g = nullptr;
  CK(cudaStreamEndCapture(x->st, &g));
  cudaGraphExec_t e = nullptr;
  cudaError_t r = cudaGraphInstantiate(&e, g, 0);
  cudaGraphDestroy(g);
  if (r != cudaSuccess) {
    err = std::string("cudaGraphInstantiate: ") + cudaGetErrorString(r);
    throw Fail{HMC_E_CUDA};
  }
  return e;
}

void build_grad_graph(hmc_ctx* x, std::string& err) {
  if (x->grad_exec) return;
  capture_begin(x, err);
  const int64_t l0 = x->launches;
  x->prof_armed = false;
  try {
    k_scatter<<<dim3((unsigned)std::min<int64_t>((x->k + 255) / 256, 1024), x->C), 256, 0, x->st>>>(x->kstate(), x->wrk_theta);
    x->launches++;
    if (x->narrow) {  // forward + gradient + prior + log pi in one cluster kernel
      launch_narrow(x, 1, 0, x->st, err);
      x->per_body = 1;
    } else {
      enqueue_body(x, x->st);
      x->per_body = x->launches - l0 - 1;
      enqueue_reduce(x, x->st, err);
      k_finalize<<<x->C, KT, 0, x->st>>>(x->kstate(), 0);
      x->launches++;
    }
  } catch (...) {
    cudaGraph_t g;
    cudaStreamEndCapture(x->st, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  x->grad_exec = capture_end(x, err);
}

void build_traj_graph(hmc_ctx* x, int L, std::string& err) {
  if (x->traj_exec && x->traj_L == L) return;
  if (x->traj_exec) {
    cudaGraphExecDestroy(x->traj_exec);
    x->traj_exec = nullptr;
  }
  x->prof_clear();
  capture_begin(x, err);
  try {
    x->prof_step = -1;
    x->prof_armed = x->prof_on;
    int id = prof_begin(x, x->st);
    k_traj_begin<<<x->C, KT, 0, x->st>>>(x->kstate(), L == 0 ? 1 : 0);
    prof_end(x, id, x->st, "traj_begin", 0.0, 0.0);
    if (x->narrow && L > 0) {
      if (x->prof_on) {  // profiled trajectory: one launch per step, each timed
        const double fl = narrow_flops(x);
        for (int s = 0; s < L; ++s) {
          x->prof_step = s;
          x->prof_armed = s == 0;
          const int idb = prof_begin(x, x->st, true);
          const int idk = prof_begin(x, x->st);  // step 0: the kernel record (same launch)
          launch_narrow(x, 1, s == L - 1 ? 2 : 1, x->st, err);
          prof_end(x, idk, x->st, "narrow_step", fl, 0.0);
          prof_end(x, idb, x->st, "body", fl, 0.0);
        }
      } else {
        launch_narrow(x, L, 2, x->st, err);  // all L leapfrog steps in one launch
      }
    } else {
      for (int s = 0; s < L; ++s) {
        x->prof_step = s;
        x->prof_armed = x->prof_on && s == 0;
        enqueue_step(x, s == L - 1 ? 2 : 1, x->st, err);
      }
    }
    x->prof_step = -1;
    x->prof_armed = x->prof_on;
    id = prof_begin(x, x->st);
    k_mh<<<x->C, KT, 0, x->st>>>(x->kstate());
    k_advance<<<1, 1, 0, x->st>>>(x->d_rec);
    x->launches += 3;
    prof_end(x, id, x->st, "mh", 0.0, 0.0);
    x->prof_armed = false;
  } catch (...) {
    x->prof_armed = false;
    cudaGraph_t g;
    cudaStreamEndCapture(x->st, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  x->traj_exec = capture_end(x, err);
  x->traj_L = L;
}

void sync_in(hmc_ctx* x, cudaStream_t user, std::string& err) {
  CK(cudaEventRecord(x->ev_in, user));
  CK(cudaStreamWaitEvent(x->st, x->ev_in, 0));
}

void sync_out(hmc_ctx* x, cudaStream_t user, bool host, std::string& err) {
  if (host) {
    CK(cudaStreamSynchronize(x->st));
    return;
  }
  CK(cudaEventRecord(x->ev_out, x->st));
  CK(cudaStreamWaitEvent(user, x->ev_out, 0));
}

void cpy(void* dst, const void* src, size_t bytes, cudaStream_t st, std::string& err) {
  if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
}

// eps > 0: every chain uses eps; eps == 0: the per-chain values already in d_eps (hmc_adapt)
void set_rec(hmc_ctx* x, float* samples, uint8_t* acc, double* dH, int64_t S, int64_t iter, double eps,
             std::string& err, int adapt = 0, double delta = 0.0) {
  CK(cudaEventSynchronize(x->ev_stage));  // previous staging copy consumed
  x->h_rec->samples = samples;
  x->h_rec->acc = acc;
  x->h_rec->dH = dH;
  x->h_rec->S = S;
  x->h_rec->sidx = 0;
  x->h_rec->iter = iter;
  x->h_rec->adapt = adapt;
  x->h_rec->delta = delta;
  CK(cudaMemcpyAsync(x->d_rec, x->h_rec, sizeof(Rec), cudaMemcpyHostToDevice, x->st));
  if (eps > 0) k_fill_d<<<1, 256, 0, x->st>>>(x->d_eps, x->C, eps);
  else if (!adapt) CK(cudaMemcpyAsync(x->d_eps, x->d_epsbar, (size_t)x->C * 8, cudaMemcpyDeviceToDevice, x->st));
  CK(cudaEventRecord(x->ev_stage, x->st));
}

// ---------------------------------------------------------------------------------------------
// Masked weight gradient (masked_wgrad.cuh): per hidden layer, the active entries grouped into
// tasks of <= MW_G entries of one output row, and the choice against the dense weight-gradient
// GEMM by a cost model (DESIGN.md §5 "masked weight gradient"):
//   dense GEMM : 2 nch rows n_out n_in FLOP at ~140 TFLOP/s (3xTF32 engine, measured cfg5) + 5 us
//   masked     : shared-memory words nch rows (T + |mask|) (T tasks) at 32 words / clk
//                / SM x 0.7, or the operand bytes at 6 TB/s, whichever is larger, x wave
//                quantisation, + 3 us (+ 3 us for the segment reduction)
// Row segments: the count with the fewest chunk-times per resident CTA slot (2 per SM).
void plan_masked_wgrad(hmc_ctx* x, const std::vector<int32_t>& slot, std::string& err) {
  // hmc_debug_set_engine(4) (tests) or HMC_MWG=1 (make DEV=1): wherever the kernel applies;
  // hmc_debug_set_engine(2) or HMC_MWG=0: never
  int force = engine_override() == 4 ? 1 : (engine_override() == 2 ? 0 : -1);
  if (const char* f = dev_env("HMC_MWG")) force = atoi(f);
  const int sms = x->tc.num_sms > 0 ? x->tc.num_sms : 148;
  bool any = false;
  for (int ni = 0; ni < x->n_nets; ++ni) {
    NetInfo& N = x->nets[ni];
    size_t part_cap = 0;
    for (int li = N.l_min < 0 ? (int)N.layers.size() : N.l_min; li < (int)N.layers.size(); ++li) {
      LayerInfo& L = x->layers[N.layers[li]];
      const bool mlp_out = (x->kind == HMC_MLP && li == (int)N.layers.size() - 1);
      if (mlp_out || !L.any_active || is_narrow(L) || L.n_in % 4 || L.n_out % 4 || L.n_in > MW_MAXW ||
          L.n_out > MW_MAXW || L.act == ACT_SIN || force == 0)
        continue;
      // tasks: the active entries of each output row (bias = input column n_in), MW_G at a time
      std::vector<std::vector<int>> tasks;
      std::vector<int> tasks_o;
      int64_t npairs = 0, lo = INT64_MAX, hi = -1;
      for (int o = 0; o < L.n_out; ++o) {
        std::vector<int> cur;
        auto note = [&](int32_t sl) { lo = std::min<int64_t>(lo, sl); hi = std::max<int64_t>(hi, sl + 1); ++npairs; };
        for (int i = 0; i <= L.n_in; ++i) {
          const int32_t sl = (i < L.n_in) ? slot[L.w_off + (int64_t)o * L.n_in + i] : (L.bias ? slot[L.b_off + o] : -1);
          if (sl < 0) continue;
          note(sl);
          cur.push_back(i);
          if ((int)cur.size() == MW_G) { tasks.push_back(cur); tasks_o.push_back(o); cur.clear(); }
        }
        if (!cur.empty()) { tasks.push_back(cur); tasks_o.push_back(o); }
      }
      const int T = (int)tasks.size();
      if (T == 0) continue;
      const int n_tb = (T + MW_NT - 1) / MW_NT;
      // row segments
      const int64_t rows = L.rows, nch = N.nch;
      const int64_t nchunk = (rows + MW_R - 1) / MW_R;
      const int64_t slots = 2LL * sms;
      int best_s = 1;
      double best_c = 1e300;
      const bool contiguous = (hi - lo == npairs);
      for (int s = 1; s <= std::min<int64_t>(64, nchunk); ++s) {
        if (s > 1 && !contiguous) break;
        const double c = (double)((nch * n_tb * s + slots - 1) / slots) * (double)((nchunk + s - 1) / s) + (s > 1 ? 2.0 : 0.0);
        if (c < best_c - 1e-9) { best_c = c; best_s = s; }
      }
      // lanes.  Warps of 32 tasks with distinct o mod 32 (conflict-free G loads), filled
      // largest task first into the warp whose input-column residues (i mod 32) stay the most
      // balanced; then each warp's lane x residue multigraph is edge-coloured (bipartite: as many
      // colours as its largest degree, Koenig) and an entry's colour is its position p, so at
      // every p the lanes read distinct banks of X.  Unused positions read a zero column whose
      // bank is free at that position (k-slot -1: not written back).
      const int pad0 = L.n_in + 1;  // zero columns n_in + 1 .. n_in + 3 (n_in: the ones)
      std::vector<int> ord(T);
      for (int t = 0; t < T; ++t) ord[t] = t;
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return tasks[a].size() > tasks[b].size(); });
      std::vector<std::vector<int>> warps;
      for (int nwarp = (T + 31) / 32; warps.empty(); ++nwarp) {
        std::vector<std::vector<int>> W(nwarp);
        std::vector<uint32_t> used(nwarp, 0);
        std::vector<std::array<int, 32>> deg(nwarp);
        for (auto& d : deg) d.fill(0);
        bool ok = true;
        for (int t : ord) {
          const uint32_t bit = 1u << (tasks_o[t] & 31);
          int best = -1;
          long long bkey = 0;
          for (int w = 0; w < nwarp; ++w) {
            if (W[w].size() >= 32 || (used[w] & bit)) continue;
            std::array<int, 32> d = deg[w];
            for (int i : tasks[t]) ++d[i & 31];
            int mx = 0;
            long long sq = 0;
            for (int v : d) { mx = std::max(mx, v); sq += (long long)v * v; }
            const long long key = ((long long)mx << 40) + (sq << 8) + (long long)W[w].size();
            if (best < 0 || key < bkey) { best = w; bkey = key; }
          }
          if (best < 0) { ok = false; break; }
          W[best].push_back(t);
          used[best] |= bit;
          for (int i : tasks[t]) ++deg[best][i & 31];
        }
        if (ok) warps = W;
      }
      const int Tp = 32 * (int)warps.size();  // lanes incl. idle ones
      std::vector<int32_t> info(Tp, 0);
      std::vector<int16_t> pi((size_t)MW_G * Tp, (int16_t)pad0);
      std::vector<int32_t> ps((size_t)MW_G * Tp, -1);
      for (int w = 0; w < (int)warps.size(); ++w) {
        const int nl = (int)warps[w].size();
        // edges: (lane, residue) per entry
        std::vector<int> el, er, ei, col;
        for (int l = 0; l < nl; ++l)
          for (int i : tasks[warps[w][l]]) { el.push_back(l); er.push_back(i & 31); ei.push_back(i); }
        const int E = (int)el.size();
        int D = 0;
        {
          std::array<int, 32> dl{}, dr{};
          for (int e = 0; e < E; ++e) { D = std::max(D, ++dl[el[e]]); D = std::max(D, ++dr[er[e]]); }
        }
        std::vector<int> cl((size_t)32 * D, -1), cr((size_t)32 * D, -1);  // [vertex][colour] -> edge
        col.assign(E, -1);
        for (int e = 0; e < E; ++e) {
          const int l = el[e], r = er[e];
          int a = 0, b = 0;
          while (cl[l * D + a] >= 0) ++a;
          while (cr[r * D + b] >= 0) ++b;
          if (cr[r * D + a] >= 0) {  // flip the a/b alternating path from r (never reaches l)
            std::vector<int> path;
            int v = r, c = a;
            bool right = true;
            for (;;) {
              const int f = right ? cr[v * D + c] : cl[v * D + c];
              if (f < 0) break;
              path.push_back(f);
              v = right ? el[f] : er[f];
              right = !right;
              c = (c == a) ? b : a;
            }
            for (int f : path) { cl[el[f] * D + col[f]] = -1; cr[er[f] * D + col[f]] = -1; }
            for (int f : path) {
              col[f] = (col[f] == a) ? b : a;
              cl[el[f] * D + col[f]] = f;
              cr[er[f] * D + col[f]] = f;
            }
          }
          col[e] = a;
          cl[l * D + a] = e;
          cr[r * D + a] = e;
        }
        if (D > MW_G) {  // (more colours than positions: first-come positions, bank conflicts accepted)
          std::array<int, 32> nxt{};
          for (int e = 0; e < E; ++e) col[e] = nxt[el[e]]++;
        }
        std::vector<int> cnt(nl, 0);
        for (int e = 0; e < E; ++e) {
          const int l = el[e], p = col[e], i = ei[e];
          const int o = tasks_o[warps[w][l]];
          const size_t q = (size_t)p * Tp + 32 * w + l;
          pi[q] = (int16_t)i;
          ps[q] = (i < L.n_in) ? slot[L.w_off + (int64_t)o * L.n_in + i] : slot[L.b_off + o];
          cnt[l] = std::max(cnt[l], p + 1);
        }
        // unused positions of busy lanes: a zero column in a bank no entry uses at that position
        for (int p = 0; p < MW_G; ++p) {
          uint32_t busy = 0;
          for (int l = 0; l < nl; ++l)
            if (ps[(size_t)p * Tp + 32 * w + l] >= 0) busy |= 1u << (pi[(size_t)p * Tp + 32 * w + l] & 31);
          int z = pad0;
          for (int j = 0; j < 3; ++j)
            if (!(busy >> ((pad0 + j) & 31) & 1u)) { z = pad0 + j; break; }
          for (int l = 0; l < 32; ++l)
            if (ps[(size_t)p * Tp + 32 * w + l] < 0) pi[(size_t)p * Tp + 32 * w + l] = (int16_t)z;
        }
        for (int l = 0; l < nl; ++l) info[32 * w + l] = tasks_o[warps[w][l]] | (cnt[l] << 16);
      }
      {  // cost: shared-memory wavefronts per row = sum over warps of (1 + its positions)
        double wf = 0;
        for (int w = 0; w < (int)warps.size(); ++w) {
          int nw = 0;
          for (int l = 0; l < 32; ++l) nw = std::max(nw, info[32 * w + l] >> 16);
          wf += 1 + nw;
        }
        const int tb = (Tp + MW_NT - 1) / MW_NT;
        const double ideal = (double)nch * tb * nchunk / slots;  // chunk-times at perfect balance
        const double quant = std::max(1.0, best_c / std::max(ideal, 1e-9));
        const double t_smem = (double)nch * rows * wf / (sms * 1.8e9 * 0.45);
        const double t_hbm = (double)nch * rows * (L.n_out + L.n_in) * 4.0 / 6e12;
        const double t_mw = std::max(t_smem, t_hbm) * quant + 3e-6 + (best_s > 1 ? 3e-6 : 0.0);
        const double t_tc = 2.0 * nch * rows * L.n_out * (double)L.n_in / (x->tc.enabled ? 140e12 : 30e12) + 5e-6;
        if (!(force == 1 || t_mw < t_tc)) continue;
      }
      int32_t* d_info = dalloc<int32_t>(x, Tp, err);
      int16_t* d_pi = dalloc<int16_t>(x, pi.size(), err);
      int32_t* d_ps = dalloc<int32_t>(x, ps.size(), err);
      CK(cudaMemcpy(d_info, info.data(), Tp * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(d_pi, pi.data(), pi.size() * 2, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(d_ps, ps.data(), ps.size() * 4, cudaMemcpyHostToDevice));
      L.mwg = true;
      L.mw = MwTasks{d_info, d_pi, d_ps, Tp};
      L.mw_seg = best_s;
      L.mw_tb = (Tp + MW_NT - 1) / MW_NT;
      L.mw_lo = lo;
      L.mw_hi = hi;
      L.mw_pairs = npairs;
      if (best_s > 1) part_cap = std::max(part_cap, (size_t)best_s * nch * x->k);
      any = true;
    }
    if (part_cap) N.mw_part = dalloc<float>(x, part_cap, err);
  }
  if (any)
    for (auto& L : x->layers)
      if (L.mwg)
        CK(cudaFuncSetAttribute(mw_kernel(L.n_out, L.n_in), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)mw_smem_bytes(MW_MAXW, MW_MAXW)));
}

void setup_impl(hmc_ctx* x, const hmc_arch* arch, const hmc_data* data, const hmc_config* cfg, std::string& err,
                bool allow_narrow = true) {
  CFG(arch && data && cfg, "arch, data and config must be non-NULL");
  CFG(arch->kind == HMC_MLP || arch->kind == HMC_DEEPONET, "arch.kind must be HMC_MLP or HMC_DEEPONET");
  x->kind = arch->kind;
  x->n_nets = arch->kind == HMC_MLP ? 1 : 2;
  CK(cudaGetDevice(&x->dev));
  // ---- architecture and flat layout ----
  int64_t off = 0;
  for (int ni = 0; ni < x->n_nets; ++ni) {
    const hmc_net& net = arch->net[ni];
    CFG(net.n_layers >= 1 && net.widths && net.acts && net.has_bias, "net needs >= 1 layer and widths/acts/has_bias");
    for (int l = 0; l < net.n_layers; ++l) {
      CFG(net.widths[l] >= 1 && net.widths[l + 1] >= 1, "layer widths must be >= 1");
      CFG(net.acts[l] >= 0 && net.acts[l] <= 2, "activation must be HMC_ACT_*");
      LayerInfo L;
      L.net = ni; L.l = l; L.n_in = net.widths[l]; L.n_out = net.widths[l + 1]; L.act = net.acts[l];
      L.bias = net.has_bias[l] != 0;
      L.w_off = off; off += (int64_t)L.n_in * L.n_out;
      if (L.bias) { L.b_off = off; off += L.n_out; }
      x->nets[ni].layers.push_back((int)x->layers.size());
      x->nets[ni].max_w = std::max(x->nets[ni].max_w, std::max(L.n_in, L.n_out));
      x->layers.push_back(L);
    }
  }
  if (x->kind == HMC_MLP) {
    const hmc_net& net = arch->net[0];
    CFG(net.widths[net.n_layers] == 1, "MLP output width must be 1 (scalar regression, P:68)");
    CFG(net.acts[net.n_layers - 1] == HMC_ACT_IDENTITY, "MLP output layer must be linear (identity)");
  } else {
    CFG(arch->net[0].widths[arch->net[0].n_layers] == arch->net[1].widths[arch->net[1].n_layers],
        "DeepONet branch and trunk output widths must be equal (S:102)");
    x->has_b0 = arch->has_b0 != 0;
    if (x->has_b0) { x->b0_off = off; off += 1; }
  }
  x->P = off;
  CFG(cfg->P == x->P, ("frozen length P=" + std::to_string(cfg->P) + " != parameter count " + std::to_string(x->P)).c_str());
  // ---- config ----
  CFG(cfg->k >= 1 && cfg->k <= x->P, "need 1 <= k <= P (an empty mask has nothing to sample)");
  x->k = cfg->k;
  CFG(std::isfinite(cfg->noise_sigma) && cfg->noise_sigma > 0, "noise_sigma must be finite and > 0");
  CFG(std::isfinite(cfg->prior_sigma) && cfg->prior_sigma > 0, "prior_sigma must be finite and > 0");
  x->sigma = cfg->noise_sigma;
  x->sigma_p = cfg->prior_sigma;
  CFG(cfg->n_chains >= 1 && cfg->n_chains <= 65535, "n_chains must be in [1, 65535]");
  x->C = cfg->n_chains;
  x->seed = cfg->seed;
  CFG(cfg->frozen && cfg->idx, "frozen and idx must be non-NULL");
  std::vector<float> h_frozen = to_host(cfg->frozen, (size_t)x->P, err);
  std::vector<int32_t> h_idx = to_host(cfg->idx, (size_t)x->k, err);
  for (int64_t j = 0; j < x->k; ++j) {
    CFG(h_idx[j] >= 0 && h_idx[j] < x->P, "idx entries must lie in [0, P)");
    CFG(j == 0 || h_idx[j] > h_idx[j - 1], "idx must be strictly ascending");
  }
  for (float v : h_frozen) CFG(std::isfinite(v), "frozen values must be finite");
  std::vector<float> h_im;
  if (cfg->inv_mass) {
    h_im = to_host(cfg->inv_mass, (size_t)x->k, err);
    for (float v : h_im) CFG(std::isfinite(v) && v > 0, "inv_mass entries must be finite and > 0");
  }
  std::vector<uint32_t> h_ch(x->C);
  if (cfg->chain_ids) h_ch = to_host(cfg->chain_ids, (size_t)x->C, err);
  else for (int c = 0; c < x->C; ++c) h_ch[c] = (uint32_t)c;
  {
    std::vector<uint32_t> s = h_ch;
    std::sort(s.begin(), s.end());
    for (size_t i = 1; i < s.size(); ++i) CFG(s[i] != s[i - 1], "chain ids must be unique");
  }
  CFG(cfg->mode >= 0 && cfg->mode <= 2, "mode must be HMC_MODE_*");
  x->mode = cfg->mode;
  x->rank = cfg->rank;
  x->world = cfg->world;
  CFG(x->world == 1 || x->world == 2 || x->world == 4 || x->world == 8, "world must be 1, 2, 4 or 8 (one node)");
  CFG(x->rank >= 0 && x->rank < x->world, "need 0 <= rank < world");
  CFG(x->mode != HMC_MODE_SINGLE || x->world == 1, "SINGLE mode needs world == 1 (DATA or CHAIN for world > 1)");
  // ---- data ----
  std::vector<float> hx, hy, hu, hq, hv;
  if (x->kind == HMC_MLP) {
    CFG(data->x && data->y && data->n >= 1, "MLP data needs x, y and n >= 1");
    x->n = data->n;
    x->d_in = arch->net[0].widths[0];
    hx = to_host(data->x, (size_t)(x->n * x->d_in), err);
    hy = to_host(data->y, (size_t)x->n, err);
    for (float v : hx) CFG(std::isfinite(v), "x must be finite");
    for (float v : hy) CFG(std::isfinite(v), "y must be finite");
    x->nets[0].rows = x->n;
    const char* e = dev_env("HMC_STREAMS");
    x->wgrad_ov = !(e && atoi(e) == 1);
  } else {
    CFG(data->u && data->q && data->v && data->n_c >= 1 && data->n_x >= 1, "DeepONet data needs u, q, v, n_c, n_x >= 1");
    x->n_c = data->n_c;
    x->n_x = data->n_x;
    x->unaligned = data->q_per_pair != 0;
    x->xb = cfg->mode == HMC_MODE_DATA && cfg->shard == HMC_SHARD_POINTS_XB;
    x->xc = cfg->mode == HMC_MODE_DATA && cfg->shard == HMC_SHARD_POINTS_XC;
    CFG(cfg->shard >= HMC_SHARD_ROWS && cfg->shard <= HMC_SHARD_POINTS_XC, "shard must be HMC_SHARD_*");
    if (x->xc) {
      CFG(!x->unaligned, "POINTS_XC needs shared query points (q_per_pair = 0)");
      CFG(cfg->world >= 1 && cfg->n_chains % cfg->world == 0, "POINTS_XC needs n_chains divisible by world");
      CFG(arch->net[0].acts[arch->net[0].n_layers - 1] != HMC_ACT_SIN,
          "POINTS_XC: the branch output layer cannot be sin (its act' is not all-gathered)");
    }
    if (x->xb) {
      CFG(!x->unaligned, "POINTS_XB needs shared query points (q_per_pair = 0)");
      CFG(cfg->world >= 1 && x->n_c % cfg->world == 0, "POINTS_XB needs n_c divisible by world");
      CFG(arch->net[0].acts[arch->net[0].n_layers - 1] != HMC_ACT_SIN,
          "POINTS_XB: the branch output layer cannot be sin (its act' is not all-gathered)");
    }
    x->n_c_loc = x->xb ? x->n_c / cfg->world : x->n_c;
    {
      const char* e = dev_env("HMC_STREAMS");
      x->two_streams = !x->unaligned && !(e && atoi(e) == 1);
      x->wgrad_ov = x->two_streams;
    }
    const int64_t q_rows = x->unaligned ? x->n_c * x->n_x : x->n_x;
    hu = to_host(data->u, (size_t)(x->n_c_loc * arch->net[0].widths[0]), err);
    hq = to_host(data->q, (size_t)(q_rows * arch->net[1].widths[0]), err);
    hv = to_host(data->v, (size_t)(x->n_c * x->n_x), err);
    for (float v : hu) CFG(std::isfinite(v), "u must be finite");
    for (float v : hq) CFG(std::isfinite(v), "q must be finite");
    for (float v : hv) CFG(std::isfinite(v), "v must be finite");
    x->nets[0].rows = x->n_c_loc;
    x->nets[1].rows = q_rows;
  }
  const int64_t n_local = x->kind == HMC_MLP ? x->n : x->n_c * x->n_x;
  x->n_global = data->n_global > 0 ? data->n_global : (x->mode == HMC_MODE_DATA ? n_local * x->world : n_local);
  if (x->mode != HMC_MODE_DATA || x->world == 1) CFG(x->n_global == n_local, "n_global must equal the local size outside DATA mode");
  // DATA mode: equal shards (SURVEY §8(b) validation): every rank holds n_global / world data
  // points (ROWS: a row block; POINTS_XB: all n_c conditions x n_x / world points)
  if (x->mode == HMC_MODE_DATA)
    CFG(n_local * x->world == x->n_global, ("DATA mode needs equal shards: local size " + std::to_string(n_local) + " x world " +
                                            std::to_string(x->world) + " != n_global " + std::to_string(x->n_global)).c_str());
  // ---- slot map, per-layer activity, l_min ----
  std::vector<int32_t> slot((size_t)x->P, -1);
  for (int64_t j = 0; j < x->k; ++j) slot[h_idx[j]] = (int32_t)j;
  for (auto& L : x->layers) {
    for (int64_t t = L.w_off; t < L.w_off + (int64_t)L.n_in * L.n_out && !L.any_active; ++t) L.any_active |= slot[t] >= 0;
    if (L.bias) for (int t = 0; t < L.n_out && !L.any_active; ++t) L.any_active |= slot[L.b_off + t] >= 0;
  }
  for (auto& L : x->layers)
    if (L.bias)
      for (int t = 0; t < L.n_out && !L.bias_active; ++t) L.bias_active |= slot[L.b_off + t] >= 0;
  if (x->has_b0) x->b0_slot = slot[x->b0_off];
  // ---- tensor-core engine: which layers keep tf32 hi/lo weight planes ----
  x->tc.init();
  std::vector<int32_t> tcpos((size_t)x->k, -1);
  for (int ni = 0; ni < x->n_nets; ++ni) {
    NetInfo& N = x->nets[ni];
    for (int i = 0; i < (int)N.layers.size(); ++i)
      if (x->layers[N.layers[i]].any_active) { N.l_min = i; break; }
  }
  x->narrow = allow_narrow && plan_narrow(x, err);
  if (x->tc.enabled && !x->narrow) {
    for (int ni = 0; ni < x->n_nets; ++ni) {
      NetInfo& N = x->nets[ni];
      for (int i = 0; i < (int)N.layers.size(); ++i) {
        LayerInfo& L = x->layers[N.layers[i]];
        const bool mlp_out = (x->kind == HMC_MLP && i == (int)N.layers.size() - 1);
        if (mlp_out || L.n_in % 4 || L.n_out % 4 || L.n_in < 32 || L.n_out < 32) continue;
        L.tc_w = true;
        // planes only when every GEMM reading these weights (forward, input gradient) takes the
        // tensor-core path: not for sin layers (their forward runs on SIMT) nor short row counts
        L.planes_only = L.act != ACT_SIN && N.rows >= 64 && !(dev_env("HMC_DENSE_W") && atoi(dev_env("HMC_DENSE_W")) == 1);
        L.q_off = x->Ptc;
        x->Ptc += (int64_t)L.n_in * L.n_out;
      }
    }
    x->Ptc = (x->Ptc + 3) / 4 * 4;
    for (int64_t j = 0; j < x->k; ++j)
      for (auto& L : x->layers)
        if (L.tc_w && h_idx[j] >= L.w_off && h_idx[j] < L.w_off + (int64_t)L.n_in * L.n_out)
          // (planes-only entries encoded as -(q + 2), see put_param)
          tcpos[j] = L.planes_only ? (int32_t)(-(L.q_off + (h_idx[j] - L.w_off)) - 2)
                                   : (int32_t)(L.q_off + (h_idx[j] - L.w_off));
  }
  for (int ni = 0; ni < x->n_nets; ++ni) {
    NetInfo& N = x->nets[ni];
    for (int i = 0; i < (int)N.layers.size(); ++i)
      if (x->layers[N.layers[i]].any_active) { N.l_min = i; break; }
  }
  // ---- device allocations ----
  const int C = x->C;
  x->d_idx = dalloc<int32_t>(x, x->k, err);
  x->d_slot = dalloc<int32_t>(x, x->P, err);
  {  // group masks / bases of the slot map, for layers whose weights leave the tensor-core engine
    std::vector<uint32_t> gm;
    std::vector<int32_t> gb;
    for (auto& L : x->layers) {
      if (!L.any_active) continue;
      const int G = (L.n_in + 31) / 32;
      L.g_off = (int64_t)gm.size();
      for (int m = 0; m < L.n_out; ++m)
        for (int g = 0; g < G; ++g) {
          uint32_t mk = 0;
          int32_t base = -1;
          for (int j = 0; j < 32 && 32 * g + j < L.n_in; ++j) {
            const int32_t sl = slot[L.w_off + (int64_t)m * L.n_in + 32 * g + j];
            if (sl >= 0) { mk |= 1u << j; if (base < 0) base = sl; }
          }
          gm.push_back(mk);
          gb.push_back(base < 0 ? 0 : base);
        }
    }
    // slot ranges, and the K split of weight-gradient GEMMs with fewer CTA-pair tiles than the
    // GPU has SM pairs (each split >= 8 K blocks of 32 rows)
    int ks_max = 1;
    for (auto& L : x->layers) {
      L.ws_lo = L.ws_hi = 0;
      bool first = true;
      for (int64_t t = L.w_off; t < L.w_off + (int64_t)L.n_in * L.n_out; ++t)
        if (slot[t] >= 0) {
          if (first) { L.ws_lo = slot[t]; first = false; }
          L.ws_hi = slot[t] + 1;
        }
      L.ksplit = 1;
      if (x->tc.enabled && L.any_active && L.n_in > 8) {
        const int64_t rows = x->nets[L.net].rows;  // (L.rows is filled in later)
        const int nch_l = (x->xc && L.net == 0) ? x->C / x->world : x->C;  // (POINTS_XC branch: its chain block)
        GemmArgs pa = gemm_base(L.n_out, L.n_in, (int)rows, nch_l);
        const int pt = TcPlanner::pair_tiles(pa);
        const int half_sms = std::max(1, x->tc.num_sms / 2);
        const int nk = (int)((rows + 31) / 32);
        if (pt < half_sms && nk >= 16) {  // fewest rounds of SM pairs per unit of K work
          double best = 1.0;
          // overlapped weight gradients (wgrad_ov) run beside the input-gradient chain, which is the
          // critical path: a split that fills every SM pair delays it, so they take at most a
          // quarter of the pairs (measured: half of the pairs cfg4 81.1k -> 85.2k evals/s, cfg3 +1 %;
          // a quarter, beside the halved input-gradient grids, cfg4 90.6k -> 92.9k)
          int ks_cap = x->wgrad_ov ? std::max(1, half_sms / 4 / std::max(1, pt)) : 16;
          if (const char* e = dev_env("HMC_KS_MAX")) ks_cap = atoi(e);
          if (const char* e = dev_env("HMC_KS_LAST"))
            if (L.l == x->nets[L.net].l_min) ks_cap = atoi(e);
          for (int ks = 2; ks <= std::min(ks_cap, nk / 8); ++ks) {
            const double cost = (double)((pt * ks + half_sms - 1) / half_sms) / ks;
            if (cost < best - 1e-12) { best = cost; L.ksplit = ks; }
          }
        }
        ks_max = std::max(ks_max, L.ksplit);
      }
    }
    if (ks_max > 1)
      for (int ni = 0; ni < x->n_nets; ++ni) x->nets[ni].gl_part = dalloc<float>(x, (size_t)ks_max * x->C * x->k, err);
    x->d_gmask = dalloc<uint32_t>(x, gm.size(), err);
    x->d_gbase = dalloc<int32_t>(x, gb.size(), err);
    if (!gm.empty()) {
      CK(cudaMemcpy(x->d_gmask, gm.data(), gm.size() * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(x->d_gbase, gb.data(), gb.size() * 4, cudaMemcpyHostToDevice));
    }
  }
  x->d_chain = dalloc<uint32_t>(x, C, err);
  if (!h_im.empty()) x->d_inv_mass = dalloc<float>(x, x->k, err);
  x->Wd = dalloc<float>(x, (size_t)C * x->P, err);
  CK(cudaMemcpy(x->d_idx, h_idx.data(), x->k * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(x->d_slot, slot.data(), x->P * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(x->d_chain, h_ch.data(), C * 4, cudaMemcpyHostToDevice));
  if (!h_im.empty()) CK(cudaMemcpy(x->d_inv_mass, h_im.data(), x->k * 4, cudaMemcpyHostToDevice));
  if (x->narrow) {  // shared-memory word of every active entry in the narrow engine's weight copy
    std::vector<int32_t> soff((size_t)x->k, -1);
    const NetInfo& N = x->nets[0];
    for (int64_t j = 0; j < x->k; ++j)
      for (int l = 0; l < x->nwa.nl; ++l) {
        const LayerInfo& L = x->layers[N.layers[l]];
        const int64_t f = h_idx[j];
        if (f >= L.w_off && f < L.w_off + (int64_t)L.n_in * L.n_out) {
          const int64_t o = (f - L.w_off) / L.n_in, i = (f - L.w_off) % L.n_in;
          soff[j] = x->nwa.sw[l] + (int32_t)(o * x->nwa.ldw[l] + i);
        } else if (L.bias && f >= L.b_off && f < L.b_off + L.n_out) {
          soff[j] = x->nwa.sb[l] + (int32_t)(f - L.b_off);
        }
      }
    x->d_soff = dalloc<int32_t>(x, x->k, err);
    CK(cudaMemcpy(x->d_soff, soff.data(), x->k * 4, cudaMemcpyHostToDevice));
    if (x->nwa.grid) {  // L2 exchange buffers of the grid mode
      nw::NarrowArgs& a = x->nwa;
      a.xpart = dalloc<float>(x, (size_t)x->C * a.nc * a.nblk * a.ksp, err);
      a.xtheta = dalloc<float>(x, (size_t)x->C * x->k, err);
      a.xsq = dalloc<double>(x, (size_t)x->C * a.nblk, err);
      a.xbar = dalloc<unsigned>(x, (size_t)x->C, err);
    }
  }
  for (int c = 0; c < C; ++c) CK(cudaMemcpy(x->Wd + (size_t)c * x->P, h_frozen.data(), x->P * 4, cudaMemcpyHostToDevice));
  if (x->Ptc > 0) {
    x->Whi = dalloc<float>(x, (size_t)C * x->Ptc, err);
    // default: tf32 hi / lo planes written by the scatter (no B conversion in the GEMM);
    // HMC_TC_RAWB=1: one raw plane split in shared memory by the converters (half the L2
    // traffic, measured 2-3 % slower: the converters are on the critical path)
    if (!(dev_env("HMC_TC_RAWB") && atoi(dev_env("HMC_TC_RAWB")) == 1)) x->Wlo = dalloc<float>(x, (size_t)C * x->Ptc, err);
    x->d_tcpos = dalloc<int32_t>(x, x->k, err);
    CK(cudaMemcpy(x->d_tcpos, tcpos.data(), x->k * 4, cudaMemcpyHostToDevice));
    for (auto& L : x->layers)
      if (L.tc_w)
        k_split_layer<<<148 * 4, 256>>>(x->Wd, x->P, L.w_off, (int64_t)L.n_in * L.n_out, x->Whi, x->Wlo, x->Ptc,
                                         L.q_off, C);
    CK(cudaGetLastError());
  }
  const size_t Ck = (size_t)C * x->k;
  x->cur_theta = dalloc<float>(x, Ck, err);
  x->cur_grad = dalloc<float>(x, Ck, err);
  x->wrk_theta = dalloc<float>(x, Ck, err);
  x->wrk_grad = dalloc<float>(x, Ck, err);
  x->p = dalloc<float>(x, Ck, err);
  x->gl = dalloc<float>(x, Ck, err);
  x->cur_logp = dalloc<double>(x, C, err);
  x->wrk_logp = dalloc<double>(x, C, err);
  x->H0 = dalloc<double>(x, C, err);
  x->lik = dalloc<double>(x, C, err);
  x->d_eps = dalloc<double>(x, C, err);
  x->d_epsbar = dalloc<double>(x, C, err);
  x->d_div = dalloc<uint32_t>(x, C, err);
  x->d_da = dalloc<double>(x, (size_t)4 * C, err);
  x->d_rec = dalloc<Rec>(x, 1, err);
  x->tmp_acc = dalloc<uint8_t>(x, C, err);
  x->tmp_dH = dalloc<double>(x, C, err);
  if (x->kind == HMC_MLP) {
    x->d_x = dalloc<float>(x, hx.size(), err);
    x->d_y = dalloc<float>(x, hy.size(), err);
    CK(cudaMemcpy(x->d_x, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(x->d_y, hy.data(), hy.size() * 4, cudaMemcpyHostToDevice));
    x->nets[0].input = x->d_x;
    x->n_part = (int)((x->n + 63) / 64);
    x->R = dalloc<float>(x, (size_t)C * x->n, err);
    x->colred_chunks = (int)((x->n + COLRED_CH - 1) / COLRED_CH);
  } else {
    x->d_u = dalloc<float>(x, hu.size(), err);
    x->d_q = dalloc<float>(x, hq.size(), err);
    x->d_v = dalloc<float>(x, hv.size(), err);
    CK(cudaMemcpy(x->d_u, hu.data(), hu.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(x->d_q, hq.data(), hq.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(x->d_v, hv.data(), hv.size() * 4, cudaMemcpyHostToDevice));
    x->nets[0].input = x->d_u;
    x->nets[1].input = x->d_q;
    x->R = dalloc<float>(x, (size_t)C * x->n_c * x->n_x, err);
    const int p = x->layers[x->nets[0].layers.back()].n_out;
    GemmArgs probe = gemm_base((int)x->n_c, (int)x->n_x, p, C);
    probe.epi = EPI_RESID;
    probe.lda = p; probe.sA = x->n_c * p; probe.ldb = p; probe.sB = x->n_x * p;
    const int bm = pick_bm((int)x->n_c, (int)x->n_x);
    // partial slots: max over both engines (unused slots stay zero); unaligned: one per function
    // (tcgen05: one slot per tile and epilogue warp)
    const int tc_slots = (int)(((x->n_c + tc::BM - 1) / tc::BM) * ((x->n_x + TcPlanner::BN - 1) / TcPlanner::BN)) * tc::NEPI;
    x->n_part = x->unaligned ? (int)x->n_c
                             : std::max(tc_slots, (int)(((x->n_x + bm - 1) / bm) * ((x->n_c + bm - 1) / bm)));
    (void)probe;
    if (x->xb) {  // all-gather / reduce-scatter staging of the branch outputs and their gradient
      const size_t blk = (size_t)C * x->n_c_loc * p;
      x->xb_recv = dalloc<float>(x, blk * x->world, err);
      x->xb_send = dalloc<float>(x, blk * x->world, err);
      x->xb_full = dalloc<float>(x, (size_t)C * x->n_c * p, err);
      x->xb_dB = dalloc<float>(x, (size_t)C * x->n_c * p, err);
    }
    if (x->xc) {
      x->xc_Ball = dalloc<float>(x, (size_t)C * x->n_c * p, err);
      x->xc_dB = dalloc<float>(x, (size_t)C * x->n_c * p, err);
      x->gl_red = dalloc<float>(x, (size_t)C * x->k, err);
    }
  }
  // per-net chain views (POINTS_XC: the branch runs this rank's chain block; its buffers keep the
  // full chain-count size, only the first nch chains are used)
  for (int ni = 0; ni < x->n_nets; ++ni) {
    NetInfo& N = x->nets[ni];
    int64_t c0 = 0;
    N.nch = C;
    if (x->xc && ni == 0) {
      N.nch = C / x->world;
      c0 = (int64_t)x->rank * N.nch;
    }
    N.wd = x->Wd + c0 * x->P;
    N.whi = x->Whi ? x->Whi + c0 * x->Ptc : nullptr;
    N.wlo = x->Wlo ? x->Wlo + c0 * x->Ptc : nullptr;
    N.gl = x->gl + c0 * x->k;
  }
  {  // two-pass column-reduction scratch: max over nets of chunks x (width + 1)
    size_t cap = 0;
    for (int ni = 0; ni < x->n_nets; ++ni) {
      const size_t chunks = (size_t)((x->nets[ni].rows + COLRED_CH - 1) / COLRED_CH);
      cap = std::max(cap, chunks * (size_t)(x->nets[ni].max_w + 1));
    }
    for (int ni = 0; ni < x->n_nets; ++ni) x->nets[ni].colred = dalloc<float>(x, (size_t)C * cap, err);
    if (x->wgrad_ov)
      for (int ni = 0; ni < x->n_nets; ++ni) x->nets[ni].colred2 = dalloc<float>(x, (size_t)C * cap, err);
  }
  {  // narrow-input weight-gradient partials: max over narrow layers of chunks x n_out x (n_in + 1)
    size_t cap = 0;
    for (int ni = 0; ni < x->n_nets; ++ni)
      for (int li : x->nets[ni].layers) {
        const LayerInfo& L = x->layers[li];
        if (is_narrow(L))
          cap = std::max(cap, (size_t)((x->nets[ni].rows + NARROW_ROWS - 1) / NARROW_ROWS) * L.n_out * (L.n_in + 1));
      }
    for (int ni = 0; ni < x->n_nets; ++ni) x->nets[ni].narrow_part = dalloc<float>(x, (size_t)C * cap, err);
  }
  x->part_sq = dalloc<double>(x, (size_t)C * x->n_part, err);
  x->part_r = dalloc<double>(x, (size_t)C * x->n_part, err);
  for (int ni = 0; ni < x->n_nets; ++ni) {
    NetInfo& N = x->nets[ni];
    const int nl = (int)N.layers.size();
    for (int i = 0; i < nl; ++i) {
      LayerInfo& L = x->layers[N.layers[i]];
      L.rows = N.rows;
      const bool mlp_out = (x->kind == HMC_MLP && i == nl - 1);
      if (!mlp_out) L.A = dalloc<float>(x, (size_t)C * L.rows * L.n_out, err);
      if (L.act == ACT_SIN && !mlp_out) L.D = dalloc<float>(x, (size_t)C * L.rows * L.n_out, err);
    }
    if (N.l_min >= 0) {
      N.G[0] = dalloc<float>(x, (size_t)C * N.rows * N.max_w, err);
      N.G[1] = dalloc<float>(x, (size_t)C * N.rows * N.max_w, err);
      if (x->tc.enabled) N.colsum = dalloc<float>(x, (size_t)C * ((N.rows + 31) / 32) * N.max_w, err);
      if (x->wgrad_ov) {  // overlapped weight gradients: one gradient buffer per layer, rotated partials
        N.nrot = std::min(NetInfo::MAXROT, std::max(3, nl));
        for (int r = 2; r < N.nrot; ++r) N.G[r] = dalloc<float>(x, (size_t)C * N.rows * N.max_w, err);
        const int top = nl - 1;
        for (int r = 0; r < N.nrot; ++r)
          N.cs[r] = (r == top % N.nrot) ? N.colsum
                                   : (x->tc.enabled ? dalloc<float>(x, (size_t)C * ((N.rows + 31) / 32) * N.max_w, err)
                                                    : nullptr);
        CK(cudaStreamCreateWithFlags(&N.ws, cudaStreamNonBlocking));
        if (!(dev_env("HMC_WS2") && atoi(dev_env("HMC_WS2")) == 0)) CK(cudaStreamCreateWithFlags(&N.ws2, cudaStreamNonBlocking));
        N.evA.resize(nl);
        N.evW.resize(nl);
        for (int i = 0; i < nl; ++i) {
          CK(cudaEventCreateWithFlags(&N.evA[i], cudaEventDisableTiming));
          CK(cudaEventCreateWithFlags(&N.evW[i], cudaEventDisableTiming));
        }
      }
    }
  }
  if (x->kind == HMC_DEEPONET && !x->unaligned && x->nets[1].l_min >= 0) {
    const int p = x->layers[x->nets[1].layers.back()].n_out;
    x->dt_ks = dt_ksplit(x, (int)x->n_x, p, (int)x->n_c, C);
    if (const char* e = dev_env("HMC_DT_KS")) { if (atoi(e) <= 1) x->dt_ks = 1; }  // dev A/B: 1 = no split
    if (x->dt_ks > 1) x->dt_part = dalloc<float>(x, (size_t)C * x->dt_ks * x->n_x * p, err);
  }
  plan_masked_wgrad(x, slot, err);
  CK(cudaMallocHost((void**)&x->h_rec, sizeof(Rec)));
  CK(cudaMallocHost((void**)&x->h_eps, sizeof(double)));
  CK(cudaEventCreateWithFlags(&x->ev_stage, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&x->ev_in, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&x->ev_out, cudaEventDisableTiming));
  CK(cudaEventRecord(x->ev_stage, 0));
  CK(cudaStreamCreateWithFlags(&x->st, cudaStreamNonBlocking));
  {
    if (x->two_streams) {
      CK(cudaStreamCreateWithFlags(&x->st2, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&x->ev_fork[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&x->ev_join[i], cudaEventDisableTiming));
      }
    }
  }
  // ---- NCCL (DATA mode) ----
  x->emulated = x->mode == HMC_MODE_DATA && cfg->exchange == 1;
  CFG(cfg->exchange >= 0 && cfg->exchange <= 2, "exchange must be 0 (NCCL), 1 (emulated phases) or 2 (timing stand-in)");
  if (x->mode == HMC_MODE_DATA && (x->world > 1 || x->xb || x->xc) && cfg->exchange == 0) {
    ncclUniqueId id;
    if (x->world > 1) {
      CFG(cfg->nccl_id, "DATA mode with world > 1 needs nccl_id");
      memcpy(&id, cfg->nccl_id, sizeof(id));
    } else {
      CKN(ncclGetUniqueId(&id));  // POINTS_XB on one rank: a communicator of one (the collectives run)
    }
    CKN(ncclCommInitRank(&x->comm, x->world, id, x->rank));
  }
  x->engine = x->narrow ? std::string("narrow-simt (") + (x->nwa.grid ? "grid " : "cluster ") + std::to_string(x->nwa.nc) + " x " + std::to_string(x->nwa.bpc) +
                              " blocks of " + std::to_string(x->nwa.rb) + " rows, " + std::to_string(x->nwa.nblk) +
                              " blocks, hw " + std::to_string(x->nw_hw) + ")"
                        : x->tc.describe();
  {
    int nm = 0, na = 0;
    for (auto& L : x->layers) { nm += L.mwg; na += L.any_active && !is_narrow(L); }
    if (nm) x->engine += " + masked wgrad (" + std::to_string(nm) + " of " + std::to_string(na) + " layers)";
  }
  if (x->dt_ks > 1) x->engine += " + dT K split " + std::to_string(x->dt_ks);
  CK(cudaDeviceSynchronize());
}

}  // namespace

// ---------------------------------------------------------------------------------------------
#define API_BEGIN(ctx)                                                                        \
  if (!(ctx)) {                                                                               \
    g_err = "NULL context";                                                                   \
    return HMC_E_STATE;                                                                       \
  }                                                                                           \
  std::string& err = (ctx)->err;                                                              \
  try {                                                                                       \
    CK(cudaSetDevice((ctx)->dev));

#define API_END                                                                               \
  }                                                                                           \
  catch (Fail f) {                                                                            \
    return f.code;                                                                            \
  }                                                                                           \
  return HMC_OK;

extern "C" {

int hmc_comm_unique_id(uint8_t id_out[128]) {
  if (!id_out) {
    g_err = "id_out is NULL";
    return HMC_E_CONFIG;
  }
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    g_err = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r);
    return HMC_E_NCCL;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
  memcpy(id_out, &id, 128);
  return HMC_OK;
}

int hmc_setup(const hmc_arch* arch, const hmc_data* data, const hmc_config* cfg, void* stream, hmc_ctx** out) {
  NvtxRange nvtx_("hmc_setup");
  (void)stream;
  if (!out) {
    g_err = "out is NULL";
    return HMC_E_CONFIG;
  }
  *out = nullptr;
  std::unique_ptr<hmc_ctx> x(new hmc_ctx());
  try {
    setup_impl(x.get(), arch, data, cfg, x->err);
  } catch (Fail f) {
    g_err = x->err;
    return f.code;
  }
  *out = x.release();
  return HMC_OK;
}

int hmc_grad(hmc_ctx* ctx, const float* theta, double* logp, float* grad, void* stream) {
  NvtxRange nvtx_("hmc_grad");
  API_BEGIN(ctx)
  if (ctx->emulated) {
    err = "state: an emulated-exchange context (hmc_config.exchange = 1) runs only hmc_debug_data_phase";
    throw Fail{HMC_E_STATE};
  }
  CFG(theta && logp && grad, "theta, logp and grad must be non-NULL");
  cudaStream_t us = (cudaStream_t)stream;
  const bool host = !is_device_ptr(theta) || !is_device_ptr(logp) || !is_device_ptr(grad);
  build_grad_graph(ctx, err);
  sync_in(ctx, us, err);
  const size_t Ck = (size_t)ctx->C * ctx->k;
  cpy(ctx->wrk_theta, theta, Ck * 4, ctx->st, err);
  CK(cudaGraphLaunch(ctx->grad_exec, ctx->st));
  cpy(grad, ctx->wrk_grad, Ck * 4, ctx->st, err);
  cpy(logp, ctx->wrk_logp, ctx->C * 8, ctx->st, err);
  sync_out(ctx, us, host, err);
  API_END
}

int hmc_logpost_const(const hmc_ctx* ctx, double* c) {
  if (!ctx) { g_err = "NULL context"; return HMC_E_STATE; }
  if (!c) return HMC_E_CONFIG;
  const double l2pi = std::log(2.0 * M_PI);
  *c = -(double)ctx->n_global * (std::log(ctx->sigma) + 0.5 * l2pi) - (double)ctx->k * (std::log(ctx->sigma_p) + 0.5 * l2pi);
  return HMC_OK;
}

static int run_traj(hmc_ctx* ctx, float* theta, double* logp, float* grad, double eps, int32_t L, int64_t iter0,
                    int32_t S, float* samples, uint8_t* acc, double* dH, void* stream, int adapt = 0,
                    double delta = 0.0, double* eps_bar = nullptr) {
  NvtxRange nvtx_(adapt ? "hmc_adapt" : (S == 1 ? "hmc_trajectory" : "hmc_sample"));
  API_BEGIN(ctx)
  if (ctx->emulated) {
    err = "state: an emulated-exchange context (hmc_config.exchange = 1) runs only hmc_debug_data_phase";
    throw Fail{HMC_E_STATE};
  }
  CFG(theta && logp && grad, "theta, logp and grad must be non-NULL");
  CFG(std::isfinite(eps) && (eps > 0 || (eps == 0 && ctx->adapted && !adapt)),
      "eps must be finite and > 0 (or 0 after hmc_adapt: the adapted per-chain steps)");
  CFG(!adapt || (delta > 0 && delta < 1), "delta must lie in (0, 1)");
  CFG(L >= 0, "L must be >= 0");
  CFG(S >= 1, "S must be >= 1");
  CFG(iter0 >= 0 && iter0 + S <= (int64_t)1 << 32, "iter must lie in [0, 2^32)");
  cudaStream_t us = (cudaStream_t)stream;
  const size_t Ck = (size_t)ctx->C * ctx->k;
  bool host = !is_device_ptr(theta) || !is_device_ptr(logp) || !is_device_ptr(grad);
  // output records: device pointers are written in place, host ones staged in device temps
  float* d_samples = nullptr;
  uint8_t* d_acc = nullptr;
  double* d_dH = nullptr;
  auto stage = [&](hmc_ctx::Stage& g, size_t bytes) -> void* {
    if (bytes > g.cap) {
      if (g.p) CK(cudaFree(g.p));
      g.p = nullptr;
      g.cap = 0;
      CK(cudaMalloc(&g.p, bytes));
      g.cap = bytes;
    }
    return g.p;
  };
  if (samples) {
    if (is_device_ptr(samples)) d_samples = samples;
    else { host = true; d_samples = (float*)stage(ctx->stage_samples, Ck * S * 4); }
  }
  if (acc) {
    if (is_device_ptr(acc)) d_acc = acc;
    else { host = true; d_acc = (S == 1) ? ctx->tmp_acc : (uint8_t*)stage(ctx->stage_acc, (size_t)ctx->C * S); }
  }
  if (dH) {
    if (is_device_ptr(dH)) d_dH = dH;
    else { host = true; d_dH = (S == 1) ? ctx->tmp_dH : (double*)stage(ctx->stage_dH, (size_t)ctx->C * S * 8); }
  }
  build_traj_graph(ctx, L, err);
  sync_in(ctx, us, err);
  cpy(ctx->cur_theta, theta, Ck * 4, ctx->st, err);
  cpy(ctx->cur_grad, grad, Ck * 4, ctx->st, err);
  cpy(ctx->cur_logp, logp, ctx->C * 8, ctx->st, err);
  if (adapt) {
    k_da_init<<<1, 256, 0, ctx->st>>>(ctx->d_eps, ctx->d_da, ctx->C, eps);
    set_rec(ctx, d_samples, d_acc, d_dH, S, iter0, 0.0, err, 1, delta);
  } else {
    set_rec(ctx, d_samples, d_acc, d_dH, S, iter0, eps, err);
  }
  for (int s = 0; s < S; ++s) CK(cudaGraphLaunch(ctx->traj_exec, ctx->st));
  if (adapt) {  // the averaged steps: kept in the context (eps == 0 later) and copied out
    k_da_finish<<<1, 256, 0, ctx->st>>>(ctx->d_eps, ctx->d_da, ctx->C, ctx->d_epsbar);
    CK(cudaMemcpyAsync(eps_bar, ctx->d_epsbar, (size_t)ctx->C * 8, cudaMemcpyDefault, ctx->st));
    host = true;
    ctx->adapted = true;
  }
  cpy(theta, ctx->cur_theta, Ck * 4, ctx->st, err);
  cpy(grad, ctx->cur_grad, Ck * 4, ctx->st, err);
  cpy(logp, ctx->cur_logp, ctx->C * 8, ctx->st, err);
  if (samples && d_samples != samples) cpy(samples, d_samples, Ck * S * 4, ctx->st, err);
  if (acc && d_acc != acc) cpy(acc, d_acc, (size_t)ctx->C * S, ctx->st, err);
  if (dH && d_dH != dH) cpy(dH, d_dH, (size_t)ctx->C * S * 8, ctx->st, err);
  sync_out(ctx, us, host, err);
  API_END
}

int hmc_trajectory(hmc_ctx* ctx, float* theta, double* logp, float* grad, double eps, int32_t L, int64_t iter,
                   uint8_t* acc, double* dH, void* stream) {
  return run_traj(ctx, theta, logp, grad, eps, L, iter, 1, nullptr, acc, dH, stream);
}

int hmc_sample(hmc_ctx* ctx, float* theta, double* logp, float* grad, double eps, int32_t L, int64_t iter0,
               int32_t S, float* samples, uint8_t* acc, double* dH, void* stream) {
  return run_traj(ctx, theta, logp, grad, eps, L, iter0, S, samples, acc, dH, stream);
}
int hmc_adapt(hmc_ctx* ctx, float* theta, double* logp, float* grad, double eps0, int32_t L, int64_t iter0,
              int32_t n_adapt, double delta, double* eps_bar, uint8_t* acc, double* dH, void* stream) {
  if (!eps_bar) {
    g_err = "config: eps_bar must be non-NULL";
    return HMC_E_CONFIG;
  }
  return run_traj(ctx, theta, logp, grad, eps0, L, iter0, n_adapt, nullptr, acc, dH, stream, 1, delta, eps_bar);
}

int hmc_predict(hmc_ctx* ctx, const float* samples, int64_t S, double* mean, double* var, void* stream) {
  NvtxRange nvtx_("hmc_predict");
  API_BEGIN(ctx)
  CFG(samples && mean && var && S >= 1, "samples, mean, var must be non-NULL and S >= 1");
  CFG(ctx->mode != HMC_MODE_DATA || ctx->world == 1, "hmc_predict runs on one rank's data (not DATA mode)");
  cudaStream_t us = (cudaStream_t)stream;
  hmc_ctx* x = ctx;
  sync_in(x, us, err);
  const int64_t N = x->kind == HMC_MLP ? x->n : x->n_c * x->n_x;
  const int C = x->C;
  DevBuf tmp;
  auto tmp_alloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    CK(cudaMalloc(&p, bytes));
    tmp.ptrs.push_back(p);
    return p;
  };
  const float* dsamp = samples;
  if (!is_device_ptr(samples)) {
    float* d = (float*)tmp_alloc((size_t)S * x->k * 4);
    CK(cudaMemcpyAsync(d, samples, (size_t)S * x->k * 4, cudaMemcpyHostToDevice, x->st));
    dsamp = d;
  }
  double* dsum = (double*)tmp_alloc((size_t)N * 8);
  double* dsq = (double*)tmp_alloc((size_t)N * 8);
  double* dmean = (double*)tmp_alloc((size_t)N * 8);
  double* dvar = (double*)tmp_alloc((size_t)N * 8);
  CK(cudaMemsetAsync(dsum, 0, (size_t)N * 8, x->st));
  CK(cudaMemsetAsync(dsq, 0, (size_t)N * 8, x->st));
  const size_t Ck = (size_t)C * x->k;
  for (int64_t s0 = 0; s0 < S; s0 += C) {
    const int nb = (int)std::min<int64_t>(C, S - s0);
    // batch of samples -> the chains' parameters (missing chains repeat the last sample)
    for (int c = 0; c < C; ++c) {
      const int64_t src = s0 + std::min(c, nb - 1);
      CK(cudaMemcpyAsync(x->wrk_theta + (size_t)c * x->k, dsamp + src * x->k, x->k * 4, cudaMemcpyDeviceToDevice,
                         x->st));
    }
    k_scatter<<<dim3((unsigned)std::min<int64_t>((x->k + 255) / 256, 1024), x->C), 256, 0, x->st>>>(x->kstate(), x->wrk_theta);
    (void)Ck;
    if (x->kind == HMC_MLP) {
      NetInfo& Nn = x->nets[0];
      const int nl = (int)Nn.layers.size();
      for (int i = 0; i < nl - 1; ++i) enqueue_forward_hidden(x, Nn, i, x->st);
      LayerInfo& O = x->layers[Nn.layers[nl - 1]];
      int64_t s_in;
      const float* in = layer_input(x, Nn, nl - 1, &s_in);
      k_out_fwd<<<dim3(x->n_part, C), 256, O.n_in * sizeof(float), x->st>>>(
          in, s_in, O.n_in, O.rows, x->Wd, x->P, O.w_off, O.b_off, nullptr, x->R, 0.0, x->part_sq, x->n_part);
    } else {
      for (int ni = 0; ni < 2; ++ni)
        for (int i = 0; i < (int)x->nets[ni].layers.size(); ++i) enqueue_forward_hidden(x, x->nets[ni], i, x->st);
      const LayerInfo& Bl = x->layers[x->nets[0].layers.back()];
      const LayerInfo& Tl = x->layers[x->nets[1].layers.back()];
      const int p = Bl.n_out;
      if (x->unaligned) {  // F per pair (no residual), b0 added by k_pred_accum
        k_pair_combine<<<dim3((unsigned)x->n_c, C), 256, p * sizeof(float), x->st>>>(
            Bl.A, Tl.A, p, x->n_c, x->n_x, nullptr, nullptr, 0, 0.0, x->R, nullptr, nullptr, 0);
      } else {
        GemmArgs a = gemm_base((int)x->n_c, (int)x->n_x, p, C);
        a.A = Bl.A; a.lda = p; a.sA = x->n_c * p;
        a.B = Tl.A; a.ldb = p; a.sB = x->n_x * p;
        a.C = x->R; a.ldc = x->n_x; a.sC = x->n_c * x->n_x;
        a.epi = EPI_STORE;
        launch_gemm(x, a, true, true, x->st, "predict");
      }
    }
    k_pred_accum<<<148 * 4, 256, 0, x->st>>>(x->R, N, nb, x->Wd, x->P, x->has_b0 ? x->b0_off : -1, dsum, dsq);
    CK(cudaGetLastError());
  }
  k_pred_final<<<148 * 4, 256, 0, x->st>>>(dsum, dsq, N, (double)S, dmean, dvar);
  CK(cudaMemcpyAsync(mean, dmean, (size_t)N * 8, cudaMemcpyDefault, x->st));
  CK(cudaMemcpyAsync(var, dvar, (size_t)N * 8, cudaMemcpyDefault, x->st));
  CK(cudaStreamSynchronize(x->st));  // temporaries are freed on return
  sync_out(x, us, true, err);
  API_END
}

int hmc_partition(const double* s2, int64_t P, double tau, int32_t rule, int32_t* active, int64_t* n_hat,
                  void* stream) {
  if (!s2 || !active || !n_hat || P < 1 || P > 0x7fffffffLL || !(tau > 0.0 && tau <= 1.0) || (rule != 0 && rule != 1)) {
    g_err = "config: s2, active, n_hat non-NULL; 1 <= P < 2^31; 0 < tau <= 1; rule 0 (ge) or 1 (le)";
    return HMC_E_CONFIG;
  }
  std::string err;
  DevBuf tmp;
  auto tmp_alloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    tmp.ptrs.push_back(p);
    return p;
  };
  cudaStream_t st = (cudaStream_t)stream;
  int64_t n2 = 1;
  while (n2 < P) n2 <<= 1;
  const int64_t nch = (P + part::CH - 1) / part::CH;
  double* ds2 = (double*)tmp_alloc((size_t)P * 8);
  double* key = (double*)tmp_alloc((size_t)n2 * 8);
  int32_t* idx = (int32_t*)tmp_alloc((size_t)n2 * 4);
  unsigned long long* res = (unsigned long long*)tmp_alloc(16);
  int32_t* flag = (int32_t*)tmp_alloc((size_t)P * 4);
  int64_t* cnt = (int64_t*)tmp_alloc((size_t)(nch + 1) * 8);
  int32_t* out = (int32_t*)tmp_alloc((size_t)P * 4);
  if (!ds2 || !key || !idx || !res || !flag || !cnt || !out) { g_err = "cuda: out of device memory"; return HMC_E_OOM; }
  auto ck = [&](cudaError_t e) { if (e != cudaSuccess && err.empty()) err = cudaGetErrorString(e); };
  ck(cudaMemcpyAsync(ds2, s2, (size_t)P * 8, cudaMemcpyDefault, st));
  const unsigned long long init[2] = {(unsigned long long)P, 0ull};
  ck(cudaMemcpyAsync(res, init, 16, cudaMemcpyHostToDevice, st));
  ck(cudaMemsetAsync(flag, 0, (size_t)P * 4, st));
  const unsigned g = (unsigned)std::min<int64_t>((n2 + 255) / 256, 148 * 16);
  part::k_init<<<g, 256, 0, st>>>(ds2, P, n2, key, idx);
  for (int64_t kk = 2; kk <= n2; kk <<= 1)
    for (int64_t j = kk >> 1; j > 0; j >>= 1) part::k_bitonic<<<g, 256, 0, st>>>(key, idx, n2, j, kk);
  const unsigned gc = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nch + 127) / 128, 148 * 4));
  double* prefix = ds2;  // (s2 is no longer needed: the keys hold the ranked copy)
  part::k_prefix_seq<<<1, 1, 0, st>>>(key, P, prefix);
  unsigned long long hres[2] = {0ull, 0ull};
  double tot = 0.0;
  ck(cudaMemcpyAsync(&tot, prefix + P - 1, 8, cudaMemcpyDeviceToHost, st));
  ck(cudaStreamSynchronize(st));
  if (tot > 0.0) part::k_nhat_seq<<<g, 256, 0, st>>>(prefix, P, tau, rule, res);
  ck(cudaMemcpyAsync(hres, res, 16, cudaMemcpyDeviceToHost, st));
  ck(cudaStreamSynchronize(st));
  if (!err.empty()) { g_err = "cuda: " + err; return HMC_E_CUDA; }
  const int64_t nh = !(tot > 0.0) ? 0 : (rule == 0 ? (int64_t)hres[0] : (int64_t)hres[1]);
  if (nh > 0) {
    part::k_flags<<<g, 256, 0, st>>>(idx, nh, flag);
    part::k_flag_count<<<gc, 128, 0, st>>>(flag, P, cnt, nch);
    part::k_count_scan<<<1, 1, 0, st>>>(cnt, nch);
    part::k_compact<<<gc, 128, 0, st>>>(flag, P, cnt, nch, out);
    ck(cudaMemcpyAsync(active, out, (size_t)nh * 4, cudaMemcpyDefault, st));
  }
  ck(cudaStreamSynchronize(st));
  ck(cudaGetLastError());
  if (!err.empty()) { g_err = "cuda: " + err; return HMC_E_CUDA; }
  *n_hat = nh;
  return HMC_OK;
}

int hmc_diagnostics(const float* samples, int32_t C, int64_t S, int64_t k, double* rhat, double* ess, void* stream) {
  if (!samples || !rhat || !ess || C < 1 || C > 1024 || S < 4 || k < 1) {
    g_err = "config: samples, rhat, ess non-NULL; 1 <= C <= 1024, S >= 4, k >= 1";
    return HMC_E_CONFIG;
  }
  std::string err;
  hmc_ctx dummy;
  hmc_ctx* x = &dummy;
  try {
    cudaStream_t st = (cudaStream_t)stream;
    const size_t tot = (size_t)C * S * k;
    const float* d = samples;
    if (!is_device_ptr(samples)) {
      float* t = dalloc<float>(x, tot, err);
      CK(cudaMemcpyAsync(t, samples, tot * 4, cudaMemcpyHostToDevice, st));
      d = t;
    }
    double* dr = dalloc<double>(x, (size_t)k, err);
    double* de = dalloc<double>(x, (size_t)k, err);
    const int grid = (int)std::min<int64_t>(k, 148 * 8);
    k_diag<<<grid, DIAG_T, 0, st>>>(d, C, S, k, dr, de);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(rhat, dr, (size_t)k * 8, cudaMemcpyDefault, st));
    CK(cudaMemcpyAsync(ess, de, (size_t)k * 8, cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
  } catch (Fail f) {
    g_err = err;
    return f.code;
  }
  return HMC_OK;
}

int hmc_sensitivity(const hmc_arch* arch, const hmc_data* data, const float* mu, const float* sigma_vi,
                    double* s2, void* stream) {
  NvtxRange nvtx_("hmc_sensitivity");
  if (!arch || !data || !mu || !sigma_vi || !s2) {
    g_err = "config: arch, data, mu, sigma_vi and s2 must be non-NULL";
    return HMC_E_CONFIG;
  }
  std::unique_ptr<hmc_ctx> x(new hmc_ctx());
  std::string& err = x->err;
  try {
    CFG(arch->kind != HMC_DEEPONET || !data->q_per_pair,
        "hmc_sensitivity: the unaligned DeepONet (q_per_pair) is not supported (its Gram-seed "
        "factorisation needs shared query points)");
    // P from the architecture (the same walk setup_impl validates)
    int64_t P = 0;
    for (int ni = 0; ni < (arch->kind == HMC_DEEPONET ? 2 : 1); ++ni) {
      const hmc_net& nt = arch->net[ni];
      CFG(nt.n_layers >= 1 && nt.widths && nt.acts && nt.has_bias, "net description incomplete");
      for (int l = 0; l < nt.n_layers; ++l)
        P += (int64_t)nt.widths[l] * nt.widths[l + 1] + (nt.has_bias[l] ? nt.widths[l + 1] : 0);
    }
    if (arch->kind == HMC_DEEPONET && arch->has_b0) P += 1;
    std::vector<int32_t> idx((size_t)P);
    for (int64_t j = 0; j < P; ++j) idx[j] = (int32_t)j;
    const std::vector<float> hmu = to_host(mu, (size_t)P, err);
    const std::vector<float> hsig = to_host(sigma_vi, (size_t)P, err);
    for (float v : hsig) CFG(std::isfinite(v) && v >= 0.f, "sigma_vi must be finite and >= 0");
    const int p = arch->kind == HMC_DEEPONET ? arch->net[0].widths[arch->net[0].n_layers] : 1;
    CFG(arch->kind != HMC_DEEPONET || p <= 1024, "DeepONet output width > 1024");
    hmc_config cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.frozen = hmu.data();
    cfg.idx = idx.data();
    cfg.P = P;
    cfg.k = P;
    cfg.noise_sigma = 1.0;
    cfg.prior_sigma = 1.0;
    cfg.n_chains = arch->kind == HMC_DEEPONET ? p : 1;
    cfg.mode = HMC_MODE_SINGLE;
    cfg.world = 1;
    setup_impl(x.get(), arch, data, &cfg, err, false);  // (the per-layer engines' squared-operand mode)
    enqueue_sensitivity(x.get(), err);
    float* dsig = dalloc<float>(x.get(), (size_t)P, err);
    double* dout = dalloc<double>(x.get(), (size_t)P, err);
    CK(cudaMemcpyAsync(dsig, hsig.data(), (size_t)P * 4, cudaMemcpyHostToDevice, x->st));
    const double n_d = x->kind == HMC_MLP ? (double)x->n : (double)x->n_c * (double)x->n_x;
    k_sens_finalize<<<148 * 4, 256, 0, x->st>>>(x->gl, x->C, P, dsig, n_d, x->has_b0 ? x->b0_off : -1, dout);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(s2, dout, (size_t)P * 8, cudaMemcpyDefault, x->st));
    CK(cudaStreamSynchronize(x->st));
    (void)stream;
  } catch (Fail f) {
    g_err = err;
    return f.code;
  }
  return HMC_OK;
}

int hmc_destroy(hmc_ctx* ctx) {
  if (!ctx) return HMC_OK;
  cudaSetDevice(ctx->dev);
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  delete ctx;
  return HMC_OK;
}

const char* hmc_last_error(const hmc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int hmc_launch_counts(const hmc_ctx* ctx, int64_t* per_grad, int64_t* per_traj_base, int64_t* per_step) {
  if (!ctx) { g_err = "NULL context"; return HMC_E_STATE; }
  hmc_ctx* x = const_cast<hmc_ctx*>(ctx);
  if (!x->grad_exec) {
    // count without executing: the body's launch count is static for a context
    std::string& err = x->err;
    try {
      CK(cudaSetDevice(x->dev));
      build_grad_graph(x, err);
    } catch (Fail f) {
      return f.code;
    }
  }
  if (x->narrow) {  // scatter + the cluster kernel; begin + one kernel for all steps + MH + advance
    if (per_grad) *per_grad = 2;
    if (per_traj_base) *per_traj_base = 4;
    if (per_step) *per_step = 0;
    return HMC_OK;
  }
  if (per_grad) *per_grad = x->per_body + 3;
  if (per_traj_base) *per_traj_base = 3;
  if (per_step) *per_step = x->per_body + 2;
  return HMC_OK;
}

int hmc_philox_words(uint64_t seed, uint32_t tag, uint32_t iter, uint32_t chain, int64_t nblocks, uint32_t* out,
                     void* stream) {
  if (!out || nblocks < 0) { g_err = "bad arguments"; return HMC_E_CONFIG; }
  cudaStream_t st = (cudaStream_t)stream;
  const bool dev = is_device_ptr(out);
  uint32_t* d = out;
  if (!dev && cudaMalloc(&d, (size_t)nblocks * 16 + 16) != cudaSuccess) { g_err = "cudaMalloc"; return HMC_E_OOM; }
  k_philox_words<<<148 * 4, 256, 0, st>>>((uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32), tag, iter, chain,
                                          nblocks, d);
  cudaError_t e = cudaGetLastError();
  if (!dev) {
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, (size_t)nblocks * 16, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d);
  }
  if (e != cudaSuccess) { g_err = cudaGetErrorString(e); return HMC_E_CUDA; }
  return HMC_OK;
}

int hmc_momentum(hmc_ctx* ctx, int64_t iter, float* p, void* stream) {
  API_BEGIN(ctx)
  CFG(p && iter >= 0 && iter < ((int64_t)1 << 32), "p non-NULL, 0 <= iter < 2^32");
  cudaStream_t us = (cudaStream_t)stream;
  const bool host = !is_device_ptr(p);
  sync_in(ctx, us, err);
  k_momentum<<<ctx->C, KT, 0, ctx->st>>>(ctx->kstate(), (uint32_t)iter, ctx->p);
  CK(cudaGetLastError());
  cpy(p, ctx->p, (size_t)ctx->C * ctx->k * 4, ctx->st, err);
  sync_out(ctx, us, host, err);
  API_END
}

const char* hmc_engine_info(const hmc_ctx* ctx) { return ctx ? ctx->engine.c_str() : ""; }

// dev build (-DHMC_DEV): narrow-engine phase cycles of CTA 0 (fwd, output, backward, barrier 1,
// reduction + update, barrier 2, tail), summed since the last reset
int hmc_debug_nw_profile(uint64_t* out, int32_t reset) {
#ifdef HMC_DEV
  unsigned long long h[10];
  if (cudaMemcpyFromSymbol(h, nw::g_nwprof, sizeof(h)) != cudaSuccess) return HMC_E_CUDA;
  if (out) for (int i = 0; i < 10; ++i) out[i] = h[i];
  if (reset) {
    memset(h, 0, sizeof(h));
    if (cudaMemcpyToSymbol(nw::g_nwprof, h, sizeof(h)) != cudaSuccess) return HMC_E_CUDA;
  }
  return HMC_OK;
#else
  (void)out; (void)reset;
  g_err = "hmc_debug_nw_profile needs a -DHMC_DEV build (make DEV=1)";
  return HMC_E_STATE;
#endif
}

// Test hook: one DATA-mode gradient evaluation split at its cross-rank steps, for contexts set
// up with hmc_config.exchange = 1 (no communicator).  The caller runs phase p on every rank's
// context and performs the collective between phases itself (include/hmc.h).
int hmc_debug_data_phase(hmc_ctx* ctx, int32_t phase, const void* in, const void* in2, void* out, void* out2,
                         void* stream) {
  API_BEGIN(ctx)
  (void)stream;
  CFG(ctx->emulated, "hmc_debug_data_phase needs a DATA-mode context set up with exchange = 1");
  CFG(phase >= 0 && phase <= 3, "phase must be 0..3");
  hmc_ctx* x = ctx;
  cudaStream_t st = x->st;
  const size_t Ck = (size_t)x->C * x->k;
  const int p = x->kind == HMC_DEEPONET ? x->layers[x->nets[0].layers.back()].n_out : 0;
  const size_t blk = (size_t)x->C * x->n_c_loc * p;
  NetInfo& Nb = x->nets[0];
  const size_t xcblk = (size_t)Nb.nch * x->n_c * p;  // POINTS_XC: this rank's chain block of branch outputs
  auto reduce_out = [&]() {
    k_reduce_partials<<<x->C, KT, 0, st>>>(x->part_sq, x->part_r, x->n_part, x->lik, x->gl, x->k, x->b0_slot);
    cpy(out, x->gl, Ck * 4, st, err);
    cpy(out2, x->lik, (size_t)x->C * 8, st, err);
  };
  if (phase == 0) {
    CFG(in && out && (x->xb || x->xc || out2), "phase 0: theta in; out (and out2 for the row layout)");
    cpy(x->wrk_theta, in, Ck * 4, st, err);
    k_scatter<<<dim3((unsigned)std::min<int64_t>((x->k + 255) / 256, 1024), x->C), 256, 0, st>>>(x->kstate(), x->wrk_theta);
    if (x->xb || x->xc) {  // forward of both nets; out = this rank's branch outputs (the all-gather's input)
      for (int ni = 0; ni < 2; ++ni)
        for (int i = 0; i < (int)x->nets[ni].layers.size(); ++i) enqueue_forward_hidden(x, x->nets[ni], i, st);
      cpy(out, x->layers[Nb.layers.back()].A, (x->xc ? xcblk : blk) * 4, st, err);
    } else {      // row layout: the whole local evaluation; out = g_lik [C x k], out2 = sum r^2 [C]
      enqueue_body(x, st);
      reduce_out();
    }
  } else if (phase == 1 && x->xc) {
    CFG(in && out, "phase 1 (POINTS_XC): in = all-gathered branch outputs, out = reduce-scatter input");
    cpy(x->xc_Ball, in, xcblk * x->world * 4, st, err);
    xb_combine(x, st, x->xc_Ball);
    if (Nb.l_min >= 0) {
      xb_dB(x, st, x->xc_Ball, x->xc_dB);
      cpy(out, x->xc_dB, xcblk * x->world * 4, st, err);
    } else {
      CK(cudaMemsetAsync(out, 0, xcblk * x->world * 4, st));
    }
  } else if (phase == 2 && x->xc) {
    CFG(in && out && out2, "phase 2 (POINTS_XC): in = reduce-scattered dB block, out / out2 = g_lik / sum r^2");
    NetInfo& Nt = x->nets[1];
    if (Nb.l_min >= 0) {
      cpy(Nb.G[0], in, xcblk * 4, st, err);
      enqueue_backward_net(x, Nb, (int)Nb.layers.size() - 1, 0, st);
    }
    if (Nt.l_min >= 0) {
      xb_dT(x, st, x->xc_Ball);
      enqueue_backward_net(x, Nt, (int)Nt.layers.size() - 1, 0, st);
    }
    reduce_out();
  } else if (phase == 1) {
    CFG(x->xb && in && out, "phase 1 (POINTS_XB): in = all-gathered branch outputs, out = reduce-scatter input");
    cpy(x->xb_recv, in, blk * x->world * 4, st, err);
    xb_mid(x, st);
    if (Nb.l_min >= 0) cpy(out, x->xb_send, blk * x->world * 4, st, err);
    else CK(cudaMemsetAsync(out, 0, blk * x->world * 4, st));
  } else if (phase == 2) {
    CFG(x->xb && in && out && out2, "phase 2 (POINTS_XB): in = reduce-scattered dB block, out / out2 = g_lik / sum r^2");
    if (Nb.l_min >= 0) cpy(Nb.G[0], in, blk * 4, st, err);
    xb_back(x, st);
    reduce_out();
  } else {
    CFG(in && in2 && out && out2, "phase 3: in / in2 = summed g_lik / sum r^2, out / out2 = grad / logp");
    cpy(x->xc ? x->gl_red : x->gl, in, Ck * 4, st, err);
    cpy(x->lik, in2, (size_t)x->C * 8, st, err);
    k_finalize<<<x->C, KT, 0, st>>>(x->kstate(), 0);
    cpy(out, x->wrk_grad, Ck * 4, st, err);
    cpy(out2, x->wrk_logp, (size_t)x->C * 8, st, err);
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  API_END
}

// Test hook: the POINTS_XB permutations alone: dir 0 = k_xb_gather ([rank][chain][i][k] ->
// [chain][rank n_loc + i][k]), dir 1 = k_xb_scatter (the inverse); device pointers, synchronous.
int hmc_debug_xb_permute(int32_t dir, int32_t C, int32_t G, int64_t n_loc, int32_t p, const float* in, float* out,
                         void* stream) {
  if (!in || !out || C < 1 || G < 1 || n_loc < 1 || p < 1 || (dir != 0 && dir != 1)) {
    g_err = "config: in / out non-NULL, C, G, n_loc, p >= 1, dir 0 or 1";
    return HMC_E_CONFIG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (dir == 0) k_xb_gather<<<148 * 4, 256, 0, st>>>(in, out, C, G, n_loc, p);
  else k_xb_scatter<<<148 * 4, 256, 0, st>>>(in, out, C, G, n_loc, p);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) { g_err = cudaGetErrorString(e); return HMC_E_CUDA; }
  return HMC_OK;
}

int hmc_debug_set_engine(int32_t mode) {
  if (mode < 0 || mode > 4) {
    g_err = "config: engine mode must be 0 (automatic), 1 (per-layer SIMT only), 2 (per-layer engines), 3 "
            "(narrow engine in cluster mode only) or 4 (masked weight gradient wherever it applies)";
    return HMC_E_CONFIG;
  }
  engine_override() = mode;
  return HMC_OK;
}

int hmc_divergences(hmc_ctx* ctx, uint32_t* counts, int32_t reset) {
  API_BEGIN(ctx)
  CFG(counts, "counts must be non-NULL");
  CK(cudaStreamSynchronize(ctx->st));
  CK(cudaMemcpy(counts, ctx->d_div, (size_t)ctx->C * 4, cudaMemcpyDefault));
  if (reset) CK(cudaMemset(ctx->d_div, 0, (size_t)ctx->C * 4));
  API_END
}

int hmc_debug_gemm(int32_t engine, int32_t a_kmajor, int32_t b_kmajor, int32_t M, int32_t N, int32_t K,
                   int32_t batch, const float* A, int64_t lda, int64_t sA, const float* B, int64_t ldb, int64_t sB,
                   float* C, int64_t ldc, int64_t sC, void* stream) {
  static TcPlanner tcp;
  static bool init = false;
  if (!init) {
    tcp.init();
    init = true;
  }
  GemmArgs a = gemm_base(M, N, K, batch);
  a.A = A; a.lda = lda; a.sA = sA; a.B = B; a.ldb = ldb; a.sB = sB; a.C = C; a.ldc = ldc; a.sC = sC;
  cudaStream_t st = (cudaStream_t)stream;
  if (engine == 1) {
    if (!tcp.accepts(a, a_kmajor != 0, b_kmajor != 0)) {
      g_err = "tcgen05 engine does not take this GEMM";
      return HMC_E_CONFIG;
    }
    const cudaError_t e = tcp.launch(a, a_kmajor != 0, b_kmajor != 0, st);
    if (e != cudaSuccess) {
      g_err = std::string("tcgen05 launch failed: ") + cudaGetErrorString(e);
      return HMC_E_CUDA;
    }
  } else {
    hmc_ctx dummy;
    launch_gemm_simt(&dummy, a, a_kmajor != 0, b_kmajor != 0, st);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = cudaGetErrorString(e);
    return HMC_E_CUDA;
  }
  return HMC_OK;
}

// dev diagnostics: per-role barrier wait cycles of the tcgen05 engine (HMC_TC_PROF=1), summed
// over CTAs since the last reset; out[16 x 16] ([kernel variant][slot], slots: tc::TcProf)
int hmc_debug_tc_profile(uint64_t* out, int32_t reset) {
  unsigned long long h[16 * 16];
  if (cudaMemcpyFromSymbol(h, tc::g_tcprof, sizeof(h)) != cudaSuccess) return HMC_E_CUDA;
  if (out) for (int i = 0; i < 16 * 16; ++i) out[i] = h[i];
  if (reset) {
    memset(h, 0, sizeof(h));
    if (cudaMemcpyToSymbol(tc::g_tcprof, h, sizeof(h)) != cudaSuccess) return HMC_E_CUDA;
  }
  return HMC_OK;
}

// dev diagnostics: CTA-0 timeline of the last tcgen05 GEMM run with HMC_TC_PROF=2, out[24 x 256]
int hmc_debug_tc_timeline(uint64_t* out) {
  if (cudaMemcpyFromSymbol(out, tc::g_tctl, sizeof(unsigned long long) * 24 * tc::TL_N) != cudaSuccess) return HMC_E_CUDA;
  return HMC_OK;
}

int hmc_profile(hmc_ctx* ctx, int32_t enable) {
  API_BEGIN(ctx)
  if ((enable != 0) != ctx->prof_on) {
    ctx->prof_on = enable != 0;
    if (ctx->traj_exec) {
      CK(cudaStreamSynchronize(ctx->st));
      cudaGraphExecDestroy(ctx->traj_exec);
      ctx->traj_exec = nullptr;
      ctx->traj_L = -1;
    }
  }
  API_END
}

int hmc_profile_read(hmc_ctx* ctx, int32_t max_recs, hmc_prof_rec* out, int32_t* n_out) {
  API_BEGIN(ctx)
  CFG(n_out && (out || max_recs == 0), "n_out must be non-NULL");
  CK(cudaStreamSynchronize(ctx->st));
  const int n = (int)ctx->prof.size();
  *n_out = n;
  for (int i = 0; i < n && i < max_recs; ++i) {
    const auto& r = ctx->prof[i];
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) {
      cudaGetLastError();
      ms = -1.f;
    }
    memset(out[i].name, 0, sizeof(out[i].name));
    strncpy(out[i].name, r.name.c_str(), sizeof(out[i].name) - 1);
    out[i].ms = ms;
    out[i].flops = r.flops;
    out[i].bytes = r.bytes;
    out[i].step = r.step;
  }
  API_END
}

}  // extern "C"
