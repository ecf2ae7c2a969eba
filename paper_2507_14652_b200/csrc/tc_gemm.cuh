// tcgen05 3xTF32 GEMM engine for the wide layers (libhmc, sm_100a only).
//
// C[b] = A[b] . B[b] with FP32 accuracy from three TF32 tensor-core products per K step:
//   A = Ah + Al, B = Bh + Bl, Ah = rna_tf32(A), Al = A - Ah (exact in fp32),
//   C ~= Al.Bh + Ah.Bl + Ah.Bh   (1xTF32 misses the 1e-5 gradient
//   tolerance, 3xTF32 meets it).  Raw (activation) B planes keep hi = the raw word (the tensor
//   core truncates a tf32 operand) and lo = rna_tf32(B - trunc(B)) beside it.
// Accumulation: the tensor core truncates its fp32 accumulator toward zero after every MMA
// (measured on B200, scripts/probe_tc_rounding.py: 1 + 1.5*2^-24 -> 1.0; 1.7e-4 relative at
// K = 16384).  Each chunk of TC_FOLD (2) K blocks of 32 accumulates in its own TMEM buffer - the
// small products of the chunk first, then its big products - and the epilogue warps fold the
// chunk partials into fp32 registers with round-to-nearest adds; two chunk buffers ping-pong so
// the MMAs of one chunk overlap the fold of the previous.
// Structure (persistent, one 512-thread CTA per SM, CTA pairs running cta_group::2 MMAs with
// M = 256 = 128 rows per CTA; each CTA holds half of the B tile):
//   warps 0-7  : epilogue  - fold (tcgen05.ld 32x32b) into BN/2 fp32 registers per thread (warp
//                w: TMEM lane quadrant w%4 = 32 tile rows, one column half), then the fused
//                epilogue (bias + tanh / act' / residual^2 / masked weight-gradient compaction
//                and bias gradient); outputs staged through 128B-swizzled smem tiles and written
//                with TMA bulk tensor stores; in the weight-gradient layout they also split the
//                raw B planes
//   warps 8-11 : converters - A rows split into hi/lo and written to TMEM (tcgen05.st); raw B
//                planes of the other layouts split in shared memory
//   warp 12/13 : TMA producers of the A ring and the B ring
//   warp 14/15 : MMA issuers of the leader CTA (alternate chunks); warp 14 allocates TMEM and,
//                in the peer CTA, relays "pre-split B half landed" to the leader
// Operand layouts: K-major or MN-major (any width: 32-wide blocks, zero-filled tails); weights
// arrive pre-split (hi/lo planes written by the scatter kernel); stride-0 operands shared by all
// batch entries; the weight gradient may split K over CTA pairs (fixed-order partial sums).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "gemm_simt.cuh"

namespace hmc {
namespace tc {

constexpr int BM = 128;    // tile rows per CTA (the pair MMA has M = 2 * BM)
constexpr int BK = 32;     // fp32 elements per K block (one 128-byte swizzle row)
constexpr int NCONV = 4;   // converter warps: one per TMEM lane quadrant (A rows -> TMEM)
constexpr int NEPI = 8;    // epilogue warps
constexpr int NT = (4 + NCONV + NEPI) * 32;  // 512 threads
// Warp roles.  The warp schedulers favour higher warp ids, so the latency-critical single-lane
// roles get the highest ids: epilogue 0-7, converters 8-11, A producer 12, B producer 13, MMA
// issuers 14 (even chunks) and 15 (odd chunks): while one issuer is blocked feeding the
// tensor pipe its chunk, the other has already passed the barriers of the next one, so the
// pipe does not drain between chunks.
constexpr int W_EPI0 = 0, W_CONV0 = NEPI, W_TMA_A = NEPI + NCONV, W_TMA_B = W_TMA_A + 1, W_MMA = W_TMA_B + 1,
              W_MMA2 = W_MMA + 1;
constexpr int STG = 4096;  // staging bytes per epilogue warp (32 rows x 32 fp32, 128B swizzle)
#ifndef TC_TANH2
#define TC_TANH2 tanh_acc2  // (tanh_mix2: 3 MUFU ops per pair)
#endif
#ifndef TC_FOLD
#define TC_FOLD 2  // K blocks per TMEM accumulator chunk (DESIGN.md §5 "accumulation")
#endif

// WG: the weight-gradient layout - no output staging (the epilogue writes the compacted k-vector
// from registers), the freed shared memory deepens the B ring, whose raw planes the epilogue
// warps split (they are idle between folds there; the converters keep A only)
template <int BN, bool WG = false>
struct Cfg {
#ifndef TC_SA
#define TC_SA 4
#endif
#ifndef TC_SB
#define TC_SB 6
#endif
#ifndef TC_SA_WG
#define TC_SA_WG 4
#endif
#ifndef TC_SB_WG
#define TC_SB_WG 10
#endif
  static constexpr int SA = WG ? TC_SA_WG : TC_SA;      // raw A ring (released by the converters)
  static constexpr int SB = WG ? TC_SB_WG : TC_SB;      // B ring (released by the MMA)
  static constexpr int A_BYTES = BM * BK * 4;           // raw fp32 A tile, 16 KB
  static constexpr int B_BYTES = (BN / 2) * BK * 4;     // this CTA's half of one B plane, 8 KB
  static constexpr int B_STAGE = 2 * B_BYTES;           // hi + lo planes
#ifndef TC_NACC
#define TC_NACC 2
#endif
  static constexpr int NACC = TC_NACC;                  // TMEM K-block accumulators (BN columns each)
  static constexpr int NAS = (512 - NACC * BN) / 64;    // TMEM A slots: [hi 32 | lo 32] columns each
  static constexpr int A_COL0 = NACC * BN;
  static_assert(NACC * BN + NAS * 64 <= 512, "TMEM budget");
  static constexpr int NC = BN / 2;                     // fp32 columns per epilogue thread
  static constexpr int NGRP = NC / 32;                  // 32-column groups per epilogue thread
  static constexpr int B_OFF = SA * A_BYTES;
  static constexpr int STG_OFF = B_OFF + SB * B_STAGE;
  static constexpr int STG_BYTES = WG ? 0 : NEPI * NGRP * STG;
  static constexpr int BAR_BYTES = 1024;
  static constexpr int SMEM = 1024 /*align*/ + STG_OFF + STG_BYTES + BAR_BYTES;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

// ---------------------------------------------------------------- PTX wrappers (sm_100a) ---
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
#ifndef TC_WAIT_MODE
#define TC_WAIT_MODE 1
#endif
// TC_WAIT_MODE 0: try_wait with the default (system-dependent) suspend time;
//              1: try_wait with a short suspend-time hint, so a sleeping waiter re-checks soon
//                 after an async-proxy completion (tcgen05.commit / TMA complete_tx);
//              2: test_wait spin (no suspension)
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity, uint32_t hint = 20) {
#if TC_WAIT_MODE == 0
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
#elif TC_WAIT_MODE == 1
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity), "r"(hint)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
#endif
}
// Optional per-role stall accounting (dev diagnostics, hmc_debug_tc_profile): cycles each role
// spends waiting on each barrier, summed over CTAs.  Slots: see TcProf below.
enum TcProf : int { P_TMA_EMPTY = 0, P_MMA_TEMPTY, P_MMA_FULLOP, P_CONV_RAW, P_CONV_AFREE, P_EPI_TFULL, P_EPI_XFULL,
                    P_EPI_OUT, P_TOTAL, P_CONV_B, P_BTMA_EMPTY, P_MMA_ISSUE, P_NPROF };
__device__ unsigned long long g_tcprof[16][16];  // [kernel variant][slot]
// timeline of CTA 0 (prof == 2): [event][k block], events: 0 MMA loop top, 1 tempty ok,
// 2 full_op ok, 3 issued, 4 epilogue tfull ok, 5 epilogue folded, 6 converter full (A) ok,
// 7 converter arrive full_op
constexpr int TL_N = 256;
__device__ unsigned long long g_tctl[24][TL_N];
// try_wait without a suspend-time hint: the thread sleeps for the hardware's own time limit per
// attempt (fewer issued instructions while waiting; slower wake-up after async-proxy arrivals)
__device__ __forceinline__ void mbar_wait_block(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_t(uint64_t* b, uint32_t parity, bool on, unsigned long long& acc,
                                            uint32_t hint = 20) {
  if (!on) {
    if (hint == 0) mbar_wait_block(b, parity);  // hint 0: blocking form
    else mbar_wait(b, parity, hint);
    return;
  }
  const unsigned long long t0 = clock64();
  mbar_wait(b, parity, hint);
  acc += clock64() - t0;
}

__device__ __forceinline__ void tma_prefetch(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)m) : "memory");
}
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          su32(dst)),
      "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// one lane of a converged warp returns true (elect.sync)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred %%px;\n"
      "elect.sync _|%%px, %1;\n"
      "@%%px mov.s32 %0, 1;\n"
      "}\n"
      : "+r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// CTA-pair TMEM (one warp of each CTA of the pair executes these)
__device__ __forceinline__ void tmem_alloc2(uint32_t* holder, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(holder)), "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}
// pair MMA (issued by the leader CTA only): D (M = 256: 128 rows in each CTA's TMEM) (+)=
// A (each CTA's TMEM, its 128 rows) . B (N columns: the first N/2 in the leader's shared memory,
// the rest at the same offset in the peer's)
__device__ __forceinline__ void mma2_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accum));
}
// pair commit: arrives on the barrier at `bar`'s offset in both CTAs once the leader's prior pair
// MMAs have completed
__device__ __forceinline__ void mma2_commit_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          su32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// arrive on the barrier at `b`'s offset in CTA `cta` of the cluster.  Default (release, CTA
// scope) semantics: a cluster-scope release costs ~1300 clocks (measured) and is not needed -
// what the leader's MMA consumes is ordered by the tcgen05 fences (TMEM) and the async-proxy
// fence (shared memory) the arriving warps execute first
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* b, uint32_t cta) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(su32(b)), "r"(cta));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void mbar_wait_cl(uint64_t* b, uint32_t parity) { mbar_wait(b, parity); }
__device__ __forceinline__ void mbar_wait_cl_t(uint64_t* b, uint32_t parity, bool on, unsigned long long& acc) {
  if (!on) { mbar_wait_cl(b, parity); return; }
  const unsigned long long t0 = clock64();
  mbar_wait_cl(b, parity);
  acc += clock64() - t0;
}
// 32 lanes x 32 consecutive 32-bit columns from registers (lane i of the warp -> TMEM lane base + i)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%"
      "28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes x 16 consecutive 32-bit columns: thread (lane i of the warp) gets TMEM lane
// (lane base + i), columns [col, col + 16).  Caller waits with tmem_wait_ld().
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// TMA bulk tensor store smem -> global (3-D map), bulk-group completion.
__device__ __forceinline__ void tma_store3(const CUtensorMap* m, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   (uint64_t)m),
               "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// rna_tf32(x) (round to nearest, ties away) by integer rounding of the 13 dropped bits; equal to
// cvt.rna.tf32.f32 for finite x (2 instructions instead of 4); non-finite inputs stay
// non-finite in hi or lo = x - hi, so NaN / Inf still propagate through the product
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// SMEM matrix descriptor, SWIZZLE_128B, sm_100 version bit.
//  K-major : rows of 128 B (32 fp32 along K), 8-row atoms at SBO = 1024 B, LBO unused (1).
//  MN-major: 128 B = 32 fp32 along M/N, 8 K-rows per atom (SBO = 1024 B between 8-row K groups),
//            32-element M/N blocks at LBO bytes.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                          uint32_t layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;            // version (sm_100)
  d |= (uint64_t)(layout & 7) << 61; // 2 = SWIZZLE_128B, 1 = SWIZZLE_128B_BASE32B
  return d;
}

// MN-major 32-bit operands: CUTLASS allows only the 128B swizzle with 32-byte atoms
// (SWIZZLE_128B_BASE32B, TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).  Descriptor parameters are
// kernel arguments so the encoding is verified on the device (tests/test_gpu_engine.py).
struct MnDesc {
  uint32_t lbo = 4096, sbo = 512, layout = 1, kstep = 1024;
  int prof = 0;  // 1: accumulate per-role wait cycles into g_tcprof[vid]; 2 + v: also record the
                 //    CTA-0 timeline of launches of kernel variant v
  int vid = 0;   // kernel variant (index in tc_variants)
  int dbg = 0;   // dev experiments: 1 = no MMAs, 2 = no converter work, 4 = no epilogue fold (results wrong)
  // raw B planes split in shared memory: hi = the raw word in place (the tensor core reads the
  // top 19 bits of a tf32 operand, i.e. trunc(x)), lo = rna_tf32(x - trunc(x)) beside it - one
  // plane written instead of two; |B - hi - lo| <= 2^-21 |B| as with the rna split
  int btrunc = 1;
  int pdl = 1;       // programmatic dependent launch (HMC_TC_PDL=0 disables)
  int emit_lead = 1;  // emit steps end (1 + emit_lead) folds before the tile end; the act' / V
                      // prefetch of the next tile follows one fold after the last store
  int tanh_end = 1;  // EPI_FWD tanh in registers at the tile end (1; +1 % with concurrent streams) or in emit steps (0)
  // mbarrier try_wait suspend-time hints (ns) of the producers / converters / epilogue waits: a
  // spinning waiter takes issue slots from the working warps of its SM sub-partition
  uint32_t hint_p = 20, hint_c = 20, hint_e = 20;
};

// Instruction descriptor for kind::tf32 with fp32 accumulation.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4)                      // D format f32
         | (2u << 7) | (2u << 10)       // A, B format tf32
         | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// ------------------------------------------------------------------------------- kernel ---
// fp32 x 32 of one tile row (columns n0 .. n0+31) from global memory, zero outside [0, N)
__device__ __forceinline__ void load_row32(const float* __restrict__ p, int n0, int N, bool vec, float (&v)[32]) {
  if (vec && n0 + 32 <= N) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(p) + q);
      v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = (n0 + i < N) ? __ldg(p + i) : 0.f;
  }
}

// A_MN: A stored M-major (A(m,k) = A[k*lda + m]);  B_MN: B stored N-major (B(k,n) = B[k*ldb + n]);
// B_PRE: B arrives as pre-split hi/lo planes (tensor maps mB / mB2).  mC: 3-D store map of the
// output (box 32 x 32 x 1, 128B swizzle) for every epilogue except EPI_WGRAD.
// A lands raw in shared memory (K-major: 128B swizzle; M-major: no swizzle), the converter warps
// split it row by row into hi/lo TMEM columns (the MMA reads A from TMEM, so A costs no
// shared-memory bandwidth beyond one read); B is read by the MMA from shared memory.
template <int BN, bool A_MN, bool B_MN, bool B_PRE, int EPI>
__global__ void __launch_bounds__(NT, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                   const __grid_constant__ CUtensorMap mB2, const __grid_constant__ CUtensorMap mC,
                   const __grid_constant__ CUtensorMap mX, GemmArgs a, MnDesc mn) {
  using C_ = Cfg<BN, EPI == EPI_WGRAD>;
  constexpr int SA = C_::SA, SB = C_::SB, NACC = C_::NACC, NC = C_::NC, NGRP = C_::NGRP;
  // raw B planes split by the epilogue warps (EPI_WGRAD), ESPLIT_D K blocks ahead of the fold
  constexpr bool ESPLIT = (EPI == EPI_WGRAD) && !B_PRE;
  constexpr uint32_t ESPLIT_D = 2 * TC_FOLD;
  // EPI_DACT reads act'(dsrc) and EPI_RESID reads V tile by tile: TMA-loaded (mX) into the
  // staging buffers while the tile's K blocks are still in flight
  const bool loadx = (EPI == EPI_RESID) || (EPI == EPI_DACT && a.act != ACT_ID);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned base, derived from the shared array by an offset so that every access
  // below compiles to LDS/STS (a pointer rebuilt from an integer would be generic)
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sAr = smem;                  // raw A ring [SA][A_BYTES]
  uint8_t* sBr = smem + C_::B_OFF;      // B ring [SB][hi | lo]
  uint8_t* stg_base = smem + C_::STG_OFF;
  uint64_t* bar = (uint64_t*)(stg_base + C_::STG_BYTES);
  uint64_t* a_full = bar;                         // [SA]   TMA -> converters
  uint64_t* a_empty = a_full + SA;                // [SA]   converters (A read) -> A producer
  uint64_t* b_full = a_empty + SA;                // [SB]   TMA -> converters
  uint64_t* b_empty = b_full + SB;                // [SB]   MMA -> B producer
  // converters -> MMA (A in TMEM, raw B split), one per TMEM A slot: the converters run ahead
  // by at most NAS K blocks (afree), so a slot's barrier can never be two phases ahead
  uint64_t* full_op = b_empty + SB;               // [NAS]
  uint64_t* afree = full_op + C_::NAS;            // [NAS]  MMA -> converters (TMEM A slot free)
  uint64_t* tfull = afree + C_::NAS;              // [NACC] MMA -> epilogue (K-block partial ready)
  uint64_t* tempty = tfull + NACC;                // [NACC] epilogue -> MMA (partial folded)
  uint64_t* xfull = tempty + NACC;                // [NEPI] per epilogue warp: mX tiles landed
  uint64_t* bsplit = xfull + NEPI;                // [SB]   epilogue (raw B split) -> MMA (ESPLIT)
  uint32_t* tmem_holder = (uint32_t*)(bsplit + SB);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // timeline (dev): kernel entry / prologue end / body end / exit of CTA 0 in the tail of row 0
  const bool tl_k = mn.prof >= 2 && mn.prof - 2 == mn.vid && blockIdx.x == 0 && threadIdx.x == 0;
  if (tl_k) g_tctl[0][TL_N - 1] = clock64();
  const int n_mt = (a.M + BM - 1) / BM, n_nt = (a.N + BN - 1) / BN;
  const int tiles_per_b = n_mt * n_nt;
  // CTA pairs (cluster of 2): the pair covers M tiles 2p and 2p+1 of the same (batch, N tile)
  // and shares the B tile, each CTA TMA-multicasting one B plane to both
  const uint32_t crank = cluster_ctarank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int n_mp = (n_mt + 1) >> 1;
  const int pairs_per_b = n_mp * n_nt;
  // EPI_WGRAD may split K (a.ksplit > 1, few output tiles): work item t = (pair tile, K split ks),
  // the split's K blocks [kbeg, kend)
  const int nk = (a.K + BK - 1) / BK;
  const int ksplit = (EPI == EPI_WGRAD && a.ksplit > 1) ? a.ksplit : 1;
  const int kper = (nk + ksplit - 1) / ksplit;
  const int total = pairs_per_b * a.batch * ksplit;  // work items
  auto tile_of = [&](int t, int& b, int& mt, int& nt) {
    t /= ksplit;
    b = t / pairs_per_b;
    const int rem = t - b * pairs_per_b;
    const int mp = rem / n_nt;
    nt = rem - mp * n_nt;
    mt = 2 * mp + (int)crank;
  };
  auto krange = [&](int t, int& kbeg, int& kend) {
    const int ks = t % ksplit;
    kbeg = ks * kper;
    kend = min(nk, kbeg + kper);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < SA; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&a_empty[s], NCONV);  // one arrive per converter warp
    }
    for (int s = 0; s < SB; ++s) {
      // pre-split planes: the leader's stage is full when its own load and the peer's (relayed)
      // have landed; raw planes: each CTA's splitters wait for their own half
      mbar_init(&b_full[s], (B_PRE && crank == 0) ? 2 : 1);
      mbar_init(&b_empty[s], 1);  // the leader's pair commit, multicast to both CTAs
    }
    for (int i = 0; i < C_::NAS; ++i) {
      mbar_init(&full_op[i], 2 * NCONV);  // both CTAs' converters arrive on the leader's
      mbar_init(&afree[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * NEPI);  // one arrive per epilogue warp of both CTAs (on the leader's)
    }
    for (int i = 0; i < NEPI; ++i) mbar_init(&xfull[i], 1);
    for (int i = 0; i < SB; ++i) mbar_init(&bsplit[i], 2 * NEPI);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tma_prefetch(&mA);
    tma_prefetch(&mB);
    if (B_PRE) tma_prefetch(&mB2);
    if (EPI != EPI_WGRAD) tma_prefetch(&mC);
    if (loadx) tma_prefetch(&mX);
  }
  if (warp == W_MMA) tmem_alloc2(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's barriers are initialised before any multicast / remote arrive
  tc_fence_after();
  // programmatic dependent launch: everything above (barrier init, TMEM allocation, tensor-map
  // prefetch) overlaps the previous kernel's tail; global memory is touched only after it has
  // completed.  The next kernel may be launched now (its CTAs get an SM as ours exit).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t tmem_base = *tmem_holder;
  unsigned long long pacc[3] = {0ull, 0ull, 0ull};
  const unsigned long long t_k0 = mn.prof ? clock64() : 0ull;
  if (tl_k) g_tctl[0][TL_N - 2] = t_k0;

  if (warp == W_TMA_A) {
    // ============================ TMA producer: A ring ============================
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = cid; t < total; t += ncl) {
        int b, mt, nt, kbeg, kend;
        tile_of(t, b, mt, nt);
        krange(t, kbeg, kend);
        for (int kb = kbeg; kb < kend; ++kb) {
          mbar_wait_t(&a_empty[s], ph ^ 1, mn.prof, pacc[0], mn.hint_p);
          uint8_t* sA = sAr + s * C_::A_BYTES;
          if (mn.dbg & 32) mbar_arrive(&a_full[s]);  // dev experiment: no A traffic
          else {
          mbar_expect_tx(&a_full[s], C_::A_BYTES);
          if (A_MN) {  // four 32-row blocks [m/32][k][m%32] (rows >= M zero-filled by the map)
#pragma unroll
            for (int i = 0; i < BM / 32; ++i)
              tma_load3(sA + i * 4096, &mA, &a_full[s], mt * BM + 32 * i, kb * BK, a.sA ? b : 0);
          }
          else tma_load3(sA, &mA, &a_full[s], kb * BK, mt * BM, a.sA ? b : 0);
          }
          if (++s == SA) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == W_TMA_B) {
    // ============================ TMA producer: B ring ============================
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const uint32_t bytes = (B_PRE ? 2 : 1) * C_::B_BYTES;
      uint32_t jq = 0;
      for (int t = cid; t < total; t += ncl) {
        int b, mt, nt, kbeg, kend;
        tile_of(t, b, mt, nt);
        krange(t, kbeg, kend);
        for (int kb = kbeg; kb < kend; ++kb, ++jq) {
          mbar_wait_t(&b_empty[s], ph ^ 1, mn.prof, pacc[0], mn.hint_p);
          if (mn.prof >= 2 && mn.prof - 2 == mn.vid && blockIdx.x == 0 && jq < TL_N) g_tctl[0][jq] = clock64();
          uint8_t* sBh = sBr + s * C_::B_STAGE;
          uint8_t* sBl = sBh + C_::B_BYTES;
          // each CTA of the pair loads its half of the B tile (columns crank * BN/2 ...): the pair
          // MMA reads the first half from the leader's shared memory, the second from the peer's
          if (mn.dbg & 16) mbar_arrive(&b_full[s]);  // dev experiment: no B traffic
          else {
          mbar_expect_tx(&b_full[s], bytes);
          const int n_half = nt * BN + (int)crank * (BN / 2);
          if (B_MN) {  // this CTA's two 32-column blocks (columns >= N zero-filled)
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load3(sBh + i * 4096, &mB, &b_full[s], n_half + 32 * i, kb * BK, (B_PRE || a.sB) ? b : 0);
          }
          else tma_load3(sBh, &mB, &b_full[s], kb * BK, n_half, (B_PRE || a.sB) ? b : 0);
          if (B_PRE) {
            if (B_MN) {
#pragma unroll
              for (int i = 0; i < BN / 64; ++i) tma_load3(sBl + i * 4096, &mB2, &b_full[s], n_half + 32 * i, kb * BK, b);
            }
            else tma_load3(sBl, &mB2, &b_full[s], kb * BK, n_half, b);
          }
          }
          if (++s == SB) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == W_MMA || warp == W_MMA2) {
    // ================================ MMA issuer ==================================
    // per chunk of TC_FOLD K blocks, into the chunk's own accumulator (folded by the epilogue):
    // the small products Al.Bh + Ah.Bl of all the chunk's blocks first (truncated relative to a
    // small partial sum), then its big ones Ah.Bh (DESIGN.md §5 "accumulation").  The two issuers
    // own alternate chunks.  The whole warp runs the loop (all values warp-uniform, so they live
    // in uniform registers); one elected lane issues the MMAs and commits.
    if (crank == 0) {
      // leader: pair MMAs M = 256 (128 rows per CTA) x N = BN
      constexpr uint32_t IDESC = idesc_tf32(2 * BM, BN, 0, B_MN ? 1 : 0);
      const uint32_t b_lbo = B_MN ? mn.lbo : 16, b_sbo = B_MN ? mn.sbo : 1024, b_lay = B_MN ? mn.layout : 2;
      // descriptor of stage 0's B hi plane; the address field (bits 0-13, addr >> 4) is advanced
      // by adding byte offsets >> 4 (all shared addresses < 256 KB)
      const uint64_t dB0 = sdesc(su32(sBr), b_lbo, b_sbo, b_lay);
      const uint32_t kstep16 = (B_MN ? mn.kstep : 32) >> 4;
      const uint32_t mine = (warp == W_MMA2) ? 1u : 0u;  // chunk parity this issuer owns
      uint32_t jb = 0, jc = 0;  // K blocks / chunks of this CTA so far (both issuers count all)
      for (int t = cid; t < total; t += ncl) {
        int kbeg, kend;
        krange(t, kbeg, kend);
        for (int kb0 = kbeg; kb0 < kend; kb0 += TC_FOLD, ++jc) {
          const int nkb = min(TC_FOLD, kend - kb0);
          if ((jc & 1u) != mine) { jb += nkb; continue; }
          const uint32_t buf = jc % NACC;
          const bool tl = mn.prof >= 2 && mn.prof - 2 == mn.vid && blockIdx.x == 0 && jc < TL_N && lane == 0;
          mbar_wait_cl_t(&tempty[buf], ((jc / NACC) & 1) ^ 1, mn.prof && lane == 0, pacc[0]);
          if (tl) g_tctl[1][jc] = clock64();
          for (int i = 0; i < nkb; ++i) {
            const uint32_t j = jb + i;
            mbar_wait_cl_t(&full_op[j % C_::NAS], (j / C_::NAS) & 1, mn.prof && lane == 0, pacc[1]);
            if (B_PRE) mbar_wait_cl(&b_full[j % SB], (j / SB) & 1u);  // (raw planes: waited for by their splitters)
            if (ESPLIT) mbar_wait_cl(&bsplit[j % SB], (j / SB) & 1u);
          }
          if (tl) g_tctl[2][jc] = clock64();
          tc_fence_after();
          const uint32_t dcol = tmem_base + buf * BN;
          const unsigned long long t_i0 = mn.prof ? clock64() : 0ull;
          if (elect_one()) {
            if (!(mn.dbg & 1)) {
              for (int i = 0; i < nkb; ++i) {
                const uint32_t j = jb + i;
                const uint32_t aH = tmem_base + C_::A_COL0 + (j % C_::NAS) * 64, aL = aH + 32;
                const uint64_t dBh = dB0 + (uint64_t)(((j % SB) * C_::B_STAGE) >> 4);
                const uint64_t dBl = dBh + (uint64_t)(C_::B_BYTES >> 4);
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                  mma2_tf32_ts(dcol, aL + 8 * kk, dBh + kk * kstep16, IDESC, (i == 0 && kk == 0) ? 0u : 1u);
                  mma2_tf32_ts(dcol, aH + 8 * kk, dBl + kk * kstep16, IDESC, 1u);
                }
              }
              for (int i = 0; i < nkb; ++i) {
                const uint32_t j = jb + i;
                const uint32_t aH = tmem_base + C_::A_COL0 + (j % C_::NAS) * 64;
                const uint64_t dBh = dB0 + (uint64_t)(((j % SB) * C_::B_STAGE) >> 4);
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) mma2_tf32_ts(dcol, aH + 8 * kk, dBh + kk * kstep16, IDESC, 1u);
              }
            }
            for (int i = 0; i < nkb; ++i) {
              mma2_commit_mc(&b_empty[(jb + i) % SB]);
              mma2_commit_mc(&afree[(jb + i) % C_::NAS]);
            }
            mma2_commit_mc(&tfull[buf]);
          }
          __syncwarp();
          jb += nkb;
          if (mn.prof) pacc[2] += clock64() - t_i0;
          if (tl) g_tctl[3][jc] = clock64();
        }
      }
    } else if (B_PRE && warp == W_MMA && lane == 0) {
      // peer: relay "my half of the pre-split B stage landed" to the leader's b_full
      uint32_t jb = 0;
      for (int t = cid; t < total; t += ncl) {
        int kbeg, kend;
        krange(t, kbeg, kend);
        for (int kb = kbeg; kb < kend; ++kb, ++jb) {
          mbar_wait(&b_full[jb % SB], (jb / SB) & 1u, mn.hint_p);
          mbar_arrive_cta(&b_full[jb % SB], 0);
        }
      }
    }
  } else if (warp >= W_CONV0) {
    // ================================ converters ==================================
    const int quad = warp & 3;          // TMEM lane quadrant = tile rows [32 quad, 32 quad + 32)
    const int r = 32 * quad + lane;     // the A row this thread splits
    const int ct = threadIdx.x - 32 * W_CONV0;  // 0..127 (B planes)
    const uint32_t ta = tmem_base + ((uint32_t)(32 * quad) << 16) + C_::A_COL0;
    int sa = 0, sb = 0;
    uint32_t pha = 0, phb = 0;
    uint32_t jb = 0;
    for (int t = cid; t < total; t += ncl) {
      int kbeg, kend;
      krange(t, kbeg, kend);
      for (int kb = kbeg; kb < kend; ++kb, ++jb) {
        // A first (the TMEM slot write is the long pole), then raw B planes if any
        mbar_wait_t(&a_full[sa], pha, mn.prof, pacc[0], mn.hint_c);
        const bool tlc = mn.prof >= 2 && mn.prof - 2 == mn.vid && blockIdx.x == 0 && jb < TL_N && lane == 0;
        if (tlc) atomicMax(&g_tctl[6][jb], clock64());  // last converter warp has A
        const uint8_t* stA = sAr + sa * C_::A_BYTES;
        uint32_t hi[32], lo[32];
        if (mn.dbg & 2) {
#pragma unroll
          for (int k = 0; k < 32; ++k) { hi[k] = 0u; lo[k] = 0u; }
        } else if (!A_MN) {  // row r: 8 x 16B chunks, chunk q at q ^ (r & 7) (128B swizzle)
          const float4* row = (const float4*)(stA + r * 128);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float4 x = row[q ^ (r & 7)];
            if (EPI == EPI_WGRAD && a.sq) { x.x *= x.x; x.y *= x.y; x.z *= x.z; x.w *= x.w; }
            // lo = x - hi on packed pairs (FADD2: half the issue slots)
            const float h0 = tf32_rna(x.x), h1 = tf32_rna(x.y), h2 = tf32_rna(x.z), h3 = tf32_rna(x.w);
            hi[4 * q + 0] = __float_as_uint(h0); hi[4 * q + 1] = __float_as_uint(h1);
            hi[4 * q + 2] = __float_as_uint(h2); hi[4 * q + 3] = __float_as_uint(h3);
            float l0, l1, l2, l3;
            upk2(fadd2(pk2(x.x, x.y), pk2(-h0, -h1)), l0, l1);
            upk2(fadd2(pk2(x.z, x.w), pk2(-h2, -h3)), l2, l3);
            lo[4 * q + 0] = __float_as_uint(l0); lo[4 * q + 1] = __float_as_uint(l1);
            lo[4 * q + 2] = __float_as_uint(l2); lo[4 * q + 3] = __float_as_uint(l3);
          }
        } else {  // [m / 32][k][m % 32], no swizzle: lanes read consecutive words
          const float* col = (const float*)stA + (r >> 5) * 1024 + (r & 31);
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            float x = col[k * 32];
            if (EPI == EPI_WGRAD && a.sq) x *= x;
            const float h = tf32_rna(x);
            hi[k] = __float_as_uint(h);
            lo[k] = __float_as_uint(x - h);
          }
        }
        const bool tc0 = tlc && warp == W_CONV0;  // converter warp 0 phase stamps
        if (tc0) g_tctl[8][jb] = clock64();
        const uint32_t as = jb % C_::NAS;
        mbar_wait_t(&afree[as], ((jb / C_::NAS) & 1) ^ 1, mn.prof, pacc[1], mn.hint_c);
        tc_fence_after();
        if (tc0) g_tctl[9][jb] = clock64();
        if (!(mn.dbg & 2)) {
          tmem_st32(ta + as * 64, hi);
          tmem_st32(ta + as * 64 + 32, lo);
        }
        if (tc0) g_tctl[10][jb] = clock64();
        if (!B_PRE && !ESPLIT) {  // B planes in shared memory: hi in place, lo beside it
          uint8_t* stB = sBr + sb * C_::B_STAGE;
          mbar_wait_t(&b_full[sb], phb, mn.prof, pacc[2], mn.hint_c);
          if (mn.prof >= 2 && mn.prof - 2 == mn.vid && blockIdx.x == 0 && jb < TL_N && lane == 0) atomicMax(&g_tctl[4][jb], clock64());
          if (tc0) g_tctl[11][jb] = clock64();
          float4* bh = (float4*)stB;
          float4* bl = (float4*)(stB + C_::B_BYTES);
#pragma unroll 4
          for (int i = ct; i < ((mn.dbg & 64) ? 0 : C_::B_BYTES / 16); i += NCONV * 32) {  // 64: dev experiment
            float4 x = bh[i];
            if (mn.btrunc && !(EPI == EPI_WGRAD && a.sq)) {
              float4 l;
              l.x = tf32_rna(x.x - tf32_trunc(x.x)); l.y = tf32_rna(x.y - tf32_trunc(x.y));
              l.z = tf32_rna(x.z - tf32_trunc(x.z)); l.w = tf32_rna(x.w - tf32_trunc(x.w));
              bl[i] = l;
              continue;
            }
            if (EPI == EPI_WGRAD && a.sq) { x.x *= x.x; x.y *= x.y; x.z *= x.z; x.w *= x.w; }
            float4 h, l;
            h.x = tf32_rna(x.x); h.y = tf32_rna(x.y); h.z = tf32_rna(x.z); h.w = tf32_rna(x.w);
            l.x = x.x - h.x; l.y = x.y - h.y; l.z = x.z - h.z; l.w = x.w - h.w;
            bh[i] = h;
            bl[i] = l;
          }
          if (tc0) g_tctl[12][jb] = clock64();
        }
        // publish: A in TMEM (wait::st), B planes visible to the async proxy (the proxy fence
        // also orders this warp's raw-A reads before the A producer's next TMA write)
        // (one elected arrive per warp after __syncwarp: per-thread arrives serialise on the
        // SM's barrier unit and cost more than the whole K block of MMAs)
        tmem_wait_st();
        if (tc0) g_tctl[13][jb] = clock64();
        fence_proxy_async();
        tc_fence_before();
        if (tc0) g_tctl[14][jb] = clock64();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_cta(&full_op[as], 0);
          mbar_arrive(&a_empty[sa]);
        }
        if (tc0) g_tctl[15][jb] = clock64();
        if (tlc) atomicMax(&g_tctl[7][jb], clock64());  // last converter warp published
        if (++sa == SA) { sa = 0; pha ^= 1; }
        if (++sb == SB) { sb = 0; phb ^= 1; }
      }
    }
  } else {
    // ================================ epilogue ====================================
    // Per tile: fold the K-block partials, then at the tile end apply the part of the fused
    // epilogue that needs the registers (act' product / residual / store of the sums) and park
    // the tile in the staging buffers; the rest (tanh for EPI_FWD, bias-gradient column sums,
    // the TMA stores) is emitted one 32-column group at a time between the folds of the NEXT
    // tile, so the MMA never waits for a tile's output work.
    const int ew = warp - W_EPI0;          // 0..7
    const int quad = warp & 3;             // TMEM lane quadrant = tile rows [32 quad, 32 quad + 32)
    const int half = ew >> 2;              // column half of the tile
    uint8_t* stg0 = stg_base + ew * NGRP * STG;  // NGRP staging tiles (32 rows x 32 fp32, 128B swizzle)
    const uint32_t t_lane = (uint32_t)(32 * quad) << 16;
    const bool vec_sl = a.slot_w && ((a.n_in & 3) == 0) && (((uintptr_t)a.slot_w & 15) == 0);
    float4* srow_base = reinterpret_cast<float4*>(stg0 + lane * 128);  // row `lane`, chunk q at q ^ (lane & 7)
    // parked tile: pend groups left (emitted in order), its batch / row block / first column
    int pend = 0, p_next = 0, p_b = 0, p_m0 = 0, p_nb = 0, p_blk = 0, p_ng = 0;
    // the parked tile is emitted in steps, one per fold of the next tile: EPI_FWD with tanh takes
    // 3 steps per 32-column group (12 / 12 / 8 columns of tanh, then the store), others 1 step;
    // with 8 K blocks per tile the last store is issued two folds before the tile end, so its
    // read of the staging tile has completed when the next tile is parked
    // tanh at the tile end in registers (mn.tanh_end: 64 independent elements per thread keep the
    // MUFU pipe busy) or in 3 emit steps per group from the staging tile (12 / 12 / 8 columns)
    const bool tanh_end = (EPI == EPI_FWD && a.act == ACT_TANH && mn.tanh_end);
    const int nstep = (EPI == EPI_FWD && a.act == ACT_TANH && !tanh_end) ? 3 : 1;
    bool tstep = false;  // timeline: stamp the end of the emit step's register work (row 23)
    uint32_t tstep_j = 0;
    auto emit_step = [&](int k) {
      if (mn.dbg & 8) return;  // dev experiment: no output traffic
      const int g = (nstep == 3) ? k / 3 : k, part = k - g * nstep;
      uint8_t* stg = stg0 + g * STG;
      float4* srow = reinterpret_cast<float4*>(stg + lane * 128);
      const int n0 = p_nb + 32 * g;
      if (EPI == EPI_FWD && a.act == ACT_TANH && nstep == 3) {
        // chunks 3 part .. 3 part + 2 (< 8) of the row: loads first (the stores would otherwise
        // order each load after the previous chunk's store), six independent tanh pairs
        const int q0 = 3 * part;
        float4 z0 = srow[q0 ^ (lane & 7)];
        float4 z1 = srow[(q0 + 1) ^ (lane & 7)];
        float4 z2 = (q0 + 2 < 8) ? srow[(q0 + 2) ^ (lane & 7)] : z1;
        TC_TANH2(z0.x, z0.y);
        TC_TANH2(z0.z, z0.w);
        TC_TANH2(z1.x, z1.y);
        TC_TANH2(z1.z, z1.w);
        if (q0 + 2 < 8) {  // (warp-uniform)
          TC_TANH2(z2.x, z2.y);
          TC_TANH2(z2.z, z2.w);
        }
        srow[q0 ^ (lane & 7)] = z0;
        srow[(q0 + 1) ^ (lane & 7)] = z1;
        if (q0 + 2 < 8) srow[(q0 + 2) ^ (lane & 7)] = z2;
      }
      if (tstep) g_tctl[23][tstep_j] = clock64();
      if (part != nstep - 1) return;
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store3(&mC, stg, n0, p_m0, p_b);
        bulk_commit();
      }
      if (EPI == EPI_DACT && a.colsum) {
        // column j of the staged 32 x 32 block summed over its rows (rows >= M hold zeros);
        // lane j reads word (r, j) at 16B chunk (j/4) ^ (r&7): 32 distinct banks per row
        const float* sf = reinterpret_cast<const float*>(stg);
        float cs = 0.f;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const float v = sf[r * 32 + ((((lane >> 2) ^ (r & 7)) << 2) | (lane & 3))];
          cs += a.sq ? v * v : v;
        }
        if (n0 + lane < a.N && p_blk * 32 < a.M)
          a.colsum[(int64_t)p_b * a.s_colsum + (int64_t)p_blk * a.N + n0 + lane] = cs;
      }
    };
    // staging free for TMA loads / new parked tiles: all groups emitted and their stores have
    // read the staging tiles (this warp's generic reads ordered before the async-proxy writes)
    auto staging_free = [&]() {
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
    };
    auto issue_prefetch = [&](int b, int mt, int nt) {
      if (lane == 0) {
        int nx = 0;
        for (int g = 0; g < NGRP; ++g) nx += (nt * BN + half * NC + 32 * g < a.N) ? 1 : 0;
        mbar_expect_tx(&xfull[ew], nx * STG);
        for (int g = 0; g < NGRP; ++g) {
          const int n0 = nt * BN + half * NC + 32 * g;
          if (n0 < a.N)
            tma_load3(stg0 + g * STG, &mX, &xfull[ew], n0, mt * BM + 32 * quad, EPI == EPI_RESID ? 0 : b);
        }
      }
      __syncwarp();
    };
    // ESPLIT: raw B stages of this CTA's K blocks [js, lim) split in place (hi) and beside (lo),
    // each warp one eighth of the stage
    uint32_t my_kb = 0;
    for (int t = cid; t < total; t += ncl) {
      int kbeg, kend;
      krange(t, kbeg, kend);
      my_kb += (uint32_t)(kend - kbeg);
    }
    uint32_t js = 0;
    auto split_upto = [&](uint32_t lim) {
      for (; js < lim && js < my_kb; ++js) {
        const int s = (int)(js % SB);
        mbar_wait(&b_full[s], (js / SB) & 1u);
        float4* bh = (float4*)(sBr + s * C_::B_STAGE);
        float4* bl = (float4*)(sBr + s * C_::B_STAGE + C_::B_BYTES);
#pragma unroll
        for (int i = ew * 32 + lane; i < C_::B_BYTES / 16; i += NEPI * 32) {
          float4 x = bh[i];
          if (mn.btrunc && !a.sq) {
            float4 l;
            l.x = tf32_rna(x.x - tf32_trunc(x.x)); l.y = tf32_rna(x.y - tf32_trunc(x.y));
            l.z = tf32_rna(x.z - tf32_trunc(x.z)); l.w = tf32_rna(x.w - tf32_trunc(x.w));
            bl[i] = l;
            continue;
          }
          if (a.sq) { x.x *= x.x; x.y *= x.y; x.z *= x.z; x.w *= x.w; }
          float4 h, l;
          h.x = tf32_rna(x.x); h.y = tf32_rna(x.y); h.z = tf32_rna(x.z); h.w = tf32_rna(x.w);
          l.x = x.x - h.x; l.y = x.y - h.y; l.z = x.z - h.z; l.w = x.w - h.w;
          bh[i] = h;
          bl[i] = l;
        }
        fence_proxy_async();  // generic-proxy writes -> the tensor core's async-proxy reads
        __syncwarp();
        if (lane == 0) mbar_arrive_cta(&bsplit[s], 0);
      }
    };
    if (ESPLIT) split_upto(ESPLIT_D);
    uint32_t jb = 0, jc = 0, jt = 0;
    for (int t = cid; t < total; t += ncl, ++jt) {
      int b, mt, nt;
      tile_of(t, b, mt, nt);
      const int rem = mt * n_nt + nt;  // tile index within the batch (residual partial slot)
      bool prefetched = false, pf_due = false;
      if (loadx && pend == 0) {
        staging_free();
        issue_prefetch(b, mt, nt);
        prefetched = true;
      }
      // ---- fold the K-block partials into round-to-nearest fp32 sums ----
      // (EPI_FWD: the warp's NC bias values are loaded now, NC/32 per lane, and only consumed at
      // the tile end - the load latency hides behind the folds instead of stalling the first)
      float acc[NC];
#pragma unroll
      for (int i = 0; i < NC; ++i) acc[i] = 0.f;
      float bias_l[NC / 32];
      // EPI_WGRAD with the compact slot map: this row's group masks / bases, loaded now and
      // consumed at the tile end (the load latency hides behind the folds)
      uint32_t gmk[NC / 32];
      int32_t gbs[NC / 32];
      if (EPI == EPI_WGRAD && a.gmask) {
        const int m = mt * BM + 32 * quad + lane;
#pragma unroll
        for (int u = 0; u < NC / 32; ++u) {
          const int n0 = nt * BN + half * NC + 32 * u;
          const bool ok = m < a.M && n0 < a.N;
          const int64_t gi = (int64_t)m * a.n_grp + (n0 >> 5);
          gmk[u] = ok ? __ldg(a.gmask + gi) : 0u;
          gbs[u] = ok ? __ldg(a.gbase + gi) : 0;
        }
      }
      {
        const int nb = nt * BN + half * NC;
        const float* bias = (EPI == EPI_FWD && a.bias) ? a.bias + (int64_t)b * a.s_bias + nb : nullptr;
#pragma unroll
        for (int u = 0; u < NC / 32; ++u) {
          const int col = u * 32 + lane;
          bias_l[u] = (bias && nb + col < a.N) ? __ldg(bias + col) : 0.f;
        }
      }
      int kbeg, kend;
      krange(t, kbeg, kend);
      const int nkt = kend - kbeg;
      const int nch = (nkt + TC_FOLD - 1) / TC_FOLD;
      for (int c = 0; c < nch; ++c, ++jc) {
        jb += min(TC_FOLD, nkt - c * TC_FOLD);  // K blocks consumed through this chunk
        const uint32_t buf = jc % NACC;
        mbar_wait_t(&tfull[buf], (jc / NACC) & 1, mn.prof, pacc[0], mn.hint_e);
        const bool tla = mn.prof >= 2 && mn.prof - 2 == mn.vid && blockIdx.x == 0 && jc < TL_N && lane == 0;
        const bool te = tla && ew == 0;  // epilogue warp 0 phase stamps (per chunk)
        if (te) g_tctl[16][jc] = clock64();
        tc_fence_after();
        const uint32_t taddr = tmem_base + t_lane + buf * BN + half * NC;
#pragma unroll
        for (int c0 = 0; c0 < ((mn.dbg & 4) ? 0 : NC); c0 += 32) {
          uint32_t r0[16], r1[16];
          tmem_ld16(taddr + c0, r0);
          tmem_ld16(taddr + c0 + 16, r1);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; i += 2) {  // packed pairs (FADD2: half the issue slots)
            upk2(fadd2(pk2(acc[c0 + i], acc[c0 + i + 1]), pk2(__uint_as_float(r0[i]), __uint_as_float(r0[i + 1]))),
                 acc[c0 + i], acc[c0 + i + 1]);
            upk2(fadd2(pk2(acc[c0 + 16 + i], acc[c0 + 17 + i]), pk2(__uint_as_float(r1[i]), __uint_as_float(r1[i + 1]))),
                 acc[c0 + 16 + i], acc[c0 + 17 + i]);
          }
        }
        if (te) g_tctl[17][jc] = clock64();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cta(&tempty[buf], 0);
        if (tla) atomicMax(&g_tctl[5][jc], clock64());  // last epilogue warp done
        if (te) g_tctl[18][jc] = clock64();
        if (ESPLIT) split_upto(jb + ESPLIT_D);  // B stages of K blocks < jb + ESPLIT_D
        if (pf_due && !prefetched) {
          // the last store of the parked tile was issued a fold ago: its read of the staging
          // tiles has (mostly) completed, the next tile's act' / V tiles can be loaded in place
          staging_free();
          issue_prefetch(b, mt, nt);
          prefetched = true;
          pf_due = false;
        }
        if (pend > 0) {
          // the parked tile's steps spread evenly over the first folds of this tile, the last one
          // (mn.emit_lead + 1) folds before the tile end
          const unsigned long long t_e0 = mn.prof ? clock64() : 0ull;
          const int left = max(1, nch - 1 - mn.emit_lead - c);
          for (int todo = (pend + left - 1) / left; todo > 0 && pend > 0; --todo) {
            tstep = te; tstep_j = jc;
            emit_step(p_next++);
            tstep = false;
            if (--pend == 0 && loadx && !prefetched) pf_due = true;
          }
          if (mn.prof) pacc[2] += clock64() - t_e0;
        }
        if (te) g_tctl[19][jc] = clock64();
      }
      const bool tt = mn.prof >= 2 && mn.prof - 2 == mn.vid && blockIdx.x == 0 && jc - 1 < TL_N && lane == 0 && ew == 0;
      const unsigned long long t_out0 = mn.prof ? clock64() : 0ull;
      while (pend > 0) {  // short K: flush the parked tile
        emit_step(p_next++);
        --pend;
      }
      if (loadx && !prefetched) {
        staging_free();
        issue_prefetch(b, mt, nt);
      }
      if (!loadx) staging_free();
      if (tt) g_tctl[20][jc - 1] = clock64();
      if (EPI == EPI_FWD) {  // + bias (column u*32 + l lives in lane l's bias_l[u])
#pragma unroll
        for (int i = 0; i < NC; ++i) acc[i] += __shfl_sync(0xffffffffu, bias_l[i >> 5], i & 31);
        if (tanh_end) {
#pragma unroll
          for (int i = 0; i < NC; i += 2) tanh_acc2(acc[i], acc[i + 1]);
        }
      }
      // ---- tile end: the register part of the fused epilogue, parked in staging ----
      if (loadx) mbar_wait_t(&xfull[ew], jt & 1, mn.prof, pacc[1]);
      if (tt) g_tctl[21][jc - 1] = clock64();
      const int m = mt * BM + 32 * quad + lane;
      const bool mrow = m < a.M;
      double psq = 0.0, pr = 0.0;
      const float b0v = (EPI == EPI_RESID && a.b0) ? a.b0[(int64_t)b * a.s_b0] : 0.f;
      int ng = 0;
#pragma unroll
      for (int g = 0; g < NC / 32; ++g) {
        const int n0 = nt * BN + half * NC + 32 * g;
        float* v = acc + 32 * g;  // compile-time offsets after unrolling: stays in registers
        if (EPI == EPI_WGRAD) {
          if (a.gmask) {  // compact slot map: one mask + one base per group (zero mask outside)
            const uint32_t mk = gmk[g];
            if (mk) {
              float* gl = (ksplit > 1 ? a.gl_part + (int64_t)(t % ksplit) * a.batch * a.k : a.gl) + (int64_t)b * a.k + gbs[g];
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if ((mk >> j) & 1u) gl[__popc(mk & ((1u << j) - 1u))] = v[j];
            }
          } else if (mrow && n0 < a.N) {
            const int32_t* sw = a.slot_w + (int64_t)m * a.n_in + n0;
            float* gl = (ksplit > 1 ? a.gl_part + (int64_t)(t % ksplit) * a.batch * a.k : a.gl) + (int64_t)b * a.k;
            const bool full = vec_sl && n0 + 32 <= a.N;
            // all 8 slot loads first (one round trip), then the scattered stores
            int4 s4[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if (full) s4[q] = __ldg(reinterpret_cast<const int4*>(sw) + q);
              else {
                s4[q].x = (n0 + 4 * q + 0 < a.N) ? __ldg(sw + 4 * q + 0) : -1;
                s4[q].y = (n0 + 4 * q + 1 < a.N) ? __ldg(sw + 4 * q + 1) : -1;
                s4[q].z = (n0 + 4 * q + 2 < a.N) ? __ldg(sw + 4 * q + 2) : -1;
                s4[q].w = (n0 + 4 * q + 3 < a.N) ? __ldg(sw + 4 * q + 3) : -1;
              }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if (s4[q].x >= 0) gl[s4[q].x] = v[4 * q];
              if (s4[q].y >= 0) gl[s4[q].y] = v[4 * q + 1];
              if (s4[q].z >= 0) gl[s4[q].z] = v[4 * q + 2];
              if (s4[q].w >= 0) gl[s4[q].w] = v[4 * q + 3];
            }
          }
          continue;
        }
        if (n0 >= a.N) continue;  // whole 32-column group outside the matrix (warp-uniform)
        ++ng;
        float4* srow = srow_base + g * (STG / 16);
        if (EPI == EPI_DACT) {
          // rows >= M and columns >= N of the loaded tile are zero-filled by TMA
          if (!mrow) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
          if (a.act != ACT_ID && !(mn.dbg & 128)) {  // (128: dev experiment, no act' product)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 d4 = srow[q ^ (lane & 7)];
              if (a.act == ACT_TANH) {  // v *= 1 - d^2 (packed pairs)
                const uint64_t one = pk2(1.f, 1.f);
                const uint64_t dxy = pk2(d4.x, d4.y), dzw = pk2(d4.z, d4.w);
                const uint64_t fxy = ffma2(fmul2(dxy, pk2(-1.f, -1.f)), dxy, one);
                const uint64_t fzw = ffma2(fmul2(dzw, pk2(-1.f, -1.f)), dzw, one);
                upk2(fmul2(pk2(v[4 * q + 0], v[4 * q + 1]), fxy), v[4 * q + 0], v[4 * q + 1]);
                upk2(fmul2(pk2(v[4 * q + 2], v[4 * q + 3]), fzw), v[4 * q + 2], v[4 * q + 3]);
              } else {
                v[4 * q + 0] *= d4.x;
                v[4 * q + 1] *= d4.y;
                v[4 * q + 2] *= d4.z;
                v[4 * q + 3] *= d4.w;
              }
            }
          }
        } else if (EPI == EPI_RESID) {
          // r = V - (acc + b0), R = r / sigma^2 (stored); per 32-column group the squares and
          // the R values are summed pairwise in fp32 (error <= 5 ulp of the group sum), the
          // group sums accumulate in fp64
          const float is2 = (float)a.inv_s2;
          float sq[32], rr[32];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 y4 = srow[q ^ (lane & 7)];
            const float yy[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i = 4 * q + e;
              const bool in = mrow && n0 + i < a.N;
              const float r = in ? yy[e] - (v[i] + b0v) : 0.f;
              v[i] = r * is2;
              sq[i] = r * r;
              rr[i] = v[i];
            }
          }
#pragma unroll
          for (int w = 16; w > 0; w >>= 1)
#pragma unroll
            for (int i = 0; i < w; ++i) {
              sq[i] += sq[i + w];
              rr[i] += rr[i + w];
            }
          psq += (double)sq[0];
          pr += (double)rr[0];
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q) srow[q ^ (lane & 7)] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
      if (EPI != EPI_WGRAD) {  // park the tile
        pend = ng * nstep; p_next = 0; p_b = b; p_m0 = mt * BM + 32 * quad; p_nb = nt * BN + half * NC;
        p_blk = mt * 4 + quad;
        __syncwarp();
      }
      if (tt) g_tctl[22][jc - 1] = clock64();
      if (mn.prof) pacc[2] += clock64() - t_out0;
      if (EPI == EPI_RESID) {
        // deterministic: warp shuffles, then one partial per (tile, epilogue warp) - slot
        // rem * NEPI + ew - summed in fixed order by the reduction kernel (no barrier across
        // the epilogue warps per tile)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          psq += __shfl_down_sync(0xffffffffu, psq, o);
          pr += __shfl_down_sync(0xffffffffu, pr, o);
        }
        if (lane == 0 && mt < n_mt) {
          a.part_sq[(int64_t)b * a.n_part + (int64_t)rem * NEPI + ew] = psq;
          a.part_r[(int64_t)b * a.n_part + (int64_t)rem * NEPI + ew] = pr;
        }
      }
    }
    while (pend > 0) {  // the last parked tile
      emit_step(p_next++);
      --pend;
    }
    if (lane == 0) bulk_wait0();
    if (EPI == EPI_WGRAD && a.bcs) {
      // the layer's bias gradient: every (chain, column) sum of the column partials, spread over
      // the epilogue threads of all CTAs (replaces a separate reduction launch)
      const int64_t tot = (int64_t)a.batch * a.M;
      for (int64_t i = (int64_t)blockIdx.x * (NEPI * 32) + ew * 32 + lane; i < tot; i += (int64_t)gridDim.x * (NEPI * 32)) {
        const int64_t c = i / a.M;
        const int o = (int)(i - c * a.M);
        const int sl = a.bcs_slot[o];
        if (sl < 0) continue;
        const float* p = a.bcs + c * a.s_bcs + o;
        float acc = 0.f;
#pragma unroll 8
        for (int blk = 0; blk < a.bcs_nblk; ++blk) acc += p[(int64_t)blk * a.M];
        a.gl[c * a.k + sl] = acc;
      }
    }
  }
  if (mn.prof && lane == 0) {
    if (warp == W_TMA_A) atomicAdd(&g_tcprof[mn.vid][P_TMA_EMPTY], pacc[0]);
    if (warp == W_MMA) {
      atomicAdd(&g_tcprof[mn.vid][P_MMA_TEMPTY], pacc[0]); atomicAdd(&g_tcprof[mn.vid][P_MMA_FULLOP], pacc[1]);
      atomicAdd(&g_tcprof[mn.vid][P_MMA_ISSUE], pacc[2]);
    }
    if (warp == W_CONV0) {
      atomicAdd(&g_tcprof[mn.vid][P_CONV_RAW], pacc[0]); atomicAdd(&g_tcprof[mn.vid][P_CONV_AFREE], pacc[1]);
      atomicAdd(&g_tcprof[mn.vid][P_CONV_B], pacc[2]);
    }
    if (warp == W_TMA_B) atomicAdd(&g_tcprof[mn.vid][P_BTMA_EMPTY], pacc[0]);
    if (warp == W_EPI0) {
      atomicAdd(&g_tcprof[mn.vid][P_EPI_TFULL], pacc[0]); atomicAdd(&g_tcprof[mn.vid][P_EPI_XFULL], pacc[1]);
      atomicAdd(&g_tcprof[mn.vid][P_EPI_OUT], pacc[2]);
    }
    if (warp == W_TMA_A) atomicAdd(&g_tcprof[mn.vid][P_TOTAL], clock64() - t_k0);
  }
  if (tl_k) g_tctl[0][TL_N - 3] = clock64();
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its peer may still multicast into it or arrive on it
  if (tl_k) g_tctl[0][TL_N - 4] = clock64();
  if (warp == W_MMA) tmem_dealloc2(tmem_base, 512);
}

// ------------------------------------------------------------------------- host side ---
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace tc

// Pre-split operand description (hi / lo planes of the weights) attached to a GemmArgs.
struct PreSplit {
  const float* hi = nullptr;
  const float* lo = nullptr;
  int64_t ld = 0, stride = 0;
  bool only = false;  // the planes are the only current copy of the weights (dense W not updated)
};

// Kernel instantiations: (A MN-major, B MN-major, B pre-split, epilogue) combinations the hot
// path uses (plus EPI_STORE for the debug GEMM on the four unsplit layouts).  Anything else runs
// on the SIMT engine.
typedef void (*TcKernel)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, GemmArgs, tc::MnDesc);
struct TcVariant {
  bool amn, bmn, pre;
  int epi;
  TcKernel fn;
  int smem;  // dynamic shared memory bytes
};
template <int BN>
inline const TcVariant* tc_variants(int* n) {
#define TV(AMN, BMN, PRE, EPI) \
  {AMN, BMN, PRE, EPI, (TcKernel)tc::tc_gemm_kernel<BN, AMN, BMN, PRE, EPI>, tc::Cfg<BN, EPI == EPI_WGRAD>::SMEM}
  static const TcVariant v[] = {
      TV(false, false, true, EPI_FWD),     // forward      Z = A W^T        (weights pre-split)
      TV(false, false, false, EPI_FWD),    // forward, raw weight plane (split in shared memory)
      TV(false, true, true, EPI_DACT),     // input grad   G = (G W) o act'  (weights pre-split)
      TV(true, true, false, EPI_WGRAD),    // weight grad  dW = G^T A, compacted into the k-vector
      TV(false, false, false, EPI_RESID),  // DeepONet combine + residual
      TV(false, true, false, EPI_DACT),    // DeepONet dB = R T
      TV(true, true, false, EPI_DACT),     // DeepONet dT = R^T B
      TV(false, false, false, EPI_STORE),  // debug GEMM
      TV(false, true, false, EPI_STORE),
      TV(true, true, false, EPI_STORE),
      TV(true, false, false, EPI_STORE),
  };
#undef TV
  *n = (int)(sizeof(v) / sizeof(v[0]));
  return v;
}

// Developer knobs (timelines, barrier profiles, A/B toggles of the engine) are read from the
// environment only in a -DHMC_DEV build (`make DEV=1`); the product library ignores them.
inline const char* dev_env(const char* name) {
#ifdef HMC_DEV
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}
// Process-wide engine override set through hmc_debug_set_engine (tests): 0 = automatic
// (tcgen05 where it takes the shape, SIMT otherwise), 1 = SIMT only.  Read at hmc_setup.
inline int& engine_override() {
  static int v = 0;
  return v;
}

struct TcPlanner {
  bool enabled = false;
  int num_sms = 148;
  tc::EncodeTiledFn encode = nullptr;
  tc::MnDesc mn;
  CUtensorMapSwizzle mn_swizzle = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
  static constexpr int BN = 128;   // tile N (UMMA N); TMEM holds 512 / BN K-block partials

  void init() {
    enabled = false;
    if (engine_override() == 1) return;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return;
    if (p.major != 10 || p.minor != 0) return;  // sm_100a binary only
    num_sms = p.multiProcessorCount;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return;
    encode = (tc::EncodeTiledFn)fn;
    if (const char* f = dev_env("HMC_TC_PROF")) mn.prof = atoi(f);
    if (const char* f = dev_env("HMC_TC_DBG")) mn.dbg = atoi(f);
    if (const char* f = dev_env("HMC_TC_BTRUNC")) mn.btrunc = atoi(f);
    if (const char* f = dev_env("HMC_TC_TANHEND")) mn.tanh_end = atoi(f);
    if (const char* f = dev_env("HMC_TC_EMITLEAD")) mn.emit_lead = atoi(f);
    if (const char* f = dev_env("HMC_TC_PDL")) mn.pdl = atoi(f);
    if (const char* f = dev_env("HMC_TC_HINT_P")) mn.hint_p = (uint32_t)atoi(f);
    if (const char* f = dev_env("HMC_TC_HINT_C")) mn.hint_c = (uint32_t)atoi(f);
    if (const char* f = dev_env("HMC_TC_HINT_E")) mn.hint_e = (uint32_t)atoi(f);
    static bool attr_done = false;
    if (!attr_done) {
      int n = 0;
      const TcVariant* v = tc_variants<BN>(&n);
      for (int i = 0; i < n; ++i)
        cudaFuncSetAttribute((const void*)v[i].fn, cudaFuncAttributeMaxDynamicSharedMemorySize, v[i].smem);
      attr_done = true;
    }
    enabled = true;
  }

  static const TcVariant* find(bool amn, bool bmn, bool pre, int epi) {
    int n = 0;
    const TcVariant* v = tc_variants<BN>(&n);
    for (int i = 0; i < n; ++i)
      if (v[i].amn == amn && v[i].bmn == bmn && v[i].pre == pre && v[i].epi == epi) return &v[i];
    return nullptr;
  }

  static bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

  // Shapes / layouts the tensor-core engine takes (everything else runs on the SIMT engine).
  bool accepts(const GemmArgs& a, bool akm, bool bkm, const PreSplit* pre = nullptr) const {
    if (!enabled) return false;
    if (a.ones_col >= 0) return false;
    if (a.M < 64 || a.N < 32 || a.K < 32) return false;
    if (a.batch > 65535) return false;
    const bool amn = !akm, bmn = !bkm;
    if (pre && !pre->lo) {  // raw weight plane: an ordinary B operand
      GemmArgs b = a;
      b.B = pre->hi; b.ldb = pre->ld; b.sB = pre->stride;
      return accepts(b, akm, bkm, nullptr);
    }
    if (!find(amn, bmn, pre != nullptr, a.epi)) return false;
    if (a.epi == EPI_FWD && a.act == ACT_SIN) return false;
    if ((a.lda % 4) || (a.sA % 4) || !al16(a.A)) return false;

    if (pre) {
      if (!pre->hi || (pre->ld % 4) || (pre->stride % 4) || !al16(pre->hi) || !al16(pre->lo)) return false;
    } else {
      if ((a.ldb % 4) || (a.sB % 4) || !al16(a.B)) return false;
    }

    if (a.epi != EPI_WGRAD) {  // TMA store of the output
      if (!a.C || (a.ldc % 4) || (a.sC % 4) || !al16(a.C)) return false;
    }
    if (a.epi == EPI_DACT && a.act != ACT_ID) {  // TMA load of act' source
      if (!a.dsrc || (a.ld_dsrc % 4) || (a.s_dsrc % 4) || !al16(a.dsrc)) return false;
    }
    if (a.epi == EPI_RESID && (!a.V || (a.ldv % 4) || !al16(a.V))) return false;
    return true;
  }

  // work items (CTA-pair tiles) of a launch without K split
  static int pair_tiles(const GemmArgs& a) {
    return (((a.M + tc::BM - 1) / tc::BM + 1) / 2) * ((a.N + BN - 1) / BN) * a.batch;
  }


  const char* describe() const { return enabled ? "tcgen05-3xtf32+simt" : "simt"; }

  // K-major operand X(row, k) = X[row*ld + k] per batch: dims (K, rows, batch), box (32, rows_box, 1)
  bool map_kmajor(CUtensorMap* m, const float* base, int64_t rows, int64_t K, int64_t ld, int64_t bstride,
                  int batch, int box_rows) const {
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)(bstride ? bstride : rows * ld) * 4};
    cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  // MN-major operand X(k, j) = X[k*ld + j] per batch: dims (MN, K, batch), box (32, 32, 1) - one
  // 32-wide MN block of 32 K rows per load, [j/32][k][j%32] in shared memory; MN need not be a
  // multiple of 32 (columns >= MN are zero-filled).  plain = no swizzle (the raw A tile only the
  // converter warps read); otherwise the MMA's SWIZZLE_128B_BASE32B layout.
  bool map_mnmajor(CUtensorMap* m, const float* base, int64_t K, int64_t MN, int64_t ld, int64_t bstride,
                   int batch, int /*box_mn*/, bool plain = false) const {
    cuuint64_t dims[3] = {(cuuint64_t)MN, (cuuint64_t)K, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)(bstride ? bstride : K * ld) * 4};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, plain ? CU_TENSOR_MAP_SWIZZLE_NONE : mn_swizzle,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  // row-major output C(m, n) = C[m*ldc + n] per batch: dims (N, M, batch), box (32, 32, 1), 128B swizzle
  bool map_store(CUtensorMap* m, float* base, int64_t M, int64_t N, int64_t ldc, int64_t bstride, int batch) const {
    cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)ldc * 4, (cuuint64_t)(bstride ? bstride : M * ldc) * 4};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }

  // Launches a GEMM accepts() took.  Returns cudaSuccess, or the error: a tensor map that could
  // not be encoded (cudaErrorInvalidValue) or the launch's own error.  Callers report it
  // (HMC_E_CUDA); there is no silent fallback to the SIMT engine.
  cudaError_t launch(const GemmArgs& a, bool akm, bool bkm, cudaStream_t st, const PreSplit* pre = nullptr) const {
    if (pre && !pre->lo) {  // raw weight plane: an ordinary B operand
      GemmArgs b = a;
      b.B = pre->hi; b.ldb = pre->ld; b.sB = pre->stride;
      return launch(b, akm, bkm, st, nullptr);
    }
    const bool amn = !akm, bmn = !bkm;
    const TcVariant* v = find(amn, bmn, pre != nullptr, a.epi);
    if (!v) return cudaErrorInvalidValue;
    CUtensorMap mA, mB, mB2, mC, mX;
    memset(&mB2, 0, sizeof(mB2));
    memset(&mC, 0, sizeof(mC));
    memset(&mX, 0, sizeof(mX));
    // an operand shared by every batch entry (stride 0, e.g. the data) is mapped once and loaded
    // at batch coordinate 0 (the kernel reads a.sA / a.sB)
    const int batA = a.sA == 0 ? 1 : a.batch, batB = a.sB == 0 ? 1 : a.batch;
    bool ok = amn ? map_mnmajor(&mA, a.A, a.K, a.M, a.lda, a.sA, batA, tc::BM, true)
                  : map_kmajor(&mA, a.A, a.M, a.K, a.lda, a.sA, batA, tc::BM);
    if (pre) {
      ok = ok && (bmn ? map_mnmajor(&mB, pre->hi, a.K, a.N, pre->ld, pre->stride, a.batch, BN / 2)
                      : map_kmajor(&mB, pre->hi, a.N, a.K, pre->ld, pre->stride, a.batch, BN / 2));
      ok = ok && (bmn ? map_mnmajor(&mB2, pre->lo, a.K, a.N, pre->ld, pre->stride, a.batch, BN / 2)
                      : map_kmajor(&mB2, pre->lo, a.N, a.K, pre->ld, pre->stride, a.batch, BN / 2));
    } else {  // (each CTA of the pair loads half of the B tile)
      ok = ok && (bmn ? map_mnmajor(&mB, a.B, a.K, a.N, a.ldb, a.sB, batB, BN / 2)
                      : map_kmajor(&mB, a.B, a.N, a.K, a.ldb, a.sB, batB, BN / 2));
      mB2 = mB;
    }
    if (a.epi != EPI_WGRAD) ok = ok && map_store(&mC, a.C, a.M, a.N, a.ldc, a.sC, a.batch);
    if (a.epi == EPI_DACT && a.act != ACT_ID)
      ok = ok && map_store(&mX, const_cast<float*>(a.dsrc), a.M, a.N, a.ld_dsrc, a.s_dsrc, a.batch);
    if (a.epi == EPI_RESID) ok = ok && map_store(&mX, const_cast<float*>(a.V), a.M, a.N, a.ldv, 0, 1);
    if (!ok) return cudaErrorInvalidValue;
    const int pairs = (((a.M + tc::BM - 1) / tc::BM + 1) / 2) * ((a.N + BN - 1) / BN) * a.batch *
                      ((a.epi == EPI_WGRAD && a.ksplit > 1) ? a.ksplit : 1);
    int pair_cap = num_sms / 2;
    if (a.max_pairs > 0 && a.max_pairs < pair_cap) pair_cap = a.max_pairs;
    // dev A/B: fewer, longer-lived CTA pairs (several tiles each) for the launches of one EPI class
    // (HMC_TC_GRIDCAP = pairs, HMC_TC_GRIDCAP_EPI = bit mask of EPI ids, default all)
    static const int gridcap = dev_env("HMC_TC_GRIDCAP") ? atoi(dev_env("HMC_TC_GRIDCAP")) : 0;
    static const int gridcap_epi = dev_env("HMC_TC_GRIDCAP_EPI") ? atoi(dev_env("HMC_TC_GRIDCAP_EPI")) : 0xff;
    if (gridcap > 0 && ((gridcap_epi >> a.epi) & 1) && gridcap < pair_cap) pair_cap = gridcap;
    const int grid = 2 * (pairs < pair_cap ? pairs : pair_cap);
    int nv = 0;
    tc::MnDesc md = mn;
    md.vid = (int)(v - tc_variants<BN>(&nv));
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tc::NT);
    cfg.dynamicSmemBytes = v->smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see griddepcontrol in the kernel
    attr[1].val.programmaticStreamSerializationAllowed = mn.pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, v->fn, mA, mB, mB2, mC, mX, a, md);
  }
};

}  // namespace hmc
