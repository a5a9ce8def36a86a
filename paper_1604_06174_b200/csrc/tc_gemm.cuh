// tcgen05 (5th-gen tensor core) GEMM for sm_100a: TMA -> shared memory (128B swizzle) ->
// tcgen05.mma (kind::f16, bf16 x bf16 -> fp32 accumulator in TMEM) -> tcgen05.ld epilogue.
//
//   D[m][n] = sum_k A(m,k) * B(n,k)      tile 128 x BN x 64, K pipelined over STAGES
//
// Operands are either K-major (rows of K contiguous: X[rows][K]) or MN-major (X[K][MN]),
// selected per operand at compile time; that covers the three contractions of a residual
// block without any transpose copies:
//   forward      D[f_out][b]  = W[f_out][:] . a[b][:]        A K-major,  B K-major
//   backward dX  D[f_in][b]   = W[:][f_in] . g[b][:]         A MN-major, B K-major
//   backward dW  D[f_in][f_out] = a[:][f_in] . g[:][f_out]    A MN-major, B MN-major
// "swap-AB": the feature dimension is M (one TMEM lane per feature), the batch is N, so the
// epilogue writes out[n*ld + m] with a warp covering 32 consecutive features (coalesced).
//
// Warp roles (128 threads, one CTA per output tile): warp 0 lane 0 = TMA producer and TMEM
// allocator, warp 1 lane 0 = MMA issuer; afterwards all 4 warps drain TMEM (warp w owns
// lanes 32w..32w+31).  Barriers: full[s]/empty[s] per stage (TMA <-> MMA), one accumulator
// barrier (MMA -> epilogue) signalled by tcgen05.commit.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "kernels_simt.cuh"  // pdl_wait / pdl_launch

namespace slmk {

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// 4-D tile load (the implicit-GEMM convolution operand: {C, W, H, image} of an NHWC tensor;
// coordinates may be negative / past the end -- those elements are zero-filled, which is the
// convolution's "same" padding)
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// Implicit-GEMM convolution operand (stride s, "same" padding p = k / 2): the im2col matrix
// col[position (i, j)][(u k + v) cin + c] = x[img][s i + u - p][s j + v - p][c] is never stored;
// its tiles are 4-D TMA boxes of the bf16 NHWC input x (map {cin, W, H, images}, element strides
// {1, s, s, 1}: a box of s wo x s rows elements loads wo x rows of them).  hw, w: the OUTPUT
// positions per image and per row.  on = 1: the K-major B operand (rows = positions, a tile = BN
// / w whole output rows, or BN / hw whole images); on = 2: the MN-major A operand of the weight
// gradient (K = positions, a 64-position K block = 64 / w output rows, or 64 / hw images).
struct ConvB {
  int on = 0, cin = 0, k = 0, hw = 0, w = 0, s = 1;
};
// bulk prefetch of one tensor-map box into L2 (no smem, no barrier)
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// ---- CTA pair (cta_group::2): two SMs of a TPC execute one M=256 MMA; each CTA stages its
// own 128 rows of A and half of the N columns of B, the leader (rank 0) issues the MMAs.
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// address of the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t cluster_map(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load into this CTA's smem whose completion is counted on the LEADER CTA's mbarrier (the
// same smem offset with the peer bit cleared)
__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the mbarrier at this smem offset in every CTA of `mask` once the leader's MMAs retire
__device__ __forceinline__ void tc_commit2(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread i of the warp gets lane (base+i).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// two 32-column loads (columns taddr .. taddr+63) behind one wait: one TMEM round trip per 64 columns
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float* v) {
  uint32_t r[64];
#define SLM_TLD(o, b)                                                                                         \
  asm volatile(                                                                                               \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"           \
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                         \
      : "=r"(r[b + 0]), "=r"(r[b + 1]), "=r"(r[b + 2]), "=r"(r[b + 3]), "=r"(r[b + 4]), "=r"(r[b + 5]),         \
        "=r"(r[b + 6]), "=r"(r[b + 7]), "=r"(r[b + 8]), "=r"(r[b + 9]), "=r"(r[b + 10]), "=r"(r[b + 11]),        \
        "=r"(r[b + 12]), "=r"(r[b + 13]), "=r"(r[b + 14]), "=r"(r[b + 15]), "=r"(r[b + 16]), "=r"(r[b + 17]),    \
        "=r"(r[b + 18]), "=r"(r[b + 19]), "=r"(r[b + 20]), "=r"(r[b + 21]), "=r"(r[b + 22]), "=r"(r[b + 23]),    \
        "=r"(r[b + 24]), "=r"(r[b + 25]), "=r"(r[b + 26]), "=r"(r[b + 27]), "=r"(r[b + 28]), "=r"(r[b + 29]),    \
        "=r"(r[b + 30]), "=r"(r[b + 31])                                                                      \
      : "r"(taddr + o));
  SLM_TLD(0, 0)
  SLM_TLD(32, 32)
#undef SLM_TLD
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared-memory matrix descriptor (tcgen05 "smem descriptor"): start address, leading and
// stride byte offsets (16-byte units), version 1 (sm_100), layout SWIZZLE_128B (= 2).
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version
  d |= (uint64_t)2 << 61;   // SWIZZLE_128B
  return d;
}

// Instruction descriptor for kind::f16: fp32 accumulate, bf16 A/B, majorness, N>>3, M>>4.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ---------------------------------------------------------------- epilogues
// Each receives (m, n0, acc[32], ks): rows m, columns n0..n0+31 of the tile, K slice ks.
struct EpiResid {  // forward, no split: out[n*ld+m] = resid[n*ld+m] + acc + bias[m]  (out may alias resid)
  static constexpr bool kTma = false;
  float* out;
  const float* resid;
  const float* bias;
  long ld;
  __device__ __forceinline__ void operator()(int m, int n0, const float* acc, int) const {
    const float bm = bias[m];
    // all 32 loads first: `out` may alias `resid` (in-place Block), so loads interleaved with
    // stores would be serialised by the compiler (one memory latency per element)
    float r[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = resid[(long)(n0 + j) * ld + m];
#pragma unroll
    for (int j = 0; j < 32; ++j) out[(long)(n0 + j) * ld + m] = __fadd_rn(r[j], __fadd_rn(acc[j], bm));
  }
};
struct EpiStoreF32 {  // out[n*ld+m] = acc
  static constexpr bool kTma = false;
  float* out;
  long ld;
  __device__ __forceinline__ void operator()(int m, int n0, const float* acc, int) const {
#pragma unroll
    for (int j = 0; j < 32; ++j) out[(long)(n0 + j) * ld + m] = acc[j];
  }
};
struct EpiStoreBF16 {  // out[n*ld+m] = bf16(acc)
  static constexpr bool kTma = false;
  __nv_bfloat16* out;
  long ld;
  __device__ __forceinline__ void operator()(int m, int n0, const float* acc, int) const {
#pragma unroll
    for (int j = 0; j < 32; ++j) out[(long)(n0 + j) * ld + m] = __float2bfloat16_rn(acc[j]);
  }
};
// split-K partial of slice ks: P[ks][n][m] (fp32, coalesced: a warp writes 32 consecutive m).
// The consumer (bn_act_rk / bn_bwd_rk) sums the slices in the fixed order 0..SK-1.
struct EpiPartial {
  static constexpr bool kTma = false;
  float* P;
  long ld;      // = M
  long slice;   // = N * M
  __device__ __forceinline__ void operator()(int m, int n0, const float* acc, int ks) const {
    float* p = P + (long)ks * slice + m;
#pragma unroll
    for (int j = 0; j < 32; ++j) p[(long)(n0 + j) * ld] = acc[j];
  }
};

// gradient accumulation in place across time steps: out[n*ld+m] += acc
struct EpiAccF32 {
  static constexpr bool kTma = false;
  float* out;
  long ld;
  __device__ __forceinline__ void operator()(int m, int n0, const float* acc, int) const {
    float r[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = out[(long)(n0 + j) * ld + m];
#pragma unroll
    for (int j = 0; j < 32; ++j) out[(long)(n0 + j) * ld + m] = __fadd_rn(r[j], acc[j]);
  }
};

// the same partials written by TMA bulk tensor stores from a smem staging box (tmC maps P
// as [slices * N rows][M] fp32, box {128, 32}); row of (ks, n) = ks * N + n
struct EpiPartialTma {
  static constexpr bool kTma = true;
  int n_rows;   // = N
  __device__ __forceinline__ int row0(int ks) const { return ks * n_rows; }
  __device__ __forceinline__ void operator()(int, int, const float*, int) const {}
};

// dW: bf16(acc) written by TMA bulk tensor stores from a smem staging box (tmC maps the output as
// [rows][M] bf16, box {128, 32}); row of column n = row_base + n (layer l's block of dW)
struct EpiStoreBF16Tma {
  static constexpr bool kTma = true;
  static constexpr bool kHalf = true;
  int row_base;
  __device__ __forceinline__ int row0(int) const { return row_base; }
  __device__ __forceinline__ void operator()(int, int, const float*, int) const {}
};
template <class E, class = void>
struct EpiHalf : std::false_type {};
template <class E>
struct EpiHalf<E, std::void_t<decltype(E::kHalf)>> : std::bool_constant<E::kHalf> {};

// ---------------------------------------------------------------- the kernel
template <int BN, bool A_MN, bool B_MN, int CG = 1>
struct TcCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;   // 16 KiB (this CTA's 128 rows of A)
  static constexpr int BNC = BN / CG;           // columns of B staged by this CTA
  static constexpr int B_BYTES = BNC * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  // as many stages as fit in ~200 KiB (up to 8): the K loop is latency bound, bytes in
  // flight per SM set its bandwidth
  // Stage caps by operand majorness (compile-time knobs, measured): the weight-gradient GEMMs
  // (both operands MN-major, short K = batch) keep 2 stages and the dX GEMMs (A = W read
  // MN-major) 4, so two CTAs share an SM and one's epilogue overlaps the other's main loop in
  // the throughput-bound backward phase (C2 34.7 -> 34.1 ms, C3 342 -> 327-331 ms); the forward
  // GEMMs keep the deep ring (their W prefetch before the dependency wait is on the critical path),
  // except the narrow ones (N tile <= 64: the LSTM gates / head GEMMs, 4 stages: C3 327 -> 321 ms)
#ifndef SLM_DW_STAGES
#define SLM_DW_STAGES 2
#endif
#ifndef SLM_DX_STAGES
#define SLM_DX_STAGES 4
#endif
#ifndef SLM_NARROW_STAGES
#define SLM_NARROW_STAGES 4
#endif
#ifndef SLM_WIDE_STAGES
#define SLM_WIDE_STAGES 8
#endif
  static constexpr int CAP = (A_MN && B_MN) ? SLM_DW_STAGES
                             : (A_MN ? SLM_DX_STAGES : (BN <= 64 ? SLM_NARROW_STAGES : SLM_WIDE_STAGES));
  static constexpr int STAGES = (200 * 1024 / STAGE) > CAP ? CAP : (200 * 1024 / STAGE);
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
};

// debug instrumentation: per-CTA %globaltimer stamps at 8 phase points (null = off)
// Two layouts: dbg bit 2 (debug hook only): [cta][8 phases] (micro-benchmarks); dbg >> 8 == slot + 1: the
// launch's start (phase 0) and end (phase 7) per CTA at [slot][1024 CTAs][2] — used to time
// every GEMM of a real step on the device clock (profile_ts option of the model).
__device__ unsigned long long* g_slm_ts = nullptr;
// the stamp buffer of this launch: the global pointer is read only when the launch is profiled
// (dbg != 0), so production launches issue no memory access for their instrumentation
__device__ __forceinline__ unsigned long long* ts_buffer(int dbg) { return dbg ? g_slm_ts : nullptr; }
// dbg bit 4 (16): phase mode of the step profile, all 8 phases of every CTA at [slot][1024 CTAs][8]
__device__ __forceinline__ void ts_mark(unsigned long long* p, int phase, int dbg, int tid = 0) {
  if (p != nullptr && threadIdx.x == tid) {
    const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int slot = (dbg >> 8) - 1;
    if (slot < 0 && !(dbg & 4)) return;   // per-CTA phase mode only from the debug hook (bit 2)
    if (slot >= 0 && !(dbg & 16) && phase != 0 && phase != 7) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (slot >= 0 && (dbg & 16))
      p[((size_t)slot * 1024 + cta) * 8 + phase] = t;
    else if (slot >= 0)
      p[((size_t)slot * 1024 + cta) * 2 + (phase == 7)] = t;
    else
      p[cta * 8 + phase] = t;
  }
}

// profile mode "after dependency" (dbg bit 3): the launch's start stamp is replaced by the
// moment this CTA's producer returns from griddepcontrol.wait (its inputs are ready), so the
// span excludes time spent overlapping the predecessor under programmatic dependent launch
__device__ __forceinline__ void ts_dep(unsigned long long* p, int dbg) {
  const int slot = (dbg >> 8) - 1;
  if (p == nullptr || slot < 0 || (dbg & 16)) return;
  const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  p[((size_t)slot * 1024 + cta) * 2] = t;
}

// a_row0/b_row0: row offsets added to the tensor-map coordinates of A / B (e.g. layer l's
// weight block inside the [n*d, d] weight tensor).
// PREFETCH_A: A is read-only for the whole step (the weights), so its first pipeline stages are
// requested before griddepcontrol.wait, i.e. while the previous kernel is still finishing
// (programmatic dependent launch); B and the epilogue inputs are read only after the wait.
// Split-K: gridDim.z = number of K slices; CTA z accumulates K range [z*K/Z, (z+1)*K/Z) and
// hands its fp32 partial to the epilogue with ks = z (EpiPartial).  Measured on B200 the
// per-SM operand ingest (~64-70 B/clk via TMA, and SS-mode tcgen05 operand reads at a
// similar rate) bounds these skinny GEMMs, so K is split until each SM ingests ~192 KiB;
// the partials are summed by the BN kernel that consumes the GEMM output anyway
// (distributed-shared-memory reduction was measured ~16 KB/us per SM: too slow).
// CG = 2: CTA pair (launched as clusters of 2 along x): CTAs 2c and 2c+1 compute the 256 x BN
// tile of rows [256c, 256c+256) with one cta_group::2 MMA per K step; each stages its own
// 128 rows of A and BN/2 columns of B (so per-SM operand ingest drops from (128+BN)*64*2 to
// (128+BN/2)*64*2 bytes per K step), the leader issues the MMAs and multicasts the commits.
template <int BN, bool A_MN, bool B_MN, bool PREFETCH_A, class Epi, int CG = 1>
__global__ void __launch_bounds__(128, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, int K, int a_row0, int b_row0, Epi epi, int dbg,
                   int pf_row0, ConvB cb) {
  unsigned long long* const tsp = ts_buffer(dbg);
  ts_mark(tsp, 0, dbg);
  using C = TcCfg<BN, A_MN, B_MN, CG>;
  uint32_t rank = 0;
  if constexpr (CG == 2) rank = cluster_ctarank();
  const bool leader = rank == 0;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps the shared space
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* accum = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * C::BM, n0 = blockIdx.y * BN;
  const int ks = (int)blockIdx.z;
  const int nk = K / C::BK / (int)gridDim.z;
  const int kbase = ks * nk * C::BK;

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      for (int s = 0; s < C::STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      mbar_init(accum, 1);
      fence_barrier_init();
    }
    __syncwarp();
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();   // the peer's barriers are initialised before use
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ts_mark(tsp, 1, dbg);
  // pf_row0 >= 0: pull this CTA's A tile of the NEXT GEMM of the chain (the next layer's
  // weights, rows a_row0 -> pf_row0) into L2 while this one runs
  if (pf_row0 >= 0 && warp == 2 && lane == 0) {
    for (int kb = 0; kb < nk; ++kb) {
      const int k0 = kbase + kb * C::BK;
      if (A_MN) {
        tma_prefetch_l2(&tmA, m0, pf_row0 + k0);
        tma_prefetch_l2(&tmA, m0 + 64, pf_row0 + k0);
      } else {
        tma_prefetch_l2(&tmA, k0, pf_row0 + m0);
      }
    }
  }

  auto tma = [&](void* dst, const CUtensorMap* map, int s, int c0, int c1) {
    if constexpr (CG == 2)
      tma_load_2d_cg2(dst, map, &full[s], c0, c1);
    else
      tma_load_2d(dst, map, &full[s], c0, c1);
  };
  // tap (u, v) and channel offset of im2col column kk, as 4-D box coordinates (c, j0, i0, img) of
  // the positions starting at q (whole image rows)
  auto conv_load = [&](void* dst, const CUtensorMap* map, int s, int kk, int q) {
    const int tap = kk / cb.cin, c0 = kk - tap * cb.cin, u = tap / cb.k, v = tap - u * cb.k, p = cb.k / 2;
    const int img = q / cb.hw, i0 = (q - img * cb.hw) / cb.w;
    tma_load_4d(dst, map, &full[s], c0, v - p, cb.s * i0 + u - p, img);
  };
  auto load_a = [&](int kb, int s) {
    uint8_t* sa = smem + s * C::STAGE;
    const int k0 = kbase + kb * C::BK;
    if (A_MN && cb.on == 2) {   // implicit im2col, A = col [positions = K][M = (tap, c)]
      conv_load(sa, &tmA, s, m0, k0);
      conv_load(sa + 8192, &tmA, s, m0 + 64, k0);
    } else if (A_MN) {  // A stored [K][M]: boxes of 64(M) x 64(K)
      tma(sa, &tmA, s, m0, a_row0 + k0);
      tma(sa + 8192, &tmA, s, m0 + 64, a_row0 + k0);
    } else {     // A stored [M][K]: one box of 64(K) x 128(M)
      tma(sa, &tmA, s, k0, a_row0 + m0);
    }
  };
  const int nb0 = n0 + (int)rank * C::BNC;   // first B column staged by this CTA
  auto load_b = [&](int kb, int s) {
    uint8_t* sb = smem + s * C::STAGE + C::A_BYTES;
    const int k0 = kbase + kb * C::BK;
    if (B_MN) {
#pragma unroll
      for (int j = 0; j < C::BNC / 64; ++j) tma(sb + j * 8192, &tmB, s, nb0 + 64 * j, b_row0 + k0);
    } else if (CG == 1 && cb.on == 1) {   // implicit im2col, B = col [N = positions][K = (tap, c)]
      conv_load(sb, &tmB, s, k0, nb0);
    } else {     // box rows = BN / CG
      tma(sb, &tmB, s, k0, b_row0 + nb0);
    }
  };
  // the leader's full barrier counts both CTAs' bytes; only it arrives (expect_tx)
  auto expect = [&](int s) {
    if (leader) mbar_expect_tx(&full[s], CG * C::STAGE);
  };

  if (CG == 1 && warp == 0 && lane == 0 && (dbg & 2)) {
    // debug probe: MMA issue rate only (no TMA, operands are whatever is in smem)
    pdl_wait();
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % C::STAGES;
      if (kb >= C::STAGES) mbar_wait(&empty[s], ((kb / C::STAGES) - 1) & 1);
      mbar_arrive(&full[s]);
    }
  } else if (warp == 0 && lane == 0) {
    // ===== TMA producer
    int kb0 = 0;
    if (PREFETCH_A) {
      kb0 = nk < C::STAGES ? nk : C::STAGES;
      for (int kb = 0; kb < kb0; ++kb) {
        expect(kb);
        load_a(kb, kb);
      }
      pdl_wait();
      if (dbg & 8) ts_dep(tsp, dbg);
      for (int kb = 0; kb < kb0; ++kb) load_b(kb, kb);
    } else {
      pdl_wait();
      if (dbg & 8) ts_dep(tsp, dbg);
    }
    for (int kb = kb0; kb < nk; ++kb) {
      const int s = kb % C::STAGES;
      if (kb >= C::STAGES) mbar_wait(&empty[s], ((kb / C::STAGES) - 1) & 1);
      expect(s);
      load_a(kb, s);
      load_b(kb, s);
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ===== MMA issuer (the leader of a CTA pair issues for both)
    constexpr uint32_t idesc = make_idesc(C::BM * CG, BN, A_MN, B_MN);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % C::STAGES;
      mbar_wait(&full[s], (kb / C::STAGES) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * C::STAGE);
      const uint32_t sb = sa + C::A_BYTES;
      if (CG == 1 && (dbg & 1)) {  // debug probe: data movement only, no MMA (bits 0-1 only; bits 8+ = ts slot)
        mbar_arrive(&empty[s]);
        continue;
      }
#pragma unroll
      for (int kk = 0; kk < C::BK / 16; ++kk) {
        // K-major SW128: +32 B per K=16 inside the 128-B row; SBO = 8 rows * 128 B.
        // MN-major SW128: +16 rows * 128 B per K=16; LBO = 64-element MN chunk (8 KiB box).
        uint64_t ad = A_MN ? make_sdesc(sa + kk * 2048, 8192, 1024) : make_sdesc(sa + kk * 32, 16, 1024);
        uint64_t bd = B_MN ? make_sdesc(sb + kk * 2048, 8192, 1024) : make_sdesc(sb + kk * 32, 16, 1024);
        if constexpr (CG == 2)
          tc_mma2(tmem, ad, bd, idesc, (kb | kk) != 0);
        else
          tc_mma(tmem, ad, bd, idesc, (kb | kk) != 0);
      }
      if constexpr (CG == 2)
        tc_commit2(&empty[s], 3);
      else
        tc_commit(&empty[s]);
    }
    if constexpr (CG == 2)
      tc_commit2(accum, 3);
    else if (dbg & 1)
      mbar_arrive(accum);
    else
      tc_commit(accum);
  }
  __syncwarp();
  // ===== epilogue: TMEM -> registers -> global
  pdl_wait();
  mbar_wait(accum, 0);
  tc_fence_after();
  // let the dependent kernel launch only now (its CTAs would otherwise sit on this kernel's SMs
  // waiting in griddepcontrol.wait for the whole main loop; measured: early trigger is slower)
  pdl_launch();
  ts_mark(tsp, 2, dbg);
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  const int m = m0 + warp * 32 + lane;
  if constexpr (Epi::kTma) {
    // fp32 (or bf16, EpiHalf) tile -> smem box [32 n][128 m] (a warp writes 128 (64) contiguous
    // bytes: conflict-free) -> cp.async.bulk.tensor store, double-buffered; the pipeline smem is
    // free after the MMAs.
    constexpr bool HALF = EpiHalf<Epi>::value;
    constexpr int BUF_BYTES = 32 * 128 * (HALF ? 2 : 4);
    // one TMEM round trip per 64 columns (two staging boxes); 4 boxes in a ring, one bulk group
    // per iteration, so iteration it reuses the boxes of iteration it - 2
    constexpr int CW = BN >= 64 ? 64 : 32;
    auto stage_box = [&](int box, const float* acc) {
      uint8_t* sbuf = smem + box * BUF_BYTES;
      if constexpr (HALF) {
        __nv_bfloat16* sp = reinterpret_cast<__nv_bfloat16*>(sbuf) + warp * 32 + lane;
#pragma unroll
        for (int j = 0; j < 32; ++j) sp[j * 128] = __float2bfloat16_rn(acc[j]);
      } else {
        float* sp = reinterpret_cast<float*>(sbuf) + warp * 32 + lane;
#pragma unroll
        for (int j = 0; j < 32; ++j) sp[j * 128] = acc[j];
      }
    };
    auto store_box = [&](int box, int c) {
      asm volatile(
          "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
              reinterpret_cast<uint64_t>(&tmC)),
          "r"(smem_u32(smem + box * BUF_BYTES)), "r"(m0), "r"(epi.row0(ks) + n0 + c)
          : "memory");
    };
#pragma unroll 1
    for (int c = 0; c < BN; c += CW) {
      const int it = c / CW;
      const int b0 = (2 * it) & 3;
      if (it >= 2) {  // the stores issued two iterations ago must have read these boxes
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
      }
      if constexpr (CW == 64) {
        float acc[64];
        tmem_ld64(trow + c, acc);
        stage_box(b0, acc);
        stage_box(b0 + 1, acc + 32);
      } else {
        float acc[32];
        tmem_ld32(trow + c, acc);
        stage_box(b0, acc);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        store_box(b0, c);
        if constexpr (CW == 64) store_box(b0 + 1, c + 32);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  } else if constexpr (BN >= 64) {
#pragma unroll 1
    for (int c = 0; c < BN; c += 64) {
      float acc[64];
      tmem_ld64(trow + c, acc);
      epi(m, n0 + c, acc, ks);
      epi(m, n0 + c + 32, acc + 32, ks);
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float acc[32];
      tmem_ld32(trow + c, acc);
      epi(m, n0 + c, acc, ks);
    }
  }
  ts_mark(tsp, 7, dbg);
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) {
    cluster_sync();
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  } else {
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  }
}

}  // namespace slmk
