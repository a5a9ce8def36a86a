// The residual Block of the chain as ONE kernel per node of V' (sm_100a): tcgen05 GEMM with
// split-K over a cluster of S CTAs, an L2 reduce-scatter of the fp32 partials inside the
// cluster, and the batch-norm work fused into the epilogue.
//
//   forward / mirror Block_l:
//     z = W_l a_l^T (swap-AB: M = 64 output features per CTA, N = B = the whole batch, K split
//     over the S CTAs of a cluster),  x_{l+1} = x_l + (z + b_l),  then the batch statistics of
//     x_{l+1} and a_{l+1} = ReLU(BN_{l+1}(x_{l+1})) (bf16) for the next Block.
//   gradient Block_l (a8): da = g W_l (dX, A = W read MN-major), then the BN backward
//     du = da 1[u > 0], dgamma = sum_b du xhat, dbeta = sum_b du,
//     dx_l = g + gamma rstd (du - dbeta/B - xhat dgamma/B), db_{l-1} = sum_b dx_l, plus the bf16
//     copies of dx_l (next dX / dW operand) and a_l (dW operand).
//
// Why this shape (measured on B200, profiles/r2_microbench.md):
//  * the whole batch is the MMA's N (the per-feature batch statistics stay inside one CTA);
//  * the layer's K is split over a cluster of S = 4 CTAs and the S fp32 partials are
//    reduce-scattered through L2 (TMA stores / loads; distributed shared memory moves only
//    ~10-20 GB/s per SM);
//  * an SM stores only ~28 B/clk to L2 (loads ~100 B/clk), so the epilogue is bound by its
//    writes: the peers' partial slices plus x_{l+1} and a_{l+1}.  M = 64 features per CTA (128
//    CTAs at d = 2048) halves every SM's writes against M = 128 (64 CTAs) at the same per-layer
//    MMA time: tcgen05 M = 64 runs at half the M = 128 rate on half the rows.
// The M = 64 accumulator holds row r in TMEM lane 32 (r / 16) + r % 16 (measured,
// scripts/mb_layout.cu): warp quarter q owns rows 16q..16q+15 in its lanes 0..15.
//
// Determinism: every sum has a fixed order (MMA K order, slice order s, the
// per-thread row loop, then the row groups in order), so mirrors (same kernel, same launch
// configuration) reproduce the forward's bits; bn_k1_kernel (the operand of the first Block of a
// run) uses the identical statistics code and thread mapping.
#pragma once
#include "tc_gemm.cuh"

namespace slmk {

// 16 warps: TMA producer / MMA issuer / TMEM owner roles, then all 16 in the epilogue (measured: the
// epilogue's latency-bound passes ran 1.4 us with 8 warps, two per scheduler)
constexpr int kBlkThreads = 512;
constexpr int kBlkNH = kBlkThreads / 128;   // warps per TMEM lane quarter (column parts of the epilogue)
template <int B, int S, bool BWD, int BM_ = 64, int CG_ = 1>
struct BlkCfg {
  static constexpr int BM = BM_, BK = 64;     // BM = output features per CTA (the MMA's M: 64 or 128)
  static constexpr int CG = CG_;              // 2: CTA pairs (cta_group::2, M = 256 over two SMs; each
                                              // SM stages half of the batch columns)
  static constexpr int FS = BM / S;           // features owned by a CTA after the reduce-scatter
  static constexpr int RG = kBlkThreads / FS; // row groups of the epilogue (threads per feature)
  static constexpr int R = B / RG;            // rows per epilogue thread (values kept in registers)
  static constexpr int A_BYTES = BM * BK * 2; // one W tile (BM x 64 bf16)
  static constexpr int B_BYTES = B / CG * BK * 2;   // one operand tile (this CTA's B / CG rows x 64 bf16)
  static constexpr int SLICE = B * FS * 4;    // one fp32 slice [B][FS] (dense rows of FS floats)
  static constexpr int AUX = SLICE;           // x_l, staged by TMA during the main loop
  static constexpr int LIMIT = 227 * 1024;
  static constexpr int STATIC = RG * FS * 4 + 64;
#ifndef SLM_BLK_NB
#define SLM_BLK_NB 3
#endif
  static constexpr int NB = SLM_BLK_NB;       // operand ring (after griddepcontrol.wait, from L2)
  // W ring: as many tiles as fit (up to 8 = a 512-wide K slice): all of them are requested
  // before griddepcontrol.wait, so the weight stream from HBM overlaps the predecessor
  static constexpr int NA_FIT = (LIMIT - 1024 - AUX - 512 - STATIC - NB * B_BYTES) / A_BYTES;
  static constexpr int NA = NA_FIT > 8 ? 8 : NA_FIT;
  static constexpr int RING_MAIN = NA * A_BYTES + NB * B_BYTES;
  static constexpr int RING = RING_MAIN > S * SLICE ? RING_MAIN : S * SLICE;
  static constexpr int SMEM = 1024 + RING + AUX + 512;
  static constexpr int TMEM_COLS = B;
  static_assert(S == 2 || S == 4, "cluster of 2 or 4 CTAs");
  static_assert(BM == 64 || BM == 128, "M tile");
  static_assert(CG == 1 || (CG == 2 && BM == 128), "CTA pairs with 128 rows per CTA");
  static_assert(B == 64 || B == 128 || B == 256, "batch tile");
  static_assert(FS % 16 == 0 && R >= 1 && R <= 32, "slice / registers");
  static_assert(NA >= 2, "pipeline");
  static_assert(SMEM + STATIC <= LIMIT, "shared memory");
};

// An fp32 slice is [B][FS] row-major: the dense layout of a {FS, rows} TMA box.  The epilogue's
// thread t handles feature t % FS, so a warp touches 128 consecutive bytes (one row at FS = 32,
// two at FS = 16): no shared-memory bank conflicts (a [FS/16][B][16] layout had two-way conflicts
// at FS = 32 and doubled the epilogue's shared-memory time, measured with ncu stall_mio).

// sum of one value per (row group rg, feature fl) over the RG row groups, in the order 0..RG-1
template <int RG, int FS>
__device__ __forceinline__ float rg_sum(float v, float (*red)[FS], int rg, int fl) {
  red[rg][fl] = v;
  __syncthreads();
  float t = red[0][fl];
#pragma unroll
  for (int r = 1; r < RG; ++r) t = __fadd_rn(t, red[r][fl]);
  __syncthreads();
  return t;
}

// Batch statistics of one feature over the B rows held by its RG threads (R each, in registers):
// two-pass mean / centred variance, per-thread serial then the row groups in order.  The forward
// epilogue, the backward epilogue and bn_k1_kernel share this exact code and mapping (thread t:
// feature t % FS, rows t / FS + RG j), so the statistics of a given x are bit-identical.
template <int B, int S, int BM>
__device__ __forceinline__ void slice_stats(const float (&v)[BlkCfg<B, S, false, BM>::R],
                                            float (*red)[BlkCfg<B, S, false, BM>::FS], int fl, int rg, float& mu,
                                            float& rstd) {
  using C = BlkCfg<B, S, false, BM>;
  constexpr float invB = 1.0f / B;   // exact: B is a power of two
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < C::R; ++j) s = __fadd_rn(s, v[j]);
  mu = __fmul_rn(rg_sum<C::RG, C::FS>(s, red, rg, fl), invB);
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < C::R; ++j) {
    const float e = __fsub_rn(v[j], mu);
    q = __fmaf_rn(e, e, q);
  }
  const float var = __fmul_rn(rg_sum<C::RG, C::FS>(q, red, rg, fl), invB);
  rstd = __frcp_rn(__fsqrt_rn(__fadd_rn(var, kEps)));
}

// a = bf16(ReLU(gamma xhat + beta)) of the slice's rows (next Block's operand)
template <int B, int S, int BM>
__device__ __forceinline__ void slice_act(const float (&v)[BlkCfg<B, S, false, BM>::R],
                                          float (*red)[BlkCfg<B, S, false, BM>::FS], int d, int f, int rg, int fl,
                                          float g, float bt, __nv_bfloat16* __restrict__ a) {
  using C = BlkCfg<B, S, false, BM>;
  float mu, rstd;
  slice_stats<B, S, BM>(v, red, fl, rg, mu, rstd);
#pragma unroll
  for (int j = 0; j < C::R; ++j)
    a[(size_t)(rg + C::RG * j) * d + f] = __float2bfloat16_rn(fmaxf(bn_u(bn_xhat(v[j], mu, rstd), g, bt), 0.f));
}

struct BlkArgs {
  int d;
  int a_row0;              // row of W_l in the [n*d][d] weight tensor (= l*d)
  int pf_row0;             // row of the next Block's W (pulled into L2 during this one), -1 none
  int x_row0;              // row of x_l in its fp32 [rows][d] tensor map
  const float* g;          // bwd: g = dx_{l+1} [B][d] fp32
  float* out;              // fwd: x_{l+1}; bwd: dx_l                   [B][d] fp32
  const float* bias;       // fwd: b_l
  const float* gamma;      // fwd: gamma_{l+1} (null: no next Block); bwd: gamma_l
  const float* beta;
  __nv_bfloat16* a_out;    // fwd: a_{l+1}; bwd: a_l (dW operand)     [B][d] bf16
  __nv_bfloat16* gq_out;   // bwd: bf16(dx_l)
  float* dgamma;           // bwd
  float* dbeta;
  float* db_prev;          // bwd: db_{l-1} (null at l = 0)
  int dbg;
};

// grid = (d/BM) * S CTAs, clusters of S along x (CTA m*S + k = K slice k of output tile m),
// kBlkThreads threads: warp 0 lane 0 TMA producer, warp 1 lane 0 MMA issuer, warp 2 owns the TMEM
// allocation; then all warps run the epilogue.
//   tmA: W, K-major {64, BM} box or MN-major {64, 64} boxes
//   tmB: the bf16 operand [B][d] (a_l fwd, bf16 dx_{l+1} bwd), {64, B} box, 128-byte swizzle
//   tmP / tmPs: the partial buffer [d/BM][S owners][S sources][B] rows of FS fp32, {FS, B} box (the
//        owner's loads) / {FS, 32} box (the chunk stores: FS features x 32 batch rows)
//   tmX: fp32 [rows][d] source of x_l, {FS, B} box
template <int B, int S, bool BWD, int BM_, int CG>
__global__ void __launch_bounds__(kBlkThreads, 1)
    blk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmPs,
               const __grid_constant__ CUtensorMap tmX, const BlkArgs args) {
  using C = BlkCfg<B, S, BWD, BM_, CG>;
  constexpr int FS = C::FS, RG = C::RG, R = C::R, NA = C::NA, NB = C::NB, BM = C::BM;
  unsigned long long* const tsp = ts_buffer(args.dbg);
  ts_mark(tsp, 0, args.dbg);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned by pointer arithmetic on the __shared__ array (not through an integer), so
  // the compiler keeps the shared address space (LDS/STS) for the epilogue's accesses
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;                                   // W tiles [NA] | operand tiles [NB]; epilogue: S slices
  uint8_t* bring = ring + NA * C::A_BYTES;
  float* xs = reinterpret_cast<float*>(smem + C::RING);   // x_l slice
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + C::RING + C::AUX);
  uint64_t* emptyA = fullA + NA;
  uint64_t* fullB = emptyA + NA;
  uint64_t* emptyB = fullB + NB;
  uint64_t* accum = emptyB + NB;
  uint64_t* auxb = accum + 1;
  uint64_t* recvb = auxb + 1;    // remote arrivals: the peers' chunks of this owner's slice are in L2
  uint64_t* recvb2 = recvb + 1;  // tx bytes of the incoming slices
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recvb2 + 1);
  __shared__ float red[RG][FS];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = args.d;
  // cluster of S * CG CTAs: rank = K slice * CG + pair half
  const uint32_t crank = cluster_ctarank();
  const uint32_t k = crank / CG, p = crank % CG;
  const bool mma_cta = p == 0;   // the pair's leader issues the MMAs (CG = 1: every CTA)
  const int m = ((int)blockIdx.x / (S * CG)) * CG + (int)p;
  const int m0 = m * BM;
  const int nk = d / 64 / S;
  const int kbase = (int)k * nk * 64;
  const int f0 = m0 + (int)k * FS;   // first feature this CTA owns after the reduce-scatter
  // this thread's feature in the epilogue and its parameters, loaded now (they are constant during
  // the step) so their latency hides under the main loop
  const int fl = threadIdx.x % FS, rg = threadIdx.x / FS;
  const int f = f0 + fl;
  const float p_bias = BWD ? 0.f : args.bias[f];
  const float p_gam = args.gamma ? args.gamma[f] : 0.f;
  const float p_bet = args.gamma ? args.beta[f] : 0.f;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmP);
    prefetch_tmap(&tmPs);
    for (int s = 0; s < NA; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < NB; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], 1);
    }
    mbar_init(accum, 1);
    mbar_init(auxb, 1);
    mbar_init(recvb, kBlkNH * (S - 1));   // one arrival per storing peer warp (one per column part)
    mbar_init(recvb2, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  cluster_sync();   // every CTA's barriers are initialised before a peer can arrive on them
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // CG = 2: both CTAs' loads complete on the leader's full barriers (it expects both halves' bytes)
  auto tma = [&](void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    if constexpr (CG == 2)
      tma_load_2d_cg2(dst, map, bar, c0, c1);
    else
      tma_load_2d(dst, map, bar, c0, c1);
  };
  auto load_a = [&](int kb) {
    const int s = kb % NA;
    uint8_t* sa = ring + s * C::A_BYTES;
    const int k0 = kbase + kb * 64;
    if (mma_cta) mbar_expect_tx(&fullA[s], CG * C::A_BYTES);
    if (BWD) {   // W stored [f_out = K][f_in = M]: 64 (M) x 64 (K) boxes
#pragma unroll
      for (int mm = 0; mm < BM; mm += 64) tma(sa + mm * 128, &tmA, &fullA[s], m0 + mm, args.a_row0 + k0);
    } else {     // W stored [f_out = M][f_in = K]: a 64 (K) x BM (M) box
      tma(sa, &tmA, &fullA[s], k0, args.a_row0 + m0);
    }
  };
  auto load_b = [&](int kb) {   // this CTA's B / CG batch rows of the operand
    const int s = kb % NB;
    if (mma_cta) mbar_expect_tx(&fullB[s], CG * C::B_BYTES);
    tma(bring + s * C::B_BYTES, &tmB, &fullB[s], kbase + kb * 64, (int)p * (B / CG));
  };

  if (warp == 0 && lane == 0) {
    // ===== TMA producer: the weights do not depend on the previous kernel, so up to NA tiles of
    // W are requested before griddepcontrol.wait (they overlap the predecessor's tail)
    const int na0 = nk < NA ? nk : NA, nb0 = nk < NB ? nk : NB;
    for (int kb = 0; kb < na0; ++kb) load_a(kb);
    pdl_wait();
    ts_mark(tsp, 1, args.dbg);
    if (args.dbg & 8) ts_dep(tsp, args.dbg);
    for (int kb = 0; kb < nb0; ++kb) load_b(kb);
    // the epilogue's x_l slice lands in its own buffer while the main loop runs
    mbar_expect_tx(auxb, C::AUX);
    tma_load_2d(xs, &tmX, auxb, f0, args.x_row0);
    // refill each ring slot as soon as the MMAs reading it retire
    for (int kb = 0; kb < nk; ++kb) {
      if (kb + NB < nk) {
        mbar_wait(&emptyB[kb % NB], (kb / NB) & 1);
        load_b(kb + NB);
      }
      if (kb + NA < nk) {
        mbar_wait(&emptyA[kb % NA], (kb / NA) & 1);
        load_a(kb + NA);
      }
    }
    // the next Block's weight tiles of this CTA into L2 (HBM -> L2 off the critical path: the next
    // kernel's requests, before and after its dependency wait, then hit L2)
    if (args.pf_row0 >= 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int k0 = kbase + kb * 64;
        if (BWD) {
#pragma unroll
          for (int mm = 0; mm < BM; mm += 64) tma_prefetch_l2(&tmA, m0 + mm, args.pf_row0 + k0);
        } else {
          tma_prefetch_l2(&tmA, k0, args.pf_row0 + m0);
        }
      }
    }
  } else if (warp == 1 && lane == 0 && mma_cta) {
    // ===== MMA issuer (CG = 2: the pair's leader issues M = 256 MMAs for both CTAs and multicasts
    // its commits to the pair's barriers)
    constexpr uint32_t idesc = make_idesc(BM * CG, B, BWD, false);
    const uint16_t pair = (uint16_t)(3u << (2 * k));
    auto commit = [&](uint64_t* bar) {
      if constexpr (CG == 2)
        tc_commit2(bar, pair);
      else
        tc_commit(bar);
    };
    for (int kb = 0; kb < nk; ++kb) {
      mbar_wait(&fullA[kb % NA], (kb / NA) & 1);
      mbar_wait(&fullB[kb % NB], (kb / NB) & 1);
#ifdef SLM_EXP_MAINLOOP
      if (kb == 0) ts_mark(tsp, 5, args.dbg, 32);
      if (kb == nk - 1) ts_mark(tsp, 6, args.dbg, 32);
#endif
      tc_fence_after();
      const uint32_t sa = smem_u32(ring + (kb % NA) * C::A_BYTES);
      const uint32_t sb = smem_u32(bring + (kb % NB) * C::B_BYTES);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = BWD ? make_sdesc(sa + kk * 2048, 8192, 1024) : make_sdesc(sa + kk * 32, 16, 1024);
        const uint64_t bd = make_sdesc(sb + kk * 32, 16, 1024);
        if constexpr (CG == 2)
          tc_mma2(tmem, ad, bd, idesc, (kb | kk) != 0);
        else
          tc_mma(tmem, ad, bd, idesc, (kb | kk) != 0);
      }
      commit(&emptyB[kb % NB]);
      commit(&emptyA[kb % NA]);
    }
    commit(accum);
  }
  __syncwarp();

  // ===== epilogue 1: accumulator -> the S feature slices (smem).  Warp (q, h) reads TMEM lane
  // quarter q (rows 16q..16q+15 in lanes 0..15) for batch columns h*B/2..: it stages its 16
  // features x 32 columns chunk by chunk and, when they belong to a peer, TMA-stores each chunk at
  // once (stores overlap the TMEM reads), waits for its stores to complete and signals the owner
  // through a remote mbarrier arrive; an owner loads its incoming slices once all its peers' warps
  // have arrived (no cluster-wide barrier)
  mbar_wait(accum, 0);
  tc_fence_after();
  ts_mark(tsp, 2, args.dbg);
  {
    // TMEM lane quarter q of the tile: BM = 128 -> rows 32q..32q+31 (lanes 0..31); BM = 64 -> rows
    // 16q..16q+15 (lanes 0..15, measured layout).  A quarter's rows belong to one owner slice;
    // QPO quarters make up a slice (2 only for BM = 64, S = 2).
    constexpr int QR = BM / 4;                 // tile rows per quarter
    constexpr int QPO = FS / QR;               // quarters per owner slice
    const int q = warp & 3, h = warp >> 2;     // lane quarter, column part h of kBlkNH
    const bool valid = QR == 32 || lane < 16;
    const int ft = QR * q + (lane & (QR - 1)); // tile row (feature) of this lane
    const int ko = (QR * q) / FS;              // owner slice of this quarter
    const bool leader = (q % QPO) == 0;        // the quarter that issues the slice's stores
    float* slot = reinterpret_cast<float*>(ring + ko * C::SLICE);
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    // 32-column chunks dealt round-robin to the kBlkNH warps of a quarter (B = 64: two warps idle)
#pragma unroll 1
    for (int c0 = h * 32; c0 < B; c0 += 32 * kBlkNH) {
      float acc[32];
      tmem_ld32(trow + c0, acc);
      if (valid) {
        float* dst = slot + c0 * FS + ft % FS;
#pragma unroll
        for (int j = 0; j < 32; ++j) dst[j * FS] = acc[j];
      }
      if (ko != (int)k) {   // a peer's rows: store this {FS features, 32 rows} chunk now
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // staged smem -> TMA (async proxy)
        if constexpr (QPO == 2)   // both quarters of the slice have staged their halves
          asm volatile("bar.sync %0, 64;" ::"r"(1 + ko * kBlkNH + h) : "memory");
        else
          __syncwarp();
        if (leader && lane == 0) {
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                           reinterpret_cast<uint64_t>(&tmPs)),
                       "r"(smem_u32(slot + c0 * FS)), "r"(0), "r"(((m * S + ko) * S + (int)k) * B + c0)
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (ko != (int)k && leader && lane == 0) {
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // this warp's chunks are in L2
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                       cluster_map(smem_u32(recvb), (uint32_t)ko * CG + p))
                   : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  ts_mark(tsp, 3, args.dbg);
  if constexpr (CG == 1) {
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  }
  if (threadIdx.x == 0) {
    mbar_wait(recvb, 0);   // every peer warp holding part of this owner's slice has stored it
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_expect_tx(recvb2, (S - 1) * C::SLICE);
    for (int s = 0; s < S; ++s) {
      if (s == (int)k) continue;
      tma_load_2d(ring + s * C::SLICE, &tmP, recvb2, 0, ((m * S + (int)k) * S + s) * B);
    }
  }

  // ===== epilogue 2: sum the S partials (slot s = K slice s, fixed order) and the fused batch norm
  const float* ringf = reinterpret_cast<const float*>(ring);
  float gv[BWD ? R : 1];
  if constexpr (BWD) {   // g = dx_{l+1}: coalesced loads issued before waiting for the slices
#pragma unroll
    for (int j = 0; j < R; ++j) gv[j] = args.g[(size_t)(rg + RG * j) * d + f];
  }
  mbar_wait(auxb, 0);
  mbar_wait(recvb2, 0);
  // the next kernel may now start its prologue and weight prefetch, hidden under the batch-norm
  // work (measured: triggering at the kernel's end instead costs 0.8 us per backward layer at C2,
  // triggering at the epilogue's start 0.3 us per forward Block)
  pdl_launch();
  ts_mark(tsp, 4, args.dbg);
  float xv[R], zv[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int off = (rg + RG * j) * FS + fl;
    float z = ringf[off];
#pragma unroll
    for (int s = 1; s < S; ++s) z = __fadd_rn(z, ringf[s * (C::SLICE / 4) + off]);
    zv[j] = z;
    xv[j] = xs[off];
  }
  if constexpr (!BWD) {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      xv[j] = __fadd_rn(xv[j], __fadd_rn(zv[j], p_bias));
#ifndef SLM_EXP_NO_XSTORE
      args.out[(size_t)(rg + RG * j) * d + f] = xv[j];
#endif
    }
#ifndef SLM_EXP_MAINLOOP
    ts_mark(tsp, 5, args.dbg);
#endif
    if (args.gamma != nullptr) slice_act<B, S, BM>(xv, red, d, f, rg, fl, p_gam, p_bet, args.a_out);
  } else {
    float mu, rstd;
    slice_stats<B, S, BM>(xv, red, fl, rg, mu, rstd);
    const float ga = p_gam, bt = p_bet;
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const float xh = bn_xhat(xv[j], mu, rstd);
      const float u = bn_u(xh, ga, bt);
      zv[j] = u > 0.f ? zv[j] : 0.f;   // du
      args.a_out[(size_t)(rg + RG * j) * d + f] = __float2bfloat16_rn(fmaxf(u, 0.f));
      s1 = __fadd_rn(s1, zv[j]);
      s2 = __fmaf_rn(zv[j], xh, s2);
    }
    ts_mark(tsp, 5, args.dbg);
    const float S1 = rg_sum<RG, FS>(s1, red, rg, fl);
    const float S2 = rg_sum<RG, FS>(s2, red, rg, fl);
    constexpr float invB = 1.0f / B;
    const float m1 = __fmul_rn(S1, invB), m2 = __fmul_rn(S2, invB);
    const float kk = __fmul_rn(ga, rstd);
    float s3 = 0.f;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const float xh = bn_xhat(xv[j], mu, rstd);
      const float v = __fadd_rn(gv[j], __fmul_rn(kk, __fsub_rn(__fsub_rn(zv[j], m1), __fmul_rn(xh, m2))));
      args.out[(size_t)(rg + RG * j) * d + f] = v;
      args.gq_out[(size_t)(rg + RG * j) * d + f] = __float2bfloat16_rn(v);
      s3 = __fadd_rn(s3, v);
    }
    const float S3 = rg_sum<RG, FS>(s3, red, rg, fl);
    if (rg == 0) {
      args.dgamma[f] = S2;
      args.dbeta[f] = S1;
      if (args.db_prev) args.db_prev[f] = S3;
    }
  }
  if constexpr (CG == 2) {   // both CTAs of the pair are done with the pair's TMEM allocation
    tc_fence_before();
    cluster_sync();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  }
  ts_mark(tsp, 7, args.dbg);
}

// K1: a = ReLU(BN(x)) for the first Block of a forward / mirror run (x_0, or a kept x_{s_j}),
// with the Block epilogue's exact mapping and statistics code: grid = d / FS CTAs of kBlkThreads,
// x read coalesced into registers.
template <int B, int S, int BM>
__global__ void __launch_bounds__(kBlkThreads) bn_k1_kernel(const float* __restrict__ x,
                                                            const float* __restrict__ gamma,
                                                            const float* __restrict__ beta, int d,
                                                            __nv_bfloat16* __restrict__ a) {
  using C = BlkCfg<B, S, false, BM>;
  __shared__ float red[C::RG][C::FS];
  pdl_wait();
  const int fl = threadIdx.x % C::FS, rg = threadIdx.x / C::FS;
  const int f = blockIdx.x * C::FS + fl;
  const float g = gamma[f], bt = beta[f];
  float v[C::R];
#pragma unroll
  for (int j = 0; j < C::R; ++j) v[j] = x[(size_t)(rg + C::RG * j) * d + f];
  pdl_launch();
  slice_act<B, S, BM>(v, red, d, f, rg, fl, g, bt, a);
}

}  // namespace slmk
