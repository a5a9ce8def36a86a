// Forward Block as ONE kernel (option blk_cluster = SK in {2, 4}, bf16, B = 256): GEMM + split-K
// reduction inside a thread-block cluster + batch-norm / ReLU epilogue.
//
//   cluster of 2 SK CTAs per 128-feature M tile: rank r = SK nt + ks, nt = batch half (N tile of
//   128 columns), ks = K slice.  Grid (d / 128) x 2 SK = 64 (SK = 2) or 128 (SK = 4) CTAs at
//   d = 2048.  The text below describes SK = 2 (FK = 128 / SK features finalised per CTA).
//
//   1. main loop (as tc_gemm_kernel): P_ks[f][b] = sum_{k in half ks} W_l[f][k] a_l[b][k] in
//      TMEM, W tiles prefetched before the dependency wait (PDL);
//   2. cluster barrier (both K halves done with their shared memory), then each CTA keeps
//      features [64 ks, 64 ks + 64) of the tile: the other half of its partial goes to the
//      K peer's shared memory over DSMEM (32 KiB), the kept half to its own;
//   3. cluster barrier, then 256 threads (feature f of 64, column quarter q of 4) finalise
//      x_{l+1} = x_l + ((P_0 + P_1) + b_l) for the CTA's 128 batch columns -> pool slot;
//   4. batch statistics of x_{l+1} over all 256 rows: per thread serial sums over its 32 rows,
//      the 4 quarters added in order q = 0..3, then the two batch halves (nt = 0 then 1, the
//      batch peer's sum arrives over DSMEM); mean first, then the centred sum of squares
//      (two-pass, like feature_stats) -> rstd;
//   5. a_{l+1} = bf16(ReLU(gamma (x - mu) rstd + beta)) -> the next Block's operand.
//
// `bn_act_cl_kernel` computes statistics and a_l from a stored x_l (the K1 before a segment's
// re-computation and before the first Block) with exactly the order of step 4, so a mirror run
// starting from a kept checkpoint reproduces the forward's operand bit for bit.
#pragma once
#include "kernels_simt.cuh"
#include "tc_gemm.cuh"

namespace slmk {

template <int SK>
struct BlkClCfg {
  static constexpr int BM = 128, BN = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = 6;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static constexpr int THREADS = 256;
  static constexpr int CL = 2 * SK;        // cluster: 2 batch halves x SK K slices
  static constexpr int FK = BM / SK;       // features kept (finalised) per CTA
  static constexpr int NQ = THREADS / FK;  // row groups per batch half
  static constexpr int RQ = BN / NQ;       // rows per thread
};

__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// per-feature statistics exchange (after the partial buffers in the stage area)
template <int FK, int NQ>
struct BlkClStats {
  float s[2][FK];     // [nt][f]: sum over the batch half nt
  float q[2][FK];     // [nt][f]: centred sum of squares
  float part[NQ][FK]; // [row group][f] per-thread partials of this CTA
};

template <int SK>
__global__ void __launch_bounds__(256, 1)
    blk_fwd_cl_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmA, int d,
                      int layer, int n_layers, const float* xin, float* xout, const float* __restrict__ bias,
                      const float* __restrict__ gamma, const float* __restrict__ beta, float* __restrict__ stats,
                      __nv_bfloat16* __restrict__ aout, int dbg) {
  using C = BlkClCfg<SK>;
  constexpr int FK = C::FK, NQ = C::NQ, RQ = C::RQ;
  using SX = BlkClStats<FK, NQ>;
  ts_mark(0, dbg);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* accum = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const uint32_t rank = cluster_ctarank();
  const int ks = (int)(rank % SK), nt = (int)(rank / SK);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = (int)(blockIdx.x / C::CL) * C::BM, n0 = nt * C::BN;
  const int nk = d / C::BK / SK;
  const int kbase = ks * nk * C::BK;

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmW);
      prefetch_tmap(&tmA);
      for (int s = 0; s < C::STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      mbar_init(accum, 1);
      fence_barrier_init();
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // ---- 1. main loop
  if (warp == 0 && lane == 0) {
    const int kb0 = nk < C::STAGES ? nk : C::STAGES;
    for (int kb = 0; kb < kb0; ++kb) {   // weights: read-only, requested before the dependency
      mbar_expect_tx(&full[kb], C::STAGE);
      tma_load_2d(smem + kb * C::STAGE, &tmW, &full[kb], kbase + kb * C::BK, layer * d + m0);
    }
    pdl_wait();
    if (dbg & 8) ts_dep(dbg);
    for (int kb = 0; kb < kb0; ++kb)
      tma_load_2d(smem + kb * C::STAGE + C::A_BYTES, &tmA, &full[kb], kbase + kb * C::BK, n0);
    for (int kb = kb0; kb < nk; ++kb) {
      const int s = kb % C::STAGES;
      mbar_wait(&empty[s], ((kb / C::STAGES) - 1) & 1);
      mbar_expect_tx(&full[s], C::STAGE);
      tma_load_2d(smem + s * C::STAGE, &tmW, &full[s], kbase + kb * C::BK, layer * d + m0);
      tma_load_2d(smem + s * C::STAGE + C::A_BYTES, &tmA, &full[s], kbase + kb * C::BK, n0);
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = make_idesc(C::BM, C::BN, false, false);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % C::STAGES;
      mbar_wait(&full[s], (kb / C::STAGES) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * C::STAGE), sb = sa + C::A_BYTES;
#pragma unroll
      for (int kk = 0; kk < C::BK / 16; ++kk)
        tc_mma(tmem, make_sdesc(sa + kk * 32, 16, 1024), make_sdesc(sb + kk * 32, 16, 1024), idesc, (kb | kk) != 0);
      tc_commit(&empty[s]);
    }
    tc_commit(accum);
  }
  __syncwarp();
  pdl_wait();
  mbar_wait(accum, 0);
  tc_fence_after();
  pdl_launch();

  // ---- 2. exchange the K-split partials: part[src ks][128 cols][FK] fp32 (64 KiB) in the stage area
  float* part = reinterpret_cast<float*>(smem);
  SX* sx = reinterpret_cast<SX*>(smem + 65536);
  cluster_sync();   // every K slice finished its MMAs: every CTA's stage area is free
  {
    const int q4 = warp & 3, ch = warp >> 2;               // TMEM lane quarter, column half
    const int fl = q4 * 32 + lane;                           // feature (lane) in the 128-row tile
    const int owner = fl / FK, fo = fl % FK;
    const uint32_t trow = tmem + ((uint32_t)(q4 * 32) << 16);
    const uint32_t dst = mapa_u32(smem_u32(part), (uint32_t)(nt * SK + owner));
#pragma unroll 1
    for (int c = ch * 64; c < ch * 64 + 64; c += 32) {
      float v[32];
      tmem_ld32(trow + c, v);
      if (owner == ks) {
#pragma unroll
        for (int j = 0; j < 32; ++j) part[(ks * C::BN + c + j) * FK + fo] = v[j];
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) st_cluster_f32(dst + (uint32_t)(((ks * C::BN + c + j) * FK + fo) * 4), v[j]);
      }
    }
  }
  tc_fence_before();
  cluster_sync();   // partials delivered
  // ---- 3. finalise x_{l+1} for features m0 + FK ks + f, rows n0 + RQ q + i
  const int f = threadIdx.x % FK, q = threadIdx.x / FK;
  const int gf = m0 + FK * ks + f;
  const float bf = bias[(size_t)layer * d + gf];
  float v[RQ];
#pragma unroll
  for (int i = 0; i < RQ; ++i) v[i] = xin[(size_t)(n0 + RQ * q + i) * d + gf];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < RQ; ++i) {
    const int c = RQ * q + i;
    float z = part[c * FK + f];
#pragma unroll
    for (int k = 1; k < SK; ++k) z = __fadd_rn(z, part[(k * C::BN + c) * FK + f]);
    v[i] = __fadd_rn(v[i], __fadd_rn(z, bf));
    xout[(size_t)(n0 + c) * d + gf] = v[i];
    s = __fadd_rn(s, v[i]);
  }
  const bool has_next = layer + 1 < n_layers;
  if (has_next) {
    // ---- 4. statistics over the 256 rows: row groups in order, then the two batch halves
    const uint32_t peer_sx = mapa_u32(smem_u32(sx), (uint32_t)((1 - nt) * SK + ks));
    sx->part[q][f] = s;
    __syncthreads();
    if (q == 0) {
      float t = sx->part[0][f];
#pragma unroll
      for (int k = 1; k < NQ; ++k) t = __fadd_rn(t, sx->part[k][f]);
      sx->s[nt][f] = t;
      st_cluster_f32(peer_sx + (uint32_t)(offsetof(SX, s) + (nt * FK + f) * 4), t);
    }
    cluster_sync();
    const float mu = __fmul_rn(__fadd_rn(sx->s[0][f], sx->s[1][f]), 1.0f / 256);
    float cq = 0.f;
#pragma unroll
    for (int i = 0; i < RQ; ++i) {
      const float c = __fsub_rn(v[i], mu);
      cq = __fmaf_rn(c, c, cq);
    }
    sx->part[q][f] = cq;
    __syncthreads();
    if (q == 0) {
      float t = sx->part[0][f];
#pragma unroll
      for (int k = 1; k < NQ; ++k) t = __fadd_rn(t, sx->part[k][f]);
      sx->q[nt][f] = t;
      st_cluster_f32(peer_sx + (uint32_t)(offsetof(SX, q) + (nt * FK + f) * 4), t);
    }
    cluster_sync();
    const float var = __fmul_rn(__fadd_rn(sx->q[0][f], sx->q[1][f]), 1.0f / 256);
    const float rstd = __frcp_rn(__fsqrt_rn(__fadd_rn(var, kEps)));
    if (nt == 0 && q == 0) {
      stats[gf] = mu;
      stats[d + gf] = rstd;
    }
    // ---- 5. the next Block's operand
    const float g = gamma[(size_t)(layer + 1) * d + gf], bt = beta[(size_t)(layer + 1) * d + gf];
#pragma unroll
    for (int i = 0; i < RQ; ++i)
      aout[(size_t)(n0 + RQ * q + i) * d + gf] = from_f32<__nv_bfloat16>(fmaxf(bn_u(bn_xhat(v[i], mu, rstd), g, bt), 0.f));
  } else {
    cluster_sync();   // keep the cluster barrier count uniform
    cluster_sync();
  }
  ts_mark(7, dbg);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::BN));
}

// K1 for the cluster lowering: statistics and a = bf16(ReLU(BN(x))) of a stored x (B = 256) in
// exactly blk_fwd_cl_kernel<SK>'s order: per feature, rows h*128 + RQ q + i summed serially over
// i, row groups q = 0..NQ-1 in order, halves h = 0 then 1.  CTA = FK features x NQ row groups.
template <int SK>
__global__ void __launch_bounds__(256) bn_act_cl_kernel(const float* __restrict__ x, const float* __restrict__ gamma,
                                                        const float* __restrict__ beta, int d,
                                                        float* __restrict__ stats, __nv_bfloat16* __restrict__ a) {
  using C = BlkClCfg<SK>;
  constexpr int FK = C::FK, NQ = C::NQ, RQ = C::RQ;
  __shared__ float part[NQ][FK];
  __shared__ float half[2][FK];
  pdl_wait();
  pdl_launch();
  const int f = threadIdx.x % FK, q = threadIdx.x / FK;
  const int gf = blockIdx.x * FK + f;
  float v[2][RQ];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < RQ; ++i) v[h][i] = x[(size_t)(h * 128 + RQ * q + i) * d + gf];
  auto combine = [&](int h, float val) {
    part[q][f] = val;
    __syncthreads();
    if (q == 0) {
      float t = part[0][f];
#pragma unroll
      for (int k = 1; k < NQ; ++k) t = __fadd_rn(t, part[k][f]);
      half[h][f] = t;
    }
    __syncthreads();
  };
  for (int h = 0; h < 2; ++h) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < RQ; ++i) s = __fadd_rn(s, v[h][i]);
    combine(h, s);
  }
  const float mu = __fmul_rn(__fadd_rn(half[0][f], half[1][f]), 1.0f / 256);
  __syncthreads();
  for (int h = 0; h < 2; ++h) {
    float cq = 0.f;
#pragma unroll
    for (int i = 0; i < RQ; ++i) {
      const float c = __fsub_rn(v[h][i], mu);
      cq = __fmaf_rn(c, c, cq);
    }
    combine(h, cq);
  }
  const float var = __fmul_rn(__fadd_rn(half[0][f], half[1][f]), 1.0f / 256);
  const float rstd = __frcp_rn(__fsqrt_rn(__fadd_rn(var, kEps)));
  if (q == 0) {
    stats[gf] = mu;
    stats[d + gf] = rstd;
  }
  const float g = gamma[gf], bt = beta[gf];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < RQ; ++i)
      a[(size_t)(h * 128 + RQ * q + i) * d + gf] = from_f32<__nv_bfloat16>(fmaxf(bn_u(bn_xhat(v[h][i], mu, rstd), g, bt), 0.f));
}

}  // namespace slmk
