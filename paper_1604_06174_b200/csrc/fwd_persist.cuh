// Persistent forward-segment kernel of the fused lowering (bf16, sm_100a).
//
// One launch runs a run of consecutive forward / mirror Block ops of V' (the whole forward pass
// in chunks, or one segment's re-computation): for each Block_l of
// the run
//
//   GEMM phase   P[ks][b][f] = sum_{k in slice ks} W_l[f][k] a_l[b][k]      (tcgen05, TMEM)
//   grid barrier
//   BN phase     x_{l+1} = x_l + (sum_ks P[ks] + b_l)  -> the node's pool slot (may alias x_l)
//                a_{l+1} = ReLU(BN_{l+1}(x_{l+1}))     -> the bf16 operand of the next Block
//   grid barrier
//
// Tiles: CTA (mt, ks) owns output features [128 mt, 128 mt + 128) x the whole batch (N = B,
// one TMEM lane per feature, "swap-AB") over K slice ks of d / S; with d = 2048, S = 8 that is
// 16 x 8 = 128 CTAs, one per SM, all resident for the whole launch (grid barriers).  The weight
// tile of layer l+1 (A operand, 128 x d/S, read-only for the whole step) is loaded into shared
// memory during layer l's BN phase, so after the barrier only the activation slice (B operand,
// B x d/S bf16) is on the critical path.  Compared with the two-kernel lowering (GEMM + bn_act_rk
// per Block) this removes two kernel boundaries (drain + launch + prologue) per Block and takes
// the weight stream off the critical path.
//
// The BN phase is the arithmetic of bn_act_rk (bn_kernels.cuh) — same thread mapping (16
// features x 32 row groups, R = B / 32 rows per thread), same fixed-order sums (slices 0..S-1,
// feature_stats) — so a_{l+1} has the bits bn_act_rk would produce from the same x_{l+1}; it
// reads with ld.global.cg because P and x are written by other CTAs of the same launch.
// Mirrors re-run this kernel with the same S, so re-computed values are bit-identical to the
// forward's.
#pragma once
#include "bn_kernels.cuh"
#include "tc_gemm.cuh"

namespace slmk {

constexpr int kSegMax = 64;   // Blocks per launch (longer runs are split into several launches)
struct FwdSegLayer {
  const float* xin;   // x_l (a pool slot or the caller's x0)
  float* xout;        // x_{l+1}'s slot
  int layer;          // l
  int dbg;            // device-clock profiling slot (ts_mark), 0 = off
};
struct FwdSegArgs {
  int nl;                   // Blocks in this launch
  int n;                    // layers of the chain (a_{l+1} is not produced after the last one)
  int d;
  unsigned lay_base;        // persistent Blocks run earlier in this step (the counters are monotonic per step)
  int phase_dbg;            // 1: per-layer, per-CTA %globaltimer stamps of 6 phase points into g_slm_ts
  unsigned* bar;            // 128 dependency counters, 128 B apart (zeroed at the start of the step)
  float* P;                 // split-K partials [S][B][d] fp32
  const float* bias;        // [n][d]
  const float* gamma;       // [n][d]
  const float* beta;        // [n][d]
  float* stats;             // [2][d] (mu, rstd of the last x produced)
  __nv_bfloat16* a;         // operand buffer [B][d] bf16 (a_l in, a_{l+1} out)
  FwdSegLayer L[kSegMax];
};

template <int B, int S>
struct FwdSegCfg {
  static constexpr int R = B / 32;
  static constexpr int A_BYTES = 128 * 64 * 2;      // 16 KiB: 128 rows of W x 64 of K
  static constexpr int B_BYTES = B * 64 * 2;        // B rows of a x 64 of K
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int MAX_KB = 4;                  // K blocks per slice (d / S / 64 <= 4)
  static constexpr int SMEM = MAX_KB * STAGE + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int THREADS = 512;
};

// dependency counters between the CTAs of one launch (all resident: one CTA per SM).  arrive:
// called by one thread after a __syncthreads that follows the CTA's stores (cumulativity through
// the CTA barrier + gpu-scope release).  wait: acquire-poll until the counter reaches `target`;
// bounded, so a dependency that can never be met (a CTA that could not become resident) traps
// instead of hanging the GPU.
__device__ __forceinline__ void ctr_arrive(unsigned* c) {
  __threadfence();
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
}
__device__ __forceinline__ void ctr_wait(const unsigned* c, unsigned target) {
  unsigned v;
  long spins = 0;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    if ((int)(v - target) >= 0) break;
    if (++spins > (1L << 28)) __trap();
  }
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void seg_mark(const FwdSegArgs& a, int j, int ph) {
  unsigned long long* p = g_slm_ts;
  if (a.phase_dbg && p != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p[((size_t)j * gridDim.x + blockIdx.x) * 8 + ph] = t;
  }
}

template <int B, int S>
__global__ void __launch_bounds__(512, 1)
    fwd_seg_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ FwdSegArgs args) {
  using C = FwdSegCfg<B, S>;
  constexpr int R = C::R;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ float red[32][kFeat + 1];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::MAX_KB * C::STAGE);
  uint64_t* accum = full + C::MAX_KB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int d = args.d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ks = (int)blockIdx.x % S, mt = (int)blockIdx.x / S;
  const int m0 = mt * 128;
  const int nkb = d / S / 64;
  const int kbase = ks * nkb * 64;
  const unsigned nblk = gridDim.x;
  const unsigned n_mt = (unsigned)d / 128;            // M tiles (GEMM CTAs per K slice)
  const unsigned gpm = 128 / kFeat;                   // BN feature groups per M tile
  const unsigned gps = (unsigned)(d / S) / kFeat;     // BN feature groups per K slice
  // dependency counters (zeroed at the start of the step, monotonic within it; G = the
  // step-global index of the Block):
  //   done1[mt] += 1  per GEMM CTA of M tile mt whose partials of Block G are stored   (S per Block)
  //   done2[ks] += 1  per BN group of K slice ks whose a_{G+1} is stored               (gps per Block)
  //   done3[mt] += 1  per BN group of M tile mt that has consumed the partials of G    (gpm per Block)
  //   done4[ks] += 1  per GEMM CTA of K slice ks whose operand loads of G completed   (n_mt per Block)
  unsigned* done1 = args.bar;
  unsigned* done2 = args.bar + 32 * 32;
  unsigned* done3 = args.bar + 64 * 32;
  unsigned* done4 = args.bar + 96 * 32;

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmW);
      prefetch_tmap(&tmA);
      for (int s = 0; s < C::MAX_KB; ++s) mbar_init(&full[s], 1);
      mbar_init(accum, 1);
      fence_barrier_init();
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(B));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const bool producer = threadIdx.x == 0;

  // weight tile of Block j (read-only during the step: may be requested before any dependency)
  auto load_w = [&](int j) {
    const int l = args.L[j].layer;
    for (int kb = 0; kb < nkb; ++kb) {
      uint8_t* sa = smem + kb * C::STAGE;
      mbar_expect_tx(&full[kb], C::STAGE);
      tma_load_2d(sa, &tmW, &full[kb], kbase + kb * 64, l * d + m0);
    }
  };
  if (producer) load_w(0);
  pdl_wait();   // x_l / a_l of the first Block come from the previous kernel of the stream

  // BN-phase thread mapping (bn_act_rk): feature lane fl of 16, row group rg of 32
  const int fl = threadIdx.x % kFeat, rg = threadIdx.x / kFeat;
  const unsigned rs = 32u * d, pslice = (unsigned)B * d;

  for (int j = 0; j < args.nl; ++j) {
    const FwdSegLayer Lj = args.L[j];
    const int l = Lj.layer;
    const unsigned G = args.lay_base + (unsigned)j;
    ts_mark(0, Lj.dbg);
    seg_mark(args, j, 0);
    // ---- GEMM phase: activation slice ks of a_l (stored by the BN groups of slice ks of Block G-1)
    if (producer) {
      ctr_wait(done2 + ks * 32, G * gps);
      fence_proxy_async_global();
      for (int kb = 0; kb < nkb; ++kb)
        tma_load_2d(smem + kb * C::STAGE + C::A_BYTES, &tmA, &full[kb], kbase + kb * 64, 0);
    } else if (warp == 1 && lane == 0) {
      constexpr uint32_t idesc = make_idesc(128, B, false, false);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[kb], j & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + kb * C::STAGE);
        const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          tc_mma(tmem, make_sdesc(sa + kk * 32, 16, 1024), make_sdesc(sb + kk * 32, 16, 1024), idesc, (kb | kk) != 0);
      }
      tc_commit(accum);
    }
    __syncwarp();
    mbar_wait(accum, j & 1);
    tc_fence_after();
    seg_mark(args, j, 1);
    if (producer) {
      ctr_arrive(done4 + ks * 32);   // this CTA no longer reads a_l: its slice may be overwritten
      // the stages are free: request the next Block's weight tile now (lands during the BN phase)
      if (j + 1 < args.nl) load_w(j + 1);
      // the partial buffer of this M tile is free once Block G-1's BN groups have read it
      ctr_wait(done3 + mt * 32, G * gpm);
    }
    __syncthreads();
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 and the 32-column chunks w/4, w/4 + 4, ...
    {
      const int q = warp & 3, cq = warp >> 2;
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
      const int m = m0 + q * 32 + lane;
      float* p = args.P + (size_t)ks * pslice + m;
#pragma unroll 1
      for (int c = cq * 32; c < B; c += 128) {
        float acc[32];
        tmem_ld32(trow + c, acc);
#pragma unroll
        for (int i = 0; i < 32; ++i) p[(size_t)(c + i) * d] = acc[i];
      }
    }
    ts_mark(7, Lj.dbg);
    tc_fence_before();
    __syncthreads();
    if (producer) ctr_arrive(done1 + mt * 32);
    seg_mark(args, j, 2);

    // ---- BN phase (finalize Block_l, produce a_{l+1}); feature groups of 16 strided over the grid
    const bool last = j + 1 == args.nl;
    if (last) pdl_launch();
    const float* ga = l + 1 < args.n ? args.gamma + (size_t)(l + 1) * d : nullptr;
    const float* be = l + 1 < args.n ? args.beta + (size_t)(l + 1) * d : nullptr;
    for (int grp = blockIdx.x; grp < d / kFeat; grp += nblk) {
      const int gmt = grp / (int)gpm, gks = grp / (int)gps;
      if (producer) ctr_wait(done1 + gmt * 32, (G + 1) * S);   // all S partials of this M tile
      __syncthreads();
      if (grp == (int)blockIdx.x) seg_mark(args, j, 3);
      const int f = grp * kFeat + fl;
      const unsigned base = (unsigned)rg * d + f;
      float v[R];
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = __ldcg(Lj.xin + base + i * rs);
      float t[S][R];
#pragma unroll
      for (int s = 0; s < S; ++s)
#pragma unroll
        for (int i = 0; i < R; ++i) t[s][i] = __ldcg(args.P + s * pslice + base + i * rs);
      const float bf = args.bias[(size_t)l * d + f];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        float z = 0.f;
#pragma unroll
        for (int s = 0; s < S; ++s) z = __fadd_rn(z, t[s][i]);
        v[i] = __fadd_rn(v[i], __fadd_rn(z, bf));
        Lj.xout[base + i * rs] = v[i];
      }
      float mu = 0.f, rstd = 0.f;
      if (ga != nullptr) feature_stats<R>(v, red, rg, fl, mu, rstd);   // contains __syncthreads
      else __syncthreads();
      if (producer) {
        ctr_arrive(done3 + gmt * 32);                 // partials consumed (used by every thread above)
        ctr_wait(done4 + gks * 32, (G + 1) * n_mt);   // no GEMM CTA still loads this slice of a_l
      }
      __syncthreads();
      if (ga != nullptr) {
        if (rg == 0) {
          args.stats[f] = mu;
          args.stats[d + f] = rstd;
        }
        const float g = ga[f], bt = be[f];
#pragma unroll
        for (int i = 0; i < R; ++i)
          args.a[base + i * rs] = from_f32<__nv_bfloat16>(fmaxf(bn_u(bn_xhat(v[i], mu, rstd), g, bt), 0.f));
      }
      fence_proxy_async_global();   // a_{l+1} (generic stores) is read by the next GEMM phase's TMA
      __syncthreads();
      if (producer) ctr_arrive(done2 + gks * 32);
    }
    seg_mark(args, j, 4);
    seg_mark(args, j, 5);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(B));
}

}  // namespace slmk
