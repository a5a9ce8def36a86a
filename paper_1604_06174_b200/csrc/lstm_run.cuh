// Persistent recurrent kernels of the unrolled LSTM (sm_100a).
//
// The per-step work of one layer is the recurrent contraction R_t = h_{t-1} W_hh^T ([B] x [4H], K = H)
// followed by the gate activations and the cell; the input projection X_t = x_t W_ih^T + b is
// independent of the recurrence and runs beforehand as ONE batched GEMM over the n steps of a run
// (N = n B instead of B; tc_gemm.cuh with EpiBiasF32).  lstm_fwd_run_kernel then runs the n steps
// of the recurrence in a single launch:
//
//   grid    H / 32 CTAs (32 at H = 1024), all resident (executor_lstm.cuh launch_run); CTA m owns hidden
//           units j0 = 32 m .. j0 + 31 and the 128 gate rows {q H + j0 + u : q = i, f, g, o}
//           (gate-interleaved M tile: four TMA boxes of 32 rows, one per gate)
//   MMA     D[128 gate rows][B] = W_hh(rows, :) . h_{t-1}^T, K = H: tcgen05 kind::f16, M = 128,
//           N = B, fp32 accumulator in TMEM; W streamed from L2 by TMA every step (256 KiB per CTA
//           does not fit next to the pipeline), h_{t-1} TMA-loaded from the exchange buffer hx
//   cell    pre = R + X_t (fp32), sigmoid / tanh -> G_t; the four gates of a unit meet in shared
//           memory; c_t = f c_{t-1} + i g stays in shared memory across steps; h_t = o tanh c_t ->
//           S_t (when materialised), bf16 h_t into hx (the next step's operand) and into the layer's
//           chunk ring (the next layer's input projection and the head read it)
//   sync    one grid-wide step barrier: a monotone counter per (layer, stream) in global memory; the
//           epilogue of every CTA publishes its h slice (generic stores, fence.proxy.async, release
//           add), the TMA producer of step t+1 spins (acquire) until all H / 32 slices are in
//
// Warp roles (10 warps): 0-7 epilogue (warp w reads TMEM lanes 32 (w % 4) = gate w % 4 of the 32
// units, half w / 4 of the batch columns; 8 warps because the activations are latency bound),
// 8 TMA producer (prefetches the next step's W stages and X_t while the epilogue runs, loads h
// only after the step barrier), 9 TMEM allocator + MMA issuer.
//
// Arithmetic (the same in every run length, so a run of n steps and n runs of one step give
// identical bits, and so do the checkpointed and the plain step): X = fl(acc_x + b) (input GEMM
// epilogue), pre = fl(R + X), act_i/f/o = 1/2 + tanh(pre/2)/2, act_g = tanh(pre),
// c = fl(fl(f c_prev) + fl(i g)), h = fl(o tanh(c)), tanh = the SFU's tanh.approx.f32.
#pragma once
#include "tc_gemm.cuh"
#include "lstm_kernels.cuh"

namespace slmk {

constexpr int kRunMax = 8;    // steps per run launch (four runs per 32-step weight-gradient chunk)

struct FwdRun {
  int H, n, t0, Kin;     // Kin: first column of W_hh inside the layer's [W_ih | W_hh] rows
  int init;              // 0 = continue from hx / cstate, 1 = zero state (t0 = 0), 2 = from s_init
  int cell;              // 0 = gates only (an isolated gates node: G_t, no cell, no state update)
  const float* s_init;   // S_{t0-1} = (h | c) [B][2H] fp32 (init = 2)
  __nv_bfloat16* hx;     // [2][B][H] bf16: h_{t-1} of step t at parity t % 2
  float* cstate;         // [B][H] fp32: c at the end of the run (the start, for init = 0)
  __nv_bfloat16* hring;  // [.][B][H] bf16 rows of step t0 .. t0 + n - 1 (null = none)
  unsigned* bar;         // step counter of this (layer, stream)
  unsigned base;         // its value when this launch starts (host-tracked)
  unsigned long long* ts; // debug (option lstm_run_ts): CTA 0's %globaltimer per step [n][16], or null
  int dbg;               // profile_ts slot (tc_gemm.cuh ts_mark): launch start / end per CTA
  float* g_out[kRunMax]; // G_t tags (null = not materialised)
  float* s_out[kRunMax]; // S_t tags
};

template <int B>
struct FwdRunCfg {
  static constexpr int NS = B == 64 ? 6 : B == 128 ? 4 : 2;   // K pipeline stages (bytes in flight
                                                             // set the W / h ingest rate)
  static constexpr int NCB = B / 64;                // 64-column blocks of the accumulator (batch)
  static constexpr int W_BYTES = 128 * 64 * 2;      // 16 KiB: 4 gates x 32 rows x 64 K
  static constexpr int H_BYTES = B * 64 * 2;        // h_{t-1}: B rows x 64 K
  static constexpr int STAGE = W_BYTES + H_BYTES;
  static constexpr int X_BYTES = 4 * 64 * 32 * 4;   // X_t of the CTA's 128 gate rows, 64 batch rows
  static constexpr int LD = 64 + 1;                 // padded rows of the gate exchange
  static constexpr int G_BYTES = 128 * LD * 4;
  static constexpr int C_BYTES = 32 * B * 4;        // c of the 32 units
  static constexpr int OFF_X = NS * STAGE;
  static constexpr int OFF_G = OFF_X + X_BYTES;
  static constexpr int OFF_C = OFF_G + G_BYTES;
  static constexpr int OFF_BAR = OFF_C + C_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static_assert(SMEM <= 232448, "shared memory");
};

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
constexpr int kRunEpiWarps = 8;   // two warps per TMEM lane quarter (gate), 32 accumulator columns each
constexpr int kRunThreads = 32 * (kRunEpiWarps + 2);
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kRunEpiWarps) : "memory"); }
// gate activation of gate q (i, f, g, o): tanh for g, sigmoid(x) = 1/2 + tanh(x/2)/2 otherwise
__device__ __forceinline__ void run_stamp(const FwdRun& a, int i, int k) {
  if (a.ts != nullptr && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.ts[i * 16 + k] = t;
  }
}
__device__ __forceinline__ float lstm_act(int q, float pre) {
  return q == 2 ? tanh_fast(pre) : __fmaf_rn(0.5f, tanh_fast(0.5f * pre), 0.5f);
}

template <int B>
__global__ void __launch_bounds__(kRunThreads, 1)
    lstm_fwd_run_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmH,
                        const __grid_constant__ CUtensorMap tmX, const __grid_constant__ FwdRun a) {
  static_assert(B == 64 || B == 128 || B == 256, "batch");
  using C = FwdRunCfg<B>;
  unsigned long long* const tsp = ts_buffer(a.dbg);
  ts_mark(tsp, 0, a.dbg);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* empty = full + C::NS;
  uint64_t* accum = empty + C::NS;
  uint64_t* tfree = accum + 1;
  uint64_t* xfull = tfree + 1;    // X_t box set (one buffer: loaded while the step's MMAs run)
  uint64_t* xempty = xfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xempty + 1);
  float* xs = reinterpret_cast<float*>(smem + C::OFF_X);
  float* gs = reinterpret_cast<float*>(smem + C::OFF_G);
  float* cs = reinterpret_cast<float*>(smem + C::OFF_C);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int H = a.H, j0 = 32 * (int)blockIdx.x, nk = H / 64;
  const unsigned ncta = gridDim.x;

  if (warp == kRunEpiWarps + 1) {
    if (lane == 0) {
      prefetch_tmap(&tmW);
      prefetch_tmap(&tmH);
      prefetch_tmap(&tmX);
      for (int s = 0; s < C::NS; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      mbar_init(accum, 1);
      mbar_init(tfree, 32 * kRunEpiWarps);
      mbar_init(xfull, 1);
      mbar_init(xempty, 32 * kRunEpiWarps);
      fence_barrier_init();
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(B));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kRunEpiWarps) {
    if (lane == 0) {
      // ===== TMA producer.  W (constant) is requested before the dependency wait and before each
      // step barrier; X_t after the dependency wait; h_{t-1} after the step barrier.
      auto load_w = [&](int kb, int s) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          tma_load_2d(smem + s * C::STAGE + q * 4096, &tmW, &full[s], a.Kin + kb * 64, q * H + j0);
      };
      auto load_h = [&](int kb, int s, int t) {
        tma_load_2d(smem + s * C::STAGE + C::W_BYTES, &tmH, &full[s], kb * 64, (t & 1) * B);
      };
      int g = 0;   // k-block counter over the whole run (ring position)
      for (int i = 0; i < a.n; ++i) {
        const int t = a.t0 + i;
        const int pre = nk < C::NS ? nk : C::NS;
        for (int kb = 0; kb < pre; ++kb) {
          const int gg = g + kb, s = gg % C::NS;
          if (gg >= C::NS) mbar_wait(&empty[s], ((gg / C::NS) - 1) & 1);
          mbar_expect_tx(&full[s], C::STAGE);
          load_w(kb, s);
        }
        if (i == 0) pdl_wait();
        if (C::NCB == 1) {   // X_t (one 64-row box set; with several column blocks the epilogue asks for them)
          if (i >= 1) mbar_wait(xempty, (i - 1) & 1);
          mbar_expect_tx(xfull, C::X_BYTES);
#pragma unroll
          for (int q = 0; q < 4; ++q) tma_load_2d(xs + q * 64 * 32, &tmX, xfull, q * H + j0, i * B);
        }
        // step barrier: every CTA has published h_{t-1} (step i-1's epilogue, or the init)
        const unsigned target = a.base + ncta * (unsigned)(i + 1);
        while ((int)(ld_acquire_gpu(a.bar) - target) < 0) {
        }
        run_stamp(a, i, 0);
        fence_proxy_async_global();
        for (int kb = 0; kb < pre; ++kb) load_h(kb, (g + kb) % C::NS, t);
        for (int kb = pre; kb < nk; ++kb) {
          const int gg = g + kb, s = gg % C::NS;
          if (gg >= C::NS) mbar_wait(&empty[s], ((gg / C::NS) - 1) & 1);
          mbar_expect_tx(&full[s], C::STAGE);
          load_w(kb, s);
          load_h(kb, s, t);
        }
        if (C::NCB > 1)   // X of every column block, each once the epilogue has consumed the previous one
          for (int cb = 0; cb < C::NCB; ++cb) {
            const int e = i * C::NCB + cb;
            if (e >= 1) mbar_wait(xempty, (e - 1) & 1);
            mbar_expect_tx(xfull, C::X_BYTES);
#pragma unroll
            for (int q = 0; q < 4; ++q) tma_load_2d(xs + q * 64 * 32, &tmX, xfull, q * H + j0, i * B + cb * 64);
          }
        g += nk;
      }
    }
  } else if (warp == kRunEpiWarps + 1) {
    if (lane == 0) {
      // ===== MMA issuer
      constexpr uint32_t idesc = make_idesc(128, B, false, false);
      int g = 0;
      for (int i = 0; i < a.n; ++i) {
        if (i > 0) mbar_wait(tfree, (i - 1) & 1);   // the epilogue has drained step i-1's accumulator
        tc_fence_after();
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % C::NS;
          mbar_wait(&full[s], (g / C::NS) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * C::STAGE), sb = sa + C::W_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma(tmem, make_sdesc(sa + kk * 32, 16, 1024), make_sdesc(sb + kk * 32, 16, 1024), idesc, (kb | kk) != 0);
          tc_commit(&empty[s]);
        }
        tc_commit(accum);
        run_stamp(a, i, 1);
      }
    }
  } else {
    // ===== epilogue (warps 0-7): warp w reads TMEM lanes 32 (w % 4) = gate q = w % 4 of the 32
    // units (lane u = unit j0 + u), accumulator columns hf*32 .. hf*32+31 of each 64-column block
    constexpr int ET = 32 * kRunEpiWarps;
    pdl_wait();
    const int q = warp & 3, hf = warp >> 2, u = lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + hf * 32;
    for (int idx = tid; idx < 32 * B; idx += ET) {   // initial state of the CTA's units
      const int uu = idx & 31, b = idx >> 5, j = j0 + uu;
      float h = 0.f, c = 0.f;
      if (a.init == 2) {
        h = a.s_init[(size_t)b * 2 * H + j];
        c = a.s_init[(size_t)b * 2 * H + H + j];
      } else if (a.init == 0 && a.cell) {
        c = a.cstate[(size_t)b * H + j];
      }
      cs[b * 32 + uu] = c;
      if (a.init != 0) a.hx[(size_t)((a.t0 & 1) * B + b) * H + j] = __float2bfloat16_rn(h);
    }
    fence_proxy_async_global();
    epi_bar();
    if (tid == 0) red_release_gpu(a.bar, 1u);
    for (int i = 0; i < a.n; ++i) {
      const int t = a.t0 + i;
      mbar_wait(accum, i & 1);
      tc_fence_after();
      if (tid == 0) run_stamp(a, i, 2);
      float* go = a.g_out[i];
      float* so = a.s_out[i];
      __nv_bfloat16* hxo = a.hx + (size_t)((t + 1) & 1) * B * H;
      __nv_bfloat16* hr = a.hring ? a.hring + (size_t)i * B * H : nullptr;
      // one 64-column block (64 batch rows) at a time: gates -> exchange -> cell.  With B = 64 the
      // step's critical path ends when h is published; G_t and S_t (when materialised) are stored
      // after the release, overlapping the next step's K loop.
      constexpr bool DEFER = C::NCB == 1;
      float acc[32], hv[8], cv[8];
      for (int cb = 0; cb < C::NCB; ++cb) {
        const int e = i * C::NCB + cb;
        tmem_ld32(trow + cb * 64, acc);
        if (DEFER) {
          tc_fence_before();
          mbar_arrive(tfree);   // the accumulator is drained: the next step's MMAs may overwrite it
        }
        if (tid == 0) run_stamp(a, i, 4);
        mbar_wait(xfull, e & 1);
        if (tid == 0) run_stamp(a, i, 5);
        const float* xq = xs + q * 64 * 32 + hf * 32 * 32;
        float xv[32];
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) xv[jj] = xq[jj * 32 + u];
        mbar_arrive(xempty);
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          acc[jj] = lstm_act(q, __fadd_rn(acc[jj], xv[jj]));
          gs[(q * 32 + u) * C::LD + hf * 32 + jj] = acc[jj];
        }
        if (!DEFER && go)
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) go[(size_t)(cb * 64 + hf * 32 + jj) * 4 * H + q * H + j0 + u] = acc[jj];
        if (tid == 0) run_stamp(a, i, 6);
        epi_bar();
        if (tid == 0) run_stamp(a, i, 7);
        if (a.cell) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int idx = tid + ET * k, uu = idx & 31, bl = idx >> 5, b = cb * 64 + bl, j = j0 + uu;
            const float ig = gs[uu * C::LD + bl], fg = gs[(32 + uu) * C::LD + bl], gg = gs[(64 + uu) * C::LD + bl],
                        og = gs[(96 + uu) * C::LD + bl];
            cv[k] = __fadd_rn(__fmul_rn(fg, cs[b * 32 + uu]), __fmul_rn(ig, gg));
            hv[k] = __fmul_rn(og, tanh_fast(cv[k]));
            cs[b * 32 + uu] = cv[k];
            const __nv_bfloat16 hb = __float2bfloat16_rn(hv[k]);
            hxo[(size_t)b * H + j] = hb;
            if (hr && !DEFER) hr[(size_t)b * H + j] = hb;
            if (!DEFER && so) {
              so[(size_t)b * 2 * H + j] = hv[k];
              so[(size_t)b * 2 * H + H + j] = cv[k];
            }
          }
        }
        if (tid == 0) run_stamp(a, i, 8);
        if (!DEFER) epi_bar();   // gs is free for the next column block
      }
      if (!DEFER) {
        tc_fence_before();
        mbar_arrive(tfree);
      }
      fence_proxy_async_global();
      if (tid == 0) run_stamp(a, i, 9);
      epi_bar();   // the CTA's h slice is complete (and gs is free for the next step)
      if (tid == 0) {
        run_stamp(a, i, 10);
        red_release_gpu(a.bar, 1u);
        run_stamp(a, i, 3);
      }
      if (DEFER) {
        if (hr && a.cell)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int idx = tid + ET * k, uu = idx & 31, b = idx >> 5;
            hr[(size_t)b * H + j0 + uu] = __float2bfloat16_rn(hv[k]);
          }
        if (go)
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) go[(size_t)(hf * 32 + jj) * 4 * H + q * H + j0 + u] = acc[jj];
        if (so && a.cell)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int idx = tid + ET * k, uu = idx & 31, b = idx >> 5, j = j0 + uu;
            so[(size_t)b * 2 * H + j] = hv[k];
            so[(size_t)b * 2 * H + H + j] = cv[k];
          }
      }
    }
    if (a.cell)
      for (int idx = tid; idx < 32 * B; idx += ET) {
        const int uu = idx & 31, b = idx >> 5;
        a.cstate[(size_t)b * H + j0 + uu] = cs[b * 32 + uu];
      }
    pdl_launch();
  }
  tc_fence_before();
  __syncthreads();
  ts_mark(tsp, 7, a.dbg);
  if (warp == kRunEpiWarps + 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(B));
}

// ============================================================================ backward runs
// lstm_bwd_run_kernel: the backward of one layer over n consecutive steps t1, t1-1, ..., t1-n+1
// (descending) in one launch.  Per step t:
//   dR_t = d_pre_{t+1} W_hh  ([B] x [H], K = 4H): the recurrent part of dh_t.  32 CTAs = 8 unit
//          tiles (m: 128 hidden units) x 4 K slices (q: the 1024 gate rows of gate q); CTA (m, q)
//          computes D[128 units][B] = W_hh(q rows, m units)^T . d_pre_{t+1}(:, q rows)^T with
//          tcgen05 (A = W read MN-major, B = d_pre K-major from the exchange buffer dpx), then
//          the four K-slice partials of a tile are summed in the fixed order q = 0..3 by the
//          unit's owner through an L2 exchange buffer (per-tile counter)
//   cell   CTA (m, q) owns units 128 m + 32 q .. +31: dh = fl(dR + dh_in) (dh_in: the gradient
//          from the layer above / the head, precomputed per chunk), the cell backward with the
//          forward's arithmetic (c re-derived from G_t and c_{t-1}, tanh on the SFU) and the dc
//          state in shared memory, d_pre_t of the 4 gates -> dpx (bf16, the next step's B
//          operand), then -- after the step barrier is released -- the chunk rings (bf16 d_pre for
//          the weight / input gradient GEMMs, fp32 d_pre for db)
// dR of the first step of the whole backward (t = T-1) is 0.
struct BwdRun {
  int H, n, t1, Kin;
  int first;                    // 1: no state yet (t1 = T - 1): dR = 0, dc = 0
  int ldh;                      // row stride of dh_in
  __nv_bfloat16* dpx;           // [2][B][4H] bf16: d_pre_t at parity t % 2
  float* dcstate;               // [B][H] fp32: dc carried into the step before the run
  float* xch;                   // [8][4][4][B][32] fp32 partial exchange
  unsigned* bar;                // step counter
  unsigned base;
  unsigned* xbar;               // [8] per-tile exchange counters
  unsigned xbase;
  unsigned long long* ts;       // debug stamps (option lstm_run_ts) or null
  int dbg;                      // profile_ts slot (tc_gemm.cuh ts_mark)
  const float* dh_in[kRunMax];  // [B] rows of step t1 - i
  const float* act[kRunMax];    // G_t tags
  const float* sprev[kRunMax];  // S_{t-1} tags (null at t = 0)
  __nv_bfloat16* dpr[kRunMax];  // d_pre ring rows [B][4H] bf16
  float* dpf[kRunMax];          // d_pre ring rows [B][4H] fp32
};

struct BwdRunCfg {
  static constexpr int B = 64;
  static constexpr int NS = 6;
  static constexpr int A_BYTES = 128 * 64 * 2;     // W: 64 gate rows (K) x 128 units, two 64-unit boxes
  static constexpr int B_BYTES = B * 64 * 2;       // d_pre: 64 batch rows x 64 gate rows
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int C_BYTES = 32 * B * 4;       // dc of the 32 owned units
  static constexpr int OFF_C = NS * STAGE;
  static constexpr int OFF_BAR = OFF_C + C_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static_assert(SMEM <= 232448, "shared memory");
};

__device__ __forceinline__ void bwd_stamp(const BwdRun& a, int i, int k) {
  if (a.ts != nullptr && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.ts[i * 16 + k] = t;
  }
}

__global__ void __launch_bounds__(kRunThreads, 1)
    lstm_bwd_run_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmD,
                        const __grid_constant__ BwdRun a) {
  using C = BwdRunCfg;
  constexpr int B = C::B, ET = 32 * kRunEpiWarps;
  unsigned long long* const tsp = ts_buffer(a.dbg);
  ts_mark(tsp, 0, a.dbg);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* empty = full + C::NS;
  uint64_t* accum = empty + C::NS;
  uint64_t* tfree = accum + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfree + 1);
  float* dcs = reinterpret_cast<float*>(smem + C::OFF_C);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int H = a.H, m = (int)blockIdx.x >> 2, q = (int)blockIdx.x & 3;
  const int u0 = 128 * m, j0 = u0 + 32 * q;   // the tile's units, this CTA's own units
  const int nk = H / 64;                       // K blocks of the gate-q slice
  const unsigned ncta = gridDim.x;
  const int mma0 = a.first ? 1 : 0;            // steps before mma0 have dR = 0

  if (warp == kRunEpiWarps + 1) {
    if (lane == 0) {
      prefetch_tmap(&tmW);
      prefetch_tmap(&tmD);
      for (int s = 0; s < C::NS; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      mbar_init(accum, 1);
      mbar_init(tfree, ET);
      fence_barrier_init();
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(B));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kRunEpiWarps) {
    if (lane == 0) {
      // ===== TMA producer: W_hh (gate-q rows, tile units; constant) ahead of the step barrier,
      // d_pre_{t+1} (gate-q columns) after it
      auto load_w = [&](int kb, int s) {
        uint8_t* sa = smem + s * C::STAGE;
        tma_load_2d(sa, &tmW, &full[s], a.Kin + u0, q * H + kb * 64);
        tma_load_2d(sa + 8192, &tmW, &full[s], a.Kin + u0 + 64, q * H + kb * 64);
      };
      auto load_d = [&](int kb, int s, int t) {
        tma_load_2d(smem + s * C::STAGE + C::A_BYTES, &tmD, &full[s], q * H + kb * 64, ((t + 1) & 1) * B);
      };
      pdl_wait();
      int g = 0;
      for (int i = mma0; i < a.n; ++i) {
        const int t = a.t1 - i;
        const int pre = nk < C::NS ? nk : C::NS;
        for (int kb = 0; kb < pre; ++kb) {
          const int gg = g + kb, s = gg % C::NS;
          if (gg >= C::NS) mbar_wait(&empty[s], ((gg / C::NS) - 1) & 1);
          mbar_expect_tx(&full[s], C::STAGE);
          load_w(kb, s);
        }
        const unsigned target = a.base + ncta * (unsigned)(i + 1);   // d_pre_{t+1} published by every CTA
        while ((int)(ld_acquire_gpu(a.bar) - target) < 0) {
        }
        bwd_stamp(a, i, 0);
        fence_proxy_async_global();
        for (int kb = 0; kb < pre; ++kb) load_d(kb, (g + kb) % C::NS, t);
        for (int kb = pre; kb < nk; ++kb) {
          const int gg = g + kb, s = gg % C::NS;
          if (gg >= C::NS) mbar_wait(&empty[s], ((gg / C::NS) - 1) & 1);
          mbar_expect_tx(&full[s], C::STAGE);
          load_w(kb, s);
          load_d(kb, s, t);
        }
        g += nk;
      }
    }
  } else if (warp == kRunEpiWarps + 1) {
    if (lane == 0) {
      // ===== MMA issuer: D[128 units][B] += W(k, unit) . d_pre(b, k), A MN-major, B K-major
      constexpr uint32_t idesc = make_idesc(128, B, true, false);
      int g = 0;
      for (int i = mma0; i < a.n; ++i) {
        if (i > mma0) mbar_wait(tfree, (i - mma0 - 1) & 1);
        tc_fence_after();
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % C::NS;
          mbar_wait(&full[s], (g / C::NS) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * C::STAGE), sb = sa + C::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma(tmem, make_sdesc(sa + kk * 2048, 8192, 1024), make_sdesc(sb + kk * 32, 16, 1024), idesc,
                   (kb | kk) != 0);
          tc_commit(&empty[s]);
        }
        tc_commit(accum);
      }
    }
  } else {
    // ===== epilogue (warps 0-7): warp w reads TMEM lanes 32 (w % 4) = tile units 32 (w % 4) ..,
    // batch columns hf*32 .. hf*32+31; the cell is per owned (unit, batch row)
    pdl_wait();
    const int qq = warp & 3, hf = warp >> 2;
    for (int idx = tid; idx < 32 * B; idx += ET) {
      const int uu = idx & 31, b = idx >> 5;
      dcs[b * 32 + uu] = a.first ? 0.f : a.dcstate[(size_t)b * H + j0 + uu];
    }
    epi_bar();
    if (tid == 0) red_release_gpu(a.bar, 1u);
    unsigned xcount = a.xbase;
    for (int i = 0; i < a.n; ++i) {
      const int t = a.t1 - i;
      const bool mma = i >= mma0;
      // ---- the step's inputs (written by earlier kernels: read-only here), loaded before waiting
      // for the MMA so their latency hides behind it
      const float* dhi = a.dh_in[i];
      const float* act = a.act[i];
      const float* sp = a.sprev[i];
      float in[8][6];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int idx = tid + ET * k, uu = idx & 31, b = idx >> 5, j = j0 + uu;
        const float* ar = act + (size_t)b * 4 * H;
        in[k][0] = __ldg(ar + j);
        in[k][1] = __ldg(ar + H + j);
        in[k][2] = __ldg(ar + 2 * H + j);
        in[k][3] = __ldg(ar + 3 * H + j);
        in[k][4] = sp ? __ldg(sp + (size_t)b * 2 * H + H + j) : 0.f;
        in[k][5] = __ldg(dhi + (size_t)b * a.ldh + j);
      }
      if (mma) {
        // ---- partial of K slice q for the tile's 128 units -> the exchange, slot (owner, q)
        mbar_wait(accum, (i - mma0) & 1);
        tc_fence_after();
        if (tid == 0) bwd_stamp(a, i, 2);
        float acc[32];
        tmem_ld32(tmem + ((uint32_t)(qq * 32) << 16) + hf * 32, acc);
        tc_fence_before();
        mbar_arrive(tfree);
        float* xo = a.xch + ((((size_t)m * 4 + qq) * 4 + q) * B + hf * 32) * 32 + lane;
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) __stcg(xo + jj * 32, acc[jj]);
        epi_bar();
        xcount += 4;
        if (tid == 0) {
          red_release_gpu(a.xbar + m, 1u);
          while ((int)(ld_acquire_gpu(a.xbar + m) - xcount) < 0) {
          }
          bwd_stamp(a, i, 4);
        }
        epi_bar();
      }
      // ---- cell backward of the owned units
      __nv_bfloat16* dpo = a.dpx + (size_t)(t & 1) * B * 4 * H;
      float dp[8][4];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int idx = tid + ET * k, uu = idx & 31, b = idx >> 5;
        float dr = 0.f;
        if (mma) {
          const float* xi = a.xch + (((size_t)m * 4 + q) * 4 * B + b) * 32 + uu;
          dr = __ldcg(xi);
#pragma unroll
          for (int s2 = 1; s2 < 4; ++s2) dr = __fadd_rn(dr, __ldcg(xi + (size_t)s2 * B * 32));
        }
        const float dh = __fadd_rn(dr, in[k][5]);
        const float ig = in[k][0], fg = in[k][1], gg = in[k][2], og = in[k][3], cp = in[k][4];
        const float c = __fadd_rn(__fmul_rn(fg, cp), __fmul_rn(ig, gg));
        const float tc = tanh_fast(c);
        const float dct = __fadd_rn(dcs[b * 32 + uu], __fmul_rn(__fmul_rn(dh, og), __fsub_rn(1.f, __fmul_rn(tc, tc))));
        dcs[b * 32 + uu] = __fmul_rn(dct, fg);
        dp[k][0] = dpre_of(0, __fmul_rn(dct, gg), ig);
        dp[k][1] = dpre_of(1, __fmul_rn(dct, cp), fg);
        dp[k][2] = dpre_of(2, __fmul_rn(dct, ig), gg);
        dp[k][3] = dpre_of(3, __fmul_rn(dh, tc), og);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int idx = tid + ET * k, uu = idx & 31, b = idx >> 5, j = j0 + uu;
#pragma unroll
        for (int g2 = 0; g2 < 4; ++g2) dpo[(size_t)b * 4 * H + g2 * H + j] = __float2bfloat16_rn(dp[k][g2]);
      }
      if (tid == 0) bwd_stamp(a, i, 8);
      fence_proxy_async_global();
      epi_bar();
      if (tid == 0) {
        red_release_gpu(a.bar, 1u);
        bwd_stamp(a, i, 3);
      }
      // ---- off the critical path: the chunk rings and the weight-gradient operand slice
      __nv_bfloat16* dr = a.dpr[i];
      float* df = a.dpf[i];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int idx = tid + ET * k, uu = idx & 31, b = idx >> 5, j = j0 + uu;
#pragma unroll
        for (int g2 = 0; g2 < 4; ++g2) {
          dr[(size_t)b * 4 * H + g2 * H + j] = __float2bfloat16_rn(dp[k][g2]);
          df[(size_t)b * 4 * H + g2 * H + j] = dp[k][g2];
        }
      }
    }
    for (int idx = tid; idx < 32 * B; idx += ET) {
      const int uu = idx & 31, b = idx >> 5;
      a.dcstate[(size_t)b * H + j0 + uu] = dcs[b * 32 + uu];
    }
    pdl_launch();
  }
  tc_fence_before();
  __syncthreads();
  ts_mark(tsp, 7, a.dbg);
  if (warp == kRunEpiWarps + 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(B));
}

// weight-gradient operand rows of n steps: out rows (i B + b) = bf16([x_t | h_{t-1}]), x_t =
// xs.p[i] (width xw, row stride xrs, zero-padded to Kin), h_{t-1} = the h half of hs.p[i] (null: 0)
struct StepPtrs {
  const float* p[kRunMax];
};
__global__ void __launch_bounds__(256) lstm_oppack_kernel(StepPtrs xs, StepPtrs hs, int n, int B, int xw, int xrs, int Kin,
                                                          int H, __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  // eight consecutive columns per thread (one 16-byte store; float4 loads where the source rows
  // allow it: the h half always, the x half when its width and row stride are multiples of 4)
  const int K = Kin + H, G = K / 8;
  const int tot = n * B * G;
  const bool xvec = xw % 8 == 0 && xrs % 4 == 0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
    const int g = e % G, r = e / G;
    const int i = r / B, b = r % B, c0 = g * 8;
    float v[8];
    if (c0 >= Kin) {
      const float* hp = hs.p[i];
      if (hp) {
        const float4 a = *reinterpret_cast<const float4*>(hp + (size_t)b * 2 * H + (c0 - Kin));
        const float4 c = *reinterpret_cast<const float4*>(hp + (size_t)b * 2 * H + (c0 - Kin) + 4);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = c.x; v[5] = c.y; v[6] = c.z; v[7] = c.w;
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = 0.f;
      }
    } else if (xvec && c0 + 8 <= xw) {
      const float* xp = xs.p[i] + (size_t)b * xrs + c0;
      const float4 a = *reinterpret_cast<const float4*>(xp), c = *reinterpret_cast<const float4*>(xp + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = c.x; v[5] = c.y; v[6] = c.z; v[7] = c.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = c0 + j < xw ? xs.p[i][(size_t)b * xrs + c0 + j] : 0.f;
    }
    __nv_bfloat162 q0 = __floats2bfloat162_rn(v[0], v[1]), q1 = __floats2bfloat162_rn(v[2], v[3]);
    __nv_bfloat162 q2 = __floats2bfloat162_rn(v[4], v[5]), q3 = __floats2bfloat162_rn(v[6], v[7]);
    reinterpret_cast<uint4*>(out)[(size_t)r * G + g] =
        make_uint4(*reinterpret_cast<uint32_t*>(&q0), *reinterpret_cast<uint32_t*>(&q1),
                   *reinterpret_cast<uint32_t*>(&q2), *reinterpret_cast<uint32_t*>(&q3));
  }
}

// input gradient of a run: out[n ld + m] = acc for the first nmax columns n (the projection runs
// over a 256-column padded N; the padding columns are not stored)
struct EpiStoreF32Lim {
  static constexpr bool kTma = false;
  float* out;
  long ld;
  int nmax;
  __device__ __forceinline__ void operator()(int m, int n0, const float* acc, int) const {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (n0 + j < nmax) out[(long)(n0 + j) * ld + m] = acc[j];
  }
};

// X_t = x_t W_ih^T + b of a run: the tcgen05 GEMM epilogue out[n ld + m] = fl(acc + bias[m])
struct EpiBiasF32 {
  static constexpr bool kTma = false;
  float* out;
  long ld;
  const float* bias;
  __device__ __forceinline__ void operator()(int m, int n0, const float* acc, int) const {
    const float bm = bias[m];
#pragma unroll
    for (int j = 0; j < 32; ++j) out[(long)(n0 + j) * ld + m] = __fadd_rn(acc[j], bm);
  }
};

// bf16 input-projection operand of layer 0 for the n steps of a run: rows i B + b = x_{t0+i}[b],
// zero-padded from I to Kin columns (x: [T][B][I] fp32, the caller's input)
__global__ void __launch_bounds__(256) lstm_xpack_kernel(const float* __restrict__ x, int I, int Kin, int B, int n,
                                                         __nv_bfloat16* __restrict__ op) {
  pdl_wait();
  pdl_launch();
  const size_t tot = (size_t)n * B * Kin;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const size_t r = e / Kin;
    const int k = (int)(e % Kin);
    op[e] = __float2bfloat16_rn(k < I ? x[r * I + k] : 0.f);
  }
}

}  // namespace slmk
