// SIMT kernels of the unrolled-LSTM step (sm_100a).  The dense contractions (gates, head
// logits, input/recurrent gradients, weight gradients) run on the tcgen05 GEMM; these kernels
// do the element-wise cell math, operand packing and the softmax head (PAPER.md:480-485,
// reading A13: PyTorch gate order i, f, g, o; h_0 = c_0 = 0).
//
// Value layouts (fp32, row-major over the batch):
//   G^l_t  [B][4H]  gate activations (i, f, g, o)
//   S^l_t  [B][2H]  (h | c)
//   gradient node of v: gradients w.r.t. v's inputs, concatenated in pred order (reading A17)
#pragma once
#include "kernels_simt.cuh"

namespace slmk {

// every LSTM SIMT kernel waits for its predecessor (griddepcontrol.wait) and then releases its
// dependent launch, so the next kernel of the chain is scheduled and runs its prologue while this
// one works (the dependent still waits for this grid's completion before reading its outputs)
__device__ __forceinline__ void lstm_entry() {
  pdl_wait();
  pdl_launch();
}

// tanh on the SFU (tanh.approx.f32, MUFU.TANH: relative error <= 2^-10.99): the forward cell and
// gate activations (lstm_run.cuh) -- reading A26 in DESIGN.md
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// S = (h, c): c = f c_prev + i g, h = o tanh(c)   (sprev null: c_prev = 0) -- an isolated cell
// node (node by node); the same arithmetic as the run kernel's cell (lstm_run.cuh).  h also goes
// as bf16 into hring [B][H] (the lane's chunk ring slot).
__global__ void __launch_bounds__(256) lstm_cell_fwd_kernel(const float* __restrict__ act,
                                                            const float* __restrict__ sprev, int H, int B,
                                                            float* __restrict__ s, __nv_bfloat16* __restrict__ hring) {
  lstm_entry();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * H; i += gridDim.x * blockDim.x) {
    const int b = i / H, j = i % H;
    const float* a = act + (size_t)b * 4 * H;
    const float cp = sprev ? sprev[(size_t)b * 2 * H + H + j] : 0.f;
    const float c = __fadd_rn(__fmul_rn(a[H + j], cp), __fmul_rn(a[j], a[2 * H + j]));
    const float h = __fmul_rn(a[3 * H + j], tanh_fast(c));
    s[(size_t)b * 2 * H + j] = h;
    s[(size_t)b * 2 * H + H + j] = c;
    hring[i] = __float2bfloat16_rn(h);
  }
}

// Back through S: dS = sum of up to 3 successor slices (dh | dc), each [B][2H] with row stride
// ld_k (null = absent), added in the fixed order 0, 1, 2.  Output rows (pred order, reading
// A17): [4H d(acts) | 2H (0 | dc_prev)] when the cell has a predecessor state, else [4H].
// A successor's contribution to dS^l_t = (dh | dc): rows of stride ld; dh = the sum of sk
// split-K slices (sstride apart, slice order) -- the dX GEMM partials of a gates gradient are
// read in place, never materialised -- and dc at column offset c_off (c_off < 0: no c part,
// adds 0).  p == null: no such successor.
struct GradSrc {
  const float* p;
  int ld, sk, c_off;
  long sstride;
};
struct GradSrcs {
  GradSrc s[3];
};
__device__ __forceinline__ void add_src(const GradSrc& g, int b, int j, float& dh, float& dc) {
  if (!g.p) return;
  const float* q = g.p + (size_t)b * g.ld + j;
  float v = q[0];
  for (int k = 1; k < g.sk; ++k) v = __fadd_rn(v, q[(size_t)k * g.sstride]);
  dh = __fadd_rn(dh, v);
  dc = __fadd_rn(dc, g.c_off >= 0 ? q[g.c_off] : 0.f);
}

__global__ void __launch_bounds__(256) lstm_cell_bwd_kernel(GradSrcs src, const float* __restrict__ act,
                                                            const float* __restrict__ sprev, int H, int B,
                                                            float* __restrict__ out) {
  lstm_entry();
  const size_t RW = (size_t)4 * H + (sprev ? 2 * H : 0);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * H; i += gridDim.x * blockDim.x) {
    const int b = i / H, j = i % H;
    float dh = 0.f, dc = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) add_src(src.s[k], b, j, dh, dc);
    const float* a = act + (size_t)b * 4 * H;
    const float ig = a[j], fg = a[H + j], gg = a[2 * H + j], og = a[3 * H + j];
    const float cp = sprev ? sprev[(size_t)b * 2 * H + H + j] : 0.f;
    const float c = __fadd_rn(__fmul_rn(fg, cp), __fmul_rn(ig, gg));
    const float tc = tanhf(c);
    const float dct = __fadd_rn(dc, __fmul_rn(__fmul_rn(dh, og), __fsub_rn(1.f, __fmul_rn(tc, tc))));
    float* da = out + (size_t)b * RW;
    da[j] = __fmul_rn(dct, gg);
    da[H + j] = __fmul_rn(dct, cp);
    da[2 * H + j] = __fmul_rn(dct, ig);
    da[3 * H + j] = __fmul_rn(dh, tc);
    if (sprev) {
      da[4 * H + j] = 0.f;
      da[4 * H + H + j] = __fmul_rn(dct, fg);
    }
  }
}

constexpr int kColGroups = 16;
// (declared before use by the fused kernels)
__device__ __forceinline__ float dpre_of(int q, float da, float a);
__device__ __forceinline__ void pack_op(const float* __restrict__ x, int xw, int xs, int Kin,
                                       const float* __restrict__ sprev, int H, int B, __nv_bfloat16* __restrict__ op);

// d_pre = d(acts) * act'  (sigmoid for i, f, o; tanh for g) -> the time-chunk rings (bf16 GEMM
// operand + fp32 for db); d(acts) rows have stride ldd.  Then the dW operand [x | h_{t-1}]
// into its ring slot.  (The unfused form of lstm_cell_bwd_dpre_kernel's second half.)
__global__ void __launch_bounds__(256) lstm_dpre_kernel(const float* __restrict__ dact, int ldd,
                                                        const float* __restrict__ act, int H, int B,
                                                        __nv_bfloat16* __restrict__ dpre, float* __restrict__ dpre_f,
                                                        const float* __restrict__ x, int xw, int xs, int Kin,
                                                        const float* __restrict__ sprev,
                                                        __nv_bfloat16* __restrict__ op) {
  lstm_entry();
  const int G4 = 4 * H;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * G4; i += gridDim.x * blockDim.x) {
    const int b = i / G4, jj = i % G4;
    const float dv = dpre_of(jj / H, dact[(size_t)b * ldd + jj], act[i]);
    dpre[i] = __float2bfloat16_rn(dv);
    dpre_f[i] = dv;
  }
  pack_op(x, xw, xs, Kin, sprev, H, B, op);
}

__device__ __forceinline__ float dpre_of(int q, float da, float a) {   // d_pre = d(act) * act'
  return q == 2 ? __fmul_rn(da, __fsub_rn(1.f, __fmul_rn(a, a))) : __fmul_rn(da, __fmul_rn(a, __fsub_rn(1.f, a)));
}
// [x | h_{t-1}] bf16 operand (lstm_pack_kernel's values), grid-stride over all threads
__device__ __forceinline__ void pack_op(const float* __restrict__ x, int xw, int xs, int Kin,
                                       const float* __restrict__ sprev, int H, int B, __nv_bfloat16* __restrict__ op) {
  const int K = Kin + H;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * K; i += gridDim.x * blockDim.x) {
    const int b = i / K, k = i % K;
    float v;
    if (k < Kin)
      v = k < xw ? x[(size_t)b * xs + k] : 0.f;
    else
      v = sprev ? sprev[(size_t)b * 2 * H + (k - Kin)] : 0.f;
    op[i] = __float2bfloat16_rn(v);
  }
}

// Fused backward of S^l_t and the element-wise part of G^l_t's backward (used when V' runs
// g[G^l_t] right after g[S^l_t]): lstm_cell_bwd_kernel's arithmetic writing g[S], d_pre of the
// four gates into the time-chunk rings (bf16 GEMM operand + fp32 for db), and the dW operand
// [x | h_{t-1}] into its ring slot.  Thread per (b, j), grid-stride.
__global__ void __launch_bounds__(256) lstm_cell_bwd_dpre_kernel(
    GradSrcs src, const float* __restrict__ act, const float* __restrict__ sprev, int H, int B, float* __restrict__ out,
    __nv_bfloat16* __restrict__ dpre, float* __restrict__ dpre_f, const float* __restrict__ x, int xw, int xs,
    int Kin, __nv_bfloat16* __restrict__ op) {
  lstm_entry();
  const size_t RW = (size_t)4 * H + (sprev ? 2 * H : 0);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * H; i += gridDim.x * blockDim.x) {
    const int b = i / H, j = i % H;
    float dh = 0.f, dc = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) add_src(src.s[k], b, j, dh, dc);
    const float* a = act + (size_t)b * 4 * H;
    const float ig = a[j], fg = a[H + j], gg = a[2 * H + j], og = a[3 * H + j];
    const float cp = sprev ? sprev[(size_t)b * 2 * H + H + j] : 0.f;
    const float cc = __fadd_rn(__fmul_rn(fg, cp), __fmul_rn(ig, gg));
    const float tc = tanhf(cc);
    const float dct = __fadd_rn(dc, __fmul_rn(__fmul_rn(dh, og), __fsub_rn(1.f, __fmul_rn(tc, tc))));
    const float da[4] = {__fmul_rn(dct, gg), __fmul_rn(dct, cp), __fmul_rn(dct, ig), __fmul_rn(dh, tc)};
    const float av[4] = {ig, fg, gg, og};
    float* o = out + (size_t)b * RW;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      o[q * H + j] = da[q];
      const float dv = dpre_of(q, da[q], av[q]);
      dpre[(size_t)b * 4 * H + q * H + j] = __float2bfloat16_rn(dv);
      dpre_f[(size_t)b * 4 * H + q * H + j] = dv;
    }
    if (sprev) {
      o[4 * H + j] = 0.f;
      o[4 * H + H + j] = __fmul_rn(dct, fg);
    }
  }
  pack_op(x, xw, xs, Kin, sprev, H, B, op);
}

// h operand of the head: bf16 [B][H] from S^{L-1}_t
__global__ void __launch_bounds__(256) lstm_hpack_kernel(const float* __restrict__ s, int H, int B,
                                                         __nv_bfloat16* __restrict__ hop) {
  lstm_entry();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * H; i += gridDim.x * blockDim.x)
    hop[i] = __float2bfloat16_rn(s[(size_t)(i / H) * 2 * H + i % H]);
}

// h operands of a batch of steps: out rows [i B + b] = bf16(h of in.p[i] (a [B][2H] state))
struct StepIn {
  const float* p[32];
};
__global__ void __launch_bounds__(256) lstm_hpack_multi_kernel(StepIn in, int n, int H, int B,
                                                               __nv_bfloat16* __restrict__ out) {
  lstm_entry();
  const size_t per = (size_t)B * H;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < (size_t)n * per;
       i += (size_t)gridDim.x * blockDim.x) {
    const int st = (int)(i / per);
    const size_t r = i % per;
    out[i] = __float2bfloat16_rn(in.p[st][(r / H) * 2 * H + r % H]);
  }
}

// Head backward finish for nsteps steps of B rows: (dh | 0) rows from the dh GEMM's split-K
// partials P [sk][N][H] (N = nsteps B rows, row stride 2H in out), and, in blocks
// 0 .. ceil(Cp/32)-1, db_o += the column sums of dlog_f step by step in descending step order
// (each step: rows b = rg (mod 16) per group, groups in order) -- the same arithmetic as one
// launch per step in the backward's descending time order.  Block = 512 threads.
__global__ void __launch_bounds__(512) lstm_head_bwd_finish_kernel(const float* __restrict__ P, int sk, int H, int N,
                                                                   float* __restrict__ out,
                                                                   const float* __restrict__ g, int Cp, int B,
                                                                   int nsteps, float* __restrict__ acc) {
  __shared__ float red[kColGroups][33];
  lstm_entry();
  // (dh | 0) rows first (the top layer's backward waits for them): the split-K partials summed in
  // slice order, four columns per thread
  const int H4 = H / 4;
  const int slice4 = N * H4;
  const float4* P4 = reinterpret_cast<const float4*>(P);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < slice4; i += gridDim.x * blockDim.x) {
    const int row = i / H4, j4 = i % H4;
    float4 a = P4[i];
    for (int s2 = 1; s2 < sk; ++s2) {
      const float4 q = P4[(size_t)s2 * slice4 + i];
      a = make_float4(__fadd_rn(a.x, q.x), __fadd_rn(a.y, q.y), __fadd_rn(a.z, q.z), __fadd_rn(a.w, q.w));
    }
    float4* o = reinterpret_cast<float4*>(out + (size_t)row * 2 * H);
    o[j4] = a;
    o[H4 + j4] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // db_o += the per-step column sums in descending step order; every step's row sums are loaded
  // up front (independent loads), then reduced over the row groups step by step
  if ((int)blockIdx.x * 32 < Cp) {
    const int c = threadIdx.x & 31, rg = threadIdx.x >> 5;
    const int j = blockIdx.x * 32 + c;
    constexpr int kMaxSteps = 32;   // kLstmChunk
    float sv[kMaxSteps];
#pragma unroll
    for (int i = 0; i < kMaxSteps; ++i) {
      float sum = 0.f;
      if (i < nsteps && j < Cp)
        for (int b = rg; b < B; b += kColGroups) sum = __fadd_rn(sum, g[((size_t)i * B + b) * Cp + j]);
      sv[i] = sum;
    }
#pragma unroll
    for (int i = kMaxSteps - 1; i >= 0; --i) {
      if (i >= nsteps) continue;
      red[rg][c] = sv[i];
      __syncthreads();
      if (rg == 0 && j < Cp) {
        float t = red[0][c];
#pragma unroll
        for (int r = 1; r < kColGroups; ++r) t = __fadd_rn(t, red[r][c]);
        acc[j] = __fadd_rn(acc[j], t);
      }
      __syncthreads();
    }
  }
}

// One block per row b: logits = sum_s P[s][b][:] + b_o (split-K partials [sk][B][Cp], slice
// order), written to the row buffer `logits`; row loss = logsumexp - logit[y] over the C real
// classes; grad (when dlog != null) = (softmax - onehot) * scale as bf16 (the GEMM operand,
// a ring slot) + fp32 (for db_o), classes >= C: 0.
// With rowloss != null the last block to finish (counter `done`, reset by it) also writes
// loss_out = sum_b rowloss[b] * scale in row order.
__global__ void __launch_bounds__(1024) lstm_head_ce_kernel(const float* __restrict__ P, int sk,
                                                           float* __restrict__ logits, const float* __restrict__ bo,
                                                           const int* __restrict__ y, int C, int Cp, int B, float scale,
                                                           float* __restrict__ rowloss, __nv_bfloat16* __restrict__ dlog,
                                                           float* __restrict__ dlog_f, unsigned* __restrict__ done,
                                                           float* __restrict__ loss_out) {
  __shared__ float sh[32];
  lstm_entry();
  const size_t slice = (size_t)B * Cp;
  float* lr = logits + (size_t)blockIdx.x * Cp;
  const float* pr = P + (size_t)blockIdx.x * Cp;
  // a row's logits and exponentials stay in registers (kPer per thread, the same element order as
  // the strided loops, so the same bits); rows wider than kPer * blockDim fall back to re-reading
  constexpr int kPer = 8;
  const bool regs = Cp <= kPer * (int)blockDim.x;
  float vv[kPer], ev[kPer];
  float mx = -INFINITY;
#pragma unroll
  for (int k = 0; k < kPer; ++k) vv[k] = ev[k] = 0.f;
  if (regs) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int c = threadIdx.x + k * blockDim.x;
      if (c < C) {
        float acc = pr[c];
        for (int s2 = 1; s2 < sk; ++s2) acc = __fadd_rn(acc, pr[s2 * slice + c]);
        const float v = __fadd_rn(acc, bo[c]);
        lr[c] = v;
        vv[k] = v;
        mx = fmaxf(mx, v);
      }
    }
  } else {
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      float acc = pr[c];
      for (int s2 = 1; s2 < sk; ++s2) acc = __fadd_rn(acc, pr[s2 * slice + c]);
      const float v = __fadd_rn(acc, bo[c]);
      lr[c] = v;
      mx = fmaxf(mx, v);
    }
  }
  mx = block_reduce_max(mx, sh);   // (block_reduce_* synchronise the block: the row is visible)
  float s = 0.f;
  if (regs) {
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if ((int)threadIdx.x + k * (int)blockDim.x < C) {
        ev[k] = expf(__fsub_rn(vv[k], mx));
        s = __fadd_rn(s, ev[k]);
      }
  } else {
    for (int c = threadIdx.x; c < C; c += blockDim.x) s = __fadd_rn(s, expf(__fsub_rn(lr[c], mx)));
  }
  s = block_reduce_sum(s, sh);
  const int yy = y[blockIdx.x];
  if (rowloss && done) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
      rowloss[blockIdx.x] = __fsub_rn(__fadd_rn(logf(s), mx), lr[yy]);
      __threadfence();
      last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      float t = 0.f;
      for (int b = threadIdx.x; b < B; b += blockDim.x) t = __fadd_rn(t, ((volatile float*)rowloss)[b]);
      t = block_reduce_sum(t, sh);
      if (threadIdx.x == 0) {
        *loss_out = __fmul_rn(t, scale);
        *done = 0u;
      }
    }
    return;
  }
  if (threadIdx.x == 0 && rowloss) rowloss[blockIdx.x] = __fsub_rn(__fadd_rn(logf(s), mx), lr[yy]);
  if (!dlog) return;
  const float inv = __frcp_rn(s);
  if (regs) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int c = threadIdx.x + k * blockDim.x;
      if (c >= Cp) continue;
      float v = 0.f;
      if (c < C) v = __fmul_rn(__fsub_rn(__fmul_rn(ev[k], inv), c == yy ? 1.f : 0.f), scale);
      dlog[(size_t)blockIdx.x * Cp + c] = __float2bfloat16_rn(v);
      dlog_f[(size_t)blockIdx.x * Cp + c] = v;
    }
    return;
  }
  for (int c = threadIdx.x; c < Cp; c += blockDim.x) {
    float v = 0.f;
    if (c < C) v = __fmul_rn(__fsub_rn(__fmul_rn(expf(__fsub_rn(lr[c], mx)), inv), c == yy ? 1.f : 0.f), scale);
    dlog[(size_t)blockIdx.x * Cp + c] = __float2bfloat16_rn(v);
    dlog_f[(size_t)blockIdx.x * Cp + c] = v;
  }
}

// Per-step losses of a batch of head steps: block i writes *out.p[i] = sum_b rowloss[i B + b] *
// scale (block_reduce_sum order, 1024 threads).
struct StepOut {
  float* p[32];
};
// (also into loss_t[i]: the per-step losses in time order, read by the Sum node)
__global__ void __launch_bounds__(1024) lstm_step_loss_kernel(const float* __restrict__ rowloss, int B, float scale,
                                                              StepOut out, float* __restrict__ loss_t) {
  __shared__ float sh[32];
  lstm_entry();
  float t = 0.f;
  for (int b = threadIdx.x; b < B; b += blockDim.x) t = __fadd_rn(t, rowloss[(size_t)blockIdx.x * B + b]);
  t = block_reduce_sum(t, sh);
  if (threadIdx.x == 0) {
    const float v = __fmul_rn(t, scale);
    *out.p[blockIdx.x] = v;
    loss_t[blockIdx.x] = v;
  }
}

// loss = sum over the step losses (pool offsets table, in time order) — the Sum node
// loss = sum over the step losses in time order -- the Sum node (the H_t values, as written
// next to their tags by lstm_step_loss_kernel into loss_t)
__global__ void __launch_bounds__(32) lstm_sum_kernel(const float* __restrict__ loss_t, int T, float* __restrict__ out) {
  lstm_entry();
  if (threadIdx.x != 0) return;
  float s = 0.f;
  for (int t = 0; t < T; ++t) s = __fadd_rn(s, loss_t[t]);
  *out = s;
}

// split-K partial sums in slice order: out[i] = sum_{ks < split} P[ks * slice + i], i < n (float4)
__global__ void __launch_bounds__(256) splitk_sum_kernel(const float4* __restrict__ P, int split, size_t slice, size_t n,
                                                         float4* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = P[i];
    for (int ks = 1; ks < split; ++ks) {
      const float4 q = P[(size_t)ks * slice + i];
      v = make_float4(__fadd_rn(v.x, q.x), __fadd_rn(v.y, q.y), __fadd_rn(v.z, q.z), __fadd_rn(v.w, q.w));
    }
    out[i] = v;
  }
}
__global__ void __launch_bounds__(256) fill_kernel(float* __restrict__ p, int n, float v) {
  lstm_entry();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

// acc[j] += sum_b g[b][j]  (column sums accumulated into a gradient; fixed order: 16 row
// groups b = rg (mod 16), then the groups in order).  Block = 32 columns x 16 groups.
__global__ void __launch_bounds__(512) colsum_acc_kernel(const float* __restrict__ g, int B, int n,
                                                         float* __restrict__ acc) {
  __shared__ float red[kColGroups][33];
  lstm_entry();
  const int c = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + c;
  float sum = 0.f;
  if (j < n)
    for (int b = rg; b < B; b += kColGroups) sum = __fadd_rn(sum, g[(size_t)b * n + j]);
  red[rg][c] = sum;
  __syncthreads();
  if (rg == 0 && j < n) {
    float t = red[0][c];
#pragma unroll
    for (int r = 1; r < kColGroups; ++r) t = __fadd_rn(t, red[r][c]);
    acc[j] = __fadd_rn(acc[j], t);
  }
}

}  // namespace slmk
