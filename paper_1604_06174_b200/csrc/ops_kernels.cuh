// SIMT kernels of the op-granularity executor (executor_ops.cuh): the network of
// Sec. 5.1 with every operation a graph node -- BN, ReLU, FC, Add, SoftmaxCE --
// so that the "drop the results of low cost operations" plan (Sec. 4.2) really
// drops and re-computes BN and ReLU outputs.  The FC contractions run on the tcgen05 GEMM
// (tc_gemm.cuh); softmax-CE and column sums reuse kernels_simt.cuh.
//
// Values are [B][w] fp32 row-major.  A gradient node holds the gradients w.r.t. all inputs of its
// forward node, concatenated along the row in pred order (reading A17).  Every reduction runs in a
// fixed order, so re-computed values and gradients are bit-identical to the plain step.
#pragma once
#include "kernels_simt.cuh"

namespace slmk {

// BN with batch statistics (reading A10: biased variance, eps 1e-5), no ReLU:
// y = gamma (x - mu) rstd + beta.
// Few-row BN (rows <= kSmallRows, e.g. the batch of an FC network): a CTA of 256 threads owns 8
// features; thread t holds feature t % 8 and rows t / 8, t / 8 + 32, ... (a warp reads 4 rows x 32
// contiguous bytes per load).  Per-feature totals: the 4 row groups of a warp by an xor-shuffle
// tree (a + b == b + a, so every lane holding the feature gets the same bits), then the 8 warps in
// warp order.  Fixed order: deterministic.  Grid d / 8.
__device__ __forceinline__ float bn8_total(float v, float (*red)[8]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 8));
  v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 16));
  if (lane < 8) red[w][lane] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) t = __fadd_rn(t, red[i][lane & 7]);
  __syncthreads();
  return t;
}
// two-pass batch statistics of feature f (mean, then the centred sum of squares; reading A10)
__device__ __forceinline__ void bn_stats8(const float* __restrict__ x, int B, int d, int f, float (*red)[8],
                                          float& mu, float& rstd) {
  const int rg = threadIdx.x >> 3;
  const float invB = __frcp_rn((float)B);
  float s = 0.f;
  for (int b = rg; b < B; b += 32) s = __fadd_rn(s, x[(size_t)b * d + f]);
  mu = __fmul_rn(bn8_total(s, red), invB);
  float v = 0.f;
  for (int b = rg; b < B; b += 32) {
    const float e = __fsub_rn(x[(size_t)b * d + f], mu);
    v = __fmaf_rn(e, e, v);
  }
  rstd = __frsqrt_rn(__fadd_rn(__fmul_rn(bn8_total(v, red), invB), kEps));
}
// out[f] = sum of g[b][f] over the B rows (bias gradients), 8 features per CTA as above
__global__ void __launch_bounds__(256) op_colsum8_kernel(const float* __restrict__ g, int B, int d,
                                                         float* __restrict__ out) {
  __shared__ float red[8][8];
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * 8 + (threadIdx.x & 7), rg = threadIdx.x >> 3;
  float s = 0.f;
  for (int b = rg; b < B; b += 32) s = __fadd_rn(s, g[(size_t)b * d + f]);
  const float t = bn8_total(s, red);
  if (threadIdx.x < 8) out[f] = t;
}
__global__ void __launch_bounds__(256) op_bn_fwd_kernel(const float* x, const float* __restrict__ gamma,
                                                        const float* __restrict__ beta, int B, int d, float* y) {
  __shared__ float red[8][8];
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * 8 + (threadIdx.x & 7), rg = threadIdx.x >> 3;
  float mu, rstd;
  bn_stats8(x, B, d, f, red, mu, rstd);
  const float g = gamma[f], bt = beta[f];
  for (int b = rg; b < B; b += 32) {
    const size_t i = (size_t)b * d + f;
    y[i] = bn_u(bn_xhat(x[i], mu, rstd), g, bt);   // y may alias x: each element is read before it is written
  }
}

// BN backward (stats re-derived from x): dgamma = sum dy xhat, dbeta = sum dy,
// dx = gamma rstd (dy - mean dy - xhat mean(dy xhat)).  dx may alias dy.
__global__ void __launch_bounds__(256) op_bn_bwd_kernel(const float* dy, const float* __restrict__ x,
                                                        const float* __restrict__ gamma, int B, int d, float* dx,
                                                        float* __restrict__ dgamma, float* __restrict__ dbeta) {
  __shared__ float red[8][8];
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * 8 + (threadIdx.x & 7), rg = threadIdx.x >> 3;
  float mu, rstd;
  bn_stats8(x, B, d, f, red, mu, rstd);
  float s1 = 0.f, s2 = 0.f;
  for (int b = rg; b < B; b += 32) {
    const size_t i = (size_t)b * d + f;
    const float g = dy[i];
    s1 = __fadd_rn(s1, g);
    s2 = __fmaf_rn(g, bn_xhat(x[i], mu, rstd), s2);
  }
  const float S1 = bn8_total(s1, red), S2 = bn8_total(s2, red);
  const float invB = __frcp_rn((float)B);
  const float m1 = __fmul_rn(S1, invB), m2 = __fmul_rn(S2, invB), k = __fmul_rn(gamma[f], rstd);
  for (int b = rg; b < B; b += 32) {
    const size_t i = (size_t)b * d + f;
    const float xh = bn_xhat(x[i], mu, rstd);
    dx[i] = __fmul_rn(k, __fsub_rn(__fsub_rn(dy[i], m1), __fmul_rn(xh, m2)));
  }
  if (threadIdx.x < 8) {
    dgamma[f] = S2;
    dbeta[f] = S1;
  }
}

// ReLU forward (y may alias x) / backward through the output (ReLU'(0) = 0; dx may alias dy)
__global__ void __launch_bounds__(256) op_relu_fwd_kernel(const float4* x, size_t n4, float4* y) {
  pdl_wait();
  pdl_launch();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = x[i];
    v.x = fmaxf(v.x, 0.f);
    v.y = fmaxf(v.y, 0.f);
    v.z = fmaxf(v.z, 0.f);
    v.w = fmaxf(v.w, 0.f);
    y[i] = v;
  }
}
__global__ void __launch_bounds__(256) op_relu_bwd_kernel(const float4* dy, const float4* __restrict__ y, size_t n4,
                                                          float4* dx) {
  pdl_wait();
  pdl_launch();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 g = dy[i], o = y[i];
    dx[i] = make_float4(o.x > 0.f ? g.x : 0.f, o.y > 0.f ? g.y : 0.f, o.z > 0.f ? g.z : 0.f, o.w > 0.f ? g.w : 0.f);
  }
}

// Add forward: y = a + b (y may alias a or b); backward: dx = [dy | dy] rows of width 2w
__global__ void __launch_bounds__(256) op_add_fwd_kernel(const float4* a, const float4* b, size_t n4, float4* y) {
  pdl_wait();
  pdl_launch();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 u = a[i], v = b[i];
    y[i] = make_float4(__fadd_rn(u.x, v.x), __fadd_rn(u.y, v.y), __fadd_rn(u.z, v.z), __fadd_rn(u.w, v.w));
  }
}
__global__ void __launch_bounds__(256) op_add_bwd_kernel(const float4* __restrict__ dy, int B, int w4,
                                                         float4* __restrict__ dx) {
  pdl_wait();
  pdl_launch();
  const size_t n4 = (size_t)B * w4;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / w4, c = i % w4;
    const float4 g = dy[i];
    dx[b * 2 * w4 + c] = g;
    dx[b * 2 * w4 + w4 + c] = g;
  }
}

// Upstream gradient of a node: the sum of its successors' gradient slices, in successor order
// (reading A17): out[b][c] = sum_k src[k][b * ld[k] + off[k] + c]
struct GradSlices {
  const float* p[8];
  int ld[8];
  int n;
};
// (widths, strides and offsets are multiples of 128 floats: float4 per thread)
__global__ void __launch_bounds__(256) op_gsum_kernel(GradSlices s, int B, int w, float* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  const int w4 = w / 4;
  const size_t n4 = (size_t)B * w4;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / w4;
    const int c = (int)(i - b * w4) * 4;
    float4 v = *reinterpret_cast<const float4*>(s.p[0] + b * s.ld[0] + c);
    for (int k = 1; k < s.n; ++k) {
      const float4 t = *reinterpret_cast<const float4*>(s.p[k] + b * s.ld[k] + c);
      v = make_float4(__fadd_rn(v.x, t.x), __fadd_rn(v.y, t.y), __fadd_rn(v.z, t.z), __fadd_rn(v.w, t.w));
    }
    reinterpret_cast<float4*>(out)[i] = v;
  }
}

// contiguous fp32 -> bf16 (RN), 8 elements per thread (n8 = elements / 8)
__global__ void __launch_bounds__(256) op_cvt_bf16_kernel(const float4* __restrict__ x, size_t n8,
                                                          uint4* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
    const float4 a = x[2 * i], e = x[2 * i + 1];
    __nv_bfloat162 t0 = __floats2bfloat162_rn(a.x, a.y), t1 = __floats2bfloat162_rn(a.z, a.w);
    __nv_bfloat162 t2 = __floats2bfloat162_rn(e.x, e.y), t3 = __floats2bfloat162_rn(e.z, e.w);
    out[i] = make_uint4(*reinterpret_cast<uint32_t*>(&t0), *reinterpret_cast<uint32_t*>(&t1),
                        *reinterpret_cast<uint32_t*>(&t2), *reinterpret_cast<uint32_t*>(&t3));
  }
}

// ---------------------------------------------------------------- many-row reductions
// Values of convolutional graphs have rows = B*H*W (NHWC) up to ~10^4-10^5 per channel: the
// per-channel sums run over row chunks of kRowChunk rows in parallel CTAs (grid (C/128, chunks)),
// each chunk's partial in a fixed order (8 row groups), then the chunk partials (block_parts_sum)
// into per-channel statistics, computed once per channel.
// Batch statistics are two-pass (mean, then the centred sum of squares), as bn_stats32.
constexpr int kRowChunk = 128;   // rows per chunk CTA (C = 128 at 64 x 32 x 32 rows: 512 CTAs)
constexpr int kSmallRows = 256;  // up to this many rows: the one-CTA-per-32-channels kernels
// Total over the chunk partials of channel f = blockIdx.x * 32 + lane, by a 1024-thread CTA (the
// partials are few KB to a few hundred KB: latency, not bandwidth): warp w sums chunks w, w + 32,
// ... (loads of consecutive channels coalesced, 4 in flight per thread), the 32 warp sums are
// added in warp order.  A fixed order, so deterministic; every thread returns the total.
constexpr int kFinThreads = 1024;
__device__ __forceinline__ float block_parts_sum(const float* __restrict__ part, int nch, int C, int f,
                                                 float (*red)[33]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float s = 0.f;
  if (f < C) {
    int ch = w;
    for (; ch + 96 < nch; ch += 128) {
      const float a = part[(size_t)ch * C + f], b = part[(size_t)(ch + 32) * C + f];
      const float c = part[(size_t)(ch + 64) * C + f], d = part[(size_t)(ch + 96) * C + f];
      s = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s, a), b), c), d);
    }
    for (; ch < nch; ch += 32) s = __fadd_rn(s, part[(size_t)ch * C + f]);
  }
  red[w][lane] = s;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) t = __fadd_rn(t, red[i][lane]);
  __syncthreads();
  return t;
}
// The chunk kernels: grid (C / 128, chunks), 256 threads; lane l of warp w holds channels
// blockIdx.x * 128 + 4 l .. + 3 (float4: a warp reads 512 contiguous bytes of a row) and rows
// r0 + w, r0 + w + 8, ... of the chunk; the eight warp partials are added in warp order.
__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 ld_f4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st_f4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
// total over the 8 warps (warp order), valid in warp 0
__device__ __forceinline__ float4 warps_sum4(float4 v, float4 (*red)[32]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  red[w][lane] = v;
  __syncthreads();
  float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
  if (w == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) t = f4_add(t, red[i][lane]);
  }
  return t;
}
// part[ch][f] = sum of x[r][f] over the rows of chunk ch
__global__ void __launch_bounds__(256) op_colpart_kernel(const float* __restrict__ x, int R, int C,
                                                         float* __restrict__ part) {
  __shared__ float4 red[8][32];
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * 128 + (threadIdx.x & 31) * 4, w = threadIdx.x >> 5, ch = blockIdx.y;
  const int r0 = ch * kRowChunk, r1 = min(R, r0 + kRowChunk);
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
  for (int r = r0 + w; r < r1; r += 8) s = f4_add(s, ld_f4(x + (size_t)r * C + f));
  const float4 t = warps_sum4(s, red);
  if (w == 0) st_f4(part + (size_t)ch * C + f, t);
}
// out[f] = total of the chunk partials (block_parts_sum); grid (C + 31) / 32, kFinThreads threads
__global__ void __launch_bounds__(kFinThreads) op_colfin_kernel(const float* __restrict__ part, int nch, int C,
                                                        float* __restrict__ out) {
  __shared__ float red[32][33];
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * 32 + (threadIdx.x & 31);
  const float t = block_parts_sum(part, nch, C, f, red);
  if (threadIdx.x < 32 && f < C) out[f] = t;
}
// per-channel statistics from the chunk partials, once per channel (reading A10): mean = total(psum)
// / R and, with psq (centred squares), rstd = 1 / sqrt(total(psq) / R + eps)
__global__ void __launch_bounds__(kFinThreads) op_bn_fin_kernel(const float* __restrict__ psum, const float* __restrict__ psq,
                                                        int nch, int R, int C, float* __restrict__ mu_out,
                                                        float* __restrict__ rstd_out) {
  __shared__ float red[32][33];
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * 32 + (threadIdx.x & 31);
  const float invR = __frcp_rn((float)R);
  if (mu_out) {
    const float t = block_parts_sum(psum, nch, C, f, red);
    if (threadIdx.x < 32 && f < C) mu_out[f] = __fmul_rn(t, invR);
  }
  if (psq) {
    const float t = block_parts_sum(psq, nch, C, f, red);
    if (threadIdx.x < 32 && f < C) rstd_out[f] = __frsqrt_rn(__fadd_rn(__fmul_rn(t, invR), kEps));
  }
}
// totals of two partial arrays (the backward sums S1, S2)
__global__ void __launch_bounds__(kFinThreads) op_parts2_kernel(const float* __restrict__ p1, const float* __restrict__ p2,
                                                        int nch, int C, float* __restrict__ s1, float* __restrict__ s2) {
  __shared__ float red[32][33];
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * 32 + (threadIdx.x & 31);
  const float a = block_parts_sum(p1, nch, C, f, red);
  const float b = block_parts_sum(p2, nch, C, f, red);
  if (threadIdx.x < 32 && f < C) {
    s1[f] = a;
    s2[f] = b;
  }
}
// psq[ch][f] = sum over chunk ch of (x - mu)^2
__global__ void __launch_bounds__(256) op_bn_sq_kernel(const float* __restrict__ x, int R, int C,
                                                       const float* __restrict__ mean, float* __restrict__ psq) {
  __shared__ float4 red[8][32];
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * 128 + (threadIdx.x & 31) * 4, w = threadIdx.x >> 5, ch = blockIdx.y;
  const int r0 = ch * kRowChunk, r1 = min(R, r0 + kRowChunk);
  const float4 mu = ld_f4(mean + f);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
  for (int r = r0 + w; r < r1; r += 8) {
    const float4 a = ld_f4(x + (size_t)r * C + f);
    const float ex = __fsub_rn(a.x, mu.x), ey = __fsub_rn(a.y, mu.y), ez = __fsub_rn(a.z, mu.z), ew = __fsub_rn(a.w, mu.w);
    v = make_float4(__fmaf_rn(ex, ex, v.x), __fmaf_rn(ey, ey, v.y), __fmaf_rn(ez, ez, v.z), __fmaf_rn(ew, ew, v.w));
  }
  const float4 t = warps_sum4(v, red);
  if (w == 0) st_f4(psq + (size_t)ch * C + f, t);
}
// y = gamma xhat + beta over chunk ch (y may alias x)
__global__ void __launch_bounds__(256) op_bn_apply_kernel(const float* x, int R, int C, const float* __restrict__ mean,
                                                          const float* __restrict__ rstdv, const float* __restrict__ gamma,
                                                          const float* __restrict__ beta, float* y) {
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * 128 + (threadIdx.x & 31) * 4, w = threadIdx.x >> 5, ch = blockIdx.y;
  const int r0 = ch * kRowChunk, r1 = min(R, r0 + kRowChunk);
  const float4 mu = ld_f4(mean + f), rs = ld_f4(rstdv + f), g = ld_f4(gamma + f), bt = ld_f4(beta + f);
#pragma unroll 4
  for (int r = r0 + w; r < r1; r += 8) {
    const size_t i = (size_t)r * C + f;
    const float4 a = ld_f4(x + i);
    st_f4(y + i, make_float4(bn_u(bn_xhat(a.x, mu.x, rs.x), g.x, bt.x), bn_u(bn_xhat(a.y, mu.y, rs.y), g.y, bt.y),
                             bn_u(bn_xhat(a.z, mu.z, rs.z), g.z, bt.z), bn_u(bn_xhat(a.w, mu.w, rs.w), g.w, bt.w)));
  }
}
// backward chunk partials: ps1 = sum dy, ps2 = sum dy xhat
__global__ void __launch_bounds__(256) op_bn_bpart_kernel(const float* dy, const float* __restrict__ x, int R, int C,
                                                          const float* __restrict__ mean, const float* __restrict__ rstdv,
                                                          float* __restrict__ ps1, float* __restrict__ ps2) {
  __shared__ float4 red[8][32];
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * 128 + (threadIdx.x & 31) * 4, w = threadIdx.x >> 5, ch = blockIdx.y;
  const int r0 = ch * kRowChunk, r1 = min(R, r0 + kRowChunk);
  const float4 mu = ld_f4(mean + f), rs = ld_f4(rstdv + f);
  float4 s1 = make_float4(0.f, 0.f, 0.f, 0.f), s2 = s1;
#pragma unroll 4
  for (int r = r0 + w; r < r1; r += 8) {
    const size_t i = (size_t)r * C + f;
    const float4 g = ld_f4(dy + i), a = ld_f4(x + i);
    s1 = f4_add(s1, g);
    s2 = make_float4(__fmaf_rn(g.x, bn_xhat(a.x, mu.x, rs.x), s2.x), __fmaf_rn(g.y, bn_xhat(a.y, mu.y, rs.y), s2.y),
                     __fmaf_rn(g.z, bn_xhat(a.z, mu.z, rs.z), s2.z), __fmaf_rn(g.w, bn_xhat(a.w, mu.w, rs.w), s2.w));
  }
  const float4 t1 = warps_sum4(s1, red);
  __syncthreads();
  const float4 t2 = warps_sum4(s2, red);
  if (w == 0) {
    st_f4(ps1 + (size_t)ch * C + f, t1);
    st_f4(ps2 + (size_t)ch * C + f, t2);
  }
}
// dx = gamma rstd (dy - mean dy - xhat mean(dy xhat)) over chunk ch (dx may alias dy); chunk 0
// writes dgamma / dbeta
__device__ __forceinline__ float bn_dx1(float g, float a, float mu, float rs, float m1, float m2, float k) {
  return __fmul_rn(k, __fsub_rn(__fsub_rn(g, m1), __fmul_rn(bn_xhat(a, mu, rs), m2)));
}
__global__ void __launch_bounds__(256) op_bn_bapply_kernel(const float* dy, const float* __restrict__ x, int R, int C,
                                                           const float* __restrict__ mean, const float* __restrict__ rstdv,
                                                           const float* __restrict__ S1v, const float* __restrict__ S2v,
                                                           const float* __restrict__ gamma, float* dx,
                                                           float* __restrict__ dgamma, float* __restrict__ dbeta) {
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * 128 + (threadIdx.x & 31) * 4, w = threadIdx.x >> 5, ch = blockIdx.y;
  const int r0 = ch * kRowChunk, r1 = min(R, r0 + kRowChunk);
  const float invR = __frcp_rn((float)R);
  const float4 mu = ld_f4(mean + f), rs = ld_f4(rstdv + f), S1 = ld_f4(S1v + f), S2 = ld_f4(S2v + f),
               gm = ld_f4(gamma + f);
  const float4 m1 = make_float4(__fmul_rn(S1.x, invR), __fmul_rn(S1.y, invR), __fmul_rn(S1.z, invR), __fmul_rn(S1.w, invR));
  const float4 m2 = make_float4(__fmul_rn(S2.x, invR), __fmul_rn(S2.y, invR), __fmul_rn(S2.z, invR), __fmul_rn(S2.w, invR));
  const float4 k = make_float4(__fmul_rn(gm.x, rs.x), __fmul_rn(gm.y, rs.y), __fmul_rn(gm.z, rs.z), __fmul_rn(gm.w, rs.w));
#pragma unroll 4
  for (int r = r0 + w; r < r1; r += 8) {
    const size_t i = (size_t)r * C + f;
    const float4 g = ld_f4(dy + i), a = ld_f4(x + i);
    st_f4(dx + i, make_float4(bn_dx1(g.x, a.x, mu.x, rs.x, m1.x, m2.x, k.x), bn_dx1(g.y, a.y, mu.y, rs.y, m1.y, m2.y, k.y),
                              bn_dx1(g.z, a.z, mu.z, rs.z, m1.z, m2.z, k.z), bn_dx1(g.w, a.w, mu.w, rs.w, m1.w, m2.w, k.w)));
  }
  if (ch == 0 && w == 0) {
    st_f4(dgamma + f, S2);
    st_f4(dbeta + f, S1);
  }
}

// ---------------------------------------------------------------- convolution
// NHWC fp32 values [B*H*W][C]; "same" padding p = k / 2, stride s; the GEMM's K index of tap (u, v)
// and channel c is (u k + v) C_in + c (W [C_out][k k C_in]).
struct ConvGeom {
  int H, W, Cin, k, s, Ho, Wo;
};
// col[r][K] (bf16, r = (b, i, j) output position) = x at the tap's input position, 0 in the padding;
// 8 consecutive K columns (one tap, C_in % 8 == 0) per thread: two float4 loads, one 16-byte store
__global__ void __launch_bounds__(256) op_im2col_kernel(const float* __restrict__ x, ConvGeom g, size_t R,
                                                        __nv_bfloat16* __restrict__ col) {
  pdl_wait();
  pdl_launch();
  // one warp per output row (position): the row's coordinates once, the lanes over its K / 8
  // 16-byte column groups (consecutive lanes write consecutive 16 B); 32-bit index arithmetic
  const int K8 = g.k * g.k * g.Cin / 8, C8 = g.Cin / 8, p = g.k / 2, hw = g.Ho * g.Wo;
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  uint4* out = reinterpret_cast<uint4*>(col);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < (int)R; r += nw) {
    const int b = r / hw, rem = r - b * hw, oi = rem / g.Wo, oj = rem - oi * g.Wo;
    const int h0 = oi * g.s - p, w0 = oj * g.s - p;
    for (int j = lane; j < K8; j += 32) {
      const int tap = j / C8, c = (j - tap * C8) * 8, u = tap / g.k, v = tap - u * g.k;
      const int h = h0 + u, w = w0 + v;
      uint4 o = make_uint4(0u, 0u, 0u, 0u);
      if (h >= 0 && h < g.H && w >= 0 && w < g.W) {
        const float4* src = reinterpret_cast<const float4*>(x + ((size_t)(b * g.H + h) * g.W + w) * g.Cin + c);
        const float4 a = src[0], e = src[1];
        __nv_bfloat162 t0 = __floats2bfloat162_rn(a.x, a.y), t1 = __floats2bfloat162_rn(a.z, a.w);
        __nv_bfloat162 t2 = __floats2bfloat162_rn(e.x, e.y), t3 = __floats2bfloat162_rn(e.z, e.w);
        o = make_uint4(*reinterpret_cast<uint32_t*>(&t0), *reinterpret_cast<uint32_t*>(&t1),
                       *reinterpret_cast<uint32_t*>(&t2), *reinterpret_cast<uint32_t*>(&t3));
      }
      out[(size_t)r * K8 + j] = o;
    }
  }
}
// dx[b][h][w][c] = sum over the taps (u, v) in order whose output position reads x[b][h][w] of
// dcol[(b, i, j)][(u k + v) C_in + c]: the gather form of col2im (no atomics; fixed order).  One
// warp per input row, the lanes over its C_in / 4 float4 groups.
__global__ void __launch_bounds__(256) op_col2im_kernel(const float* __restrict__ dcol, ConvGeom g, size_t Rin,
                                                        float* __restrict__ dx) {
  pdl_wait();
  pdl_launch();
  const int K = g.k * g.k * g.Cin, C4 = g.Cin / 4, p = g.k / 2, hw = g.H * g.W;
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < (int)Rin; r += nw) {
    const int b = r / hw, rem = r - b * hw, h = rem / g.W, w = rem - h * g.W;
    for (int c4 = lane; c4 < C4; c4 += 32) {
      const int c = c4 * 4;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int u = 0; u < g.k; ++u) {
        const int ih = h + p - u;
        if (ih < 0 || ih % g.s) continue;
        const int oi = ih / g.s;
        if (oi >= g.Ho) continue;
        for (int v = 0; v < g.k; ++v) {
          const int iw = w + p - v;
          if (iw < 0 || iw % g.s) continue;
          const int oj = iw / g.s;
          if (oj >= g.Wo) continue;
          const float4 d = *reinterpret_cast<const float4*>(dcol + ((size_t)(b * g.Ho + oi) * g.Wo + oj) * K +
                                                            (u * g.k + v) * g.Cin + c);
          acc = make_float4(__fadd_rn(acc.x, d.x), __fadd_rn(acc.y, d.y), __fadd_rn(acc.z, d.z),
                            __fadd_rn(acc.w, d.w));
        }
      }
      reinterpret_cast<float4*>(dx)[(size_t)r * C4 + c4] = acc;
    }
  }
}
// The flipped, transposed kernel of a k x k stride-1 convolution: Wt[c][t' C_out + o] =
// W[o][(k k - 1 - t') C_in + c] (tap t' = u' k + v' reads tap (k-1-u', k-1-v')), so that
// dx = im2col(dy) Wt^T -- the input gradient of a stride-1 "same" convolution is the same
// convolution of dy with the spatially flipped kernel, input and output channels exchanged.
// 32 x 32 tiles through shared memory per tap: grid (C_in / 32, C_out / 32, k k), 256 threads.
__global__ void __launch_bounds__(256) op_wflip_kernel(const __nv_bfloat16* __restrict__ W, int k, int Cin, int Cout,
                                                       __nv_bfloat16* __restrict__ Wt) {
  __shared__ __nv_bfloat16 tile[32][34];
  pdl_wait();
  pdl_launch();
  const int c0 = blockIdx.x * 32, o0 = blockIdx.y * 32, tp = blockIdx.z, t = k * k - 1 - tp;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const size_t K = (size_t)k * k * Cin, Kt = (size_t)k * k * Cout;
  for (int i = ty; i < 32; i += 8) tile[i][tx] = W[(size_t)(o0 + i) * K + (size_t)t * Cin + c0 + tx];   // [o][c]
  __syncthreads();
  for (int i = ty; i < 32; i += 8) Wt[(size_t)(c0 + i) * Kt + (size_t)tp * Cout + o0 + tx] = tile[tx][i];
}
// split-K partial sums -> bf16: out[i] = bf16(sum_{ks < split} P[ks * n + i]) in ks order
// (n % 4 == 0: 4 elements per thread, float4 loads, 8-byte stores)
__global__ void __launch_bounds__(256) op_splitk_bf16_kernel(const float* __restrict__ P, int split, size_t n,
                                                             __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  const size_t n4 = n / 4;
  const float4* P4 = reinterpret_cast<const float4*>(P);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = P4[i];
#pragma unroll 4
    for (int ks = 1; ks < split; ++ks) {
      const float4 t = P4[(size_t)ks * n4 + i];
      v = make_float4(__fadd_rn(v.x, t.x), __fadd_rn(v.y, t.y), __fadd_rn(v.z, t.z), __fadd_rn(v.w, t.w));
    }
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    reinterpret_cast<uint2*>(out)[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
}
// global average pool: y[b][c] = (sum over the HW positions in order) / HW; backward dx = dy / HW
__global__ void __launch_bounds__(256) op_pool_fwd_kernel(const float* __restrict__ x, int B, int HW, int C,
                                                          float* __restrict__ y) {
  pdl_wait();
  pdl_launch();
  const int n = B * C;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int b = i / C, c = i % C;
    float s = 0.f;
    for (int q = 0; q < HW; ++q) s = __fadd_rn(s, x[((size_t)b * HW + q) * C + c]);
    y[i] = __fdiv_rn(s, (float)HW);
  }
}
__global__ void __launch_bounds__(256) op_pool_bwd_kernel(const float* __restrict__ dy, int B, int HW, int C,
                                                          float* __restrict__ dx) {
  pdl_wait();
  pdl_launch();
  const size_t n = (size_t)B * HW * C;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t c = i % C, b = i / ((size_t)HW * C);
    dx[i] = __fdiv_rn(dy[b * C + c], (float)HW);
  }
}

}  // namespace slmk
