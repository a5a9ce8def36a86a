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
// y = gamma (x - mu) rstd + beta.  Block = 32 features x 8 row groups (the bn_act_kernel order).
__device__ __forceinline__ void bn_stats32(const float* __restrict__ x, int B, int d, int f, bool ok, float (*red)[33],
                                           float& mu, float& rstd) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float s = 0.f;
  if (ok)
    for (int b = w; b < B; b += 8) s = __fadd_rn(s, x[(size_t)b * d + f]);
  red[w][lane] = s;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) tot = __fadd_rn(tot, red[i][lane]);
  mu = __fmul_rn(tot, __frcp_rn((float)B));
  __syncthreads();
  float v = 0.f;
  if (ok)
    for (int b = w; b < B; b += 8) {
      const float dx = __fsub_rn(x[(size_t)b * d + f], mu);
      v = __fmaf_rn(dx, dx, v);
    }
  red[w][lane] = v;
  __syncthreads();
  float var = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) var = __fadd_rn(var, red[i][lane]);
  var = __fmul_rn(var, __frcp_rn((float)B));
  rstd = __frsqrt_rn(__fadd_rn(var, kEps));
  __syncthreads();
}

__global__ void __launch_bounds__(256) op_bn_fwd_kernel(const float* __restrict__ x, const float* __restrict__ gamma,
                                                        const float* __restrict__ beta, int B, int d,
                                                        float* __restrict__ y) {
  __shared__ float red[8][33];
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f = blockIdx.x * 32 + lane;
  const bool ok = f < d;
  float mu, rstd;
  bn_stats32(x, B, d, f, ok, red, mu, rstd);
  if (!ok) return;
  const float g = gamma[f], bt = beta[f];
  for (int b = w; b < B; b += 8) {
    const size_t i = (size_t)b * d + f;
    y[i] = bn_u(bn_xhat(x[i], mu, rstd), g, bt);   // y may alias x: each element is read once before
  }
}

// BN backward (stats re-derived from x): dgamma = sum dy xhat, dbeta = sum dy,
// dx = gamma rstd (dy - mean dy - xhat mean(dy xhat)).  dx may alias dy.
__global__ void __launch_bounds__(256) op_bn_bwd_kernel(const float* dy, const float* __restrict__ x,
                                                        const float* __restrict__ gamma, int B, int d, float* dx,
                                                        float* __restrict__ dgamma, float* __restrict__ dbeta) {
  __shared__ float red[8][33];
  __shared__ float red2[8][33];
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f = blockIdx.x * 32 + lane;
  const bool ok = f < d;
  float mu, rstd;
  bn_stats32(x, B, d, f, ok, red, mu, rstd);
  float s1 = 0.f, s2 = 0.f;
  if (ok)
    for (int b = w; b < B; b += 8) {
      const size_t i = (size_t)b * d + f;
      const float g = dy[i];
      s1 = __fadd_rn(s1, g);
      s2 = __fmaf_rn(g, bn_xhat(x[i], mu, rstd), s2);
    }
  red[w][lane] = s1;
  red2[w][lane] = s2;
  __syncthreads();
  float S1 = 0.f, S2 = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    S1 = __fadd_rn(S1, red[i][lane]);
    S2 = __fadd_rn(S2, red2[i][lane]);
  }
  if (!ok) return;
  const float invB = __frcp_rn((float)B);
  const float m1 = __fmul_rn(S1, invB), m2 = __fmul_rn(S2, invB), k = __fmul_rn(gamma[f], rstd);
  for (int b = w; b < B; b += 8) {
    const size_t i = (size_t)b * d + f;
    const float xh = bn_xhat(x[i], mu, rstd);
    dx[i] = __fmul_rn(k, __fsub_rn(__fsub_rn(dy[i], m1), __fmul_rn(xh, m2)));
  }
  if (w == 0) {
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
__global__ void __launch_bounds__(256) op_gsum_kernel(GradSlices s, int B, int w, float* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  const size_t n = (size_t)B * w;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / w, c = i % w;
    float v = s.p[0][b * s.ld[0] + c];
    for (int k = 1; k < s.n; ++k) v = __fadd_rn(v, s.p[k][b * s.ld[k] + c]);
    out[i] = v;
  }
}

// bf16 GEMM operand (round to nearest even): rows of width w from a source of row stride ld
__global__ void __launch_bounds__(256) op_pack_kernel(const float* __restrict__ x, int B, int w, int ld,
                                                      __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  const size_t n = (size_t)B * w;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(x[(i / w) * ld + i % w]);
}

// ---------------------------------------------------------------- many-row reductions
// Values of convolutional graphs have rows = B*H*W (NHWC) up to ~10^4-10^5 per channel: the
// per-channel sums run over row chunks of kRowChunk rows in parallel CTAs (grid (C/32, chunks)),
// each chunk's partial in a fixed order (8 row groups), then the chunk partials in chunk order.
// Batch statistics are two-pass (mean, then the centred sum of squares), as bn_stats32.
constexpr int kRowChunk = 256;
__device__ __forceinline__ float chunk_colsum(const float* __restrict__ x, int R, int C, int f, int r0, int r1,
                                              float (*red)[33]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float s = 0.f;
  if (f < C)
    for (int r = r0 + w; r < r1; r += 8) s = __fadd_rn(s, x[(size_t)r * C + f]);
  red[w][lane] = s;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) t = __fadd_rn(t, red[i][lane]);
  __syncthreads();
  return t;
}
__device__ __forceinline__ float parts_sum(const float* __restrict__ part, int nch, int C, int f) {
  float t = 0.f;
  for (int ch = 0; ch < nch; ++ch) t = __fadd_rn(t, part[(size_t)ch * C + f]);
  return t;
}
// part[ch][f] = sum of x[r][f] over the rows of chunk ch
__global__ void __launch_bounds__(256) op_colpart_kernel(const float* __restrict__ x, int R, int C,
                                                         float* __restrict__ part) {
  __shared__ float red[8][33];
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * 32 + (threadIdx.x & 31), ch = blockIdx.y;
  const int r0 = ch * kRowChunk, r1 = min(R, r0 + kRowChunk);
  const float t = chunk_colsum(x, R, C, f, r0, r1, red);
  if (threadIdx.x < 32 && f < C) part[(size_t)ch * C + f] = t;
}
// out[f] = sum of the chunk partials in chunk order
__global__ void __launch_bounds__(256) op_colfin_kernel(const float* __restrict__ part, int nch, int C,
                                                        float* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < C) out[f] = parts_sum(part, nch, C, f);
}
// mean and rstd of channel f from the chunk partials (sum, centred squares)
__device__ __forceinline__ void parts_stats(const float* __restrict__ psum, const float* __restrict__ psq, int nch,
                                            int R, int C, int f, float& mu, float& rstd) {
  const float invR = __frcp_rn((float)R);
  mu = __fmul_rn(parts_sum(psum, nch, C, f), invR);
  if (psq) rstd = __frsqrt_rn(__fadd_rn(__fmul_rn(parts_sum(psq, nch, C, f), invR), kEps));
}
// psq[ch][f] = sum over chunk ch of (x - mu)^2, mu from psum
__global__ void __launch_bounds__(256) op_bn_sq_kernel(const float* __restrict__ x, int R, int C,
                                                       const float* __restrict__ psum, float* __restrict__ psq) {
  __shared__ float red[8][33];
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f = blockIdx.x * 32 + lane, ch = blockIdx.y, nch = gridDim.y;
  const int r0 = ch * kRowChunk, r1 = min(R, r0 + kRowChunk);
  float mu = 0.f, dummy;
  if (f < C) parts_stats(psum, nullptr, nch, R, C, f, mu, dummy);
  float v = 0.f;
  if (f < C)
    for (int r = r0 + w; r < r1; r += 8) {
      const float e = __fsub_rn(x[(size_t)r * C + f], mu);
      v = __fmaf_rn(e, e, v);
    }
  red[w][lane] = v;
  __syncthreads();
  if (w != 0 || f >= C) return;
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) t = __fadd_rn(t, red[i][lane]);
  psq[(size_t)ch * C + f] = t;
}
// y = gamma xhat + beta over chunk ch (y may alias x)
__global__ void __launch_bounds__(256) op_bn_apply_kernel(const float* x, int R, int C, const float* __restrict__ psum,
                                                          const float* __restrict__ psq, const float* __restrict__ gamma,
                                                          const float* __restrict__ beta, float* y) {
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f = blockIdx.x * 32 + lane, ch = blockIdx.y, nch = gridDim.y;
  if (f >= C) return;
  const int r0 = ch * kRowChunk, r1 = min(R, r0 + kRowChunk);
  float mu, rstd;
  parts_stats(psum, psq, nch, R, C, f, mu, rstd);
  const float g = gamma[f], bt = beta[f];
  for (int r = r0 + w; r < r1; r += 8) {
    const size_t i = (size_t)r * C + f;
    y[i] = bn_u(bn_xhat(x[i], mu, rstd), g, bt);
  }
}
// backward chunk partials: ps1 = sum dy, ps2 = sum dy xhat
__global__ void __launch_bounds__(256) op_bn_bpart_kernel(const float* dy, const float* __restrict__ x, int R, int C,
                                                          const float* __restrict__ psum, const float* __restrict__ psq,
                                                          float* __restrict__ ps1, float* __restrict__ ps2) {
  __shared__ float red[8][33];
  __shared__ float red2[8][33];
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f = blockIdx.x * 32 + lane, ch = blockIdx.y, nch = gridDim.y;
  const int r0 = ch * kRowChunk, r1 = min(R, r0 + kRowChunk);
  float mu = 0.f, rstd = 0.f, s1 = 0.f, s2 = 0.f;
  if (f < C) {
    parts_stats(psum, psq, nch, R, C, f, mu, rstd);
    for (int r = r0 + w; r < r1; r += 8) {
      const size_t i = (size_t)r * C + f;
      const float g = dy[i];
      s1 = __fadd_rn(s1, g);
      s2 = __fmaf_rn(g, bn_xhat(x[i], mu, rstd), s2);
    }
  }
  red[w][lane] = s1;
  red2[w][lane] = s2;
  __syncthreads();
  if (w != 0 || f >= C) return;
  float t1 = 0.f, t2 = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    t1 = __fadd_rn(t1, red[i][lane]);
    t2 = __fadd_rn(t2, red2[i][lane]);
  }
  ps1[(size_t)ch * C + f] = t1;
  ps2[(size_t)ch * C + f] = t2;
}
// dx = gamma rstd (dy - mean dy - xhat mean(dy xhat)) over chunk ch (dx may alias dy); chunk 0
// writes dgamma / dbeta
__global__ void __launch_bounds__(256) op_bn_bapply_kernel(const float* dy, const float* __restrict__ x, int R, int C,
                                                           const float* __restrict__ psum, const float* __restrict__ psq,
                                                           const float* __restrict__ ps1, const float* __restrict__ ps2,
                                                           const float* __restrict__ gamma, float* dx,
                                                           float* __restrict__ dgamma, float* __restrict__ dbeta) {
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f = blockIdx.x * 32 + lane, ch = blockIdx.y, nch = gridDim.y;
  if (f >= C) return;
  const int r0 = ch * kRowChunk, r1 = min(R, r0 + kRowChunk);
  float mu, rstd;
  parts_stats(psum, psq, nch, R, C, f, mu, rstd);
  const float S1 = parts_sum(ps1, nch, C, f), S2 = parts_sum(ps2, nch, C, f);
  const float invR = __frcp_rn((float)R);
  const float m1 = __fmul_rn(S1, invR), m2 = __fmul_rn(S2, invR), k = __fmul_rn(gamma[f], rstd);
  for (int r = r0 + w; r < r1; r += 8) {
    const size_t i = (size_t)r * C + f;
    const float xh = bn_xhat(x[i], mu, rstd);
    dx[i] = __fmul_rn(k, __fsub_rn(__fsub_rn(dy[i], m1), __fmul_rn(xh, m2)));
  }
  if (ch == 0 && w == 0) {
    dgamma[f] = S2;
    dbeta[f] = S1;
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
  const int K = g.k * g.k * g.Cin, K8 = K / 8, p = g.k / 2;
  const size_t n = R * (size_t)K8;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / K8;
    const int q = (int)(i % K8) * 8, tap = q / g.Cin, c = q % g.Cin, u = tap / g.k, v = tap % g.k;
    const int hw = g.Ho * g.Wo, b = (int)(r / hw), rem = (int)(r % hw), oi = rem / g.Wo, oj = rem % g.Wo;
    const int h = oi * g.s + u - p, w = oj * g.s + v - p;
    uint4 o = make_uint4(0u, 0u, 0u, 0u);
    if (h >= 0 && h < g.H && w >= 0 && w < g.W) {
      const float4* src = reinterpret_cast<const float4*>(x + ((size_t)(b * g.H + h) * g.W + w) * g.Cin + c);
      const float4 a = src[0], e = src[1];
      __nv_bfloat162 t0 = __floats2bfloat162_rn(a.x, a.y), t1 = __floats2bfloat162_rn(a.z, a.w);
      __nv_bfloat162 t2 = __floats2bfloat162_rn(e.x, e.y), t3 = __floats2bfloat162_rn(e.z, e.w);
      o = make_uint4(*reinterpret_cast<uint32_t*>(&t0), *reinterpret_cast<uint32_t*>(&t1),
                     *reinterpret_cast<uint32_t*>(&t2), *reinterpret_cast<uint32_t*>(&t3));
    }
    reinterpret_cast<uint4*>(col)[i] = o;
  }
}
// dx[b][h][w][c] = sum over the taps (u, v) in order whose output position reads x[b][h][w] of
// dcol[(b, i, j)][(u k + v) C_in + c]: the gather form of col2im (no atomics; fixed order)
__global__ void __launch_bounds__(256) op_col2im_kernel(const float* __restrict__ dcol, ConvGeom g, size_t Rin,
                                                        float* __restrict__ dx) {
  pdl_wait();
  pdl_launch();
  const int K = g.k * g.k * g.Cin, C4 = g.Cin / 4, p = g.k / 2;
  const size_t n = Rin * (size_t)C4;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / C4;
    const int c = (int)(i % C4) * 4;
    const int hw = g.H * g.W, b = (int)(r / hw), rem = (int)(r % hw), h = rem / g.W, w = rem % g.W;
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
        acc = make_float4(__fadd_rn(acc.x, d.x), __fadd_rn(acc.y, d.y), __fadd_rn(acc.z, d.z), __fadd_rn(acc.w, d.w));
      }
    }
    reinterpret_cast<float4*>(dx)[i] = acc;
  }
}
// split-K partial sums -> bf16: out[i] = bf16(sum_{ks < split} P[ks * n + i]) in ks order
__global__ void __launch_bounds__(256) op_splitk_bf16_kernel(const float* __restrict__ P, int split, size_t n,
                                                             __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float v = P[i];
    for (int ks = 1; ks < split; ++ks) v = __fadd_rn(v, P[(size_t)ks * n + i]);
    out[i] = __float2bfloat16_rn(v);
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
