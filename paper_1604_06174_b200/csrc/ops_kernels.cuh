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

}  // namespace slmk
