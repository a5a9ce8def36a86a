// SIMT kernels of the chain step (sm_100a): batch-norm/ReLU operand production, batch-norm
// backward, softmax cross-entropy, column reductions, and an exact-fp32 FFMA GEMM used for
// the f32 configuration (tcgen05 has no fp32 kind; TF32 cannot meet 1e-4, SURVEY hard part 6).
//
// Determinism: every reduction runs in a fixed order (per-thread serial loop, then a fixed
// smem tree), no atomics, no fast-math — re-running a kernel on the same input reproduces
// its output bit for bit, which is what makes the checkpointed step equal the
// non-checkpointed step.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace slmk {

constexpr float kEps = 1e-5f;

// Programmatic dependent launch: every kernel of the step waits for its predecessor's memory
// before touching data the predecessor may have written (a no-op without the PDL attribute),
// and lets its successor start its prologue early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <class T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }

// u = gamma * (x - mu) * rstd + beta — the one definition used by forward, re-computation
// and backward (mask and xhat), so all three see identical bits.
__device__ __forceinline__ float bn_xhat(float x, float mu, float rstd) {
  return __fmul_rn(__fsub_rn(x, mu), rstd);
}
__device__ __forceinline__ float bn_u(float xhat, float g, float b) { return __fmaf_rn(g, xhat, b); }

// ------------------------------------------------------------------ K1 bn_act
// Per feature f: mu = mean_b x[b,f], var = mean_b (x-mu)^2 (two-pass), rstd = 1/sqrt(var+eps);
// a[b,f] = ReLU(gamma (x-mu) rstd + beta) stored as T (bf16 operand or fp32).
// Block = 32 features x 8 row-groups (256 threads); warp w sums rows w, w+8, ...; the 8
// partials are combined in a fixed order.  Coalesced: a warp reads 32 consecutive floats.
template <class T>
__global__ void __launch_bounds__(256) bn_act_kernel(const float* __restrict__ x,
                                                     const float* __restrict__ gamma,
                                                     const float* __restrict__ beta, int B, int d,
                                                     float* __restrict__ stats, T* __restrict__ a) {
  __shared__ float red[8][33];
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f = blockIdx.x * 32 + lane;
  const bool ok = f < d;
  float s = 0.f;
  if (ok)
    for (int b = w; b < B; b += 8) s = __fadd_rn(s, x[(size_t)b * d + f]);
  red[w][lane] = s;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) tot = __fadd_rn(tot, red[i][lane]);
  const float mu = __fdiv_rn(tot, (float)B);
  __syncthreads();
  float q = 0.f;
  if (ok)
    for (int b = w; b < B; b += 8) {
      float c = __fsub_rn(x[(size_t)b * d + f], mu);
      q = __fmaf_rn(c, c, q);
    }
  red[w][lane] = q;
  __syncthreads();
  float qt = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) qt = __fadd_rn(qt, red[i][lane]);
  const float var = __fdiv_rn(qt, (float)B);
  const float rstd = __frcp_rn(__fsqrt_rn(__fadd_rn(var, kEps)));
  if (!ok) return;
  if (w == 0) {
    stats[f] = mu;
    stats[d + f] = rstd;
  }
  const float g = gamma[f], bt = beta[f];
  for (int b = w; b < B; b += 8) {
    float u = bn_u(bn_xhat(x[(size_t)b * d + f], mu, rstd), g, bt);
    a[(size_t)b * d + f] = from_f32<T>(fmaxf(u, 0.f));
  }
}

// ------------------------------------------------------------------ batch-norm backward
// Inputs: da = g W (fp32 [B,d]), x = x_l, stats of x_l, gamma, beta, g = dx_{l+1}.
// du = da * 1[u > 0];  dgamma = sum_b du xhat;  dbeta = sum_b du;
// dx = g + gamma rstd (du - dbeta/B - xhat dgamma/B)   (written to dx, may alias g)
// db_prev = sum_b dx (= db of layer l-1), gq = bf16(dx) (next GEMM operand) when non-null.
template <class GQ>
__global__ void __launch_bounds__(256) bn_bwd_kernel(
    const float* __restrict__ da, const float* __restrict__ x, const float* __restrict__ stats,
    const float* __restrict__ gamma, const float* __restrict__ beta, const float* g, float* dx,
    int B, int d, float* __restrict__ dgamma, float* __restrict__ dbeta,
    float* __restrict__ db_prev, GQ* __restrict__ gq) {
  __shared__ float red[2][8][33];
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f = blockIdx.x * 32 + lane;
  const bool ok = f < d;
  float mu = 0.f, rstd = 0.f, ga = 0.f, bt = 0.f;
  if (ok) {
    mu = stats[f];
    rstd = stats[d + f];
    ga = gamma[f];
    bt = beta[f];
  }
  float s1 = 0.f, s2 = 0.f;
  if (ok)
    for (int b = w; b < B; b += 8) {
      size_t i = (size_t)b * d + f;
      float xh = bn_xhat(x[i], mu, rstd);
      float du = bn_u(xh, ga, bt) > 0.f ? da[i] : 0.f;
      s1 = __fadd_rn(s1, du);
      s2 = __fmaf_rn(du, xh, s2);
    }
  red[0][w][lane] = s1;
  red[1][w][lane] = s2;
  __syncthreads();
  float S1 = 0.f, S2 = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    S1 = __fadd_rn(S1, red[0][i][lane]);
    S2 = __fadd_rn(S2, red[1][i][lane]);
  }
  __syncthreads();
  const float invB = __frcp_rn((float)B);
  const float m1 = __fmul_rn(S1, invB), m2 = __fmul_rn(S2, invB);
  const float k = __fmul_rn(ga, rstd);
  float s3 = 0.f;
  if (ok)
    for (int b = w; b < B; b += 8) {
      size_t i = (size_t)b * d + f;
      float xh = bn_xhat(x[i], mu, rstd);
      float du = bn_u(xh, ga, bt) > 0.f ? da[i] : 0.f;
      float v = __fadd_rn(g[i], __fmul_rn(k, __fsub_rn(__fsub_rn(du, m1), __fmul_rn(xh, m2))));
      dx[i] = v;
      s3 = __fadd_rn(s3, v);
      if (gq) gq[i] = from_f32<GQ>(v);
    }
  red[0][w][lane] = s3;
  __syncthreads();
  if (!ok || w != 0) return;
  float S3 = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) S3 = __fadd_rn(S3, red[0][i][lane]);
  dgamma[f] = S2;
  dbeta[f] = S1;
  if (db_prev) db_prev[f] = S3;
}

// ------------------------------------------------------------------ column sum (db_{n-1})
__global__ void __launch_bounds__(256) colsum_kernel(const float* __restrict__ g, int B, int d,
                                                     float* __restrict__ out) {
  __shared__ float red[8][33];
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (f < d)
    for (int b = w; b < B; b += 8) s = __fadd_rn(s, g[(size_t)b * d + f]);
  red[w][lane] = s;
  __syncthreads();
  if (w != 0 || f >= d) return;
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) t = __fadd_rn(t, red[i][lane]);
  out[f] = t;
}

// ------------------------------------------------------------------ softmax cross-entropy
__device__ __forceinline__ float block_reduce_max(float v, float* sh) {
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float r = sh[0];
  for (int i = 1; i < nw; ++i) r = fmaxf(r, sh[i]);
  return r;
}
__device__ __forceinline__ float block_reduce_sum(float v, float* sh) {
  for (int o = 16; o; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float r = sh[0];
  for (int i = 1; i < nw; ++i) r = __fadd_rn(r, sh[i]);
  return r;
}

// One block per row: row_loss[b] = logsumexp(x[b,:]) - x[b, y_b].
__global__ void __launch_bounds__(256) ce_fwd_kernel(const float* __restrict__ x,
                                                     const int* __restrict__ labels, int d,
                                                     float* __restrict__ row_loss) {
  __shared__ float sh[32];
  pdl_wait();
  pdl_launch();
  const float* xr = x + (size_t)blockIdx.x * d;
  float mx = -INFINITY;
  for (int f = threadIdx.x; f < d; f += blockDim.x) mx = fmaxf(mx, xr[f]);
  mx = block_reduce_max(mx, sh);
  float s = 0.f;
  for (int f = threadIdx.x; f < d; f += blockDim.x) s = __fadd_rn(s, expf(__fsub_rn(xr[f], mx)));
  s = block_reduce_sum(s, sh);
  if (threadIdx.x == 0) row_loss[blockIdx.x] = __fsub_rn(__fadd_rn(logf(s), mx), xr[labels[blockIdx.x]]);
}

// loss = sum_b row_loss[b] / B_global (single block, fixed order).
__global__ void __launch_bounds__(256) ce_reduce_kernel(const float* __restrict__ row_loss, int B,
                                                        float inv_bg, float* __restrict__ loss) {
  __shared__ float sh[32];
  pdl_wait();
  pdl_launch();
  float s = 0.f;
  for (int b = threadIdx.x; b < B; b += blockDim.x) s = __fadd_rn(s, row_loss[b]);
  s = block_reduce_sum(s, sh);
  if (threadIdx.x == 0) *loss = __fmul_rn(s, inv_bg);
}

// One block per row: dx[b,:] = (softmax(x[b,:]) - onehot(y_b)) / B_global; dx may alias x
// (the whole row is read before it is written).  gq = bf16 copy when non-null.
template <class GQ>
__global__ void __launch_bounds__(256) ce_bwd_kernel(const float* x, const int* __restrict__ labels,
                                                     int d, float inv_bg, float* dx,
                                                     GQ* __restrict__ gq) {
  __shared__ float sh[32];
  pdl_wait();
  pdl_launch();
  const size_t row = (size_t)blockIdx.x * d;
  const float* xr = x + row;
  float mx = -INFINITY;
  for (int f = threadIdx.x; f < d; f += blockDim.x) mx = fmaxf(mx, xr[f]);
  mx = block_reduce_max(mx, sh);
  float s = 0.f;
  for (int f = threadIdx.x; f < d; f += blockDim.x) s = __fadd_rn(s, expf(__fsub_rn(xr[f], mx)));
  s = block_reduce_sum(s, sh);
  const float inv = __frcp_rn(s);
  const int y = labels[blockIdx.x];
  __syncthreads();  // every thread has consumed xr[] through the reductions above
  // each thread rewrites only the elements it reads here
  for (int f = threadIdx.x; f < d; f += blockDim.x) {
    float p = __fmul_rn(expf(__fsub_rn(xr[f], mx)), inv);
    float v = __fmul_rn(__fsub_rn(p, f == y ? 1.f : 0.f), inv_bg);
    dx[row + f] = v;
    if (gq) gq[row + f] = from_f32<GQ>(v);
  }
}

// ------------------------------------------------------------------ FFMA GEMM (SIMT)
// C(m, n) = sum_k A(m, k) B(n, k), fp32 accumulation in increasing k (deterministic),
// A(m,k) = A[m*sAm + k*sAk], B(n,k) = B[n*sBn + k*sBk].  64x64 tile, 256 threads, 4x4 per
// thread, k-tile 16 staged in shared memory.  Epilogue modes:
//   EPI_RESID: out[m*ldo + n] = resid[m*ldo + n] + acc + bias[n]   (forward block)
//   EPI_STORE: out[m*ldo + n] = acc                                  (da, dW)
enum { EPI_RESID = 0, EPI_STORE = 1 };
template <class TA, class TB, class TO, int EPI>
__global__ void __launch_bounds__(256) simt_gemm_kernel(
    int M, int N, int K, const TA* __restrict__ A, long sAm, long sAk, const TB* __restrict__ Bm,
    long sBn, long sBk, TO* out, long ldo, const float* resid, const float* __restrict__ bias) {
  __shared__ float As[16][64 + 1];
  __shared__ float Bs[16][64 + 1];
  pdl_wait();
  pdl_launch();
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      int kk = i / 64, r = i % 64;
      int m = m0 + r, n = n0 + r, k = k0 + kk;
      As[kk][r] = (m < M && k < K) ? to_f32(A[m * sAm + k * sAk]) : 0.f;
      Bs[kk][r] = (n < N && k < K) ? to_f32(Bm[n * sBn + k * sBk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        av[i] = As[kk][ty * 4 + i];
        bv[i] = Bs[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m >= M || n >= N) continue;
      long o = (long)m * ldo + n;
      if (EPI == EPI_RESID)
        out[o] = from_f32<TO>(__fadd_rn(resid[o], __fadd_rn(acc[i][j], bias[n])));
      else
        out[o] = from_f32<TO>(acc[i][j]);
    }
}

}  // namespace slmk
