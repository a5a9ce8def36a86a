// Register-resident batch-norm kernels of the fused lowering (sm_100a SIMT).
//
// One CTA = 16 features x 32 row groups (512 threads, 128 CTAs at d = 2048): thread t has
// feature t%16 of row group rg = t/16 and owns rows rg, rg+32, ..., rg+32(R-1) of the batch
// (B = 32 R exactly, d % 16 == 0: no bounds tests), all values in registers, so every input is
// read once with all loads in flight (a warp touches two 64-byte row segments per load).  The batch and the
// number of split-K slices are compile-time: the previous generic version was instruction
// bound (64-bit index arithmetic and guards around every load; ncu: 0.67 IPC/scheduler, 11 us).
//
// Per-feature reductions always run in the same order (per-thread serial over its rows, then
// the 32 warp partials in order), so the statistics of a given x are bit-identical whichever
// kernel computes them (forward finalize, plain K1 before a mirror, backward) — the property
// that makes the checkpointed step equal the non-checkpointed one.
#pragma once
#include "kernels_simt.cuh"

namespace slmk {

constexpr int kFeat = 16;   // features per CTA
constexpr int kThreads = 512;
template <int F = kFeat>
__device__ __forceinline__ float cta_feature_sum(float v, float (*red)[F + 1], int rg, int fl) {
  red[rg][fl] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) t = __fadd_rn(t, red[i][fl]);
  __syncthreads();
  return t;
}

// mean (two-pass) and rstd of this thread's feature over the whole batch
template <int R, int F = kFeat>
__device__ __forceinline__ void feature_stats(const float (&v)[R], float (*red)[F + 1], int w, int lane, float& mu,
                                              float& rstd) {
  constexpr float invB = 1.0f / (32 * R);   // exact: B is a power of two
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < R; ++i) s = __fadd_rn(s, v[i]);
  mu = __fmul_rn(cta_feature_sum<F>(s, red, w, lane), invB);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const float c = __fsub_rn(v[i], mu);
    q = __fmaf_rn(c, c, q);
  }
  const float var = __fmul_rn(cta_feature_sum<F>(q, red, w, lane), invB);
  rstd = __frcp_rn(__fsqrt_rn(__fadd_rn(var, kEps)));
}

// z[i] = sum_{s < NS} P[s][row_i][f] in the fixed order s = 0, 1, ...  (p = P + f + w*d)
template <int R, int NS>
__device__ __forceinline__ void sum_slices(const float* __restrict__ p, unsigned rowstride, unsigned pslice,
                                           float (&z)[R]) {
  constexpr int CH = NS < 1 ? 1 : NS;   // every slice's loads in flight at once (<= 64 values)
#pragma unroll
  for (int i = 0; i < R; ++i) z[i] = 0.f;
#pragma unroll
  for (int s0 = 0; s0 < NS; s0 += CH) {
    float t[CH][R];
#pragma unroll
    for (int s = 0; s < CH; ++s)
#pragma unroll
      for (int i = 0; i < R; ++i) t[s][i] = p[(s0 + s) * pslice + i * rowstride];
#pragma unroll
    for (int s = 0; s < CH; ++s)
#pragma unroll
      for (int i = 0; i < R; ++i) z[i] = __fadd_rn(z[i], t[s][i]);
  }
}

// K1 (+ forward finalize).  NS > 0: x = xin + (sum_s P[s] + bias) is stored to xout (may alias
// xin: element-wise).  Then, if gamma != null: stats[2][d] and a = ReLU(gamma xhat + beta) (T).
// F = features per CTA (16: 512 threads, 8: 256 threads — option bn_feat); the per-feature
// reduction order (32 row groups) does not depend on F.
template <class T, int R, int NS, int F = kFeat>
__global__ void __launch_bounds__(F * 32) bn_act_rk(const float* xin, const float* __restrict__ P, unsigned pslice,
                                                  const float* __restrict__ bias, float* xout,
                                                  const float* __restrict__ gamma, const float* __restrict__ beta,
                                                  int d, float* __restrict__ stats, T* __restrict__ a) {
  __shared__ float red[32][F + 1];
  pdl_wait();
  const int lane = threadIdx.x % F, w = threadIdx.x / F;   // feature in CTA, row group
  const int f = blockIdx.x * F + lane;
  const unsigned base = (unsigned)w * d + f, rs = 32u * d;
  float v[R];
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = xin[base + i * rs];
  if (NS > 0) {
    float z[R];
    sum_slices<R, NS>(P + base, rs, pslice, z);
    const float bf = bias[f];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      v[i] = __fadd_rn(v[i], __fadd_rn(z[i], bf));
      xout[base + i * rs] = v[i];
    }
  }
  pdl_launch();   // all inputs are loaded
  if (gamma == nullptr) return;
  float mu, rstd;
  feature_stats<R, F>(v, red, w, lane, mu, rstd);
  if (w == 0) {
    stats[f] = mu;
    stats[d + f] = rstd;
  }
  const float g = gamma[f], bt = beta[f];
#pragma unroll
  for (int i = 0; i < R; ++i) a[base + i * rs] = from_f32<T>(fmaxf(bn_u(bn_xhat(v[i], mu, rstd), g, bt), 0.f));
}

// Batch-norm backward of Block_l with its statistics recomputed from x_l (no separate K1):
//   da = sum_{s<NS} P[s] (split-K dX partials, fixed order),  du = da * 1[u > 0],
//   dgamma = sum_b du xhat,  dbeta = sum_b du,  dx = g + gamma rstd (du - dbeta/B - xhat dgamma/B)
//   -> dx (may alias g);  db_prev = sum_b dx;  gq = bf16(dx) (next dX / dW operand);
//   a = ReLU(u) (this layer's dW operand; the same bits as the forward's a_l).
template <class GQ, class TA, int R, int NS, int F = kFeat>
__global__ void __launch_bounds__(F * 32) bn_bwd_rk(const float* __restrict__ P, unsigned pslice,
                                                  const float* __restrict__ x, const float* __restrict__ gamma,
                                                  const float* __restrict__ beta, const float* g, float* dx, int d,
                                                  float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                  float* __restrict__ db_prev, GQ* __restrict__ gq,
                                                  TA* __restrict__ a_out) {
  __shared__ float red[32][F + 1];
  pdl_wait();
  const int lane = threadIdx.x % F, w = threadIdx.x / F;   // feature in CTA, row group
  const int f = blockIdx.x * F + lane;
  const unsigned base = (unsigned)w * d + f, rs = 32u * d;
  float xv[R], du[R];
#pragma unroll
  for (int i = 0; i < R; ++i) xv[i] = x[base + i * rs];
  sum_slices<R, NS>(P + base, rs, pslice, du);   // du <- da
  float mu, rstd;
  feature_stats<R, F>(xv, red, w, lane, mu, rstd);
  const float ga = gamma[f], bt = beta[f];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const float xh = bn_xhat(xv[i], mu, rstd);
    const float u = bn_u(xh, ga, bt);
    du[i] = u > 0.f ? du[i] : 0.f;
    a_out[base + i * rs] = from_f32<TA>(fmaxf(u, 0.f));
    s1 = __fadd_rn(s1, du[i]);
    s2 = __fmaf_rn(du[i], xh, s2);
  }
  const float S1 = cta_feature_sum<F>(s1, red, w, lane);
  const float S2 = cta_feature_sum<F>(s2, red, w, lane);
  constexpr float invB = 1.0f / (32 * R);
  const float m1 = __fmul_rn(S1, invB), m2 = __fmul_rn(S2, invB);
  const float k = __fmul_rn(ga, rstd);
  float gv[R];
#pragma unroll
  for (int i = 0; i < R; ++i) gv[i] = g[base + i * rs];
  pdl_launch();   // all inputs are loaded
  float s3 = 0.f;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const float xh = bn_xhat(xv[i], mu, rstd);
    const float v = __fadd_rn(gv[i], __fmul_rn(k, __fsub_rn(__fsub_rn(du[i], m1), __fmul_rn(xh, m2))));
    dx[base + i * rs] = v;
    gq[base + i * rs] = from_f32<GQ>(v);
    s3 = __fadd_rn(s3, v);
  }
  const float S3 = cta_feature_sum<F>(s3, red, w, lane);
  if (w != 0) return;
  dgamma[f] = S2;
  dbeta[f] = S1;
  if (db_prev) db_prev[f] = S3;
}

}  // namespace slmk

namespace slmk {

// ---------------------------------------------------------------- vectorised K1 / finalize (option bn_vec)
// CTA = 16 features x 128 row groups (512 threads): thread t holds features 4 (t % 4) .. +3 of
// rows rg, rg + 128, ... (rg = t / 4, R4 = B / 128 rows), loaded as float4 (a warp covers 8 rows
// x 64 contiguous bytes per instruction, 4x fewer memory instructions than bn_act_rk).  Per
// feature reductions in a fixed order: serial over the thread's rows, xor-shuffle tree over the
// 8 row groups of a warp (offsets 4, 8, 16), then the 16 warps' partials added in warp order.
// The forward finalize and the K1 before a mirror run both use this kernel, so their statistics
// are bit-identical; it is not bit-identical to bn_act_rk (another order).
__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 f4_shfl_tree(float4 v) {
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    float4 u;
    u.x = __shfl_xor_sync(0xffffffffu, v.x, o);
    u.y = __shfl_xor_sync(0xffffffffu, v.y, o);
    u.z = __shfl_xor_sync(0xffffffffu, v.z, o);
    u.w = __shfl_xor_sync(0xffffffffu, v.w, o);
    // fixed operand order (lower lane first) so every lane of the group computes the same bits
    const bool lo = (threadIdx.x & o) == 0;
    v = lo ? f4_add(v, u) : f4_add(u, v);
  }
  return v;
}
// sum over the CTA's 128 row groups of this thread's 4 features (result valid in every thread)
__device__ __forceinline__ float4 cta_quad_sum(float4 v, float4 (*red)[4]) {
  v = f4_shfl_tree(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane < 4) red[warp][lane] = v;
  __syncthreads();
  float4 t = red[0][lane & 3];
#pragma unroll
  for (int w = 1; w < 16; ++w) t = f4_add(t, red[w][lane & 3]);
  __syncthreads();
  return t;
}

template <int R4, int NS>
__global__ void __launch_bounds__(512) bn_act_v4(const float* xin, const float* __restrict__ P, unsigned pslice,
                                                 const float* __restrict__ bias, float* xout,
                                                 const float* __restrict__ gamma, const float* __restrict__ beta,
                                                 int d, float* __restrict__ stats, __nv_bfloat16* __restrict__ a) {
  __shared__ float4 red[16][4];
  pdl_wait();
  const int fq = threadIdx.x & 3, rg = threadIdx.x >> 2;
  const int f0 = blockIdx.x * 16 + 4 * fq;
  const unsigned base = (unsigned)rg * d + f0, rs = 128u * d;
  float4 v[R4];
#pragma unroll
  for (int i = 0; i < R4; ++i) v[i] = *reinterpret_cast<const float4*>(xin + base + i * rs);
  if (NS > 0) {
    float4 t[NS > 0 ? NS : 1][R4];
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int i = 0; i < R4; ++i) t[s][i] = *reinterpret_cast<const float4*>(P + s * pslice + base + i * rs);
    const float4 bf = *reinterpret_cast<const float4*>(bias + f0);
#pragma unroll
    for (int i = 0; i < R4; ++i) {
      float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int s = 0; s < NS; ++s) z = f4_add(z, t[s][i]);
      v[i] = f4_add(v[i], f4_add(z, bf));
      *reinterpret_cast<float4*>(xout + base + i * rs) = v[i];
    }
  }
  pdl_launch();
  if (gamma == nullptr) return;
  constexpr float invB = 1.0f / (128 * R4);
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int i = 0; i < R4; ++i) s = f4_add(s, v[i]);
  const float4 S = cta_quad_sum(s, red);
  const float4 mu = make_float4(__fmul_rn(S.x, invB), __fmul_rn(S.y, invB), __fmul_rn(S.z, invB), __fmul_rn(S.w, invB));
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int i = 0; i < R4; ++i) {
    const float cx = __fsub_rn(v[i].x, mu.x), cy = __fsub_rn(v[i].y, mu.y), cz = __fsub_rn(v[i].z, mu.z),
                cw = __fsub_rn(v[i].w, mu.w);
    q = make_float4(__fmaf_rn(cx, cx, q.x), __fmaf_rn(cy, cy, q.y), __fmaf_rn(cz, cz, q.z), __fmaf_rn(cw, cw, q.w));
  }
  const float4 Q = cta_quad_sum(q, red);
  float rstd[4];
  const float* Qp = &Q.x;
  const float* mp = &mu.x;
#pragma unroll
  for (int k = 0; k < 4; ++k) rstd[k] = __frcp_rn(__fsqrt_rn(__fadd_rn(__fmul_rn(Qp[k], invB), kEps)));
  if (rg == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      stats[f0 + k] = mp[k];
      stats[d + f0 + k] = rstd[k];
    }
  }
  const float4 g = *reinterpret_cast<const float4*>(gamma + f0), bt = *reinterpret_cast<const float4*>(beta + f0);
  const float* gp = &g.x;
  const float* bp = &bt.x;
#pragma unroll
  for (int i = 0; i < R4; ++i) {
    const float* vp = &v[i].x;
    __nv_bfloat16 o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = __float2bfloat16_rn(fmaxf(bn_u(bn_xhat(vp[k], mp[k], rstd[k]), gp[k], bp[k]), 0.f));
    uint2 pk;
    pk.x = (uint32_t)__bfloat16_as_ushort(o[0]) | ((uint32_t)__bfloat16_as_ushort(o[1]) << 16);
    pk.y = (uint32_t)__bfloat16_as_ushort(o[2]) | ((uint32_t)__bfloat16_as_ushort(o[3]) << 16);
    *reinterpret_cast<uint2*>(a + base + i * rs) = pk;
  }
}

}  // namespace slmk
