/* slm_debug.h — test-only entry points of libslm (not part of the product API).
 *
 * slm_debug_gemm runs ONE of the three block contractions through a chosen implementation
 * so tests can compare the tcgen05 kernel against the SIMT FFMA kernel on the device:
 *   kind 0 (forward)   out[n][m] = resid[n][m] + bias[m] + sum_k A[m][k] B[n][k]
 *                       A bf16 [M][K], B bf16 [N][K], out/resid fp32 [N][M]
 *   kind 1 (dX)        out[n][m] = sum_k A[k][m] B[n][k]
 *                       A bf16 [K][M], B bf16 [N][K], out fp32 [N][M]
 *   kind 2 (dW)        out[n][m] = bf16(sum_k A[k][m] B[k][n])
 *                       A bf16 [K][M], B bf16 [K][N], out bf16 [N][M]
 * impl 0 = tcgen05/TMA (bn = N tile: 32|64|128|256; M % 128 == 0, N % bn == 0, K % 64 == 0),
 * impl 1 = SIMT, impl 2 = tcgen05 data movement only (no MMA), impl 3 = tcgen05 MMA only (no
 * TMA) — the last two are bandwidth / issue-rate probes with meaningless results —, impl 4 =
 * tcgen05 CTA pair (cta_group::2, clusters of 2 along M: M % 256 == 0, bn in {128, 256}).
 * split = split-K factor of the tcgen05 kernel (K % (64 split) == 0); with split > 1, kinds 0
 * and 1 write the fp32 partial tiles out[s][n][m] (split x N x M; the caller sums over s, kind 0
 * then ignores resid/bias).  All pointers are device pointers; asynchronous on `stream`.
 */
#ifndef SLM_DEBUG_H_
#define SLM_DEBUG_H_
#include "slm.h"
#ifdef __cplusplus
extern "C" {
#endif
slm_status slm_debug_gemm(int kind, int impl, int bn, int split, int M, int N, int K, const void* A,
                          const void* B, void* out, const float* resid, const float* bias,
                          void* stream);
/* slm_debug_block runs ONE fused Block kernel (paper_1604_06174_b200/csrc/blk_fused.cuh) for a
 * single layer with W bf16 [d][d] (row = output feature):
 *   bwd = 0 (forward Block): opnd = a_l bf16 [B][d]; out = x + (a W^T + bias)
 *           fp32 [B][d]; if gamma != NULL also a_out = bf16 ReLU(BN(out)) with (gamma, beta)
 *   bwd = 1 (gradient Block): opnd = bf16(g) [B][d], x = x_l, g = dx_{l+1} fp32;
 *           out = dx_l, a_out = bf16 ReLU(BN(x)), gq_out = bf16(dx_l), dgamma, dbeta [d],
 *           db_prev [d] (may be NULL)
 * P: exchange buffer of blk_split(B, d) * B * d fp32 (workspace).  dbg != 0: per-CTA phase stamps
 * into the slm_debug_timestamps buffer ([cta][8]).  B in {64, 128, 256}, d % 128 == 0 (B = 256:
 * d % 256 == 0).  Device pointers, asynchronous on `stream`. */
slm_status slm_debug_block(int bwd, int B, int d, const void* W, const void* opnd, const float* x, const float* g,
                           const float* bias, const float* gamma, const float* beta, float* out, void* a_out,
                           void* gq_out, float* dgamma, float* dbeta, float* db_prev, void* P, int dbg,
                           void* stream);
/* slm_debug_plan_alias makes `node` of the plan's G' write into the pool tag of `onto` (test hook:
 * a deliberately clobbering plan, for the poison option of slm_model_set_option). */
slm_status slm_debug_plan_alias(slm_plan* p, int32_t node, int32_t onto);
/* Per-CTA %globaltimer stamps (8 per CTA, phases of tc_gemm_kernel) written to dev_buf
 * (uint64, >= 8 * CTAs of the next launches); NULL switches the instrumentation off. */
slm_status slm_debug_timestamps(void* dev_buf);
/* Metadata of the GEMM launches stamped by the last step run with profile_ts (test hook):
 * per slot the kernel kind (SLM_K_*) and an executor tag (LSTM: stream * 4 + {0 fwd, 1 mirror,
 * 2 grad}); *n = number of stamped launches; cap = 0 queries n. */
slm_status slm_debug_ts_meta(const slm_model* m, int32_t* kind, int32_t* aux, int32_t cap, int32_t* n);
#ifdef __cplusplus
}
#endif
#endif
