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
