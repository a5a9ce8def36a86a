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
 * impl 1 = SIMT.  All pointers are device pointers; asynchronous on `stream`.
 */
#ifndef SLM_DEBUG_H_
#define SLM_DEBUG_H_
#include "slm.h"
#ifdef __cplusplus
extern "C" {
#endif
slm_status slm_debug_gemm(int kind, int impl, int bn, int M, int N, int K, const void* A,
                          const void* B, void* out, const float* resid, const float* bias,
                          void* stream);
#ifdef __cplusplus
}
#endif
#endif
