// Stand-alone calibration of per-kernel overheads on B200 (not part of the library):
// empty kernel, 2 MiB copy, and the BN kernels of the fused lowering, each timed as a CUDA
// graph of back-to-back launches (with and without programmatic dependent launch).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "bn_kernels.cuh"

using namespace slmk;

__global__ void empty_kernel() {}
__global__ void empty_pdl_kernel() {
  pdl_wait();
  pdl_launch();
}
__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, int n) {
  pdl_wait();
  pdl_launch();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = a[i];
}

template <class F>
float time_graph(F launch, int reps) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int i = 0; i < 3; ++i) launch(s);
  cudaStreamSynchronize(s);
  cudaGraph_t g;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < reps; ++i) launch(s);
  cudaStreamEndCapture(s, &g);
  cudaGraphExec_t ge;
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < 5; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms * 1000.f / (5 * reps);
}

template <class... KArgs, class... Args>
void lk(void (*k)(KArgs...), dim3 g, dim3 b, cudaStream_t s, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

int main() {
  const int B = 256, d = 2048, reps = 200;
  float *x, *x2, *P, *stats, *gam, *bet, *bias;
  __nv_bfloat16* a;
  cudaMalloc(&x, B * d * 4);
  cudaMalloc(&x2, B * d * 4);
  cudaMalloc(&P, 8 * B * d * 4);
  cudaMalloc(&stats, 2 * d * 4);
  cudaMalloc(&gam, d * 4);
  cudaMalloc(&bet, d * 4);
  cudaMalloc(&bias, d * 4);
  cudaMalloc(&a, B * d * 2);
  cudaMemset(x, 0, B * d * 4);
  cudaMemset(P, 0, 8 * B * d * 4);
  cudaMemset(gam, 0, d * 4);
  for (int pdl = 0; pdl < 2; ++pdl) {
    printf("pdl=%d\n", pdl);
    printf("  empty            %7.2f us\n", time_graph([&](cudaStream_t s) { lk(empty_pdl_kernel, dim3(1), dim3(32), s, pdl); }, reps));
    printf("  empty 148x1024   %7.2f us\n", time_graph([&](cudaStream_t s) { lk(empty_pdl_kernel, dim3(148), dim3(1024), s, pdl); }, reps));
    for (int nb : {64, 148, 296, 592}) {
      int n4 = B * d / 4;
      printf("  copy 2MiB g=%3d  %7.2f us\n", nb,
             time_graph([&](cudaStream_t s) { lk(copy_kernel, dim3(nb), dim3(512), s, pdl, (const float4*)x, (float4*)x2, n4); }, reps));
    }
    printf("  bn_act_rk NS=0   %7.2f us\n",
           time_graph([&](cudaStream_t s) {
             lk(bn_act_rk<__nv_bfloat16, 8, 0>, dim3(d / kFeat), dim3(kThreads), s, pdl, (const float*)x, (const float*)P,
                (unsigned)(B * d), (const float*)bias, x2, (const float*)gam, (const float*)bet, d, stats, a);
           }, reps));
    printf("  bn_act_rk NS=8   %7.2f us\n",
           time_graph([&](cudaStream_t s) {
             lk(bn_act_rk<__nv_bfloat16, 8, 8>, dim3(d / kFeat), dim3(kThreads), s, pdl, (const float*)x, (const float*)P,
                (unsigned)(B * d), (const float*)bias, x2, (const float*)gam, (const float*)bet, d, stats, a);
           }, reps));
  }
  return 0;
}
