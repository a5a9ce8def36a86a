// Empirical TMEM layout of a tcgen05.mma kind::f16 accumulator with M = 64 (cta_group::1):
// A[i][0] = i + 1, B[j][0] = 1 (all other K zero) => D[i][j] = i + 1; every TMEM lane of the 4
// sub-partitions is read back (32x32b.x1, column 0 and column 8) to see where row i lives.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
template <int M>
__global__ void k(float* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __nv_bfloat16* A = reinterpret_cast<__nv_bfloat16*>(sm);          // 128 rows x 64 K (SW128)
  __nv_bfloat16* Bm = reinterpret_cast<__nv_bfloat16*>(sm + 16384);  // 256 rows x 64 K
  for (int i = threadIdx.x; i < (16384 + 32768) / 2; i += blockDim.x) reinterpret_cast<__nv_bfloat16*>(sm)[i] = __float2bfloat16(0.f);
  __syncthreads();
  if (threadIdx.x < M) {   // element (i, 0): chunk 0 of row i lands at chunk (i % 8)
    const int i = threadIdx.x;
    A[((i / 8) * 1024 + (i % 8) * 128 + (i % 8) * 16) / 2] = __float2bfloat16((float)(i + 1));
  }
  for (int j = threadIdx.x; j < 256; j += blockDim.x) Bm[((j / 8) * 1024 + (j % 8) * 128 + (j % 8) * 16) / 2] = __float2bfloat16(1.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint64_t ad = make_sdesc(smem_u32(A), 16, 1024), bd = make_sdesc(smem_u32(Bm), 16, 1024);
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = threadIdx.x / 32;
  for (int c : {0, 8, 255}) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    out[(c == 0 ? 0 : (c == 8 ? 1 : 2)) * 128 + threadIdx.x] = __uint_as_float(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}
int main() {
  float* d;
  cudaMalloc(&d, 3 * 128 * 4);
  cudaFuncSetAttribute(k<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  cudaFuncSetAttribute(k<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  float h[3 * 128];
  for (int M : {128, 64}) {
    cudaMemset(d, 0, 3 * 128 * 4);
    if (M == 64) k<64><<<1, 128, 60 * 1024>>>(d); else k<128><<<1, 128, 60 * 1024>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("M=%d (%s): lane -> D value at column 0 / 8 / 255 (row + 1; 0 = empty)\n", M, cudaGetErrorString(e));
    for (int l = 0; l < 128; ++l) printf("%3d:%g/%g/%g%s", l, h[l], h[128 + l], h[256 + l], (l % 8 == 7) ? "\n" : "  ");
  }
  return 0;
}
