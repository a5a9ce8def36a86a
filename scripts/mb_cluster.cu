// Micro-benchmarks of the primitives the fused chain Block depends on (not part of the library):
//   1. distributed shared memory bulk copies (cp.async.bulk.shared::cluster.shared::cta) inside a
//      cluster of CS CTAs: every CTA sends CS-1 chunks to its peers (an all-to-all, the split-K
//      reduce-scatter pattern) -> bytes per SM-cycle
//   2. the same with scalar st.shared::cluster.v4 stores
//   3. a flag-based grid barrier over G persistent CTAs (red.release.gpu + ld.acquire.gpu spin)
//   4. max active clusters of size 8 / 16 with ~200 KB shared memory per CTA
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/mb_cluster.cu -o /tmp/mb_cluster
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);    \
      exit(1);                                                                           \
    }                                                                                    \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- 1. bulk all-to-all: CTA r sends chunk j (CHUNK bytes) to CTA j's receive slot r
template <int CS>
__global__ void __launch_bounds__(128, 1) k_dsmem_bulk(int chunk, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* send = sm;                        // CS chunks
  uint8_t* recv = sm + CS * chunk;           // CS slots
  __shared__ __align__(8) uint64_t bar;
  const uint32_t r = ctarank();
  for (int i = threadIdx.x; i < CS * chunk / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(send)[i] = i + r;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  csync();
  uint64_t t0 = 0, t1 = 0;
  for (int it = 0; it < reps; ++it) {
    if (it == 1) t0 = gtime();
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                   "r"((CS - 1) * chunk)
                   : "memory");
    }
    csync();   // every receiver armed its barrier
    if (threadIdx.x < CS && threadIdx.x != r) {
      const uint32_t j = threadIdx.x;
      const uint32_t dst = mapa(smem_u32(recv + r * chunk), j);
      const uint32_t rb = mapa(smem_u32(&bar), j);
      asm volatile(
          "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
          "r"(smem_u32(send + j * chunk)), "r"(chunk), "r"(rb)
          : "memory");
    }
    mbar_wait(smem_u32(&bar), it & 1);
  }
  t1 = gtime();
  csync();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = t0;
    out[blockIdx.x * 2 + 1] = t1;
  }
}

// ---- 2. scalar remote stores (v4) for comparison
template <int CS>
__global__ void __launch_bounds__(256, 1) k_dsmem_st(int chunk, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* recv = sm + CS * chunk;
  const uint32_t r = ctarank();
  csync();
  uint64_t t0 = 0;
  for (int it = 0; it < reps; ++it) {
    if (it == 1) t0 = gtime();
    for (int j = 0; j < CS; ++j) {
      if (j == (int)r) continue;
      const uint32_t dst = mapa(smem_u32(recv + r * chunk), j);
      for (int i = threadIdx.x; i < chunk / 16; i += blockDim.x) {
        asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 16 * i), "r"(i), "r"(j), "r"(it),
                     "r"(r)
                     : "memory");
      }
    }
    csync();
  }
  const uint64_t t1 = gtime();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = t0;
    out[blockIdx.x * 2 + 1] = t1;
  }
}

// ---- 3. grid barrier
__global__ void k_gridbar(unsigned* cnt, int reps, unsigned long long* out) {
  const unsigned G = gridDim.x;
  uint64_t t0 = 0;
  for (int it = 0; it < reps; ++it) {
    if (it == 1) t0 = gtime();
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      const unsigned target = (unsigned)(it + 1) * G;
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
      } while (v < target);
    }
    __syncthreads();
  }
  const uint64_t t1 = gtime();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = t0;
    out[blockIdx.x * 2 + 1] = t1;
  }
}

static double span_us(const std::vector<unsigned long long>& h, int n) {
  unsigned long long a = ~0ull, b = 0;
  for (int i = 0; i < n; ++i) {
    if (h[2 * i] < a) a = h[2 * i];
    if (h[2 * i + 1] > b) b = h[2 * i + 1];
  }
  return (b - a) / 1000.0;
}

template <int CS>
void run_bulk(int chunk, int nclusters, int reps, bool scalar) {
  const int grid = CS * nclusters;
  const int smem = 2 * CS * chunk;
  unsigned long long* d;
  CK(cudaMalloc(&d, grid * 16));
  auto k = scalar ? k_dsmem_st<CS> : k_dsmem_bulk<CS>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (CS > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(scalar ? 256 : 128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  CK(cudaOccupancyMaxActiveClusters(&ncl, k, &cfg));
  CK(cudaLaunchKernelEx(&cfg, k, chunk, reps, d));
  CK(cudaDeviceSynchronize());
  std::vector<unsigned long long> h(grid * 2);
  CK(cudaMemcpy(h.data(), d, grid * 16, cudaMemcpyDeviceToHost));
  const double us = span_us(h, grid) / (reps - 1);
  const double bytes_per_cta = (double)(CS - 1) * chunk;   // sent (= received) per CTA per rep
  printf("%s CS=%2d chunk=%6d clusters=%3d (max active %3d): %.3f us/rep, %.1f GB/s per SM out, %.1f B/clk@1.9GHz\n",
         scalar ? "dsmem st.v4 " : "dsmem bulk  ", CS, chunk, nclusters, ncl, us, bytes_per_cta / us / 1e3,
         bytes_per_cta / (us * 1e-6) / 1.9e9);
  CK(cudaFree(d));
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  printf("SMs %d\n", sms);
  for (int chunk : {4096, 8192, 16384}) {
    run_bulk<8>(chunk, 16, 50, false);
    run_bulk<8>(chunk, 1, 50, false);
    run_bulk<16>(chunk / 2, 8, 50, false);
  }
  run_bulk<8>(16384, 16, 20, true);
  run_bulk<4>(16384, 32, 50, false);
  run_bulk<2>(32768, 64, 50, false);
  // grid barrier
  for (int G : {64, 128, 148}) {
    unsigned* cnt;
    unsigned long long* d;
    CK(cudaMalloc(&cnt, 4));
    CK(cudaMemset(cnt, 0, 4));
    CK(cudaMalloc(&d, G * 16));
    const int reps = 2000;
    k_gridbar<<<G, 128>>>(cnt, reps, d);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(G * 2);
    CK(cudaMemcpy(h.data(), d, G * 16, cudaMemcpyDeviceToHost));
    printf("grid barrier G=%d: %.3f us per barrier\n", G, span_us(h, G) / (reps - 1));
    cudaFree(cnt);
    cudaFree(d);
  }
  return 0;
}
