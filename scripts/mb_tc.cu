// Micro-benchmarks for the chain Block redesign (not part of the library):
//   mma     tcgen05.mma issue rate in SS mode (operands in shared memory, no TMA) for the tile
//           shapes the Block can use: cta_group::1 M=128 x N in {64,128,256}, cta_group::2 M=256 x
//           N in {128,256}; one CTA (pair) alone and the whole chip
//   ingest  TMA operand streaming of a forward layer: W slices streamed from HBM (a different
//           layer every iteration, 512 MiB > L2) + the activation K-slice (1 MiB, L2 resident),
//           no MMA; optional multicast of the activation across a cluster along M
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/mb_tc.cu -o scripts/mb_tc
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
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
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* b, uint32_t rank) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(smem_u32(b), rank)) : "memory");
}
__device__ __forceinline__ uint64_t clk() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ================================================================ MMA issue rate
template <int N, int CG, int MC = 128>
__global__ void __launch_bounds__(128, 1) k_mma(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t done[4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = CG == 2 ? ctarank() : 0;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&done[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "n"(N));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                   "n"(N < 32 ? 32 : N));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CG == 2) csync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  uint64_t t0 = 0, t1 = 0;
  if (threadIdx.x == 0 && rank == 0) {
    constexpr uint32_t idesc = make_idesc(MC * CG, N);
    const uint32_t sa = smem_u32(sm), sb = sa + 16384;
    t0 = clk();
    for (int it = 0; it < iters; ++it) {
      const int s = it & 3;
      if (it >= 4) mbar_wait(&done[s], ((it >> 2) - 1) & 1);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = make_sdesc(sa + kk * 32, 16, 1024), bd = make_sdesc(sb + kk * 32, 16, 1024);
        if (CG == 2)
          asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(ad), "l"(bd),
                       "r"(idesc)
                       : "memory");
        else
          asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(ad), "l"(bd),
                       "r"(idesc)
                       : "memory");
      }
      if (CG == 2)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&done[s])),
            "h"((uint16_t)1)
            : "memory");
      else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&done[s]))
                     : "memory");
    }
    for (int it = iters - 4 > 0 ? iters - 4 : 0; it < iters; ++it) mbar_wait(&done[it & 3], (it >> 2) & 1);
    t1 = clk();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CG == 2) csync();
  if (warp == 0) {
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(N));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(N < 32 ? 32 : N));
  }
}

template <int N, int CG, int MC = 128>
void run_mma(int grid, int iters) {
  auto k = k_mma<N, CG, MC>;
  const int smem = 64 * 1024;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long* d;
  CK(cudaMalloc(&d, grid * 8));
  CK(cudaMemset(d, 0, grid * 8));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = CG > 1 ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, k, iters, d));
  CK(cudaDeviceSynchronize());
  std::vector<unsigned long long> h(grid);
  CK(cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost));
  double mx = 0, sum = 0;
  int cnt = 0;
  for (int i = 0; i < grid; ++i)
    if (h[i]) {
      mx = h[i] > mx ? h[i] : mx;
      sum += h[i];
      ++cnt;
    }
  const double per = (sum / cnt) / (iters * 4.0);   // cycles per K=16 MMA
  const double macs_sm = (double)MC * CG * N * 16 / per / CG;
  printf("mma CG=%d M=%3d N=%3d grid=%3d: %.1f clk per K16 MMA (max %.1f), %.0f MAC/clk/SM (peak 4096)\n", CG, MC * CG,
         N, grid, per, mx / (iters * 4.0), macs_sm);
  cudaFree(d);
}

// ================================================================ TMA ingest
// Each CTA streams, for `layers` layers, its W slice (rows m0..m0+127 of the layer, K range
// kslice) and the activation K-slice (NB rows of act, same K range): nkb K-blocks of 64 per layer.
// CS > 1: cluster along M; the activation box is split into CS row groups, CTA r loads group r
// and multicasts it to the whole cluster.
template <int NB, int CS, int STAGES>
__global__ void __launch_bounds__(128, 1) k_ingest(const __grid_constant__ CUtensorMap tmW,
                                                    const __grid_constant__ CUtensorMap tmX, int nkb, int layers,
                                                    int mtiles, int d, unsigned long long* out) {
  constexpr int A_BYTES = 128 * 64 * 2, B_BYTES = NB * 64 * 2, STAGE = A_BYTES + B_BYTES;
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const uint32_t rank = CS > 1 ? ctarank() : 0;
  const int cta = blockIdx.x;
  const int mt = cta % mtiles, ks = cta / mtiles;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (CS > 1) csync();
  const int total = layers * nkb;
  uint64_t t0 = gtime();
  if (threadIdx.x == 0) {
    for (int i = 0; i < total; ++i) {
      const int s = i % STAGES;
      if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
      const int layer = i / nkb, kb = i % nkb;
      const int k0 = (ks * nkb + kb) * 64;
      uint8_t* sa = sm + s * STAGE;
      mbar_expect_tx(&full[s], STAGE);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              smem_u32(sa)),
          "l"((uint64_t)&tmW), "r"(smem_u32(&full[s])), "r"(k0), "r"(layer * d + mt * 128)
          : "memory");
      if (CS == 1) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                smem_u32(sa + A_BYTES)),
            "l"((uint64_t)&tmX), "r"(smem_u32(&full[s])), "r"(k0), "r"(0)
            : "memory");
      } else {
        constexpr int R = NB / CS;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, "
            "{%3, %4}], [%2], %5;" ::"r"(smem_u32(sa + A_BYTES + rank * R * 128)),
            "l"((uint64_t)&tmX), "r"(smem_u32(&full[s])), "r"(k0), "r"((int)rank * R), "h"((uint16_t)((1u << CS) - 1))
            : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < total; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      if (CS == 1)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
      else
        for (int r = 0; r < CS; ++r) mbar_arrive_remote(&empty[s], r);
    }
  }
  __syncthreads();
  if (CS > 1) csync();
  const uint64_t t1 = gtime();
  if (threadIdx.x == 0) {
    out[cta * 2] = t0;
    out[cta * 2 + 1] = t1;
  }
}


// ================================================================ epilogue components
// mode 0: tcgen05.ld of the whole 128 x 256 fp32 accumulator into registers (8 warps, x32 loads)
// mode 1: + stores into a 128-byte-swizzled [b][32] smem layout (the Block kernel's slices)
// mode 2: + TMA bulk tensor stores of 3 of the 4 slices (96 KiB) to global and wait_group 0
// mode 3: TMA loads of 3 slices (96 KiB) from global into smem only
__device__ __forceinline__ int swo(int B_, int c, int b, int f32) {
  return (c * B_ + b) * 32 + ((((f32 >> 2) ^ (b & 7))) << 2) + (f32 & 3);
}
__global__ void __launch_bounds__(256, 1) k_epi(const __grid_constant__ CUtensorMap tmP, int mode, int reps,
                                                 unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  float sink = 0.f;
  const uint64_t t0 = clk();
  for (int r = 0; r < reps; ++r) {
    if (mode <= 2) {
      const int q = warp & 3, h = warp >> 2;
      float* slot = reinterpret_cast<float*>(sm + q * 32768);
      for (int c0 = h * 128; c0 < h * 128 + 128; c0 += 32) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
            "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(tmem + ((uint32_t)(q * 32) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (mode == 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) sink += __uint_as_float(v[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) slot[swo(256, 0, c0 + j, lane)] = __uint_as_float(v[j]);
        }
      }
      if (mode == 2) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
          for (int s = 1; s < 4; ++s)
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                             (uint64_t)&tmP),
                         "r"(smem_u32(sm + s * 32768)), "r"(0), "r"((int)(blockIdx.x * 4 + s) * 256)
                         : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
      }
      __syncthreads();
    } else {
      if (threadIdx.x == 0) {
        mbar_expect_tx(&bar, 3 * 32768);
        for (int s = 1; s < 4; ++s)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
              "[%2];" ::"r"(smem_u32(sm + s * 32768)),
              "l"((uint64_t)&tmP), "r"(smem_u32(&bar)), "r"(0), "r"((int)(blockIdx.x * 4 + s) * 256)
              : "memory");
      }
      mbar_wait(&bar, r & 1);
      __syncthreads();
    }
  }
  const uint64_t t1 = clk();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps + (sink == 12345.f);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}


// store-path variants for the 96 KiB partial exchange (per CTA), completion included:
// mode 0: TMA bulk tensor store (3 boxes of 32 KiB), wait_group 0
// mode 1: st.global.v4 from registers (256 threads, 24 x 16 B each), then fence.acq_rel.gpu
// mode 2: st.global.b32 coalesced (a warp writes 128 B per instruction), then fence.acq_rel.gpu
// mode 3: 1-D bulk copies cp.async.bulk.global.shared::cta (3 x 32 KiB), wait_group 0
__global__ void __launch_bounds__(256, 1) k_store(const __grid_constant__ CUtensorMap tmP, float* P, int mode, int reps,
                                                   unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  float* dst = P + (size_t)blockIdx.x * 4 * 8192;
  const uint64_t t0 = clk();
  for (int r = 0; r < reps; ++r) {
    if (mode == 0 || mode == 3) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int s = 1; s < 4; ++s) {
          if (mode == 0)
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                             (uint64_t)&tmP),
                         "r"(smem_u32(sm + s * 32768)), "r"(0), "r"((int)(blockIdx.x * 4 + s) * 256)
                         : "memory");
          else
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + s * 8192),
                         "r"(smem_u32(sm + s * 32768)), "r"(32768)
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
      __syncthreads();
    } else if (mode == 1) {
      float4 v = make_float4(r, 1, 2, 3);
      float4* d4 = reinterpret_cast<float4*>(dst + 8192);
      for (int i = threadIdx.x; i < 3 * 8192 / 4; i += 256) d4[i] = v;
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      __syncthreads();
    } else {
      for (int i = threadIdx.x; i < 3 * 8192; i += 256) dst[8192 + i] = (float)r;
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      __syncthreads();
    }
  }
  const uint64_t t1 = clk();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn enc() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    fn = (EncodeTiledFn)p;
  }
  return fn;
}
static CUtensorMap map2d(void* base, uint64_t inner, uint64_t rows, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

template <int NB, int CS, int STAGES>
void run_ingest(void* W, void* X, int d, int nlay, int mtiles, int ksplit, const char* tag) {
  const int nkb = d / 64 / ksplit;
  const int grid = mtiles * ksplit;
  CUtensorMap tw = map2d(W, d, (uint64_t)nlay * d, 128), tx = map2d(X, d, 256, NB / CS);
  auto k = k_ingest<NB, CS, STAGES>;
  const int smem = STAGES * (128 + NB) * 128 + 1024;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  unsigned long long* dd;
  CK(cudaMalloc(&dd, grid * 16));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = CS > 1 ? 1 : 0;
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaLaunchKernelEx(&cfg, k, tw, tx, nkb, nlay, mtiles, d, dd));
    CK(cudaDeviceSynchronize());
  }
  std::vector<unsigned long long> h(grid * 2);
  CK(cudaMemcpy(h.data(), dd, grid * 16, cudaMemcpyDeviceToHost));
  unsigned long long a = ~0ull, b = 0;
  for (int i = 0; i < grid; ++i) {
    a = h[2 * i] < a ? h[2 * i] : a;
    b = h[2 * i + 1] > b ? h[2 * i + 1] : b;
  }
  const double us = (b - a) / 1000.0 / nlay;
  const double per_cta = (double)nkb * (128 + NB) * 128;
  const double wbytes = (double)d * d * 2, xbytes = (double)mtiles / CS * ksplit * nkb * 64 * NB * 2;
  printf("ingest %-28s grid=%3d NB=%3d CS=%d st=%d: %.3f us/layer  per-SM %.0f KiB -> %.1f B/clk@1.9GHz; "
         "W %.2f TB/s, L2 reads of act %.1f MiB\n",
         tag, grid, NB, CS, STAGES, us, per_cta / 1024, per_cta / (us * 1e-6) / 1.9e9, wbytes / (us * 1e-6) / 1e12,
         xbytes / (1 << 20));
  cudaFree(dd);
}

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  printf("SMs %d\n", sms);
  const int iters = 2048;
  run_mma<256, 1, 64>(1, iters);
  run_mma<256, 2, 64>(2, iters);
  run_mma<128, 2, 64>(2, iters);
  run_mma<256, 1, 64>(148, iters);
  run_mma<256, 2, 64>(148, iters);
  run_mma<64, 1>(1, iters);
  run_mma<128, 1>(1, iters);
  run_mma<256, 1>(1, iters);
  run_mma<128, 2>(2, iters);
  run_mma<256, 2>(2, iters);
  run_mma<128, 1>(148, iters);
  run_mma<256, 1>(148, iters);
  run_mma<256, 2>(148, iters);


  // epilogue components at 64 CTAs (the Block kernel's grid at C2)
  {
    float* Pb;
    const int grid = 64;
    CK(cudaMalloc(&Pb, (size_t)grid * 4 * 256 * 32 * 4));
    CUtensorMap tp;
    cuuint64_t dims[2] = {32, (cuuint64_t)grid * 4 * 256};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {32, 256};
    cuuint32_t es[2] = {1, 1};
    CUresult rr = enc()(&tp, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Pb, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rr != CUDA_SUCCESS) printf("encode P failed %d\n", (int)rr);
    CK(cudaFuncSetAttribute(k_epi, cudaFuncAttributeMaxDynamicSharedMemorySize, 129 * 1024));
    unsigned long long* dd;
    CK(cudaMalloc(&dd, grid * 8));
    const char* names[4] = {"TMEM ld 128 KiB (8 warps)", "+ STS swizzled", "+ TMA store 96 KiB + wait", "TMA load 96 KiB"};
    for (int mode = 0; mode < 4; ++mode) {
      k_epi<<<grid, 256, 129 * 1024>>>(tp, mode, 20, dd);
      CK(cudaDeviceSynchronize());
      std::vector<unsigned long long> h(grid);
      CK(cudaMemcpy(h.data(), dd, grid * 8, cudaMemcpyDeviceToHost));
      double sum = 0;
      for (auto v : h) sum += v;
      printf("epilogue %-28s: %.0f clk per rep (mean over %d CTAs) = %.2f us @1.9GHz\n", names[mode], sum / grid, grid,
             sum / grid / 1900.0);
    }
    CK(cudaFuncSetAttribute(k_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 129 * 1024));
    const char* sn[4] = {"TMA tensor store 3x32KiB", "st.global.v4 + fence", "st.global.b32 + fence", "bulk 1-D store 3x32KiB"};
    for (int g : {64, 16})
      for (int mode = 0; mode < 4; ++mode) {
        k_store<<<g, 256, 129 * 1024>>>(tp, Pb, mode, 20, dd);
        CK(cudaDeviceSynchronize());
        std::vector<unsigned long long> h(g);
        CK(cudaMemcpy(h.data(), dd, g * 8, cudaMemcpyDeviceToHost));
        double sum = 0;
        for (auto v : h) sum += v;
        printf("store %-26s grid %2d: %.0f clk per 96 KiB = %.2f us\n", sn[mode], g, sum / g, sum / g / 1900.0);
      }

  }
  const int d = 2048, nlay = 64;
  void *W, *X;
  CK(cudaMalloc(&W, (size_t)nlay * d * d * 2));
  CK(cudaMalloc(&X, (size_t)256 * d * 2));
  CK(cudaMemset(W, 0, (size_t)nlay * d * d * 2));
  CK(cudaMemset(X, 0, (size_t)256 * d * 2));
  // forward-layer operand streams (W from HBM, act from L2)
  run_ingest<128, 1, 6>(W, X, d, nlay, 16, 2, "r1 default 16x2(Ntile128)");
  run_ingest<256, 1, 4>(W, X, d, nlay, 16, 8, "16 mt x 8 ks, N=256");
  run_ingest<256, 2, 4>(W, X, d, nlay, 16, 8, "16 mt x 8 ks, N=256, MC2");
  run_ingest<256, 4, 4>(W, X, d, nlay, 16, 8, "16 mt x 8 ks, N=256, MC4");
  run_ingest<256, 8, 4>(W, X, d, nlay, 16, 8, "16 mt x 8 ks, N=256, MC8");
  run_ingest<128, 1, 6>(W, X, d, nlay, 16, 8, "16 mt x 8 ks, N=128 (pair half)");
  run_ingest<128, 2, 6>(W, X, d, nlay, 16, 8, "16 mt x 8 ks, N=128, MC2");
  run_ingest<128, 4, 6>(W, X, d, nlay, 16, 8, "16 mt x 8 ks, N=128, MC4");
  run_ingest<128, 1, 6>(W, X, d, nlay, 16, 4, "16 mt x 4 ks, N=128");
  run_ingest<256, 1, 4>(W, X, d, nlay, 16, 4, "16 mt x 4 ks, N=256");
  run_ingest<256, 4, 4>(W, X, d, nlay, 16, 4, "16 mt x 4 ks, N=256, MC4");
  return 0;
}
