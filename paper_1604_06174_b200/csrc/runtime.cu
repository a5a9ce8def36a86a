// Device runtime of the chain training step on sm_100a (slm_model_*, slm_step*, slm_comm_*).
//
// slm_step executes V' (Alg. 2's order) node by node, each node writing
// into the pool slot of its temporal tag (Fig. 2):
//   forward / mirror Block_l   K1 bn_act(x_l) -> a_l ; GEMM fwd x_{l+1} = x_l + a_l W_l^T + b_l
//   SoftmaxCE (loss)           ce_fwd + ce_reduce
//   grad SoftmaxCE             ce_bwd -> dx_n (+ bf16 copy) ; colsum -> db_{n-1}
//   grad Block_l               K1 bn_act(x_l) ; GEMM dX da = g W_l ; GEMM dW = g^T a_l ;
//                              bn_bwd -> dx_l (+ bf16 copy), dgamma_l, dbeta_l, db_{l-1}
// Re-computation is just the mirror nodes of V': the same
// kernels with the same launch configuration, so recomputed values are bit-identical.
// The whole step is captured once into a CUDA graph per (plan, model, buffers) and
// replayed (no host work per node after the first call).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "kernels_simt.cuh"
#include "slm_internal.h"
#include "tc_gemm.cuh"

using namespace slm;

namespace {

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                \
      return SLM_E_CUDA;                                                            \
    }                                                                               \
  } while (0)

// ---------------------------------------------------------------- NCCL (loaded at run time)
typedef struct { char internal[128]; } nccl_uid;
typedef void* nccl_comm_t;
struct Nccl {
  void* h = nullptr;
  int (*GetUniqueId)(nccl_uid*) = nullptr;
  int (*CommInitRank)(nccl_comm_t*, int, nccl_uid, int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*CommDestroy)(nccl_comm_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool load() {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
    AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
    CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
    GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
    GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
    GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
    return GetUniqueId && CommInitRank && AllReduce && CommDestroy && GroupStart && GroupEnd;
  }
};
Nccl g_nccl;
enum { NCCL_FLOAT32 = 7, NCCL_BF16 = 9, NCCL_SUM = 0 };

// ---------------------------------------------------------------- tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// bf16 2-D tensor [rows][inner] (inner contiguous), box {64, box_rows}, 128-byte swizzle.
slm_status make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows, uint32_t box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SLM_E_CUDA;
  }
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return SLM_E_CUDA;
  }
  return SLM_OK;
}

// ---------------------------------------------------------------- GEMM launchers
enum GemmKind { G_FWD = 0, G_DX = 1, G_DW = 2 };

// Every kernel of the step is launched with programmatic stream serialization (PDL) when
// `pdl` is set: it may start while its predecessor drains and synchronises on it with
// griddepcontrol.wait before touching dependent data.
template <class... KArgs, class... Args>
cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                     Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

template <int BN, bool AMN, bool BMN, bool PRE, class Epi>
slm_status launch_tc(const CUtensorMap& a, const CUtensorMap& b, int M, int N, int K, int a_row0,
                     int b_row0, Epi epi, cudaStream_t st, bool pdl) {
  using C = slmk::TcCfg<BN, AMN, BMN>;
  auto kern = slmk::tc_gemm_kernel<BN, AMN, BMN, PRE, Epi>;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  CK(launch_k(kern, dim3(M / 128, N / BN), dim3(128), C::SMEM, st, pdl, a, b, K, a_row0, b_row0, epi));
  return SLM_OK;
}

template <class Epi, bool AMN, bool BMN, bool PRE>
slm_status launch_tc_bn(int bn, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int K,
                        int a_row0, int b_row0, Epi epi, cudaStream_t st, bool pdl) {
  switch (bn) {
    case 32: if (!BMN) return launch_tc<32, AMN, BMN, PRE>(a, b, M, N, K, a_row0, b_row0, epi, st, pdl); break;
    case 64: return launch_tc<64, AMN, BMN, PRE>(a, b, M, N, K, a_row0, b_row0, epi, st, pdl);
    case 128: return launch_tc<128, AMN, BMN, PRE>(a, b, M, N, K, a_row0, b_row0, epi, st, pdl);
    case 256: return launch_tc<256, AMN, BMN, PRE>(a, b, M, N, K, a_row0, b_row0, epi, st, pdl);
  }
  set_error("unsupported GEMM N tile " + std::to_string(bn));
  return SLM_E_UNSUPPORTED;
}

}  // namespace

// ====================================================================== model
struct slm_comm {
  nccl_comm_t comm = nullptr;
  int rank = 0, world = 1;
  int64_t bucket_bytes = 256ll << 20;
  cudaStream_t stream = nullptr;
  std::vector<cudaEvent_t> events;
};

struct Op {
  int type;      // 0 fwd block, 1 ce fwd, 2 ce bwd, 3 bwd block
  int layer;
  int in_tag;    // fwd: x_l ; ce: x_n ; bwd block: g = dx_{l+1}
  int aux_tag;   // bwd block: x_l
  int out_tag;
};

struct GraphKey {
  const void* plan;
  const void *x0, *labels, *pool, *ws, *loss;
  cudaStream_t stream;
  const void* comm;
  bool operator<(const GraphKey& o) const {
    return std::tie(plan, x0, labels, pool, ws, loss, stream, comm) <
           std::tie(o.plan, o.x0, o.labels, o.pool, o.ws, o.loss, o.stream, o.comm);
  }
};

struct slm_model {
  slm_chain_desc d{};
  int kind = SLM_MODEL_CHAIN;
  int use_graph = 1;
  int gemm_impl = 0;      // 0 tcgen05 (bf16), 1 SIMT
  int pdl = 1;            // programmatic dependent launch between the step's kernels
  int bn_fwd = 64, bn_dx = 64, bn_dw = 128;
  // tensor maps bound to the current workspace / weights
  const void* maps_ws = nullptr;
  CUtensorMap mW_K, mW_MN, mA_K, mA_MN, mG_K[2], mG_MN[2];
  std::map<GraphKey, cudaGraphExec_t> graphs;
  int64_t last_launches = 0;
  // profile_events: (start, end, kind) per kernel, read by slm_model_kernel_times
  int profile = 0;
  struct EvPair {
    cudaEvent_t a, b;
    int kind;
  };
  std::vector<EvPair> ev_live;
  std::vector<cudaEvent_t> ev_free;
  double acc_ms[SLM_K_COUNT] = {};
  int64_t acc_cnt[SLM_K_COUNT] = {};
  cudaEvent_t get_event() {
    if (!ev_free.empty()) {
      cudaEvent_t e = ev_free.back();
      ev_free.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  ~slm_model() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    for (auto& p : ev_live) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    for (auto e : ev_free) cudaEventDestroy(e);
  }
};

namespace {

struct WsLayout {
  size_t a, stats, gq0, gq1, da, rowloss, total;
};
WsLayout ws_layout(const slm_model& m) {
  const size_t B = m.d.batch, d = m.d.width;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  WsLayout L{};
  size_t off = 0;
  L.a = off;
  off += al(B * d * 4);
  L.stats = off;
  off += al(2 * d * 4);
  L.gq0 = off;
  off += al(B * d * 2);
  L.gq1 = off;
  off += al(B * d * 2);
  L.da = off;
  off += al(B * d * 4);
  L.rowloss = off;
  off += al(B * 4);
  L.total = off;
  return L;
}

bool tc_ok(const slm_model& m) {
  const int B = m.d.batch, d = m.d.width;
  return m.d.dtype == SLM_BF16 && m.gemm_impl == 0 && d % 128 == 0 && B % 64 == 0 && B <= 4096 &&
         B % m.bn_fwd == 0 && B % m.bn_dx == 0 && d % m.bn_dw == 0;
}

slm_status lower(const slm_plan* p, std::vector<Op>* ops) {
  ops->clear();
  const int n = p->dims[0];
  for (int v : p->order) {
    const int kind = p->kind[v], op = p->op[v], orig = p->orig[v];
    const int* pr = &p->preds[p->pred_ptr[v]];
    const int npr = p->pred_ptr[v + 1] - p->pred_ptr[v];
    if (op == SLM_OP_INPUT) continue;
    if (kind != SLM_KIND_GRAD) {
      if (op == SLM_OP_BLOCK)
        ops->push_back({0, orig - 1, p->node_tag[pr[0]], -1, p->node_tag[v]});
      else if (op == SLM_OP_SOFTMAX_CE)
        ops->push_back({1, n, p->node_tag[pr[0]], -1, p->node_tag[v]});
      else {
        set_error("unsupported op in chain plan");
        return SLM_E_UNSUPPORTED;
      }
    } else {
      if (op == SLM_OP_SOFTMAX_CE) {
        if (npr != 1) return SLM_E_UNSUPPORTED;
        ops->push_back({2, n, p->node_tag[pr[0]], -1, p->node_tag[v]});
      } else if (op == SLM_OP_BLOCK) {
        if (npr != 2) return SLM_E_UNSUPPORTED;
        ops->push_back({3, orig - 1, p->node_tag[pr[0]], p->node_tag[pr[1]], p->node_tag[v]});
      } else {
        set_error("unsupported gradient op in chain plan");
        return SLM_E_UNSUPPORTED;
      }
    }
  }
  return SLM_OK;
}

slm_status bind_maps(slm_model& m, void* ws) {
  if (m.maps_ws == ws) return SLM_OK;
  const uint64_t B = m.d.batch, d = m.d.width, n = m.d.n_layers;
  WsLayout L = ws_layout(m);
  uint8_t* w = (uint8_t*)ws;
  slm_status st;
  if ((st = make_map(&m.mW_K, m.d.W, d, n * d, 128)) != SLM_OK) return st;
  if ((st = make_map(&m.mW_MN, m.d.W, d, n * d, 64)) != SLM_OK) return st;
  if ((st = make_map(&m.mA_K, w + L.a, d, B, m.bn_fwd)) != SLM_OK) return st;
  if ((st = make_map(&m.mA_MN, w + L.a, d, B, 64)) != SLM_OK) return st;
  for (int i = 0; i < 2; ++i) {
    uint8_t* g = w + (i ? L.gq1 : L.gq0);
    if ((st = make_map(&m.mG_K[i], g, d, B, m.bn_dx)) != SLM_OK) return st;
    if ((st = make_map(&m.mG_MN[i], g, d, B, 64)) != SLM_OK) return st;
  }
  m.maps_ws = ws;
  return SLM_OK;
}

// Enqueue the whole step on `st`; counts kernel launches into *launches.
slm_status enqueue(const slm_plan* p, slm_model& m, const void* x0, const int32_t* labels, void* pool,
                   void* ws, float* loss, cudaStream_t st, slm_comm* comm, int64_t* launches) {
  using namespace slmk;
  const int B = m.d.batch, d = m.d.width, n = m.d.n_layers;
  const bool bf16 = m.d.dtype == SLM_BF16;
  const bool tc = tc_ok(m);
  const int Bg = m.d.batch_global > 0 ? m.d.batch_global : B;
  const float inv_bg = 1.0f / (float)Bg;
  WsLayout L = ws_layout(m);
  uint8_t* w = (uint8_t*)ws;
  float* stats = (float*)(w + L.stats);
  void* abuf = w + L.a;
  __nv_bfloat16* gq[2] = {(__nv_bfloat16*)(w + L.gq0), (__nv_bfloat16*)(w + L.gq1)};
  float* da = (float*)(w + L.da);
  float* rowloss = (float*)(w + L.rowloss);

  std::vector<Op> ops;
  slm_status s = lower(p, &ops);
  if (s != SLM_OK) return s;
  if (tc && (s = bind_maps(m, ws)) != SLM_OK) return s;

  // tag -> pointer: pool offset, or the caller buffer bound to an external tag
  std::vector<void*> tp(p->tag_size.size(), nullptr);
  for (size_t t = 0; t < tp.size(); ++t)
    if (p->tag_offset[t] >= 0) tp[t] = (uint8_t*)pool + p->tag_offset[t];
  for (int v = 0; v < p->n_fwd; ++v) {
    int t = p->node_tag[v];
    if (t < 0 || p->tag_offset[t] >= 0) continue;
    if (p->op[v] == SLM_OP_INPUT) tp[t] = const_cast<void*>(x0);
    else if (p->op[v] == SLM_OP_SOFTMAX_CE) tp[t] = loss;
  }
  auto X = [&](int tag) { return (float*)tp[tag]; };

  const size_t Wl = (size_t)d * d;
  const float* bvec = m.d.b;
  const float* gam = m.d.gamma;
  const float* bet = m.d.beta;
  const dim3 colgrid((d + 31) / 32), blk(256);
  int64_t nl = 0;
  int gpar = 0;  // which gq buffer holds the current upstream gradient copy
  // data-parallel buckets: layers [lo, hi] are reduced after layer lo's backward
  int bucket_hi = n - 1;
  const int64_t per_layer = (int64_t)Wl * (bf16 ? 2 : 4);
  const int bucket_layers =
      comm ? (int)std::max<int64_t>(1, std::min<int64_t>(n, comm->bucket_bytes / per_layer)) : 0;
  int ev_i = 0;

  const bool pdl = m.pdl != 0;
  auto simt_gemm = [&](auto* A, long sAm, long sAk, auto* Bp, long sBn, long sBk, auto* out, long ldo,
                       int M, int N, int K, const float* resid, const float* bias, bool resid_epi) -> cudaError_t {
    dim3 grid((N + 63) / 64, (M + 63) / 64);
    using TA = std::remove_const_t<std::remove_pointer_t<decltype(A)>>;
    using TB = std::remove_const_t<std::remove_pointer_t<decltype(Bp)>>;
    using TO = std::remove_pointer_t<decltype(out)>;
    if (resid_epi)
      return launch_k(simt_gemm_kernel<TA, TB, TO, EPI_RESID>, grid, dim3(256), 0, st, pdl, M, N, K, A, sAm, sAk,
                      Bp, sBn, sBk, out, ldo, resid, bias);
    return launch_k(simt_gemm_kernel<TA, TB, TO, EPI_STORE>, grid, dim3(256), 0, st, pdl, M, N, K, A, sAm, sAk, Bp,
                    sBn, sBk, out, ldo, resid, bias);
  };
  // batch-norm kernels: register-resident variant when the batch fits (B <= 256)
  const bool rk = B <= 256;
  const dim3 rkblk(1024);
  auto bn_act = [&](const float* xin, int l) -> cudaError_t {
    const float* ga = gam + (size_t)l * d;
    const float* be = bet + (size_t)l * d;
    if (bf16)
      return rk ? launch_k(bn_act_rk<__nv_bfloat16, 8>, colgrid, rkblk, 0, st, pdl, xin, ga, be, B, d, stats,
                           (__nv_bfloat16*)abuf)
                : launch_k(bn_act_kernel<__nv_bfloat16>, colgrid, blk, 0, st, pdl, xin, ga, be, B, d, stats,
                           (__nv_bfloat16*)abuf);
    return rk ? launch_k(bn_act_rk<float, 8>, colgrid, rkblk, 0, st, pdl, xin, ga, be, B, d, stats, (float*)abuf)
              : launch_k(bn_act_kernel<float>, colgrid, blk, 0, st, pdl, xin, ga, be, B, d, stats, (float*)abuf);
  };

  // optional per-kernel CUDA events (profile_events), recorded on the launching stream
  cudaEvent_t ev0 = nullptr;
  auto pbeg = [&]() {
    if (m.profile) {
      ev0 = m.get_event();
      cudaEventRecord(ev0, st);
    }
  };
  auto pend = [&](int kind) {
    if (m.profile) {
      cudaEvent_t e1 = m.get_event();
      cudaEventRecord(e1, st);
      m.ev_live.push_back({ev0, e1, kind});
    }
  };

  for (const Op& o : ops) {
    const int l = o.layer;
    if (o.type == 0 || o.type == 3) {
      // K1: statistics + activation operand of x_l (forward input, or x_l in the backward)
      pbeg();
      CK(bn_act(X(o.type == 0 ? o.in_tag : o.aux_tag), l));
      pend(SLM_K_BN_ACT);
      ++nl;
    }
    if (o.type == 0) {
      const float* xin = X(o.in_tag);
      float* xout = X(o.out_tag);
      pbeg();
      if (tc) {
        slmk::EpiResid epi{xout, xin, bvec + (size_t)l * d, d};
        if ((s = launch_tc_bn<slmk::EpiResid, false, false, true>(m.bn_fwd, m.mW_K, m.mA_K, d, B, d, l * d, 0, epi,
                                                                  st, pdl)) != SLM_OK)
          return s;
      } else if (bf16) {
        CK(simt_gemm((const __nv_bfloat16*)abuf, (long)d, 1L, (const __nv_bfloat16*)m.d.W + l * Wl, (long)d, 1L,
                     xout, (long)d, B, d, d, xin, bvec + (size_t)l * d, true));
      } else {
        CK(simt_gemm((const float*)abuf, (long)d, 1L, (const float*)m.d.W + l * Wl, (long)d, 1L, xout, (long)d,
                     B, d, d, xin, bvec + (size_t)l * d, true));
      }
      pend(SLM_K_GEMM_FWD);
      ++nl;
    } else if (o.type == 1) {
      pbeg();
      CK(launch_k(ce_fwd_kernel, dim3(B), blk, 0, st, pdl, (const float*)X(o.in_tag), labels, d, rowloss));
      CK(launch_k(ce_reduce_kernel, dim3(1), blk, 0, st, pdl, (const float*)rowloss, B, inv_bg, X(o.out_tag)));
      pend(SLM_K_CE);
      nl += 2;
    } else if (o.type == 2) {
      float* dxn = X(o.out_tag);
      pbeg();
      if (bf16)
        CK(launch_k(ce_bwd_kernel<__nv_bfloat16>, dim3(B), blk, 0, st, pdl, (const float*)X(o.in_tag), labels, d,
                    inv_bg, dxn, gq[0]));
      else
        CK(launch_k(ce_bwd_kernel<float>, dim3(B), blk, 0, st, pdl, (const float*)X(o.in_tag), labels, d, inv_bg,
                    dxn, (float*)nullptr));
      CK(launch_k(colsum_kernel, colgrid, blk, 0, st, pdl, (const float*)dxn, B, d, m.d.db + (size_t)(n - 1) * d));
      pend(SLM_K_CE);
      gpar = 0;
      nl += 2;
    } else {  // type 3: backward of Block_l
      const float* g = X(o.in_tag);
      const float* xl = X(o.aux_tag);
      float* dxl = X(o.out_tag);
      if (tc) {
        // da[b][f_in] = sum_k g[b][k] W_l[k][f_in]
        slmk::EpiStoreF32 e1{da, d};
        pbeg();
        if ((s = launch_tc_bn<slmk::EpiStoreF32, true, false, true>(m.bn_dx, m.mW_MN, m.mG_K[gpar], d, B, d, l * d,
                                                                    0, e1, st, pdl)) != SLM_OK)
          return s;
        pend(SLM_K_GEMM_DX);
        // dW_l[f_out][f_in] = sum_b g[b][f_out] a[b][f_in]
        slmk::EpiStoreBF16 e2{(__nv_bfloat16*)m.d.dW + l * Wl, d};
        pbeg();
        if ((s = launch_tc_bn<slmk::EpiStoreBF16, true, true, false>(m.bn_dw, m.mA_MN, m.mG_MN[gpar], d, d, B, 0,
                                                                     0, e2, st, pdl)) != SLM_OK)
          return s;
        pend(SLM_K_GEMM_DW);
      } else if (bf16) {
        const __nv_bfloat16* gqp = gq[gpar];
        pbeg();
        CK(simt_gemm(gqp, (long)d, 1L, (const __nv_bfloat16*)m.d.W + l * Wl, 1L, (long)d, da, (long)d, B, d, d,
                     (const float*)nullptr, (const float*)nullptr, false));
        pend(SLM_K_GEMM_DX);
        pbeg();
        CK(simt_gemm(gqp, 1L, (long)d, (const __nv_bfloat16*)abuf, 1L, (long)d,
                     (__nv_bfloat16*)m.d.dW + l * Wl, (long)d, d, d, B, (const float*)nullptr,
                     (const float*)nullptr, false));
        pend(SLM_K_GEMM_DW);
      } else {
        pbeg();
        CK(simt_gemm(g, (long)d, 1L, (const float*)m.d.W + l * Wl, 1L, (long)d, da, (long)d, B, d, d,
                     (const float*)nullptr, (const float*)nullptr, false));
        pend(SLM_K_GEMM_DX);
        pbeg();
        CK(simt_gemm(g, 1L, (long)d, (const float*)abuf, 1L, (long)d, (float*)m.d.dW + l * Wl, (long)d, d, d,
                     B, (const float*)nullptr, (const float*)nullptr, false));
        pend(SLM_K_GEMM_DW);
      }
      float* dbp = l > 0 ? m.d.db + (size_t)(l - 1) * d : nullptr;
      const float* ga = gam + (size_t)l * d;
      const float* be = bet + (size_t)l * d;
      float* dga = m.d.dgamma + (size_t)l * d;
      float* dbe = m.d.dbeta + (size_t)l * d;
      pbeg();
      if (bf16)
        CK(rk ? launch_k(bn_bwd_rk<__nv_bfloat16, 8>, colgrid, rkblk, 0, st, pdl, (const float*)da, xl,
                         (const float*)stats, ga, be, g, dxl, B, d, dga, dbe, dbp, gq[gpar ^ 1])
              : launch_k(bn_bwd_kernel<__nv_bfloat16>, colgrid, blk, 0, st, pdl, (const float*)da, xl,
                         (const float*)stats, ga, be, g, dxl, B, d, dga, dbe, dbp, gq[gpar ^ 1]));
      else
        CK(rk ? launch_k(bn_bwd_rk<float, 8>, colgrid, rkblk, 0, st, pdl, (const float*)da, xl, (const float*)stats,
                         ga, be, g, dxl, B, d, dga, dbe, dbp, (float*)nullptr)
              : launch_k(bn_bwd_kernel<float>, colgrid, blk, 0, st, pdl, (const float*)da, xl, (const float*)stats,
                         ga, be, g, dxl, B, d, dga, dbe, dbp, (float*)nullptr));
      pend(SLM_K_BN_BWD);
      gpar ^= 1;
      nl += 3;
      // data-parallel: all-reduce the bucket [l, bucket_hi] once its last layer is done
      if (comm && comm->world > 1 && (bucket_hi - l + 1 >= bucket_layers || l == 0)) {
        const int lo = l, cnt = bucket_hi - l + 1;
        cudaEvent_t ev = comm->events[ev_i++ % comm->events.size()];
        CK(cudaEventRecord(ev, st));
        CK(cudaStreamWaitEvent(comm->stream, ev, 0));
        g_nccl.GroupStart();
        int r = 0;
        r |= g_nccl.AllReduce((uint8_t*)m.d.dW + (size_t)lo * per_layer, (uint8_t*)m.d.dW + (size_t)lo * per_layer,
                              (size_t)cnt * Wl, bf16 ? NCCL_BF16 : NCCL_FLOAT32, NCCL_SUM, comm->comm,
                              comm->stream);
        r |= g_nccl.AllReduce(m.d.dgamma + (size_t)lo * d, m.d.dgamma + (size_t)lo * d, (size_t)cnt * d,
                              NCCL_FLOAT32, NCCL_SUM, comm->comm, comm->stream);
        r |= g_nccl.AllReduce(m.d.dbeta + (size_t)lo * d, m.d.dbeta + (size_t)lo * d, (size_t)cnt * d,
                              NCCL_FLOAT32, NCCL_SUM, comm->comm, comm->stream);
        g_nccl.GroupEnd();
        if (r) {
          set_error("ncclAllReduce failed");
          return SLM_E_NCCL;
        }
        bucket_hi = l - 1;
      }
    }
  }
  if (comm && comm->world > 1) {
    // db (all layers; db_0 is final after the last backward) and the loss, then join
    g_nccl.GroupStart();
    int r = 0;
    cudaEvent_t ev = comm->events[ev_i++ % comm->events.size()];
    CK(cudaEventRecord(ev, st));
    CK(cudaStreamWaitEvent(comm->stream, ev, 0));
    r |= g_nccl.AllReduce(m.d.db, m.d.db, (size_t)n * d, NCCL_FLOAT32, NCCL_SUM, comm->comm, comm->stream);
    r |= g_nccl.AllReduce(loss, loss, 1, NCCL_FLOAT32, NCCL_SUM, comm->comm, comm->stream);
    g_nccl.GroupEnd();
    if (r) {
      set_error("ncclAllReduce failed");
      return SLM_E_NCCL;
    }
    cudaEvent_t ev2 = comm->events[ev_i++ % comm->events.size()];
    CK(cudaEventRecord(ev2, comm->stream));
    CK(cudaStreamWaitEvent(st, ev2, 0));
  }
  CK(cudaGetLastError());
  if (launches) *launches = nl;
  return SLM_OK;
}

slm_status check_plan_model(const slm_plan* p, const slm_model* m) {
  if (!p || !m) {
    set_error("null plan/model");
    return SLM_E_ARG;
  }
  if (p->graph_kind != SLM_MODEL_CHAIN || p->dims[0] != m->d.n_layers || p->dims[1] != m->d.batch ||
      p->dims[2] != m->d.width) {
    set_error("plan was not built for this chain's dims (use slm_graph_chain)");
    return SLM_E_SHAPE;
  }
  return SLM_OK;
}

}  // namespace

extern "C" {

const char* slm_version(void) { return "slm 0.1 sm_100a"; }

slm_status slm_model_chain(const slm_chain_desc* desc, slm_model** out) {
  if (!desc || !out) {
    set_error("null argument");
    return SLM_E_ARG;
  }
  *out = nullptr;
  if (desc->n_layers < 0 || desc->batch <= 0 || desc->width <= 0 ||
      (desc->dtype != SLM_F32 && desc->dtype != SLM_BF16)) {
    set_error("bad chain dims/dtype");
    return SLM_E_ARG;
  }
  if (!desc->W || !desc->b || !desc->gamma || !desc->beta || !desc->dW || !desc->db || !desc->dgamma ||
      !desc->dbeta) {
    set_error("null parameter/gradient pointer");
    return SLM_E_ARG;
  }
  auto* m = new slm_model();
  m->d = *desc;
  const int B = desc->batch;
  m->bn_fwd = B >= 64 ? 64 : 32;
  m->bn_dx = m->bn_fwd;
  m->bn_dw = desc->width % 256 == 0 ? 256 : 128;
  *out = m;
  return SLM_OK;
}

void slm_model_destroy(slm_model* m) { delete m; }

slm_status slm_model_set_option(slm_model* m, const char* key, int64_t value) {
  if (!m || !key) {
    set_error("null argument");
    return SLM_E_ARG;
  }
  std::string k(key);
  if (k == "use_graph") m->use_graph = (int)value;
  else if (k == "gemm_impl") m->gemm_impl = (int)value;
  else if (k == "bn_fwd") m->bn_fwd = (int)value;
  else if (k == "bn_dx") m->bn_dx = (int)value;
  else if (k == "bn_dw") m->bn_dw = (int)value;
  else if (k == "profile_events") m->profile = (int)value;
  else if (k == "pdl") m->pdl = (int)value;
  else {
    set_error("unknown option " + k);
    return SLM_E_ARG;
  }
  for (auto& kv : m->graphs) cudaGraphExecDestroy(kv.second);
  m->graphs.clear();
  m->maps_ws = nullptr;
  return SLM_OK;
}

slm_status slm_model_kernel_times(slm_model* m, float* ms, int64_t* count, int32_t n_kinds, int32_t reset) {
  if (!m) {
    set_error("null model");
    return SLM_E_ARG;
  }
  for (auto& p : m->ev_live) {
    CK(cudaEventSynchronize(p.b));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, p.a, p.b));
    m->acc_ms[p.kind] += t;
    m->acc_cnt[p.kind] += 1;
    m->ev_free.push_back(p.a);
    m->ev_free.push_back(p.b);
  }
  m->ev_live.clear();
  for (int k = 0; k < n_kinds && k < SLM_K_COUNT; ++k) {
    if (ms) ms[k] = (float)m->acc_ms[k];
    if (count) count[k] = m->acc_cnt[k];
  }
  if (reset)
    for (int k = 0; k < SLM_K_COUNT; ++k) {
      m->acc_ms[k] = 0;
      m->acc_cnt[k] = 0;
    }
  return SLM_OK;
}

slm_status slm_workspace_bytes(const slm_plan* p, const slm_model* m, size_t* bytes) {
  slm_status s = check_plan_model(p, m);
  if (s != SLM_OK) return s;
  if (!bytes) return SLM_E_ARG;
  *bytes = ws_layout(*m).total;
  return SLM_OK;
}

slm_status slm_step_launches(const slm_plan* p, const slm_model* m, int64_t* launches) {
  slm_status s = check_plan_model(p, m);
  if (s != SLM_OK) return s;
  std::vector<Op> ops;
  if ((s = lower(p, &ops)) != SLM_OK) return s;
  int64_t nl = 0;
  for (auto& o : ops) nl += (o.type == 3) ? 4 : 2;
  *launches = nl;
  return SLM_OK;
}

slm_status slm_step(const slm_plan* p, slm_model* m, const void* x0, const int32_t* labels, void* pool,
                    size_t pool_bytes, void* ws, size_t ws_bytes, float* loss, void* stream, slm_comm* comm) {
  slm_status s = check_plan_model(p, m);
  if (s != SLM_OK) return s;
  if (!x0 || !labels || !loss || (!pool && p->pool_bytes > 0) || !ws) {
    set_error("null device buffer");
    return SLM_E_ARG;
  }
  if ((int64_t)pool_bytes < p->pool_bytes || ws_bytes < ws_layout(*m).total) {
    set_error("pool or workspace smaller than required");
    return SLM_E_BUFFER_TOO_SMALL;
  }
  if (((uintptr_t)pool & 255) || ((uintptr_t)ws & 255)) {
    set_error("pool and workspace must be 256-byte aligned");
    return SLM_E_ARG;
  }
  int dev = 0;
  CK(cudaGetDevice(&dev));
  int major = 0, minor = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  if (major != 10 || minor != 0) {
    set_error("slm kernels are built for sm_100a only");
    return SLM_E_UNSUPPORTED;
  }
  if (m->d.dtype == SLM_BF16 && m->gemm_impl == 0 && !tc_ok(*m)) {
    set_error("bf16 tcgen05 path needs width % 128 == 0 and batch % 64 == 0 (or gemm_impl=1)");
    return SLM_E_UNSUPPORTED;
  }
  if (comm && comm->world > 1 && m->d.batch_global <= 0) {
    set_error("data parallel step needs batch_global");
    return SLM_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (!m->use_graph || st == nullptr || m->profile) return enqueue(p, *m, x0, labels, pool, ws, loss, st, comm, &m->last_launches);
  GraphKey key{p, x0, labels, pool, ws, loss, st, comm};
  auto it = m->graphs.find(key);
  if (it == m->graphs.end()) {
    // the first call runs eagerly (sets kernel attributes, tensor maps) then captures
    s = enqueue(p, *m, x0, labels, pool, ws, loss, st, comm, &m->last_launches);
    if (s != SLM_OK) return s;
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    s = enqueue(p, *m, x0, labels, pool, ws, loss, st, comm, &m->last_launches);
    cudaError_t e = cudaStreamEndCapture(st, &graph);
    if (s != SLM_OK) return s;
    if (e != cudaSuccess) {
      set_error(std::string("graph capture: ") + cudaGetErrorString(e));
      return SLM_E_CUDA;
    }
    cudaGraphExec_t exec;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      set_error(std::string("graph instantiate: ") + cudaGetErrorString(e));
      return SLM_E_CUDA;
    }
    m->graphs[key] = exec;
    return SLM_OK;  // this call already executed the step eagerly
  }
  CK(cudaGraphLaunch(it->second, st));
  return SLM_OK;
}

slm_status slm_step_host(const slm_plan* p, slm_model* m, const float* x0_host, const int32_t* labels_host,
                         void* x0_dev, int32_t* labels_dev, void* pool, size_t pool_bytes, void* ws,
                         size_t ws_bytes, float* loss_dev, float* loss_host, void* stream, slm_comm* comm) {
  slm_status s = check_plan_model(p, m);
  if (s != SLM_OK) return s;
  if (!x0_host || !labels_host || !x0_dev || !labels_dev || !loss_host) {
    set_error("null host/staging buffer");
    return SLM_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t B = m->d.batch, d = m->d.width;
  CK(cudaMemcpyAsync(x0_dev, x0_host, B * d * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(labels_dev, labels_host, B * 4, cudaMemcpyHostToDevice, st));
  s = slm_step(p, m, x0_dev, labels_dev, pool, pool_bytes, ws, ws_bytes, loss_dev, stream, comm);
  if (s != SLM_OK) return s;
  CK(cudaMemcpyAsync(loss_host, loss_dev, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return SLM_OK;
}

// ---------------------------------------------------------------- data parallel
slm_status slm_comm_unique_id(void* id128) {
  if (!id128) return SLM_E_ARG;
  if (!g_nccl.load()) {
    set_error("libnccl.so.2 not loadable");
    return SLM_E_NCCL;
  }
  nccl_uid u;
  if (g_nccl.GetUniqueId(&u) != 0) {
    set_error("ncclGetUniqueId failed");
    return SLM_E_NCCL;
  }
  std::memcpy(id128, &u, 128);
  return SLM_OK;
}

slm_status slm_comm_init(int32_t rank, int32_t world, const void* id128, int64_t bucket_bytes, slm_comm** out) {
  if (!out || !id128 || world < 1 || rank < 0 || rank >= world) {
    set_error("bad comm arguments");
    return SLM_E_ARG;
  }
  *out = nullptr;
  if (!g_nccl.load()) {
    set_error("libnccl.so.2 not loadable");
    return SLM_E_NCCL;
  }
  auto* c = new slm_comm();
  c->rank = rank;
  c->world = world;
  if (bucket_bytes > 0) c->bucket_bytes = bucket_bytes;
  nccl_uid u;
  std::memcpy(&u, id128, 128);
  int r = g_nccl.CommInitRank(&c->comm, world, u, rank);
  if (r != 0) {
    set_error(std::string("ncclCommInitRank: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
    delete c;
    return SLM_E_NCCL;
  }
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    set_error("cudaStreamCreate failed");
    return SLM_E_CUDA;
  }
  c->events.resize(4096);
  for (auto& e : c->events) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  *out = c;
  return SLM_OK;
}

void slm_comm_destroy(slm_comm* c) {
  if (!c) return;
  for (auto& e : c->events) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  delete c;
}

// ---------------------------------------------------------------- test hook
// slm_debug_gemm: one GEMM of the three kinds through the chosen implementation
// (impl 0 = tcgen05 with N tile bn, 1 = SIMT); declared in include/slm_debug.h.
slm_status slm_debug_gemm(int kind, int impl, int bn, int M, int N, int K, const void* A, const void* Bm,
                          void* out, const float* resid, const float* bias, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  using bf = __nv_bfloat16;
  if (impl == 0) {
    CUtensorMap ma, mb;
    slm_status s;
    if (kind == G_FWD) {  // A = W [M][K], B = act [N][K]; out[n][m] = resid + acc + bias[m]
      if ((s = make_map(&ma, A, K, M, 128)) || (s = make_map(&mb, Bm, K, N, bn))) return s;
      slmk::EpiResid e{(float*)out, resid, bias, M};
      return launch_tc_bn<slmk::EpiResid, false, false, true>(bn, ma, mb, M, N, K, 0, 0, e, st, false);
    } else if (kind == G_DX) {  // A = W [K][M] (MN), B = g [N][K]; out[n][m] fp32
      if ((s = make_map(&ma, A, M, K, 64)) || (s = make_map(&mb, Bm, K, N, bn))) return s;
      slmk::EpiStoreF32 e{(float*)out, M};
      return launch_tc_bn<slmk::EpiStoreF32, true, false, true>(bn, ma, mb, M, N, K, 0, 0, e, st, false);
    } else {  // DW: A = act [K][M] (MN), B = g [K][N] (MN); out[n][m] bf16
      if ((s = make_map(&ma, A, M, K, 64)) || (s = make_map(&mb, Bm, N, K, 64))) return s;
      slmk::EpiStoreBF16 e{(bf*)out, M};
      return launch_tc_bn<slmk::EpiStoreBF16, true, true, false>(bn, ma, mb, M, N, K, 0, 0, e, st, false);
    }
  }
  dim3 grid((M + 63) / 64, (N + 63) / 64);  // SIMT computes C(n, m) with n as the row
  if (kind == G_FWD)
    slmk::simt_gemm_kernel<bf, bf, float, slmk::EPI_RESID><<<grid, 256, 0, st>>>(
        N, M, K, (const bf*)Bm, (long)K, 1L, (const bf*)A, (long)K, 1L, (float*)out, (long)M, resid, bias);
  else if (kind == G_DX)
    slmk::simt_gemm_kernel<bf, bf, float, slmk::EPI_STORE><<<grid, 256, 0, st>>>(
        N, M, K, (const bf*)Bm, (long)K, 1L, (const bf*)A, 1L, (long)M, (float*)out, (long)M, nullptr, nullptr);
  else
    slmk::simt_gemm_kernel<bf, bf, bf, slmk::EPI_STORE><<<grid, 256, 0, st>>>(
        N, M, K, (const bf*)Bm, 1L, (long)N, (const bf*)A, 1L, (long)M, (bf*)out, (long)M, nullptr, nullptr);
  CK(cudaGetLastError());
  return SLM_OK;
}

}  // extern "C"
