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
#include <array>
#include <cstdio>
#include <type_traits>
#include <cstring>
#include <map>
#include <set>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "kernels_simt.cuh"
#include "slm_internal.h"
#include "tc_gemm.cuh"
#include "blk_fused.cuh"

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
  int (*GetVersion)(int*) = nullptr;
  int version = 0;
  // SLM_NCCL_LIB (an explicit path) first, else the process's libnccl.so.2 (the one torch loaded,
  // NCCL 2.28.9 in this image); NCCL >= 2.27 is required (ncclGetVersion)
  bool load() {
    if (h) return true;
    const char* env = getenv("SLM_NCCL_LIB");
    h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    GetVersion = (decltype(GetVersion))dlsym(h, "ncclGetVersion");
    if (!GetVersion || GetVersion(&version) != 0 || version < 22700) {
      dlclose(h);
      h = nullptr;
      return false;
    }
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

// bf16 NHWC tensor [images][h][w][c] as a 4-D map {c, w, h, images}, element strides {1, s, s, 1},
// box {64, s wo, s rows, nimg}, 128-byte swizzle: one box = `rows` whole output rows of wo
// positions (every s-th input column / row) of 64 channels -- or nimg whole images (rows = the
// output height) -- laid out in shared memory as the 2-D box {64, wo rows nimg} (the
// implicit-GEMM convolution operand, slmk::ConvB; rows of a box never wrap into the next image:
// out-of-bounds rows are zero-filled)
slm_status make_map4(CUtensorMap* map, const void* base, uint64_t c, uint64_t w, uint64_t h, uint64_t imgs,
                     uint32_t wo, uint32_t rows, uint32_t s, uint32_t nimg) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SLM_E_CUDA;
  }
  cuuint64_t dims[4] = {c, w, h, imgs};
  cuuint64_t strides[3] = {c * 2, w * c * 2, h * w * c * 2};
  cuuint32_t box[4] = {64, s * wo, s * rows, nimg};
  cuuint32_t es[4] = {1, s, s, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (4-D conv operand) failed: " + std::to_string((int)r));
    return SLM_E_CUDA;
  }
  return SLM_OK;
}

}  // namespace

#include "executor.cuh"
#include "lstm_kernels.cuh"
#include "lstm_run.cuh"
#include "executor_lstm.cuh"
#include "executor_ops.cuh"

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

slm_status slm_model_lstm(const slm_lstm_desc* desc, slm_model** out) {
  if (!desc || !out) {
    set_error("null argument");
    return SLM_E_ARG;
  }
  *out = nullptr;
  const slm_lstm_desc& d = *desc;
  if (d.n_layers <= 0 || d.steps <= 0 || d.n_in <= 0 || d.n_classes <= 0 ||
      !(d.batch == 64 || d.batch == 128 || d.batch == 256) || d.hidden <= 0 || d.hidden % 128) {
    set_error("bad lstm dims (batch in {64,128,256}, hidden % 128 == 0)");
    return SLM_E_ARG;
  }
  if (!d.W || !d.b || !d.W_o || !d.b_o || !d.dW || !d.db || !d.dW_o || !d.db_o) {
    set_error("null parameter/gradient pointer");
    return SLM_E_ARG;
  }
  auto* m = new slm_model();
  m->kind = SLM_MODEL_LSTM;
  m->ld = d;
  *out = m;
  return SLM_OK;
}

slm_status slm_model_ops(const slm_graph* g, const slm_ops_desc* desc, slm_model** out) {
  if (!g || !desc || !out) {
    set_error("null argument");
    return SLM_E_ARG;
  }
  *out = nullptr;
  const slm_ops_desc& d = *desc;
  const int n = (int)g->nodes.size();
  if (d.n_nodes != n || d.batch <= 0 || d.batch % 64) {
    set_error("slm_model_ops: n_nodes must match the graph, batch % 64 == 0");
    return SLM_E_ARG;
  }
  if (!d.W || !d.b || !d.gamma || !d.beta || !d.dW || !d.db || !d.dgamma || !d.dbeta) {
    set_error("slm_model_ops: null parameter array");
    return SLM_E_ARG;
  }
  auto m = std::make_unique<slm_model>();
  m->kind = SLM_MODEL_OPS;
  slm_ops_model& o = m->od;
  o.batch = d.batch;
  o.batch_global = d.batch_global;
  auto bad = [&](int v, const std::string& why) {
    set_error("slm_model_ops: node " + std::to_string(v) + ": " + why);
    return SLM_E_UNSUPPORTED;
  };
  for (int v = 0; v < n; ++v) {
    const slm::Node& nd = g->nodes[v];
    if (!ops_supported(nd.op)) return bad(v, "unsupported op " + std::to_string(nd.op));
    const bool loss = nd.op == SLM_OP_SOFTMAX_CE;
    std::array<int, 5> sh{1, 1, 0, 0, 0};
    if (d.shape) {
      for (int i = 0; i < 5; ++i) sh[i] = d.shape[5 * v + i];
      if (sh[0] <= 0 || sh[1] <= 0 || (!loss && sh[2] <= 0)) return bad(v, "bad shape");
    } else if (!loss) {
      if (nd.out_bytes % (4 * (int64_t)d.batch)) return bad(v, "out_bytes is not a multiple of 4 batch");
      sh[2] = (int)(nd.out_bytes / (4 * (int64_t)d.batch));
    }
    const int64_t rows = (int64_t)d.batch * sh[0] * sh[1];
    if (!loss && (sh[2] % 128 || (int64_t)sh[2] * rows * 4 != nd.out_bytes))
      return bad(v, "width must be a multiple of 128 and out_bytes = 4 batch H W C");
    const bool has_in = !nd.preds.empty();
    const std::array<int, 5> in = has_in && d.shape ? std::array<int, 5>{d.shape[5 * nd.preds[0]], d.shape[5 * nd.preds[0] + 1],
                                                                            d.shape[5 * nd.preds[0] + 2], 0, 0}
                                                    : std::array<int, 5>{1, 1, 0, 0, 0};
    if (nd.op == SLM_OP_CONV) {
      if (!d.shape) return bad(v, "Conv needs shapes");
      const int k = sh[3], st = sh[4];
      if (!(k == 1 || k == 3) || !(st == 1 || st == 2)) return bad(v, "Conv k in {1, 3}, stride in {1, 2}");
      if (sh[0] != (in[0] - 1) / st + 1 || sh[1] != (in[1] - 1) / st + 1 || in[2] % 128)
        return bad(v, "Conv output size / input channels");
      if (!d.W[v] || !d.b[v] || !d.dW[v] || !d.db[v]) return bad(v, "Conv without W / b / dW / db");
      m->od.max_col = std::max(m->od.max_col, rows * (int64_t)k * k * in[2]);
      if (k == 3 && st == 1) {   // dx as the convolution of dy with the flipped kernel (executor_ops.cuh)
        m->od.max_colT = std::max(m->od.max_colT, rows * (int64_t)k * k * sh[2]);
        m->od.max_wt = std::max(m->od.max_wt, (int64_t)k * k * in[2] * sh[2]);
      }
    }
    if (nd.op == SLM_OP_POOL && (sh[0] != 1 || sh[1] != 1 || sh[2] != in[2])) return bad(v, "Pool output [batch][C]");
    if ((nd.op == SLM_OP_FC || nd.op == SLM_OP_SOFTMAX_CE) && (in[0] != 1 || in[1] != 1))
      return bad(v, "FC / SoftmaxCE need an input with H = W = 1");
    if ((nd.op == SLM_OP_ADD) && d.shape &&
        (d.shape[5 * nd.preds[1]] != in[0] || d.shape[5 * nd.preds[1] + 1] != in[1] || d.shape[5 * nd.preds[1] + 2] != in[2]))
      return bad(v, "Add of different shapes");
    if (rows >= (int64_t)1 << 31) return bad(v, "more than 2^31 - 1 rows (batch * H * W)");
    m->od.rows.push_back(rows);
    m->od.shape.push_back(sh);
    if (!loss) {
      m->od.max_elems = std::max(m->od.max_elems, rows * sh[2]);
      m->od.max_parts = std::max(m->od.max_parts, ((rows + slmk::kRowChunk - 1) / slmk::kRowChunk) * sh[2]);
    }
    if (loss && nd.out_bytes != 4) {
      set_error("slm_model_ops: the SoftmaxCE node's output is the 4-byte loss");
      return SLM_E_ARG;
    }
    if (nd.op == SLM_OP_FC && (!d.W[v] || !d.b[v] || !d.dW[v] || !d.db[v])) {
      set_error("slm_model_ops: FC node " + std::to_string(v) + " without W / b / dW / db");
      return SLM_E_ARG;
    }
    if (nd.op == SLM_OP_BN && (!d.gamma[v] || !d.beta[v] || !d.dgamma[v] || !d.dbeta[v])) {
      set_error("slm_model_ops: BN node " + std::to_string(v) + " without gamma / beta / dgamma / dbeta");
      return SLM_E_ARG;
    }
    o.W.push_back(d.W[v]);
    o.b.push_back(d.b[v]);
    o.gamma.push_back(d.gamma[v]);
    o.beta.push_back(d.beta[v]);
    o.dW.push_back(d.dW[v]);
    o.db.push_back(d.db[v]);
    o.dgamma.push_back(d.dgamma[v]);
    o.dbeta.push_back(d.dbeta[v]);
    o.op.push_back(nd.op);
    o.out_bytes.push_back(nd.out_bytes);
    if (!loss) m->ops_maxw = std::max(m->ops_maxw, sh[2]);
  }
  *out = m.release();
  return SLM_OK;
}

void slm_model_destroy(slm_model* m) { delete m; }

// workspace bytes of a model's step
size_t model_ws_bytes(const slm_model& m) {
  if (m.kind == SLM_MODEL_LSTM) return lstm_ws_layout(m.ld, m.lstm_sk, m.lstm_skx).total;
  if (m.kind == SLM_MODEL_OPS) return ops_ws_layout(m).total;
  return ws_layout(m).total;
}

slm_status slm_model_get_option(const slm_model* m, const char* key, int64_t* value) {
  if (!m || !key || !value) {
    set_error("null argument");
    return SLM_E_ARG;
  }
  const std::string k(key);
  if (k == "last_overlap") *value = m->last_overlap ? 1 : 0;
  else if (k == "overlap") *value = m->overlap;
  else if (k == "fused") *value = m->fused;
  else if (k == "use_graph") *value = m->use_graph;
  else if (k == "block_split") *value = m->kind == SLM_MODEL_CHAIN && fused_ok(*m) ? blk_shape(m->d.batch, m->d.width, m->block_cfg).S : 0;
  else if (k == "block_m") *value = m->kind == SLM_MODEL_CHAIN && fused_ok(*m) ? blk_shape(m->d.batch, m->d.width, m->block_cfg).BM : 0;
  else {
    set_error("unknown or write-only option: " + k);
    return SLM_E_ARG;
  }
  return SLM_OK;
}

// Lowering options (include/slm.h lists them).  Every change drops the captured CUDA graphs.
slm_status slm_model_set_option(slm_model* m, const char* key, int64_t value) {
  if (!m || !key) {
    set_error("null argument");
    return SLM_E_ARG;
  }
  std::string k(key);
  if (k == "use_graph") m->use_graph = (int)value;
  else if (k == "gemm_impl") m->gemm_impl = (int)value;
  else if (k == "fused") m->fused = (int)value;
  else if (k == "overlap") m->overlap = (int)value;
  else if (k == "block_cfg") m->block_cfg = (int)value;
  else if (k == "poison") m->poison = (int)value;
  else if (k == "pdl") m->pdl = (int)value;
  else if (k == "lstm_streams") m->lstm_streams = (int)value;
  else if (k == "lstm_fuse_runs") m->lstm_fuse_runs = (int)value;
  else if (k == "lstm_run_ts") m->lstm_run_ts = reinterpret_cast<void*>(value);
  else if (k == "lstm_run_ts_n") m->lstm_run_ts_n = (int)value;
  // measurement hooks
  else if (k == "profile_ts") {
    m->profile_ts = (int)value;
    if (value <= 0) {   // detach the device-clock buffer: the caller may free it now
      m->ts_buf = nullptr;
      unsigned long long* z = nullptr;
      CK(cudaMemcpyToSymbol(slmk::g_slm_ts, &z, sizeof(z)));
    }
  }
  else if (k == "profile_ts_buffer") {
    m->ts_buf = reinterpret_cast<void*>(value);
    unsigned long long* p = (unsigned long long*)m->ts_buf;
    CK(cudaMemcpyToSymbol(slmk::g_slm_ts, &p, sizeof(p)));
  }
  else if (k == "profile_events") m->profile = (int)value;
  else if (k == "profile_ts_dep") m->profile_ts_dep = (int)value;
  else {
    set_error("unknown option " + k);
    return SLM_E_ARG;
  }
  for (auto& kv : m->graphs) cudaGraphExecDestroy(kv.second);
  m->graphs.clear();
  m->maps_ws = nullptr;
  m->lst.maps.ws = nullptr;
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
  // device-clock GEMM spans of the last step (profile_ts): max end - min start over the CTAs
  if (m->profile_ts > 0 && m->ts_buf && m->ts_used > 0 && m->profile_ts_dep != 2) {
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> h((size_t)m->ts_used * 1024 * 2);
    CK(cudaMemcpy(h.data(), m->ts_buf, h.size() * 8, cudaMemcpyDeviceToHost));
    for (int s = 0; s < m->ts_used; ++s) {
      unsigned long long t0 = ~0ull, t1 = 0;
      for (int c = 0; c < 1024; ++c) {
        unsigned long long a = h[((size_t)s * 1024 + c) * 2], b = h[((size_t)s * 1024 + c) * 2 + 1];
        if (a == 0 || b == 0) continue;
        t0 = std::min(t0, a);
        t1 = std::max(t1, b);
      }
      if (t1 > t0 && t0 != ~0ull) {
        m->acc_ms[m->ts_kind[s]] += (double)(t1 - t0) * 1e-6;
        m->acc_cnt[m->ts_kind[s]] += 1;
      }
    }
    CK(cudaMemset(m->ts_buf, 0, h.size() * 8));
  }
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
  *bytes = model_ws_bytes(*m);
  return SLM_OK;
}

slm_status slm_step_launches(const slm_plan* p, const slm_model* m, int64_t* launches) {
  slm_status s = check_plan_model(p, m);
  if (s != SLM_OK) return s;
  if (m->kind == SLM_MODEL_LSTM) {
    *launches = lstm_launches(p, *m);
    return SLM_OK;
  }
  if (m->kind == SLM_MODEL_OPS) {   // a dry run of the executor
    int64_t n = 0;
    s = enqueue_ops(p, const_cast<slm_model&>(*m), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &n, true);
    *launches = n;
    return s;
  }
  std::vector<Op> ops;
  if ((s = lower(p, &ops)) != SLM_OK) return s;
  // mirrors enqueue(): K1 only when the operand is not already resident
  const bool fz = fused_ok(*m);
  const int n = m->d.n_layers;
  int64_t nl = 0;
  int act_node = -1;
  for (auto& o : ops) {
    if (o.type == 0) {
      nl += (act_node != o.in_node ? 1 : 0) + 1;
      act_node = fz && o.layer + 1 < n ? o.node : -1;
    } else if (o.type == 3) {
      nl += fz ? 2 : 4;
      if (!fz) act_node = -1;
    } else {
      nl += 2;
    }
  }
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
  const bool is_lstm = m->kind == SLM_MODEL_LSTM, is_ops = m->kind == SLM_MODEL_OPS;
  if ((int64_t)pool_bytes < p->pool_bytes || ws_bytes < model_ws_bytes(*m)) {
    set_error("pool or workspace smaller than required");
    return SLM_E_BUFFER_TOO_SMALL;
  }
  if (((uintptr_t)pool & 255) || ((uintptr_t)ws & 255)) {
    set_error("pool and workspace must be 256-byte aligned");
    return SLM_E_ARG;
  }
  if ((is_lstm || is_ops) && comm) {
    set_error("the LSTM and op-graph steps run replicas-only (comm must be NULL)");
    return SLM_E_UNSUPPORTED;
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
  if (!is_lstm && !is_ops && m->d.dtype == SLM_BF16 && m->gemm_impl == 0 && !tc_ok(*m)) {
    set_error("bf16 tcgen05 path needs width % 128 == 0 and batch % 64 == 0 (or gemm_impl=1)");
    return SLM_E_UNSUPPORTED;
  }
  if (!is_lstm && !is_ops && comm && comm->world > 1 && m->d.batch_global <= 0) {
    set_error("data parallel step needs batch_global");
    return SLM_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  auto run = [&]() {
    if (is_ops) return enqueue_ops(p, *m, x0, labels, pool, ws, loss, st, &m->last_launches);
    return is_lstm ? enqueue_lstm(p, *m, x0, labels, pool, ws, loss, st, &m->last_launches)
                   : enqueue(p, *m, x0, labels, pool, ws, loss, st, comm, &m->last_launches);
  };
  if (!m->use_graph || st == nullptr || m->profile) return run();
  GraphKey key{p->uid, x0, labels, pool, ws, loss, st, comm};
  auto it = m->graphs.find(key);
  if (it == m->graphs.end()) {
    // the first call runs eagerly (sets kernel attributes, tensor maps) then captures
    s = run();
    if (s != SLM_OK) return s;
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    s = run();
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
  size_t xb, lb;
  if (m->kind == SLM_MODEL_LSTM) {
    xb = (size_t)m->ld.steps * m->ld.batch * m->ld.n_in * 4;
    lb = (size_t)m->ld.steps * m->ld.batch * 4;
  } else if (m->kind == SLM_MODEL_OPS) {
    xb = (size_t)m->od.out_bytes[0];   // node 0 is the input (slm_graph_create keeps ids)
    for (size_t v = 0; v < m->od.op.size(); ++v)
      if (m->od.op[v] == SLM_OP_INPUT) {
        xb = (size_t)m->od.out_bytes[v];
        break;
      }
    lb = (size_t)m->od.batch * 4;
  } else {
    xb = (size_t)m->d.batch * m->d.width * 4;
    lb = (size_t)m->d.batch * 4;
  }
  CK(cudaMemcpyAsync(x0_dev, x0_host, xb, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(labels_dev, labels_host, lb, cudaMemcpyHostToDevice, st));
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
    set_error("libnccl.so.2 (or SLM_NCCL_LIB) not loadable or older than NCCL 2.27");
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
    set_error("libnccl.so.2 (or SLM_NCCL_LIB) not loadable or older than NCCL 2.27");
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

// ---------------------------------------------------------------- test hooks
slm_status slm_debug_ts_meta(const slm_model* m, int32_t* kind, int32_t* aux, int32_t cap, int32_t* n) {
  if (!m || !n) return SLM_E_ARG;
  *n = m->ts_used;
  if (cap < m->ts_used) return cap == 0 ? SLM_OK : SLM_E_BUFFER_TOO_SMALL;
  for (int i = 0; i < m->ts_used; ++i) {
    if (kind) kind[i] = m->ts_kind[i];
    if (aux) aux[i] = i < (int)m->ts_aux.size() ? m->ts_aux[i] : 0;
  }
  return SLM_OK;
}

slm_status slm_debug_timestamps(void* dev_buf) {
  unsigned long long* p = (unsigned long long*)dev_buf;
  CK(cudaMemcpyToSymbol(slmk::g_slm_ts, &p, sizeof(p)));
  return SLM_OK;
}

// slm_debug_block: one fused Block kernel (blk_fused.cuh) on caller buffers; declared in
// include/slm_debug.h.
slm_status slm_debug_block(int bwd, int B, int d, const void* W, const void* opnd, const float* x, const float* g,
                           const float* bias, const float* gamma, const float* beta, float* out, void* a_out,
                           void* gq_out, float* dgamma, float* dbeta, float* db_prev, void* P, int dbg, void* stream) {
  const BlkShape sh = blk_shape(B, d, dbg >> 4);   // dbg bits 4..: block_cfg
  const int S = sh.S;
  if (S == 0) {
    set_error("slm_debug_block: unsupported (B, d)");
    return SLM_E_UNSUPPORTED;
  }
  CUtensorMap ma, mb, mp[2], mx;
  slm_status s;
  const uint64_t prow = blk_prows(B, d, S, sh.BM);
  if ((s = make_map(&ma, W, d, d, bwd ? 64u : (uint32_t)sh.BM)) ||
      (s = make_map(&mb, opnd, d, B, (uint32_t)(B / sh.CG))) ||
      (s = make_map_f32_box(&mp[0], P, (uint32_t)(sh.BM / S), prow, (uint32_t)(sh.BM / S), (uint32_t)B)) ||
      (s = make_map_f32_box(&mp[1], P, (uint32_t)(sh.BM / S), prow, (uint32_t)(sh.BM / S), 32u)) ||
      (s = make_map_f32_box(&mx, x, d, B, (uint32_t)(sh.BM / S), (uint32_t)B)))
    return s;
  slmk::BlkArgs a{};
  a.d = d;
  a.pf_row0 = -1;
  a.g = g;
  a.out = out;
  a.bias = bias;
  a.gamma = gamma;
  a.beta = beta;
  a.a_out = (__nv_bfloat16*)a_out;
  a.gq_out = (__nv_bfloat16*)gq_out;
  a.dgamma = dgamma;
  a.dbeta = dbeta;
  a.db_prev = db_prev;
  a.dbg = (dbg & 1) ? 4 : 0;
  return launch_blk(B, sh, bwd != 0, ma, mb, mp, mx, a, (cudaStream_t)stream, false);
}

// slm_debug_plan_alias: make `node` write into `onto`'s tag (a deliberately clobbering plan for the
// poison test); declared in include/slm_debug.h.
slm_status slm_debug_plan_alias(slm_plan* p, int32_t node, int32_t onto) {
  if (!p || node < 0 || onto < 0 || node >= (int)p->node_tag.size() || onto >= (int)p->node_tag.size()) {
    set_error("slm_debug_plan_alias: bad node");
    return SLM_E_ARG;
  }
  const int t = p->node_tag[onto];
  if (t < 0 || p->node_tag[node] < 0 || p->tag_size[t] < p->tag_size[p->node_tag[node]]) {
    set_error("slm_debug_plan_alias: nodes not in V' or tag too small");
    return SLM_E_ARG;
  }
  p->node_tag[node] = t;
  p->uid |= 1ull << 63;   // never matches a captured graph of the intact plan
  return SLM_OK;
}

// slm_debug_gemm: one GEMM of the three kinds through the chosen implementation
// (impl 0 = tcgen05 with N tile bn, 1 = SIMT); declared in include/slm_debug.h.
slm_status slm_debug_gemm(int kind, int impl, int bn, int split, int M, int N, int K, const void* A, const void* Bm,
                          void* out, const float* resid, const float* bias, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  using bf = __nv_bfloat16;
  if (impl == 0 || impl >= 2) {
    const int dbg = (impl == 2 ? 1 : (impl == 3 ? 2 : 0)) | 4;   // 2: data movement only, 3: MMA only; 4: phase stamps
    const int cg = impl == 4 ? 2 : 1;                       // 4: CTA-pair (cta_group::2) tcgen05
    const uint32_t bbox = (uint32_t)(bn / cg);              // K-major B box rows
    CUtensorMap ma, mb;
    slm_status s;
    if (kind == G_FWD && split == 1) {  // A = W [M][K], B = act [N][K]; out[n][m] = resid + acc + bias[m]
      if ((s = make_map(&ma, A, K, M, 128)) || (s = make_map(&mb, Bm, K, N, bbox))) return s;
      slmk::EpiResid e{(float*)out, resid, bias, M};
      return launch_tc_bn<slmk::EpiResid, false, false, true>(bn, split, ma, mb, M, N, K, 0, 0, e, st, false, dbg,
                                                              nullptr, cg);
    } else if (kind == G_FWD) {  // split-K partials: out[s][n][m] (fp32, split x N x M)
      CUtensorMap mc;
      if ((s = make_map(&ma, A, K, M, 128)) || (s = make_map(&mb, Bm, K, N, bbox)) ||
          (s = make_map_f32(&mc, out, M, (uint64_t)split * N)))
        return s;
      slmk::EpiPartialTma e{N};
      return launch_tc_bn<slmk::EpiPartialTma, false, false, true>(bn, split, ma, mb, M, N, K, 0, 0, e, st, false, dbg,
                                                                   &mc, cg);
    } else if (kind == G_DX) {  // A = W [K][M] (MN), B = g [N][K]; out[s][n][m] fp32 (split partials)
      CUtensorMap mc;
      if ((s = make_map(&ma, A, M, K, 64)) || (s = make_map(&mb, Bm, K, N, bbox)) ||
          (s = make_map_f32(&mc, out, M, (uint64_t)split * N)))
        return s;
      slmk::EpiPartialTma e{N};
      return launch_tc_bn<slmk::EpiPartialTma, true, false, true>(bn, split, ma, mb, M, N, K, 0, 0, e, st, false, dbg,
                                                                  &mc, cg);
    } else {  // DW: A = act [K][M] (MN), B = g [K][N] (MN); out[n][m] bf16
      if ((s = make_map(&ma, A, M, K, 64)) || (s = make_map(&mb, Bm, N, K, 64))) return s;
      slmk::EpiStoreBF16 e{(bf*)out, M};
      return launch_tc_bn<slmk::EpiStoreBF16, true, true, false>(bn, split, ma, mb, M, N, K, 0, 0, e, st, false, dbg,
                                                                 nullptr, cg);
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
