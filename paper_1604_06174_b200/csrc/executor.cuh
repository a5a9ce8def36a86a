// Executor of V' for the residual chain (included by runtime.cu; not a standalone TU).
//
// Every node of V' (Alg. 2's order) writes its value into the pool slot of
// its temporal tag (Fig. 2).  Two lowerings:
//
// * fused (bf16, tcgen05; the product path at B <= 256):
//     forward/mirror Block_l   [K1 bn_act(x_l) only if a_l is not already resident]
//                              GEMM  P[s] = W_l a_l^T over K slice s   (split-K, 128 CTAs)
//                              finalize+K1  x_{l+1} = x_l + (sum_s P[s] + b_l) -> slot,
//                                           stats/a_{l+1} for the next Block (same kernel code as K1)
//     grad Block_l             GEMM  P[s] = g_{l+1} W_l over K slice s (dX, split-K)
//                              bn_bwd  da = sum_s P[s], stats of x_l, a_l, dx_l, dgamma, dbeta,
//                                      db_{l-1}, bf16 copy of dx_l
//                              GEMM  dW_l = g_{l+1}^T a_l   on a second stream (off the critical
//                                      path; joined by events two layers later)
// * basic (f32 FFMA path, SIMT GEMMs, or B > 256): K1 + GEMM with residual epilogue; K1 + dX +
//   dW + bn_bwd in the backward.
//
// Mirrors re-run exactly the forward kernels with the same launch configuration, and every
// reduction has a fixed order, so re-computed values are bit-identical.

namespace {

// ---------------------------------------------------------------- launchers
// Every kernel of the step is launched with programmatic stream serialization (PDL) when
// `pdl` is set: it may start while its predecessor drains and synchronises on it with
// griddepcontrol.wait before touching dependent data.
template <class... KArgs, class... Args>
cudaError_t launch_kc(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                      int cluster_x, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster_x > 1) {   // thread-block cluster (CTA pairs of the cta_group::2 GEMM)
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster_x;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
template <class... KArgs, class... Args>
cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                     Args... args) {
  return launch_kc(k, grid, block, smem, st, pdl, 1, args...);
}

enum GemmKind { G_FWD = 0, G_DX = 1, G_DW = 2 };

template <int BN, bool AMN, bool BMN, bool PRE, class Epi, int CG = 1>
slm_status launch_tc(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, int M, int N, int K, int split,
                     int a_row0, int b_row0, Epi epi, cudaStream_t st, bool pdl, int dbg, int pf_row0 = -1,
                     slmk::ConvB cb = {}) {
  using C = slmk::TcCfg<BN, AMN, BMN, CG>;
  auto kern = slmk::tc_gemm_kernel<BN, AMN, BMN, PRE, Epi, CG>;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  if (split < 1 || K % (64 * split) || M % (128 * CG) || N % BN) {
    set_error("GEMM shape not tileable: M % (128 * cta_group), N % BN, K % (64 * split)");
    return SLM_E_UNSUPPORTED;
  }
  CK(launch_kc(kern, dim3(M / 128, N / BN, split), dim3(128), C::SMEM, st, pdl, CG, a, b, c, K, a_row0, b_row0, epi,
               dbg, pf_row0, cb));
  return SLM_OK;
}

// c: tensor map of the output for TMA-store epilogues (Epi::kTma), else ignored.
// cg = 2: CTA-pair GEMM (cta_group::2); a K-major B map must then have box rows bn / 2.
template <class Epi, bool AMN, bool BMN, bool PRE>
slm_status launch_tc_bn(int bn, int split, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int K,
                        int a_row0, int b_row0, Epi epi, cudaStream_t st, bool pdl, int dbg = 0,
                        const CUtensorMap* c = nullptr, int cg = 1, int pf = -1, slmk::ConvB cb = {}) {
  const CUtensorMap& cm = c ? *c : a;
  if (cg == 2) {
    switch (bn) {
      case 128:
        return launch_tc<128, AMN, BMN, PRE, Epi, 2>(a, b, cm, M, N, K, split, a_row0, b_row0, epi, st, pdl, dbg, pf, cb);
      case 256:
        return launch_tc<256, AMN, BMN, PRE, Epi, 2>(a, b, cm, M, N, K, split, a_row0, b_row0, epi, st, pdl, dbg, pf, cb);
    }
    set_error("unsupported CTA-pair GEMM N tile " + std::to_string(bn));
    return SLM_E_UNSUPPORTED;
  }
  switch (bn) {
    case 32:
      if (!BMN) return launch_tc<32, AMN, BMN, PRE>(a, b, cm, M, N, K, split, a_row0, b_row0, epi, st, pdl, dbg, pf, cb);
      break;
    case 64: return launch_tc<64, AMN, BMN, PRE>(a, b, cm, M, N, K, split, a_row0, b_row0, epi, st, pdl, dbg, pf, cb);
    case 128: return launch_tc<128, AMN, BMN, PRE>(a, b, cm, M, N, K, split, a_row0, b_row0, epi, st, pdl, dbg, pf, cb);
    case 256: return launch_tc<256, AMN, BMN, PRE>(a, b, cm, M, N, K, split, a_row0, b_row0, epi, st, pdl, dbg, pf, cb);
  }
  set_error("unsupported GEMM N tile " + std::to_string(bn));
  return SLM_E_UNSUPPORTED;
}

// bf16 2-D tensor [rows][inner], box {128, 32}, no swizzle (dW epilogue bulk stores)
slm_status make_map_bf16_store(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SLM_E_CUDA;
  }
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {128, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (bf16 store) failed: " + std::to_string((int)r));
    return SLM_E_CUDA;
  }
  return SLM_OK;
}

// fp32 2-D tensor [rows][inner], box {128, 32}, no swizzle (epilogue bulk stores)
slm_status make_map_f32(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SLM_E_CUDA;
  }
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 4};
  cuuint32_t box[2] = {128, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (f32) failed: " + std::to_string((int)r));
    return SLM_E_CUDA;
  }
  return SLM_OK;
}

// fp32 2-D tensor [rows][inner], box {box_inner, box_rows}, no swizzle: the Block kernel's x slices
// and its partial-exchange buffer (blk_fused.cuh)
slm_status make_map_f32_box(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows, uint32_t box_inner,
                            uint32_t box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SLM_E_CUDA;
  }
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 4};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (f32 box) failed: " + std::to_string((int)r));
    return SLM_E_CUDA;
  }
  return SLM_OK;
}
// rows of FS = BM / S floats in the Block kernel's partial buffer: [d/BM][S][S][B]
uint64_t blk_prows(int B, int d, int S, int BM) { return (uint64_t)(d / BM) * S * S * B; }

// Shape of the fused Block (blk_fused.cuh): BM output features per CTA (the MMA's M) and the
// cluster split S of K; option block_cfg: 0 = default, 1 = (64, 4), 2 = (128, 4), 3 = (64, 2),
// 4 = (128, 4) as CTA pairs (cta_group::2: clusters of 8, each SM stages half of the batch).
// Default: (128, 4) at B = 256 (64 CTAs at d = 2048), (64, 4) below; (64, 2) when d % 256 != 0.
// Measured at C2 (scripts/chain_timeline.py, profiles/r2_block_shapes.md): (128, 4) 29.9 ms/step,
// (64, 2) 31.6, (64, 4) 35.1 — the 128-CTA Blocks run the forward pass faster (10.5 vs 11.4 us per
// Block) but leave no room for the concurrent recompute and dW streams of the backward phase.
// {0, 0} = not supported (basic lowering).
struct BlkShape {
  int BM, S, CG;   // CG = 2: CTA pairs (cta_group::2), clusters of S * CG
};
BlkShape blk_shape(int B, int d, int cfg) {
  if (!(B == 64 || B == 128 || B == 256) || d % 128) return {0, 0, 1};
  static const BlkShape tab[5] = {{128, 4, 1}, {64, 4, 1}, {128, 4, 1}, {64, 2, 1}, {128, 4, 2}};
  BlkShape sh = tab[(cfg >= 0 && cfg <= 4) ? cfg : 0];
  if (sh.BM == 128 && B != 256) sh = {64, sh.S, 1};
  if (sh.CG == 2 && (d / sh.BM) % 2) sh.CG = 1;
  if ((d / sh.S) % 64 || d % sh.BM) sh = {64, 2, 1};   // K slice of whole 64-column blocks
  if (d % sh.BM || (d / sh.S) % 64) return {0, 0, 1};
  return sh;
}
int blk_split(int B, int d) { return blk_shape(B, d, 0).S; }

template <int B_, int S_, bool BWD, int BM_, int CG_ = 1>
slm_status launch_blk_t(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& p, const CUtensorMap& ps,
                        const CUtensorMap& x, const slmk::BlkArgs& args, cudaStream_t st, bool pdl) {
  using C = slmk::BlkCfg<B_, S_, BWD, BM_, CG_>;
  auto kern = slmk::blk_kernel<B_, S_, BWD, BM_, CG_>;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  CK(launch_kc(kern, dim3(args.d / BM_ * S_), dim3(slmk::kBlkThreads), C::SMEM, st, pdl, S_ * CG_, a, b, p, ps, x,
               args));
  return SLM_OK;
}
slm_status launch_blk(int B, BlkShape sh, bool bwd, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap* p,
                      const CUtensorMap& x, const slmk::BlkArgs& args, cudaStream_t st, bool pdl) {
#define SLM_BLK(B_, S_, BM_, CG_)                                                              \
  if (B == B_ && sh.S == S_ && sh.BM == BM_ && sh.CG == CG_)                                   \
    return bwd ? launch_blk_t<B_, S_, true, BM_, CG_>(a, b, p[0], p[1], x, args, st, pdl)      \
               : launch_blk_t<B_, S_, false, BM_, CG_>(a, b, p[0], p[1], x, args, st, pdl);
  SLM_BLK(64, 2, 64, 1) SLM_BLK(64, 4, 64, 1) SLM_BLK(128, 2, 64, 1) SLM_BLK(128, 4, 64, 1) SLM_BLK(256, 2, 64, 1)
  SLM_BLK(256, 4, 64, 1) SLM_BLK(256, 4, 128, 1) SLM_BLK(256, 4, 128, 2)
#undef SLM_BLK
  set_error("unsupported fused Block configuration");
  return SLM_E_UNSUPPORTED;
}
cudaError_t launch_k1(int B, BlkShape sh, const float* x, const float* gam, const float* bet, int d, __nv_bfloat16* a,
                      cudaStream_t st, bool pdl) {
#define SLM_K1(B_, S_, BM_)                                                                                      \
  if (B == B_ && sh.S == S_ && sh.BM == BM_)                                                                    \
    return launch_k(slmk::bn_k1_kernel<B_, S_, BM_>, dim3(d / (BM_ / S_)), dim3(slmk::kBlkThreads), 0, st, pdl, x, \
                    gam, bet, d, a);
  SLM_K1(64, 2, 64) SLM_K1(64, 4, 64) SLM_K1(128, 2, 64) SLM_K1(128, 4, 64) SLM_K1(256, 2, 64) SLM_K1(256, 4, 64)
  SLM_K1(256, 4, 128)
#undef SLM_K1
  return cudaErrorInvalidValue;
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
  int in_node;   // fwd block: the node whose value is x_l
  int node;      // this node of G'
  int aux_node = -1;   // bwd block: the node whose value is g (in_node then holds x_l's node)
};

// CUDA-graph cache key: the plan's process-unique id (never reused, unlike its address), the
// caller's buffers, stream and communicator
struct GraphKey {
  uint64_t plan;
  const void *x0, *labels, *pool, *ws, *loss;
  cudaStream_t stream;
  const void* comm;
  bool operator<(const GraphKey& o) const {
    return std::tie(plan, x0, labels, pool, ws, loss, stream, comm) <
           std::tie(o.plan, o.x0, o.labels, o.pool, o.ws, o.loss, o.stream, o.comm);
  }
};

// LSTM executor state (executor_lstm.cuh): tensor maps bound to the weights / workspace and
// the Sum node's pool-offset table
struct LstmMaps {
  // per layer: W_l K-major / MN-major, forward operand [B][K_l], the time-chunk rings of the
  // backward operands (op K-major/MN-major, d_pre K-major/MN-major), the dX partials
  std::vector<CUtensorMap> wK, wK32, wMN, opRK, opRMN, dpRK, dpRMN, pX, pG, pGm, pXd;   // partials of layer l's streams
  CUtensorMap woK, woMN, hopRK, hopRMN, dlRK, dlRMN, pL, pH, hopRKb[3], dlRKb[3], pHB;            // pL / pH over the head's
  // per forward lane (lstm_run.cuh): hx [2B][H] (box 64 x B), X [kRunMax B][4H] f32 (box 32 x 64),
  // the chunk ring [2 CH B][H] and the packed operand [kRunMax B][Kin] as GEMM B operands (box
  // rows 64 / 256)
  std::vector<CUtensorMap> hxM, xpM, ringM[2], xopM[2];
  // backward runs: the d_pre ring as a 256-row B operand, the d_pre exchange (box 64 x B)
  std::vector<CUtensorMap> dpR256, dpxM;
  // the second (odd-chunk) half of the backward rings when the weight gradients run on their own
  // stream (executor_lstm.cuh: chunk-parity double buffering)
  std::vector<CUtensorMap> opRMN1, dpRMN1, dpR2561;
  std::vector<CUtensorMap> xpM1;   // the second half of each lane's double-buffered projection X
  const void* ws = nullptr;
};
struct slm_lstm_state {
  LstmMaps maps;
  // layer-wavefront execution (option lstm_streams): one stream per layer + one for the head,
  // a ring of events per stream, fork/join events
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> ev;
  cudaEvent_t fork = nullptr;
  std::vector<cudaEvent_t> join;
  ~slm_lstm_state() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    for (auto e : join) cudaEventDestroy(e);
    if (fork) cudaEventDestroy(fork);
    for (auto x : streams) cudaStreamDestroy(x);
  }
};

// dW ring (fused lowering): the dW GEMM of backward k reads ab[k % kNA] and gq[k % kNG]; the
// gradient Block of backward k overwrites gq[(k+1) % kNG] and ab[k % kNA], so it waits for dW of
// backward k - kNA: kNA layers of slack between the dX chain and the dW stream
#ifndef SLM_KNA
#define SLM_KNA 2
#endif
constexpr int kNA = SLM_KNA, kNG = kNA + 1;

// op-granularity model (executor_ops.cuh): per forward node parameters, the graph it was built for
struct slm_ops_model {
  int batch = 0, batch_global = 0;
  std::vector<const void*> W;
  std::vector<const float*> b, gamma, beta;
  std::vector<void*> dW;
  std::vector<float*> db, dgamma, dbeta;
  std::vector<int> op;
  std::vector<int64_t> out_bytes;
  // per node: rows (batch H W) and (H, W, C, k, s) (convolutional graphs)
  std::vector<int64_t> rows;
  std::vector<std::array<int, 5>> shape;
  int64_t max_elems = 0, max_col = 0, max_parts = 0, max_colT = 0, max_wt = 0;   // workspace sizing
};

struct slm_model {
  slm_chain_desc d{};
  slm_lstm_desc ld{};
  slm_ops_model od;
  int ops_maxw = 0;
  slm_lstm_state lst;
  int kind = SLM_MODEL_CHAIN;
  int use_graph = 1;
  int gemm_impl = 0;      // 0 tcgen05 (bf16), 1 SIMT
  int pdl = 1;            // programmatic dependent launch between the step's kernels
  int fused = 1;          // fused lowering (one Block kernel per node, blk_fused.cuh)
  int dw_stream = 1;      // dW GEMMs on a second stream (fixed; measured: serial dW 41 vs 27.9 ms/step)
  int bn_fwd = 64, bn_dx = 64, bn_dw = 256;   // N tiles of the basic lowering's GEMMs (bn_dw: also the fused dW)
  int poison = 0;         // debug: fill a pool tag with NaN once its value is dead (sequential schedule)
  int block_cfg = 0;      // fused Block shape (blk_shape: 0 default, 1..4 explicit (BM, S))
  int overlap = 1;        // segment recompute on its own stream, concurrent with the backward of
                          // the next segment, when the plan allows it (SLM_ALLOC_MIRROR_PARITY)
  int lstm_streams = 2;   // LSTM: layer wavefront over L+1 streams (2: + L mirror streams)
  int lstm_sk = 1;        // LSTM: split-K of the gates GEMMs (0 = auto; 1 measured best with the wavefront)
  int lstm_skx = 4;       // LSTM: split-K of the dX GEMMs (0 = auto; 4 measured best with the wavefront)
  int lstm_fuse_runs = 1; // LSTM: forward / recompute phases as chunk x layer runs (0: node by node in V' order)
  void* lstm_run_ts = nullptr;   // debug: per-step device clock of CTA 0 of the first runs ([run][kRunMax][4] u64)
  int lstm_run_ts_n = 0;
  // tensor maps bound to the current workspace / weights
  const void* maps_ws = nullptr;
  int maps_key = -1;
  CUtensorMap mW_K, mW_K64, mW_MN, mdW_st, mA_K, mA_MN, mAct[2], mAct3[2], mPf[2], mPf3[2], mG_K[kNG], mG_MN[kNG], mAb_MN[kNA];
  std::map<GraphKey, cudaGraphExec_t> graphs;
  int64_t last_launches = 0;
  bool last_overlap = false;           // the last enqueued step ran its recompute on s3
  cudaStream_t s2 = nullptr;           // second stream (dW)
  cudaStream_t s3 = nullptr;           // recompute stream (option overlap)
  std::vector<cudaEvent_t> ov_ev;      // its fork/join events
  std::vector<cudaEvent_t> sync_ev;    // fork/join events (reused every step)
  // profile_ts: device-clock (%globaltimer) start/end of every CTA of the first profile_ts Block /
  // GEMM launches of a step, in the caller's buffer ts_buf ([slot][1024][2] uint64, zeroed)
  int profile_ts = 0;
  int profile_ts_dep = 0;   // 1: stamp the start after the dependency wait (ts_dep); 2: all 8 phases
                            // of every CTA, [slot][1024][8] (scripts/chain_timeline.py PHASES=1)
  void* ts_buf = nullptr;
  std::vector<int> ts_kind;
  std::vector<int> ts_aux;    // per slot: the LSTM stream of the launch (slm_debug_ts_meta)
  int ts_cur_aux = 0;
  int ts_used = 0;
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
    for (auto e : sync_ev) cudaEventDestroy(e);
    if (s2) cudaStreamDestroy(s2);
    if (s3) cudaStreamDestroy(s3);
    for (auto e : ov_ev) cudaEventDestroy(e);
  }
};

namespace {

bool tc_ok(const slm_model& m) {
  const int B = m.d.batch, d = m.d.width;
  return m.d.dtype == SLM_BF16 && m.gemm_impl == 0 && d % 128 == 0 && B % 64 == 0 && B <= 4096 &&
         B % m.bn_fwd == 0 && B % m.bn_dx == 0 && d % m.bn_dw == 0;
}
// the fused lowering (blk_fused.cuh): the whole batch per Block CTA (N = B <= 256), K split over a
// cluster of blk_shape() CTAs
bool fused_ok(const slm_model& m) { return tc_ok(m) && m.fused && blk_shape(m.d.batch, m.d.width, m.block_cfg).S > 0; }

struct WsLayout {
  size_t act[2], act3[2], stats, gq[kNG], ab[kNA], P, P3, da, rowloss, a, total;
};
WsLayout ws_layout(const slm_model& m) {
  const size_t B = m.d.batch, d = m.d.width;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  WsLayout L{};
  const bool fz = fused_ok(m);
  const size_t S = fz ? (size_t)blk_shape((int)B, (int)d, m.block_cfg).S : 0;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += al(bytes);
    return o;
  };
  L.a = take(B * d * 4);                  // basic lowering: a_l (fp32 or bf16)
  L.stats = take(2 * d * 4);
  for (int i = 0; i < kNG; ++i) L.gq[i] = take(B * d * 2);
  for (int i = 0; i < kNA; ++i) L.ab[i] = take(fz ? B * d * 2 : 0);
  for (int i = 0; i < 2; ++i) L.act[i] = take(fz ? B * d * 2 : 0);
  L.P = take(S * B * d * 4);              // partial exchange of the Block kernels ([d/64][S][S][.][B][16])
  L.da = take(fz ? 0 : B * d * 4);
  L.rowloss = take(B * 4);
  // the recompute stream's own operands and partial buffer (option overlap)
  const bool ovw = fz && m.overlap;
  for (int i = 0; i < 2; ++i) L.act3[i] = take(ovw ? B * d * 2 : 0);
  L.P3 = take(ovw ? S * B * d * 4 : 0);
  L.total = off;
  return L;
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
        ops->push_back({0, orig - 1, p->node_tag[pr[0]], -1, p->node_tag[v], pr[0], v});
      else if (op == SLM_OP_SOFTMAX_CE)
        ops->push_back({1, n, p->node_tag[pr[0]], -1, p->node_tag[v], pr[0], v});
      else {
        set_error("unsupported op in chain plan");
        return SLM_E_UNSUPPORTED;
      }
    } else {
      if (op == SLM_OP_SOFTMAX_CE) {
        if (npr != 1) return SLM_E_UNSUPPORTED;
        ops->push_back({2, n, p->node_tag[pr[0]], -1, p->node_tag[v], pr[0], v});
      } else if (op == SLM_OP_BLOCK) {
        if (npr != 2) return SLM_E_UNSUPPORTED;
        ops->push_back({3, orig - 1, p->node_tag[pr[0]], p->node_tag[pr[1]], p->node_tag[v], pr[1], v, pr[0]});
      } else {
        set_error("unsupported gradient op in chain plan");
        return SLM_E_UNSUPPORTED;
      }
    }
  }
  return SLM_OK;
}

slm_status bind_maps(slm_model& m, void* ws) {
  const int key = m.bn_fwd * 7 + m.bn_dx * 131 + m.fused + m.bn_dw * 1009 + m.overlap * 5 + m.block_cfg * 100003;
  if (m.maps_ws == ws && m.maps_key == key) return SLM_OK;
  const uint64_t B = m.d.batch, d = m.d.width, n = m.d.n_layers;
  WsLayout L = ws_layout(m);
  uint8_t* w = (uint8_t*)ws;
  const bool fz = fused_ok(m);
  slm_status st;
  if ((st = make_map(&m.mW_K, m.d.W, d, n * d, 128)) != SLM_OK) return st;
  if ((st = make_map(&m.mW_MN, m.d.W, d, n * d, 64)) != SLM_OK) return st;
  if (fz) {
    const BlkShape sh = blk_shape((int)B, (int)d, m.block_cfg);
    const uint64_t prow = blk_prows((int)B, (int)d, sh.S, sh.BM);
    if ((st = make_map(&m.mW_K64, m.d.W, d, n * d, (uint32_t)sh.BM)) != SLM_OK) return st;
    const uint32_t brows = (uint32_t)(B / sh.CG);   // K-major operand box rows: this CTA's batch rows
    if ((st = make_map_bf16_store(&m.mdW_st, m.d.dW, d, n * d)) != SLM_OK) return st;
    for (int i = 0; i < 2; ++i)
      if ((st = make_map(&m.mAct[i], w + L.act[i], d, B, brows)) != SLM_OK) return st;
    // partial exchange: {32, B} box for the owner's loads, {32, 32} for a warp's chunk stores
    const uint32_t FS = (uint32_t)(sh.BM / sh.S);
    if ((st = make_map_f32_box(&m.mPf[0], w + L.P, FS, prow, FS, (uint32_t)B)) != SLM_OK) return st;
    if ((st = make_map_f32_box(&m.mPf[1], w + L.P, FS, prow, FS, 32u)) != SLM_OK) return st;
    if (m.overlap) {
      for (int i = 0; i < 2; ++i)
        if ((st = make_map(&m.mAct3[i], w + L.act3[i], d, B, brows)) != SLM_OK) return st;
      if ((st = make_map_f32_box(&m.mPf3[0], w + L.P3, FS, prow, FS, (uint32_t)B)) != SLM_OK) return st;
      if ((st = make_map_f32_box(&m.mPf3[1], w + L.P3, FS, prow, FS, 32u)) != SLM_OK) return st;
    }
    for (int i = 0; i < kNA; ++i)
      if ((st = make_map(&m.mAb_MN[i], w + L.ab[i], d, B, 64)) != SLM_OK) return st;
  } else {
    if ((st = make_map(&m.mA_K, w + L.a, d, B, (uint32_t)m.bn_fwd)) != SLM_OK) return st;
    if ((st = make_map(&m.mA_MN, w + L.a, d, B, 64)) != SLM_OK) return st;
  }
  const uint32_t grows = fz ? (uint32_t)(B / blk_shape((int)B, (int)d, m.block_cfg).CG) : (uint32_t)m.bn_dx;
  for (int i = 0; i < kNG; ++i) {
    if ((st = make_map(&m.mG_K[i], w + L.gq[i], d, B, grows)) != SLM_OK) return st;
    if ((st = make_map(&m.mG_MN[i], w + L.gq[i], d, B, 64)) != SLM_OK) return st;
  }
  m.maps_ws = ws;
  m.maps_key = key;
  return SLM_OK;
}

slm_status ensure_streams(slm_model& m, int n_layers) {
  if (!m.s2) CK(cudaStreamCreateWithFlags(&m.s2, cudaStreamNonBlocking));
  if (m.overlap && !m.s3) CK(cudaStreamCreateWithFlags(&m.s3, cudaStreamNonBlocking));
  const size_t need = 2 * (size_t)n_layers + 8;
  while (m.sync_ev.size() < need) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    m.sync_ev.push_back(e);
  }
  return SLM_OK;
}

// Enqueue the whole step on `st`; counts kernel launches into *launches.
slm_status enqueue(const slm_plan* p, slm_model& m, const void* x0, const int32_t* labels, void* pool, void* ws,
                   float* loss, cudaStream_t st, slm_comm* comm, int64_t* launches) {
  using namespace slmk;
  using bf = __nv_bfloat16;
  const int B = m.d.batch, d = m.d.width, n = m.d.n_layers;
  const bool bf16 = m.d.dtype == SLM_BF16;
  const bool tc = tc_ok(m);
  const bool fz = fused_ok(m);
  const BlkShape bsh = fz ? blk_shape(B, d, m.block_cfg) : BlkShape{0, 0, 1};
  const int Bg = m.d.batch_global > 0 ? m.d.batch_global : B;
  const float inv_bg = 1.0f / (float)Bg;
  const WsLayout L = ws_layout(m);
  uint8_t* w = (uint8_t*)ws;
  float* stats = (float*)(w + L.stats);
  void* abuf = w + L.a;
  bf* gq[kNG];
  bf* ab[kNA];
  for (int i = 0; i < kNG; ++i) gq[i] = (bf*)(w + L.gq[i]);
  for (int i = 0; i < kNA; ++i) ab[i] = (bf*)(w + L.ab[i]);
  float* da = (float*)(w + L.da);
  float* rowloss = (float*)(w + L.rowloss);
  const bool pdl = m.pdl != 0;
  const bool side = fz && m.dw_stream;

  std::vector<Op> ops;
  slm_status s = lower(p, &ops);
  if (s != SLM_OK) return s;
  if (tc && (s = bind_maps(m, ws)) != SLM_OK) return s;
  if (side && (s = ensure_streams(m, n)) != SLM_OK) return s;

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

  // fp32 [rows][d] views of the pool and of x_0 for the Block kernels' x / g slice loads: every
  // pool tag of a chain plan holds one [B][d] fp32 value (A9 offsets are sums of B*d*4-byte tags)
  CUtensorMap mx_pool, mx_x0;
  const uint64_t row_bytes = (uint64_t)d * 4;
  if (fz) {
    const uint64_t prows = std::max<uint64_t>((uint64_t)p->pool_bytes / row_bytes, (uint64_t)B);
    const uint32_t FS = (uint32_t)(bsh.BM / bsh.S);
    if ((s = make_map_f32_box(&mx_pool, pool ? pool : x0, d, prows, FS, (uint32_t)B)) != SLM_OK) return s;
    if ((s = make_map_f32_box(&mx_x0, x0, d, (uint64_t)B, FS, (uint32_t)B)) != SLM_OK) return s;
  }
  auto xsrc = [&](const float* ptr, const CUtensorMap** map, int* row) -> slm_status {
    if (ptr == (const float*)x0) {
      *map = &mx_x0;
      *row = 0;
      return SLM_OK;
    }
    const uint64_t off = (uint64_t)((const uint8_t*)ptr - (const uint8_t*)pool);
    if (!pool || off % row_bytes || off + (uint64_t)B * row_bytes > (uint64_t)p->pool_bytes) {
      set_error("pool slot not addressable as [rows][d] fp32");
      return SLM_E_UNSUPPORTED;
    }
    *map = &mx_pool;
    *row = (int)(off / row_bytes);
    return SLM_OK;
  };

  const size_t Wl = (size_t)d * d;
  const float* bvec = m.d.b;
  const float* gam = m.d.gamma;
  const float* bet = m.d.beta;
  const dim3 colgrid((d + 31) / 32), blk(256);
  int64_t nl = 0;

  // optional per-kernel CUDA events (profile_events), recorded on the launching stream
  cudaEvent_t ev0 = nullptr;
  auto pbeg = [&](cudaStream_t ss) {
    if (m.profile) {
      ev0 = m.get_event();
      cudaEventRecord(ev0, ss);
    }
  };
  auto pend = [&](int kind, cudaStream_t ss) {
    if (m.profile) {
      cudaEvent_t e1 = m.get_event();
      cudaEventRecord(e1, ss);
      m.ev_live.push_back({ev0, e1, kind});
    }
  };

  auto simt_gemm = [&](auto* A, long sAm, long sAk, auto* Bp, long sBn, long sBk, auto* out, long ldo, int M, int N,
                       int K, const float* resid, const float* bias, bool resid_epi) -> cudaError_t {
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
  // K1 of the basic lowering
  auto bn_act = [&](const float* xin, int l) -> cudaError_t {
    const float* ga = gam + (size_t)l * d;
    const float* be = bet + (size_t)l * d;
    if (bf16) return launch_k(bn_act_kernel<bf>, colgrid, blk, 0, st, pdl, xin, ga, be, B, d, stats, (bf*)abuf);
    return launch_k(bn_act_kernel<float>, colgrid, blk, 0, st, pdl, xin, ga, be, B, d, stats, (float*)abuf);
  };

  int ts_slot = 0;
  if (m.profile_ts > 0 && (int)m.ts_kind.size() < m.profile_ts) m.ts_kind.resize(m.profile_ts);
  auto gdbg = [&](int kind) -> int {   // launch slot for the device-clock timing
    if (m.profile_ts <= 0 || m.ts_buf == nullptr || ts_slot >= m.profile_ts) return 0;
    m.ts_kind[ts_slot] = kind;
    return ((++ts_slot) << 8) | (m.profile_ts_dep == 1 ? 8 : 0) | (m.profile_ts_dep == 2 ? 16 : 0);
  };
  int kb = 0;             // backward index: the k-th gradient Block node
  int gcur = 0;           // gq buffer holding the bf16 copy of the current upstream gradient
  int ev_i = 0;
  std::vector<int> dw_event(n + 2, -1);   // sync_ev index recorded after dW of backward k
  // data-parallel buckets: layers [lo, hi] are reduced after layer lo's backward
  int bucket_hi = n - 1;
  const int64_t per_layer = (int64_t)Wl * (bf16 ? 2 : 4);
  const int bucket_layers =
      comm ? (int)std::max<int64_t>(1, std::min<int64_t>(n, comm->bucket_bytes / per_layer)) : 0;
  int cev_i = 0;

  // ---- option overlap (reading A24): after the first mirror, V' alternates mirror runs M_r and
  // gradient runs N_r.  M_r runs on s3 as soon as M_{r-1} and N_{r-2} are done, i.e. concurrently
  // with N_{r-1}; N_r waits for M_r.  Enabled only when the plan makes that sound: no tag written
  // by M_r is touched by N_{r-1}, no tag written by N_{r-1} is read by M_r (SLM_ALLOC_MIRROR_PARITY
  // plans satisfy it; other plans run sequentially).
  std::vector<int> run_of(ops.size(), -1);
  std::vector<char> is_m(ops.size(), 0);
  bool ov = false;
  int n_runs = 0;
  if (fz && side && m.overlap && m.s3 && !m.poison) {
    size_t i = 0;
    auto mir = [&](size_t k) { return ops[k].type == 0 && p->kind[ops[k].node] == SLM_KIND_MIRROR; };
    while (i < ops.size() && !mir(i)) ++i;
    int r = -1;
    bool prev = false;
    for (; i < ops.size(); ++i) {
      const bool im = mir(i);
      if (im && !prev) ++r;
      run_of[i] = r;
      is_m[i] = im;
      prev = im;
    }
    n_runs = r + 1;
    std::vector<std::set<int>> mw(n_runs), mr(n_runs), nw(n_runs), nrd(n_runs);
    for (size_t k = 0; k < ops.size(); ++k) {
      if (run_of[k] < 0) continue;
      const int q = run_of[k];
      (is_m[k] ? mw : nw)[q].insert(ops[k].out_tag);
      (is_m[k] ? mr : nrd)[q].insert(ops[k].in_tag);
      if (ops[k].aux_tag >= 0) (is_m[k] ? mr : nrd)[q].insert(ops[k].aux_tag);
    }
    ov = n_runs > 1;
    for (int q = 1; q < n_runs && ov; ++q) {
      for (int t : mw[q])
        if (nw[q - 1].count(t) || nrd[q - 1].count(t)) ov = false;
      for (int t : nw[q - 1])
        if (mr[q].count(t)) ov = false;
    }
    while (ov && m.ov_ev.size() < (size_t)(2 * n_runs + 2)) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      m.ov_ev.push_back(e);
    }
  }
  m.last_overlap = ov;
  // fused lowering: the bf16 operand a = ReLU(BN(x)) of the next forward Block lives in one of two
  // buffers per stream (a Block reads one and writes the other); node = the x node it belongs to
  struct ActState {
    int node = -1, cur = 0;
  } act_main, act_rec;
  bf* act_ptr[2][2] = {{(bf*)(w + L.act[0]), (bf*)(w + L.act[1])}, {(bf*)(w + L.act3[0]), (bf*)(w + L.act3[1])}};
  int abuf_node = -1;   // basic lowering: node whose operand is resident in abuf

  // debug option poison ("ad hoc application ... can lead to errors"): after the op
  // that reads a value for the last time in V', its pool tag is filled with NaN (0xFF bytes), so
  // a plan that lets a later op read a recycled slot it should not see produces NaN instead of
  // silently wrong numbers.  Runs with the sequential schedule (one stream).
  std::vector<int> last_read;
  if (m.poison) {
    last_read.assign(p->kind.size(), -1);
    for (size_t i = 0; i < ops.size(); ++i) {
      last_read[ops[i].in_node] = (int)i;
      if (ops[i].aux_node >= 0) last_read[ops[i].aux_node] = (int)i;
    }
  }
  auto poison_after = [&](size_t oi) -> slm_status {
    if (!m.poison) return SLM_OK;
    const Op& o = ops[oi];
    for (int v : {o.in_node, o.aux_node}) {
      if (v < 0 || last_read[v] != (int)oi) continue;
      const int t = p->node_tag[v];
      if (t < 0 || p->tag_offset[t] < 0 || t == o.out_tag) continue;   // caller buffer or overwritten in place
      CK(cudaMemsetAsync((uint8_t*)pool + p->tag_offset[t], 0xFF, (size_t)p->tag_size[t], st));
      ++nl;
    }
    return SLM_OK;
  };

  for (size_t oi = 0; oi < ops.size(); ++oi) {
    if (oi > 0 && (s = poison_after(oi - 1)) != SLM_OK) return s;
    const Op& o = ops[oi];
    const int l = o.layer;
    if (ov && run_of[oi] >= 0 && (oi == 0 || run_of[oi - 1] != run_of[oi] || is_m[oi - 1] != is_m[oi])) {
      const int r = run_of[oi];
      if (is_m[oi]) {            // start of M_r on s3: st holds everything through N_{r-1}
        CK(cudaEventRecord(m.ov_ev[2 * r], st));   // E_N[r-1] (r = 0: the forward prefix)
        if (r == 0) CK(cudaStreamWaitEvent(m.s3, m.ov_ev[0], 0));
        if (r >= 2) CK(cudaStreamWaitEvent(m.s3, m.ov_ev[2 * (r - 1)], 0));   // E_N[r-2]
      } else {                   // start of N_r on st: M_r done
        CK(cudaEventRecord(m.ov_ev[2 * r + 1], m.s3));
        CK(cudaStreamWaitEvent(st, m.ov_ev[2 * r + 1], 0));
      }
    }
    if (o.type == 0) {  // ---------------- forward / mirror Block_l
      const float* xin = X(o.in_tag);
      float* xout = X(o.out_tag);
      if (fz) {
        const bool on3 = ov && is_m[oi];
        cudaStream_t fs = on3 ? m.s3 : st;
        ActState& as = on3 ? act_rec : act_main;
        bf* const* ap = act_ptr[on3 ? 1 : 0];
        if (as.node != o.in_node) {   // K1: a_l from x_l (first Block of a run)
          pbeg(fs);
          CK(launch_k1(B, bsh, xin, gam + (size_t)l * d, bet + (size_t)l * d, d, ap[as.cur], fs, pdl));
          pend(SLM_K_BN_ACT, fs);
          ++nl;
        }
        const CUtensorMap* xm;
        int xrow;
        if ((s = xsrc(xin, &xm, &xrow)) != SLM_OK) return s;
        BlkArgs a{};
        a.d = d;
        a.a_row0 = l * d;
        a.pf_row0 = l + 1 < n ? (l + 1) * d : -1;
        a.x_row0 = xrow;
        a.out = xout;
        a.bias = bvec + (size_t)l * d;
        a.gamma = l + 1 < n ? gam + (size_t)(l + 1) * d : nullptr;
        a.beta = l + 1 < n ? bet + (size_t)(l + 1) * d : nullptr;
        a.a_out = ap[as.cur ^ 1];
        a.dbg = gdbg(SLM_K_GEMM_FWD);
        pbeg(fs);
        if ((s = launch_blk(B, bsh, false, m.mW_K64, (on3 ? m.mAct3 : m.mAct)[as.cur], on3 ? m.mPf3 : m.mPf, *xm, a, fs,
                            pdl)) != SLM_OK)
          return s;
        pend(SLM_K_GEMM_FWD, fs);
        as.cur ^= 1;
        as.node = a.gamma ? o.node : -1;
        ++nl;
      } else {
        if (abuf_node != o.in_node) {
          pbeg(st);
          CK(bn_act(xin, l));
          pend(SLM_K_BN_ACT, st);
          ++nl;
        }
        pbeg(st);
        if (tc) {
          slmk::EpiResid epi{xout, xin, bvec + (size_t)l * d, d};
          if ((s = launch_tc_bn<slmk::EpiResid, false, false, true>(m.bn_fwd, 1, m.mW_K, m.mA_K, d, B, d, l * d, 0,
                                                                    epi, st, pdl)) != SLM_OK)
            return s;
        } else if (bf16) {
          CK(simt_gemm((const bf*)abuf, (long)d, 1L, (const bf*)m.d.W + l * Wl, (long)d, 1L, xout, (long)d, B, d, d,
                       xin, bvec + (size_t)l * d, true));
        } else {
          CK(simt_gemm((const float*)abuf, (long)d, 1L, (const float*)m.d.W + l * Wl, (long)d, 1L, xout, (long)d, B,
                       d, d, xin, bvec + (size_t)l * d, true));
        }
        pend(SLM_K_GEMM_FWD, st);
        abuf_node = -1;
        ++nl;
      }
    } else if (o.type == 1) {  // ---------------- loss
      pbeg(st);
      CK(launch_k(ce_fwd_kernel, dim3(B), blk, 0, st, pdl, (const float*)X(o.in_tag), labels, d, rowloss));
      CK(launch_k(ce_reduce_kernel, dim3(1), blk, 0, st, pdl, (const float*)rowloss, B, inv_bg, X(o.out_tag)));
      pend(SLM_K_CE, st);
      nl += 2;
    } else if (o.type == 2) {  // ---------------- gradient of the loss
      float* dxn = X(o.out_tag);
      pbeg(st);
      if (bf16)
        CK(launch_k(ce_bwd_kernel<bf>, dim3(B), blk, 0, st, pdl, (const float*)X(o.in_tag), labels, d, inv_bg, dxn,
                    gq[0]));
      else
        CK(launch_k(ce_bwd_kernel<float>, dim3(B), blk, 0, st, pdl, (const float*)X(o.in_tag), labels, d, inv_bg,
                    dxn, (float*)nullptr));
      CK(launch_k(colsum_kernel, colgrid, blk, 0, st, pdl, (const float*)dxn, B, d, m.d.db + (size_t)(n - 1) * d));
      pend(SLM_K_CE, st);
      gcur = 0;
      nl += 2;
    } else {  // ---------------- backward of Block_l
      const float* g = X(o.in_tag);
      const float* xl = X(o.aux_tag);
      float* dxl = X(o.out_tag);
      float* dbp = l > 0 ? m.d.db + (size_t)(l - 1) * d : nullptr;
      const float* ga = gam + (size_t)l * d;
      const float* be = bet + (size_t)l * d;
      float* dga = m.d.dgamma + (size_t)l * d;
      float* dbe = m.d.dbeta + (size_t)l * d;
      if (fz) {
        const int gnext = (gcur + 1) % kNG, abi = kb % kNA;
        // the Block overwrites gq[(k+1) % kNG] and ab[k % kNA], last read by dW of backward k - kNA
        if (side && kb >= kNA && dw_event[kb - kNA] >= 0)
          CK(cudaStreamWaitEvent(st, m.sync_ev[dw_event[kb - kNA]], 0));
        const CUtensorMap* xm;
        int xrow;
        if ((s = xsrc(xl, &xm, &xrow)) != SLM_OK) return s;
        BlkArgs a{};
        a.d = d;
        a.a_row0 = l * d;
        a.pf_row0 = l > 0 ? (l - 1) * d : -1;
        a.x_row0 = xrow;
        a.g = g;
        a.out = dxl;
        a.gamma = ga;
        a.beta = be;
        a.a_out = ab[abi];
        a.gq_out = gq[gnext];
        a.dgamma = dga;
        a.dbeta = dbe;
        a.db_prev = dbp;
        a.dbg = gdbg(SLM_K_GEMM_DX);
        pbeg(st);
        if ((s = launch_blk(B, bsh, true, m.mW_MN, m.mG_K[gcur], m.mPf, *xm, a, st, pdl)) != SLM_OK) return s;
        pend(SLM_K_GEMM_DX, st);
        // dW_l[f_out][f_in] = sum_b g[b][f_out] a[b][f_in]  (second stream)
        cudaStream_t sw = st;
        if (side) {
          cudaEvent_t ef = m.sync_ev[ev_i++];
          CK(cudaEventRecord(ef, st));
          CK(cudaStreamWaitEvent(m.s2, ef, 0));
          sw = m.s2;
        }
        pbeg(sw);
        slmk::EpiStoreBF16Tma e2{l * d};
        if ((s = launch_tc_bn<slmk::EpiStoreBF16Tma, true, true, false>(m.bn_dw, 1, m.mAb_MN[abi], m.mG_MN[gcur], d, d,
                                                                        B, 0, 0, e2, sw, pdl && !side,
                                                                        gdbg(SLM_K_GEMM_DW), &m.mdW_st)) != SLM_OK)
          return s;
        pend(SLM_K_GEMM_DW, sw);
        if (side) {
          dw_event[kb] = ev_i;
          CK(cudaEventRecord(m.sync_ev[ev_i++], m.s2));
        }
        gcur = gnext;
        nl += 2;
      } else {
        pbeg(st);
        CK(bn_act(xl, l));
        pend(SLM_K_BN_ACT, st);
        if (tc) {
          slmk::EpiStoreF32 e1{da, d};
          pbeg(st);
          if ((s = launch_tc_bn<slmk::EpiStoreF32, true, false, true>(m.bn_dx, 1, m.mW_MN, m.mG_K[gcur], d, B, d,
                                                                      l * d, 0, e1, st, pdl)) != SLM_OK)
            return s;
          pend(SLM_K_GEMM_DX, st);
          slmk::EpiStoreBF16 e2{(bf*)m.d.dW + l * Wl, d};
          pbeg(st);
          if ((s = launch_tc_bn<slmk::EpiStoreBF16, true, true, false>(m.bn_dw, 1, m.mA_MN, m.mG_MN[gcur], d, d, B,
                                                                       0, 0, e2, st, pdl)) != SLM_OK)
            return s;
          pend(SLM_K_GEMM_DW, st);
        } else if (bf16) {
          const bf* gqp = gq[gcur];
          pbeg(st);
          CK(simt_gemm(gqp, (long)d, 1L, (const bf*)m.d.W + l * Wl, 1L, (long)d, da, (long)d, B, d, d,
                       (const float*)nullptr, (const float*)nullptr, false));
          pend(SLM_K_GEMM_DX, st);
          pbeg(st);
          CK(simt_gemm(gqp, 1L, (long)d, (const bf*)abuf, 1L, (long)d, (bf*)m.d.dW + l * Wl, (long)d, d, d, B,
                       (const float*)nullptr, (const float*)nullptr, false));
          pend(SLM_K_GEMM_DW, st);
        } else {
          pbeg(st);
          CK(simt_gemm(g, (long)d, 1L, (const float*)m.d.W + l * Wl, 1L, (long)d, da, (long)d, B, d, d,
                       (const float*)nullptr, (const float*)nullptr, false));
          pend(SLM_K_GEMM_DX, st);
          pbeg(st);
          CK(simt_gemm(g, 1L, (long)d, (const float*)abuf, 1L, (long)d, (float*)m.d.dW + l * Wl, (long)d, d, d, B,
                       (const float*)nullptr, (const float*)nullptr, false));
          pend(SLM_K_GEMM_DW, st);
        }
        pbeg(st);
        if (bf16)
          CK(launch_k(bn_bwd_kernel<bf>, colgrid, blk, 0, st, pdl, (const float*)da, xl, (const float*)stats, ga, be,
                      g, dxl, B, d, dga, dbe, dbp, gq[(gcur + 1) % kNG]));
        else
          CK(launch_k(bn_bwd_kernel<float>, colgrid, blk, 0, st, pdl, (const float*)da, xl, (const float*)stats, ga,
                      be, g, dxl, B, d, dga, dbe, dbp, (float*)nullptr));
        pend(SLM_K_BN_BWD, st);
        gcur = (gcur + 1) % kNG;
        abuf_node = -1;
        nl += 4;
      }
      // data-parallel: all-reduce the bucket [l, bucket_hi] once its last layer is done
      if (comm && (bucket_hi - l + 1 >= bucket_layers || l == 0)) {   // (world 1: identity, same path)
        const int lo = l, cnt = bucket_hi - l + 1;
        cudaEvent_t ev = comm->events[cev_i++ % comm->events.size()];
        CK(cudaEventRecord(ev, side ? m.s2 : st));
        CK(cudaStreamWaitEvent(comm->stream, ev, 0));
        cudaEvent_t ev1 = comm->events[cev_i++ % comm->events.size()];
        CK(cudaEventRecord(ev1, st));
        CK(cudaStreamWaitEvent(comm->stream, ev1, 0));
        g_nccl.GroupStart();
        int r = 0;
        r |= g_nccl.AllReduce((uint8_t*)m.d.dW + (size_t)lo * per_layer, (uint8_t*)m.d.dW + (size_t)lo * per_layer,
                              (size_t)cnt * Wl, bf16 ? NCCL_BF16 : NCCL_FLOAT32, NCCL_SUM, comm->comm, comm->stream);
        r |= g_nccl.AllReduce(m.d.dgamma + (size_t)lo * d, m.d.dgamma + (size_t)lo * d, (size_t)cnt * d,
                              NCCL_FLOAT32, NCCL_SUM, comm->comm, comm->stream);
        r |= g_nccl.AllReduce(m.d.dbeta + (size_t)lo * d, m.d.dbeta + (size_t)lo * d, (size_t)cnt * d, NCCL_FLOAT32,
                              NCCL_SUM, comm->comm, comm->stream);
        g_nccl.GroupEnd();
        if (r) {
          set_error("ncclAllReduce failed");
          return SLM_E_NCCL;
        }
        bucket_hi = l - 1;
      }
      ++kb;
    }
  }
  // join the dW stream
  if (side && kb > 0 && dw_event[kb - 1] >= 0) CK(cudaStreamWaitEvent(st, m.sync_ev[dw_event[kb - 1]], 0));
  if (comm) {
    // db (all layers; db_0 is final after the last backward) and the loss, then join
    cudaEvent_t ev = comm->events[cev_i++ % comm->events.size()];
    CK(cudaEventRecord(ev, st));
    CK(cudaStreamWaitEvent(comm->stream, ev, 0));
    g_nccl.GroupStart();
    int r = 0;
    r |= g_nccl.AllReduce(m.d.db, m.d.db, (size_t)n * d, NCCL_FLOAT32, NCCL_SUM, comm->comm, comm->stream);
    r |= g_nccl.AllReduce(loss, loss, 1, NCCL_FLOAT32, NCCL_SUM, comm->comm, comm->stream);
    g_nccl.GroupEnd();
    if (r) {
      set_error("ncclAllReduce failed");
      return SLM_E_NCCL;
    }
    cudaEvent_t ev2 = comm->events[cev_i++ % comm->events.size()];
    CK(cudaEventRecord(ev2, comm->stream));
    CK(cudaStreamWaitEvent(st, ev2, 0));
  }
  CK(cudaGetLastError());
  if (launches) *launches = nl;
  m.ts_used = ts_slot;
  return SLM_OK;
}

slm_status check_plan_model(const slm_plan* p, const slm_model* m) {
  if (!p || !m) {
    set_error("null plan/model");
    return SLM_E_ARG;
  }
  if (m->kind == SLM_MODEL_OPS) {
    const slm_ops_model& o = m->od;
    bool ok = p->graph_kind == -1 && p->n_fwd == (int)o.op.size();
    for (int v = 0; ok && v < p->n_fwd; ++v) ok = p->op[v] == o.op[v] && p->out_bytes[v] == o.out_bytes[v];
    if (!ok) {
      set_error("plan was not built for this op graph");
      return SLM_E_SHAPE;
    }
    return SLM_OK;
  }
  if (m->kind == SLM_MODEL_LSTM) {
    const slm_lstm_desc& d = m->ld;
    if (p->graph_kind != SLM_MODEL_LSTM || p->dims[0] != d.n_layers || p->dims[1] != d.steps ||
        p->dims[2] != d.batch || p->dims[3] != d.hidden || p->dims[4] != d.n_in) {
      set_error("plan was not built for this LSTM's dims (use slm_graph_lstm)");
      return SLM_E_SHAPE;
    }
    return SLM_OK;
  }
  if (p->graph_kind != SLM_MODEL_CHAIN || p->dims[0] != m->d.n_layers || p->dims[1] != m->d.batch ||
      p->dims[2] != m->d.width) {
    set_error("plan was not built for this chain's dims (use slm_graph_chain)");
    return SLM_E_SHAPE;
  }
  return SLM_OK;
}

}  // namespace
