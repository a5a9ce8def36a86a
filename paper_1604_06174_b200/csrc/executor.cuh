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
                     int a_row0, int b_row0, Epi epi, cudaStream_t st, bool pdl, int dbg, int pf_row0 = -1) {
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
               dbg, pf_row0));
  return SLM_OK;
}

// c: tensor map of the output for TMA-store epilogues (Epi::kTma), else ignored.
// cg = 2: CTA-pair GEMM (cta_group::2); a K-major B map must then have box rows bn / 2.
template <class Epi, bool AMN, bool BMN, bool PRE>
slm_status launch_tc_bn(int bn, int split, const CUtensorMap& a, const CUtensorMap& b, int M, int N, int K,
                        int a_row0, int b_row0, Epi epi, cudaStream_t st, bool pdl, int dbg = 0,
                        const CUtensorMap* c = nullptr, int cg = 1, int pf = -1) {
  const CUtensorMap& cm = c ? *c : a;
  if (cg == 2) {
    switch (bn) {
      case 128:
        return launch_tc<128, AMN, BMN, PRE, Epi, 2>(a, b, cm, M, N, K, split, a_row0, b_row0, epi, st, pdl, dbg, pf);
      case 256:
        return launch_tc<256, AMN, BMN, PRE, Epi, 2>(a, b, cm, M, N, K, split, a_row0, b_row0, epi, st, pdl, dbg, pf);
    }
    set_error("unsupported CTA-pair GEMM N tile " + std::to_string(bn));
    return SLM_E_UNSUPPORTED;
  }
  switch (bn) {
    case 32:
      if (!BMN) return launch_tc<32, AMN, BMN, PRE>(a, b, cm, M, N, K, split, a_row0, b_row0, epi, st, pdl, dbg, pf);
      break;
    case 64: return launch_tc<64, AMN, BMN, PRE>(a, b, cm, M, N, K, split, a_row0, b_row0, epi, st, pdl, dbg, pf);
    case 128: return launch_tc<128, AMN, BMN, PRE>(a, b, cm, M, N, K, split, a_row0, b_row0, epi, st, pdl, dbg, pf);
    case 256: return launch_tc<256, AMN, BMN, PRE>(a, b, cm, M, N, K, split, a_row0, b_row0, epi, st, pdl, dbg, pf);
  }
  set_error("unsupported GEMM N tile " + std::to_string(bn));
  return SLM_E_UNSUPPORTED;
}

// forward Block as one cluster kernel (blk_cluster.cuh), split-K SK in {2, 4}
template <int SK>
slm_status launch_blk_cl_t(const CUtensorMap& w, const CUtensorMap& a, int d, int l, int n, const float* xin,
                           float* xout, const float* bias, const float* gam, const float* bet, float* stats,
                           __nv_bfloat16* aout, cudaStream_t st, bool pdl, int dbg) {
  using C = slmk::BlkClCfg<SK>;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(slmk::blk_fwd_cl_kernel<SK>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  CK(launch_kc(slmk::blk_fwd_cl_kernel<SK>, dim3(d / 128 * C::CL), dim3(C::THREADS), C::SMEM, st, pdl, C::CL, w, a, d,
               l, n, xin, xout, bias, gam, bet, stats, aout, dbg));
  return SLM_OK;
}
slm_status launch_blk_cl(int sk, const CUtensorMap& w, const CUtensorMap& a, int d, int l, int n, const float* xin,
                         float* xout, const float* bias, const float* gam, const float* bet, float* stats,
                         __nv_bfloat16* aout, cudaStream_t st, bool pdl, int dbg) {
  (void)sk;
  return launch_blk_cl_t<2>(w, a, d, l, n, xin, xout, bias, gam, bet, stats, aout, st, pdl, dbg);
}
cudaError_t launch_bn_act_cl(int sk, const float* x, const float* gam, const float* bet, int d, float* stats,
                             __nv_bfloat16* a, cudaStream_t st, bool pdl) {
  (void)sk;
  return launch_k(slmk::bn_act_cl_kernel<2>, dim3(d / slmk::BlkClCfg<2>::FK), dim3(256), 0, st, pdl, x, gam, bet, d,
                  stats, a);
}

// persistent forward run (fwd_persist.cuh): B in {64, 128, 256}, S in {4, 8, 16}
template <int B_, int S_>
slm_status launch_fwd_seg_t(const CUtensorMap& w, const CUtensorMap& a, const slmk::FwdSegArgs& A, int grid,
                            cudaStream_t st, bool pdl) {
  using C = slmk::FwdSegCfg<B_, S_>;
  auto kern = slmk::fwd_seg_kernel<B_, S_>;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  CK(launch_k(kern, dim3(grid), dim3(C::THREADS), C::SMEM, st, pdl, w, a, A));
  return SLM_OK;
}
slm_status launch_fwd_seg(int B, int S, const CUtensorMap& w, const CUtensorMap& a, const slmk::FwdSegArgs& A,
                          int grid, cudaStream_t st, bool pdl) {
#define SLM_FS(B_, S_) \
  if (B == B_ && S == S_) return launch_fwd_seg_t<B_, S_>(w, a, A, grid, st, pdl);
#define SLM_FS_B(B_) SLM_FS(B_, 4) SLM_FS(B_, 8) SLM_FS(B_, 16)
  SLM_FS_B(64) SLM_FS_B(128) SLM_FS_B(256)
#undef SLM_FS_B
#undef SLM_FS
  set_error("unsupported persistent forward configuration");
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

// register-resident BN kernels: compile-time rows per warp R = B/32, split count NS and features
// per CTA F (option bn_feat: 16 -> 512-thread CTAs, 8 -> 256-thread CTAs, same arithmetic)
template <int R, int NS, int F>
cudaError_t launch_act_rk(cudaStream_t st, bool pdl, int d, const float* xin, const float* P, unsigned pslice,
                          const float* bias, float* xout, const float* ga, const float* be, float* stats,
                          __nv_bfloat16* a) {
  return launch_k(slmk::bn_act_rk<__nv_bfloat16, R, NS, F>, dim3(d / F), dim3(F * 32), 0, st, pdl, xin, P, pslice, bias,
                  xout, ga, be, d, stats, a);
}
cudaError_t act_rk(int R, int ns, int F, cudaStream_t st, bool pdl, int d, const float* xin, const float* P,
                   unsigned pslice, const float* bias, float* xout, const float* ga, const float* be, float* stats,
                   __nv_bfloat16* a) {
#define SLM_ACT(R_, NS_, F_)                                                                                 \
  if (R == R_ && ns == NS_ && F == F_)                                                                      \
    return launch_act_rk<R_, NS_, F_>(st, pdl, d, xin, P, pslice, bias, xout, ga, be, stats, a);
#define SLM_ACT_R(R_, F_) SLM_ACT(R_, 0, F_) SLM_ACT(R_, 1, F_) SLM_ACT(R_, 2, F_) SLM_ACT(R_, 4, F_) SLM_ACT(R_, 8, F_)
  SLM_ACT_R(2, 16) SLM_ACT_R(4, 16) SLM_ACT_R(8, 16) SLM_ACT_R(8, 8)
#undef SLM_ACT_R
#undef SLM_ACT
  return cudaErrorInvalidValue;
}
// vectorised K1 / finalize (option bn_vec): B in {128, 256}
cudaError_t act_v4(int B, int ns, cudaStream_t st, bool pdl, int d, const float* xin, const float* P,
                   unsigned pslice, const float* bias, float* xout, const float* ga, const float* be, float* stats,
                   __nv_bfloat16* a) {
#define SLM_AV(R_, NS_)                                                                                      \
  if (B == 128 * R_ && ns == NS_)                                                                           \
    return launch_k(slmk::bn_act_v4<R_, NS_>, dim3(d / 16), dim3(512), 0, st, pdl, xin, P, pslice, bias, xout, ga, \
                    be, d, stats, a);
#define SLM_AV_R(R_) SLM_AV(R_, 0) SLM_AV(R_, 1) SLM_AV(R_, 2) SLM_AV(R_, 4) SLM_AV(R_, 8)
  SLM_AV_R(1) SLM_AV_R(2)
#undef SLM_AV_R
#undef SLM_AV
  return cudaErrorInvalidValue;
}

template <int R, int NS, int F>
cudaError_t launch_bwd_rk(cudaStream_t st, bool pdl, int d, const float* P, unsigned pslice, const float* x,
                          const float* ga, const float* be, const float* g, float* dx, float* dga, float* dbe,
                          float* dbp, __nv_bfloat16* gq, __nv_bfloat16* a) {
  return launch_k(slmk::bn_bwd_rk<__nv_bfloat16, __nv_bfloat16, R, NS, F>, dim3(d / F), dim3(F * 32), 0, st, pdl, P,
                  pslice, x, ga, be, g, dx, d, dga, dbe, dbp, gq, a);
}
cudaError_t bwd_rk(int R, int ns, int F, cudaStream_t st, bool pdl, int d, const float* P, unsigned pslice,
                   const float* x, const float* ga, const float* be, const float* g, float* dx, float* dga, float* dbe,
                   float* dbp, __nv_bfloat16* gq, __nv_bfloat16* a) {
#define SLM_BWD(R_, NS_, F_)                                                                                 \
  if (R == R_ && ns == NS_ && F == F_)                                                                      \
    return launch_bwd_rk<R_, NS_, F_>(st, pdl, d, P, pslice, x, ga, be, g, dx, dga, dbe, dbp, gq, a);
#define SLM_BWD_R(R_, F_) SLM_BWD(R_, 1, F_) SLM_BWD(R_, 2, F_) SLM_BWD(R_, 4, F_) SLM_BWD(R_, 8, F_)
  SLM_BWD_R(2, 16) SLM_BWD_R(4, 16) SLM_BWD_R(8, 16) SLM_BWD_R(8, 8)
#undef SLM_BWD_R
#undef SLM_BWD
  return cudaErrorInvalidValue;
}

}  // namespace

constexpr int kMaxLag = 8;

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

// LSTM executor state (executor_lstm.cuh): tensor maps bound to the weights / workspace and
// the Sum node's pool-offset table
struct LstmMaps {
  // per layer: W_l K-major / MN-major, forward operand [B][K_l], the time-chunk rings of the
  // backward operands (op K-major/MN-major, d_pre K-major/MN-major), the dX partials
  std::vector<CUtensorMap> wK, wK32, wMN, opK, opRK, opRMN, dpRK, dpRMN, pX, pG, pGm, pXd;   // partials of layer l's streams
  CUtensorMap woK, woMN, hopRK, hopRMN, dlRK, dlRMN, pL, pH, hfK[2][2], hopRKb[3], dlRKb[3], pHB;            // pL / pH over the head's
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

struct slm_model {
  slm_chain_desc d{};
  slm_lstm_desc ld{};
  slm_lstm_state lst;
  int kind = SLM_MODEL_CHAIN;
  int use_graph = 1;
  int gemm_impl = 0;      // 0 tcgen05 (bf16), 1 SIMT
  int pdl = 1;            // programmatic dependent launch between the step's kernels
  int fused = 1;          // fused lowering (split-K partials reduced in the BN kernels)
  int dw_stream = 1;      // dW GEMMs on a second stream
  int bn_fwd = 64, bn_dx = 64, bn_dw = 256;  // N tiles (basic lowering; the fused one uses bn = B)
  int sk_fwd = 0, sk_dx = 0;                  // split-K of the fused forward / dX GEMMs (0 = auto)
  int fused_bn = 0;                           // N tile of the fused forward / dX GEMMs (0 = batch)
  int cta_pair = 0;                           // fused forward / dX GEMMs as CTA pairs (cta_group::2)
  int bn_vec = 0;                             // vectorised forward BN kernel (bn_act_v4; another reduction order;
                                              // measured slower at C2: 14.3 vs 13.1 us per forward Block)
  int bn_feat = 16;                           // features per CTA of the BN kernels (16 | 8; same bits; 8 measured slower)
  int tile_dx = 0, tile_mir = 0;              // N tiles of the dX / recompute-stream GEMMs (0 = fused_bn rule)
  int blk_cluster = 0;                        // forward Block as one cluster kernel (blk_cluster.cuh; B = 256;
                                              // measured 35.2 vs 35.3 ms/step at C2: within noise, default off)
  int dw_lag = 2;                             // dW ring depth: layers the dW stream may lag the dX chain (2..8)
  int dw_tma = 1;                             // dW epilogue: bf16 TMA bulk stores (0 = per-thread stores)
  int s3_prio = 0;                            // priority of the recompute stream above the lowest (set before the first step)
  int overlap = 1;                            // segment recompute on its own stream, concurrent with the backward of
                                              // the next segment, when the plan allows it (SLM_ALLOC_MIRROR_PARITY)
  int persist_dbg = 0;                        // persistent kernel phase stamps (scripts/persist_phases.py)
  int persist = 0;                            // runs of forward / mirror Blocks as one persistent kernel (fwd_persist.cuh;
                                              // measured slower at C2: 47.4 / 50.9 ms/step vs 43.2)
  int lstm_streams = 2;                       // LSTM: layer wavefront over L+1 streams (2: + L mirror streams)
  int lstm_grid = 1;                          // LSTM element-wise grids sized to the work
  int l2_prefetch = 0;                        // chain GEMMs pull the next layer's W tile into L2 (measured: no gain)
  int lstm_sk = 1;                            // LSTM: split-K of the gates GEMMs (0 = auto; 1 measured best with the wavefront)
  int lstm_fuse_cell = 0;                     // LSTM: gates + cell in the GEMM epilogue (needs lstm_sk = 1; measured slower)
  int lstm_skx = 4;                           // LSTM: split-K of the dX GEMMs (0 = auto; 4 measured best with the wavefront)
  // tensor maps bound to the current workspace / weights
  const void* maps_ws = nullptr;
  int maps_key = -1;
  CUtensorMap mW_K, mW_MN, mA_K, mA_K3, mP3, mdW_st, mA_Kf, mA_MN, mG_K[kMaxLag + 1], mG_MN[kMaxLag + 1], mAb_MN[kMaxLag], mP;
  std::map<GraphKey, cudaGraphExec_t> graphs;
  int64_t last_launches = 0;
  bool last_overlap = false;           // the last enqueued step ran its recompute on s3
  cudaStream_t s2 = nullptr;           // second stream (dW)
  cudaStream_t s3 = nullptr;           // recompute stream (option overlap)
  std::vector<cudaEvent_t> ov_ev;      // its fork/join events
  cudaStream_t s1 = nullptr;           // high-priority critical-path stream (option prio)
  cudaEvent_t prio_ev[2] = {nullptr, nullptr};
  int prio = 0;                        // 1: critical path on s1 (highest priority), dW on s2 (lowest)
  std::vector<cudaEvent_t> sync_ev;    // fork/join events (reused every step)
  // profile_ts: device-clock (%globaltimer) start/end of every CTA of the first profile_ts GEMM
  // launches of a step, in the caller's buffer ts_buf ([slot][1024][2] uint64, zeroed)
  int profile_ts = 0;
  int profile_ts_dep = 0;   // 1: stamp the start after the dependency wait (ts_dep)
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
    if (s1) cudaStreamDestroy(s1);
    for (auto e : prio_ev)
      if (e) cudaEventDestroy(e);
  }
};

namespace {

bool tc_ok(const slm_model& m) {
  const int B = m.d.batch, d = m.d.width;
  return m.d.dtype == SLM_BF16 && m.gemm_impl == 0 && d % 128 == 0 && B % 64 == 0 && B <= 4096 &&
         B % m.bn_fwd == 0 && B % m.bn_dx == 0 && d % m.bn_dw == 0;
}
// the fused lowering: full batch per GEMM tile (N = B <= 256), split-K partials
bool fused_ok(const slm_model& m) {
  const int B = m.d.batch;
  return tc_ok(m) && m.fused && (B == 64 || B == 128 || B == 256) && m.d.width % 256 == 0;
}
// N tile of the fused GEMMs: 128 (measured best at C2: 43.7 ms/step vs 45.1 with the full
// batch of 256 per tile; profiles/README.md sweep), or the batch when smaller
int fused_n(const slm_model& m) { return m.fused_bn > 0 ? m.fused_bn : std::min(m.d.batch, 128); }
// N tiles of the dX GEMMs and of the recompute-stream mirror GEMMs (options tile_dx, tile_mir; 0 =
// fused_n).  The N tile does not change any element's accumulation order (one tcgen05 MMA per
// K = 16 step, K blocks in order), so mirrors with another tile reproduce the forward's bits.
int dx_tile(const slm_model& m) { return m.tile_dx > 0 ? std::min(m.tile_dx, m.d.batch) : fused_n(m); }
int mir_tile(const slm_model& m) { return m.tile_mir > 0 ? std::min(m.tile_mir, m.d.batch) : fused_n(m); }
// split-K factor: as many K slices as keep <= ~148 CTAs and >= 64 of K per slice
int auto_split(int M, int K, int req, int n_tiles = 1) {
  if (req > 0) return req;
  const int tiles = M / 128 * n_tiles;
  int s = 1;
  // ~64 CTAs: measured best at C2 (split 4: 44.7 ms/step vs 56.1 with split 8 under PDL — the
  // remaining SMs run the dependent BN kernel's early CTAs and the off-path dW GEMM)
  while (s < 8 && tiles * s * 2 <= 80 && K % (64 * s * 2) == 0) s *= 2;
  return s;
}

// split-K factor S of the persistent forward kernel (fwd_persist.cuh), 0 = not applicable:
// the largest S with (d / 128) x S CTAs <= one per SM, a K slice of 64..256 (all of it resident
// in shared memory)
int persist_split(const slm_model& m) {
  if (!m.persist || !fused_ok(m)) return 0;
  const int d = m.d.width, tiles = d / 128;
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int s : {16, 8, 4})
    if (tiles * s <= sms && d % (s * 64) == 0 && d / s >= 64 && d / s <= 256) return s;
  return 0;
}

// dW lag ring (fused lowering): the dW GEMM of backward k reads ab[k % NA] and gq[k % NG]; bn_bwd of
// backward k overwrites gq[(k+1) % NG] and ab[k % NA], so it waits for dW of backward k - NA
// (NG = NA + 1): NA layers of slack between the dX chain and the dW stream (option dw_lag)
int dw_na(const slm_model& m) { return std::max(2, std::min(kMaxLag, m.dw_lag)); }
int dw_ng(const slm_model& m) { return dw_na(m) + 1; }

struct WsLayout {
  size_t a, stats, gq[kMaxLag + 1], ab[kMaxLag], P, da, rowloss, bar, a3, stats3, P3, total;
  int sk_fwd, sk_dx, sk_persist;
};
WsLayout ws_layout(const slm_model& m) {
  const size_t B = m.d.batch, d = m.d.width;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  WsLayout L{};
  const int nt = fused_ok(m) ? (int)B / fused_n(m) : 1;
  L.sk_fwd = auto_split((int)d, (int)d, m.sk_fwd, nt);
  L.sk_dx = auto_split((int)d, (int)d, m.sk_dx, nt);
  L.sk_persist = persist_split(m);
  size_t off = 0;
  L.a = off;
  off += al(B * d * 4);
  L.stats = off;
  off += al(2 * d * 4);
  for (int i = 0; i < dw_ng(m); ++i) {
    L.gq[i] = off;
    off += al(B * d * 2);
  }
  for (int i = 0; i < dw_na(m); ++i) {
    L.ab[i] = off;
    off += al(B * d * 2);
  }
  L.P = off;
  off += al((size_t)std::max({L.sk_fwd, L.sk_dx, L.sk_persist}) * B * d * 4);
  L.da = off;
  off += al(B * d * 4);
  L.rowloss = off;
  off += al(B * 4);
  L.bar = off;
  off += 128 * 128;
  // the recompute stream's own operand / statistics / partial buffers (option overlap)
  const bool ovw = fused_ok(m) && m.overlap;
  L.a3 = off;
  off += ovw ? al(B * d * 4) : 0;
  L.stats3 = off;
  off += ovw ? al(2 * d * 4) : 0;
  L.P3 = off;
  off += ovw ? al((size_t)L.sk_fwd * B * d * 4) : 0;
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
        ops->push_back({3, orig - 1, p->node_tag[pr[0]], p->node_tag[pr[1]], p->node_tag[v], pr[1], v});
      } else {
        set_error("unsupported gradient op in chain plan");
        return SLM_E_UNSUPPORTED;
      }
    }
  }
  return SLM_OK;
}

slm_status bind_maps(slm_model& m, void* ws) {
  const int key = m.bn_fwd * 7 + m.bn_dx * 131 + m.fused + m.fused_bn * 1009 + m.cta_pair * 100003 + m.persist * 3 +
                  m.overlap * 5 + m.dw_tma * 11 + m.dw_lag * 13 + m.blk_cluster * 17 + m.tile_dx * 19 +
                  m.tile_mir * 23;
  if (m.maps_ws == ws && m.maps_key == key) return SLM_OK;
  const uint64_t B = m.d.batch, d = m.d.width, n = m.d.n_layers;
  WsLayout L = ws_layout(m);
  uint8_t* w = (uint8_t*)ws;
  const bool fz = fused_ok(m);
  // fused: N tile fused_n() (K-major B box rows = tile / cta group)
  const uint32_t fb = (uint32_t)(fused_n(m) / (m.cta_pair ? 2 : 1));
  const uint32_t cgd = m.cta_pair ? 2 : 1;
  const uint32_t bnf = fz ? fb : (uint32_t)m.bn_fwd, bnx = fz ? (uint32_t)dx_tile(m) / cgd : (uint32_t)m.bn_dx;
  slm_status st;
  if ((st = make_map(&m.mW_K, m.d.W, d, n * d, 128)) != SLM_OK) return st;
  if ((st = make_map(&m.mW_MN, m.d.W, d, n * d, 64)) != SLM_OK) return st;
  if ((st = make_map(&m.mA_K, w + L.a, d, B, bnf)) != SLM_OK) return st;
  if (fz && (st = make_map(&m.mA_Kf, w + L.a, d, B, (uint32_t)B)) != SLM_OK) return st;
  if (fz && m.dw_tma && (st = make_map_bf16_store(&m.mdW_st, m.d.dW, d, n * d)) != SLM_OK) return st;
  if (fz && m.overlap) {
    if ((st = make_map(&m.mA_K3, w + L.a3, d, B, (uint32_t)mir_tile(m) / cgd)) != SLM_OK) return st;
    if ((st = make_map_f32(&m.mP3, w + L.P3, d, (uint64_t)L.sk_fwd * B)) != SLM_OK) return st;
  }
  if ((st = make_map(&m.mA_MN, w + L.a, d, B, 64)) != SLM_OK) return st;
  for (int i = 0; i < dw_ng(m); ++i) {
    if ((st = make_map(&m.mG_K[i], w + L.gq[i], d, B, bnx)) != SLM_OK) return st;
    if ((st = make_map(&m.mG_MN[i], w + L.gq[i], d, B, 64)) != SLM_OK) return st;
  }
  for (int i = 0; i < dw_na(m); ++i)
    if ((st = make_map(&m.mAb_MN[i], w + L.ab[i], d, B, 64)) != SLM_OK) return st;
  if ((st = make_map_f32(&m.mP, w + L.P, d, (uint64_t)std::max({L.sk_fwd, L.sk_dx, L.sk_persist}) * B)) != SLM_OK)
    return st;
  m.maps_ws = ws;
  m.maps_key = key;
  return SLM_OK;
}

slm_status ensure_streams(slm_model& m, int n_layers) {
  if (!m.s2) {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&m.s2, cudaStreamNonBlocking, m.prio ? lo : 0));
    if (m.prio) {
      CK(cudaStreamCreateWithPriority(&m.s1, cudaStreamNonBlocking, hi));
      for (auto& e : m.prio_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
  }
  if (m.overlap && !m.s3) {
    // s3_prio = k > 0: the recompute stream k levels above the lowest priority
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&m.s3, cudaStreamNonBlocking, std::max(hi, lo - m.s3_prio)));
  }
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
  const int Bg = m.d.batch_global > 0 ? m.d.batch_global : B;
  const float inv_bg = 1.0f / (float)Bg;
  const WsLayout L = ws_layout(m);
  uint8_t* w = (uint8_t*)ws;
  float* stats = (float*)(w + L.stats);
  void* abuf = w + L.a;
  const int NA = dw_na(m), NG = dw_ng(m);
  bf* gq[kMaxLag + 1];
  bf* ab[kMaxLag];
  for (int i = 0; i < NG; ++i) gq[i] = (bf*)(w + L.gq[i]);
  for (int i = 0; i < NA; ++i) ab[i] = (bf*)(w + L.ab[i]);
  float* P = (float*)(w + L.P);
  const long pslice = (long)B * d;
  float* da = (float*)(w + L.da);
  float* rowloss = (float*)(w + L.rowloss);
  const bool pdl = m.pdl != 0;
  const bool side = fz && m.dw_stream;

  std::vector<Op> ops;
  slm_status s = lower(p, &ops);
  if (s != SLM_OK) return s;
  if (tc && (s = bind_maps(m, ws)) != SLM_OK) return s;
  if (side && (s = ensure_streams(m, n)) != SLM_OK) return s;
  // option prio: the critical path runs on a high-priority internal stream forked from the caller's
  cudaStream_t caller = st;
  const bool use_s1 = side && m.prio && m.s1 != nullptr && st != nullptr;
  if (use_s1) {
    CK(cudaEventRecord(m.prio_ev[0], caller));
    CK(cudaStreamWaitEvent(m.s1, m.prio_ev[0], 0));
    st = m.s1;
  }

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
  // features per CTA of the BN kernels (option bn_feat = 8 only at B = 256)
  auto bnf_ = [&]() { return m.bn_feat == 8 && B == 256 ? 8 : 16; };
  // K1 (optionally fused with the forward finalize from split-K partials)
  auto bn_act = [&](const float* xin, const float* Pp, int nsplit, const float* bias, float* xout, int l,
                    cudaStream_t fs = nullptr, void* fa = nullptr, float* fstats = nullptr) -> cudaError_t {
    const float* ga = l < n ? gam + (size_t)l * d : nullptr;
    const float* be = l < n ? bet + (size_t)l * d : nullptr;
    if (fz && m.bn_vec && (B == 128 || B == 256))
      return act_v4(B, Pp ? nsplit : 0, fs ? fs : st, pdl, d, xin, Pp, (unsigned)pslice, bias, xout, ga, be,
                    fstats ? fstats : stats, (bf*)(fa ? fa : abuf));
    if (fz)
      return act_rk(B / 32, Pp ? nsplit : 0, bnf_(), fs ? fs : st, pdl, d, xin, Pp, (unsigned)pslice, bias, xout, ga, be,
                    fstats ? fstats : stats, (bf*)(fa ? fa : abuf));
    if (bf16)
      return launch_k(bn_act_kernel<bf>, colgrid, blk, 0, st, pdl, xin, ga, be, B, d, stats, (bf*)abuf);
    return launch_k(bn_act_kernel<float>, colgrid, blk, 0, st, pdl, xin, ga, be, B, d, stats, (float*)abuf);
  };

  int ts_slot = 0;
  if (m.profile_ts > 0 && (int)m.ts_kind.size() < m.profile_ts) m.ts_kind.resize(m.profile_ts);
  auto gdbg = [&](int kind) -> int {   // launch slot for the device-clock GEMM timing
    if (m.profile_ts <= 0 || m.ts_buf == nullptr || ts_slot >= m.profile_ts) return 0;
    m.ts_kind[ts_slot] = kind;
    return ((++ts_slot) << 8) | (m.profile_ts_dep ? 8 : 0);
  };
  int abuf_node = -1;     // node whose activation operand a = ReLU(BN(x)) is resident in abuf
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

  // persistent forward runs: grid-barrier counter, zeroed once per step (monotonic within it)
  const int PS = L.sk_persist;
  unsigned* bar = (unsigned*)(w + L.bar);
  unsigned bar_count = 0;
  if (PS > 0) CK(cudaMemsetAsync(bar, 0, 128 * 128, st));

  // ---- option overlap (reading A24): after the first mirror, V' alternates mirror runs M_r and
  // gradient runs N_r.  M_r runs on s3 as soon as M_{r-1} and N_{r-2} are done, i.e. concurrently
  // with N_{r-1}; N_r waits for M_r.  Enabled only when the plan makes that sound: no tag written
  // by M_r is touched by N_{r-1}, no tag written by N_{r-1} is read by M_r (SLM_ALLOC_MIRROR_PARITY
  // plans satisfy it; other plans run sequentially as before).
  std::vector<int> run_of(ops.size(), -1);
  std::vector<char> is_m(ops.size(), 0);
  bool ov = false;
  int n_runs = 0;
  if (fz && side && m.overlap && PS == 0 && m.s3) {
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
  int abuf3_node = -1;   // abuf_node of the recompute stream's operand buffer
  float* stats3 = (float*)(w + L.stats3);
  void* abuf3 = w + L.a3;
  float* P3 = (float*)(w + L.P3);

  for (size_t oi = 0; oi < ops.size(); ++oi) {
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
      const bool on3 = ov && is_m[oi];
      cudaStream_t fs = on3 ? m.s3 : st;
      void* fa = on3 ? abuf3 : abuf;
      float* fstats = on3 ? stats3 : stats;
      float* fP = on3 ? P3 : P;
      int& fnode = on3 ? abuf3_node : abuf_node;
      // split-K 2 only: SK = 4 (clusters of 8) measured 19.7 us per Block at C2 and did not match the
      // default lowering at d = 2048 (test_cluster_block_option); not dispatched
      const int csk = 2;
      const bool clk = fz && m.blk_cluster && B == 256 && PS == 0 && fused_n(m) == 128 && !m.cta_pair;
      if (!fz || fnode != o.in_node) {
        pbeg(fs);
        if (clk)
          CK(launch_bn_act_cl(csk, xin, gam + (size_t)l * d, bet + (size_t)l * d, d, fstats, (bf*)fa, fs, pdl));
        else
          CK(bn_act(xin, nullptr, 0, nullptr, nullptr, l, fs, fa, fstats));
        pend(SLM_K_BN_ACT, fs);
        ++nl;
      }
      if (clk) {
        pbeg(fs);
        if ((s = launch_blk_cl(csk, m.mW_K, on3 ? m.mA_K3 : m.mA_K, d, l, n, xin, xout, bvec, gam, bet, fstats, (bf*)fa,
                               fs, pdl, gdbg(SLM_K_GEMM_FWD))) != SLM_OK)
          return s;
        pend(SLM_K_GEMM_FWD, fs);
        fnode = o.node;
        ++nl;
      } else
      if (PS > 0) {
        // the run of chained forward / mirror Blocks starting here (each reads the previous one's
        // output), up to kSegMax per launch
        slmk::FwdSegArgs A{};
        A.n = n;
        A.d = d;
        A.bar = bar;
        A.P = P;
        A.bias = bvec;
        A.gamma = gam;
        A.beta = bet;
        A.stats = stats;
        A.a = (bf*)abuf;
        A.phase_dbg = m.persist_dbg;
        int cnt = 0;
        size_t oj = oi;
        for (;;) {
          const Op& q = ops[oj];
          A.L[cnt++] = {X(q.in_tag), X(q.out_tag), q.layer, gdbg(SLM_K_GEMM_FWD)};
          if (cnt == slmk::kSegMax || oj + 1 >= ops.size()) break;
          const Op& nx = ops[oj + 1];
          if (nx.type != 0 || nx.in_node != q.node) break;
          ++oj;
        }
        A.nl = cnt;
        const int grid = d / 128 * PS;
        A.lay_base = bar_count;
        bar_count += (unsigned)cnt;
        pbeg(st);
        if ((s = launch_fwd_seg(B, PS, m.mW_K, m.mA_Kf, A, grid, st, pdl)) != SLM_OK) return s;
        pend(SLM_K_GEMM_FWD, st);
        abuf_node = ops[oj].node;
        oi = oj;
        ++nl;
      } else if (fz) {
        slmk::EpiPartialTma epi{B};
        pbeg(fs);
        if ((s = launch_tc_bn<slmk::EpiPartialTma, false, false, true>(
                 on3 ? mir_tile(m) : fused_n(m), L.sk_fwd, m.mW_K, on3 ? m.mA_K3 : m.mA_K, d, B, d, l * d, 0, epi, fs, pdl,
                 gdbg(SLM_K_GEMM_FWD), on3 ? &m.mP3 : &m.mP, m.cta_pair ? 2 : 1,
                 m.l2_prefetch && l + 1 < n ? (l + 1) * d : -1)) != SLM_OK)
          return s;
        pend(SLM_K_GEMM_FWD, fs);
        // finalize x_{l+1} and produce a_{l+1} for the next Block (BN of layer l+1)
        pbeg(fs);
        CK(bn_act(xin, fP, L.sk_fwd, bvec + (size_t)l * d, xout, l + 1, fs, fa, fstats));
        pend(SLM_K_BN_ACT, fs);
        fnode = o.node;
        nl += 2;
      } else {
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
        const int gnext = (gcur + 1) % NG, abi = kb % NA;
        // dX: P[s] = g_{l+1} W_l over K slice s
        slmk::EpiPartialTma e1{B};
        pbeg(st);
        if ((s = launch_tc_bn<slmk::EpiPartialTma, true, false, true>(
                 dx_tile(m), L.sk_dx, m.mW_MN, m.mG_K[gcur], d, B, d, l * d, 0, e1, st, pdl, gdbg(SLM_K_GEMM_DX), &m.mP,
                 m.cta_pair ? 2 : 1, m.l2_prefetch && l > 0 ? (l - 1) * d : -1)) != SLM_OK)
          return s;
        pend(SLM_K_GEMM_DX, st);
        // bn_bwd(k) overwrites gq[(k+1)%NG] and ab[k%NA], last read by dW of backward k-NA
        if (side && kb >= NA && dw_event[kb - NA] >= 0) CK(cudaStreamWaitEvent(st, m.sync_ev[dw_event[kb - NA]], 0));
        pbeg(st);
        CK(bwd_rk(B / 32, L.sk_dx, bnf_(), st, pdl, d, (const float*)P, (unsigned)pslice, xl, ga, be, g, dxl, dga, dbe, dbp,
                  gq[gnext], ab[abi]));
        pend(SLM_K_BN_BWD, st);
        // dW_l[f_out][f_in] = sum_b g[b][f_out] a[b][f_in]  (second stream)
        cudaStream_t sw = st;
        if (side) {
          cudaEvent_t ef = m.sync_ev[ev_i++];
          CK(cudaEventRecord(ef, st));
          CK(cudaStreamWaitEvent(m.s2, ef, 0));
          sw = m.s2;
        }
        pbeg(sw);
        if (m.dw_tma) {
          slmk::EpiStoreBF16Tma e2{l * d};
          if ((s = launch_tc_bn<slmk::EpiStoreBF16Tma, true, true, false>(m.bn_dw, 1, m.mAb_MN[abi], m.mG_MN[gcur], d,
                                                                          d, B, 0, 0, e2, sw, pdl && !side,
                                                                          gdbg(SLM_K_GEMM_DW), &m.mdW_st)) != SLM_OK)
            return s;
        } else {
          slmk::EpiStoreBF16 e2{(bf*)m.d.dW + l * Wl, d};
          if ((s = launch_tc_bn<slmk::EpiStoreBF16, true, true, false>(m.bn_dw, 1, m.mAb_MN[abi], m.mG_MN[gcur], d,
                                                                       d, B, 0, 0, e2, sw, pdl && !side,
                                                                       gdbg(SLM_K_GEMM_DW))) != SLM_OK)
            return s;
        }
        pend(SLM_K_GEMM_DW, sw);
        if (side) {
          dw_event[kb] = ev_i;
          CK(cudaEventRecord(m.sync_ev[ev_i++], m.s2));
        }
        gcur = gnext;
        nl += 3;
      } else {
        pbeg(st);
        CK(bn_act(xl, nullptr, 0, nullptr, nullptr, l));
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
                      g, dxl, B, d, dga, dbe, dbp, gq[(gcur + 1) % 3]));
        else
          CK(launch_k(bn_bwd_kernel<float>, colgrid, blk, 0, st, pdl, (const float*)da, xl, (const float*)stats, ga,
                      be, g, dxl, B, d, dga, dbe, dbp, (float*)nullptr));
        pend(SLM_K_BN_BWD, st);
        gcur = (gcur + 1) % 3;
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
  if (use_s1) {   // join the critical-path stream back into the caller's
    CK(cudaEventRecord(m.prio_ev[1], st));
    CK(cudaStreamWaitEvent(caller, m.prio_ev[1], 0));
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
