// Executor of V' for the unrolled LSTM (included by runtime.cu after executor.cuh).
//
// Node semantics (graph: oracle.graph.lstm_graph / slm_graph_lstm, time-major ids):
//   X_t      Input [B][n_in]                 bound to x + t*B*n_in (caller buffer)
//   G^l_t    gates  [B][4H] = act([x | h_{t-1}] W_l^T + b_l)        pack + tcgen05 GEMM
//   S^l_t    cell   [B][2H] = (h, c)                                SIMT
//   H_t      head   scalar  = sum_b CE(h W_o^T + b_o, y_t) / (T B)  tcgen05 GEMM + SIMT
//   Sum      loss   scalar  (caller buffer)
// and one gradient node per non-Input node holding d(inputs) concatenated in pred order;
// weight gradients accumulate in place across time steps with fp32
// read-modify-write GEMM epilogues.  Re-computed (mirror) nodes run the same kernels with the
// same configuration, so the checkpointed step is bit-identical to the plain one.

namespace {

struct LstmWs {
  size_t op, dpre_bf, dpre_f, gx, logits, dlog_bf, dlog_f, hop, rowloss, offs, total;
};

inline int lstm_kin0(int n_in) { return (n_in + 127) / 128 * 128; }   // keeps K_0 = Kin0 + H a multiple of 128
inline int lstm_cpad(int C) { return (C + 127) / 128 * 128; }

LstmWs lstm_ws_layout(const slm_lstm_desc& d) {
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  const size_t B = d.batch, H = d.hidden, T = d.steps;
  const size_t Kmax = std::max<size_t>(lstm_kin0(d.n_in), H) + H, Cp = lstm_cpad(d.n_classes);
  LstmWs L{};
  size_t off = 0;
  L.op = off;       off += al(B * Kmax * 2);
  L.dpre_bf = off;  off += al(B * 4 * H * 2);
  L.dpre_f = off;   off += al(B * 4 * H * 4);
  L.gx = off;       off += al(B * Kmax * 4);
  L.logits = off;   off += al(B * Cp * 4);
  L.dlog_bf = off;  off += al(B * Cp * 2);
  L.dlog_f = off;   off += al(B * Cp * 4);
  L.hop = off;      off += al(B * H * 2);
  L.rowloss = off;  off += al(B * 4);
  L.offs = off;     off += al(T * 8);
  L.total = off;
  return L;
}


size_t lstm_w_offset(const slm_lstm_desc& d, int l) {   // elements
  const size_t H = d.hidden, k0 = lstm_kin0(d.n_in) + H;
  return l == 0 ? 0 : 4 * H * k0 + (size_t)(l - 1) * 4 * H * 2 * H;
}

slm_status lstm_bind_maps(const slm_lstm_desc& d, LstmMaps& M, void* ws) {
  if (M.ws == ws) return SLM_OK;
  const uint64_t B = d.batch, H = d.hidden, Cp = lstm_cpad(d.n_classes);
  const LstmWs L = lstm_ws_layout(d);
  uint8_t* w = (uint8_t*)ws;
  const __nv_bfloat16* W = (const __nv_bfloat16*)d.W;
  M.wK.resize(d.n_layers);
  M.wMN.resize(d.n_layers);
  slm_status st;
  for (int l = 0; l < d.n_layers; ++l) {
    const uint64_t K = (l == 0 ? lstm_kin0(d.n_in) : H) + H;
    if ((st = make_map(&M.wK[l], W + lstm_w_offset(d, l), K, 4 * H, 128)) != SLM_OK) return st;
    if ((st = make_map(&M.wMN[l], W + lstm_w_offset(d, l), K, 4 * H, 64)) != SLM_OK) return st;
  }
  if ((st = make_map(&M.woK, d.W_o, H, Cp, 128)) != SLM_OK) return st;
  if ((st = make_map(&M.woMN, d.W_o, H, Cp, 64)) != SLM_OK) return st;
  const uint64_t K0 = lstm_kin0(d.n_in) + H;
  // operand [B][K]: the GEMM's B operand (K-major, box rows = B) and the dW's A (MN-major)
  if ((st = make_map(&M.dpK, w + L.dpre_bf, 4 * H, B, (uint32_t)B)) != SLM_OK) return st;
  if ((st = make_map(&M.dpMN, w + L.dpre_bf, 4 * H, B, 64)) != SLM_OK) return st;
  if ((st = make_map(&M.hopK, w + L.hop, H, B, (uint32_t)B)) != SLM_OK) return st;
  if ((st = make_map(&M.hopMN, w + L.hop, H, B, 64)) != SLM_OK) return st;
  if ((st = make_map(&M.dlK, w + L.dlog_bf, Cp, B, (uint32_t)B)) != SLM_OK) return st;
  if ((st = make_map(&M.dlMN, w + L.dlog_bf, Cp, B, 64)) != SLM_OK) return st;
  M.ws = ws;
  return SLM_OK;
}

// the operand buffer is [B][K_l] with a per-layer K: encode its maps per call (host only)
slm_status lstm_op_maps(const slm_lstm_desc& d, void* ws, int l, CUtensorMap* k, CUtensorMap* mn) {
  const uint64_t B = d.batch, H = d.hidden, K = (l == 0 ? lstm_kin0(d.n_in) : H) + H;
  uint8_t* w = (uint8_t*)ws + lstm_ws_layout(d).op;
  slm_status st;
  if ((st = make_map(k, w, K, B, (uint32_t)B)) != SLM_OK) return st;
  return make_map(mn, w, K, B, 64);
}

struct LstmNode {
  int t, l;     // time, layer (-1 for X_t, L for H_t / Sum)
};

slm_status enqueue_lstm(const slm_plan* p, slm_model& m, const void* xin, const int32_t* labels, void* pool,
                        void* ws, float* loss, cudaStream_t st, int64_t* launches) {
  using namespace slmk;
  const slm_lstm_desc& d = m.ld;
  slm_lstm_state& S = m.lst;
  const bool pdl = m.pdl != 0;
  int ts_slot = 0;
  if (m.profile_ts > 0 && (int)m.ts_kind.size() < m.profile_ts) m.ts_kind.resize(m.profile_ts);
  auto gdbg = [&](int kind) -> int {   // launch slot for the device-clock GEMM timing
    if (m.profile_ts <= 0 || m.ts_buf == nullptr || ts_slot >= m.profile_ts) return 0;
    m.ts_kind[ts_slot] = kind;
    return (++ts_slot) << 8;
  };
  using bf = __nv_bfloat16;
  const int L = d.n_layers, T = d.steps, B = d.batch, H = d.hidden, I = d.n_in, C = d.n_classes;
  const int Cp = lstm_cpad(C), K0 = lstm_kin0(I);
  const LstmWs W = lstm_ws_layout(d);
  uint8_t* w = (uint8_t*)ws;
  bf* op = (bf*)(w + W.op);
  bf* dpre_bf = (bf*)(w + W.dpre_bf);
  float* dpre_f = (float*)(w + W.dpre_f);
  float* gx = (float*)(w + W.gx);
  float* logits = (float*)(w + W.logits);
  bf* dlog_bf = (bf*)(w + W.dlog_bf);
  float* dlog_f = (float*)(w + W.dlog_f);
  bf* hop = (bf*)(w + W.hop);
  float* rowloss = (float*)(w + W.rowloss);
  long* offs = (long*)(w + W.offs);
  const float scale = 1.0f / ((float)T * (float)B);
  slm_status s;
  if ((s = lstm_bind_maps(d, S.maps, ws)) != SLM_OK) return s;
  std::vector<CUtensorMap> opK(L), opMN(L);
  for (int l = 0; l < L; ++l)
    if ((s = lstm_op_maps(d, ws, l, &opK[l], &opMN[l])) != SLM_OK) return s;

  const int N = p->n_fwd;
  const int per_t = 2 * L + 2;
  auto info = [&](int v) -> LstmNode {   // forward node id -> (t, l), time-major layout
    if (v == N - 1) return {T - 1, L};
    const int t = v / per_t, r = v % per_t;
    if (r == 0) return {t, -1};
    if (r == per_t - 1) return {t, L};
    return {t, (r - 1) / 2};
  };
  // tag -> pointer
  std::vector<void*> tp(p->tag_size.size(), nullptr);
  for (size_t t = 0; t < tp.size(); ++t)
    if (p->tag_offset[t] >= 0) tp[t] = (uint8_t*)pool + p->tag_offset[t];
  for (int v = 0; v < N; ++v) {
    const int t = p->node_tag[v];
    if (t < 0 || p->tag_offset[t] >= 0) continue;
    if (p->op[v] == SLM_OP_INPUT) tp[t] = (uint8_t*)const_cast<void*>(xin) + (size_t)info(v).t * B * I * 4;
    else if (p->op[v] == SLM_OP_SUM) tp[t] = loss;
  }
  auto V = [&](int node) -> float* { return node < 0 ? nullptr : (float*)tp[p->node_tag[node]]; };
  const int* pred = p->preds.data();
  auto preds_of = [&](int v) { return std::make_pair(pred + p->pred_ptr[v], p->pred_ptr[v + 1] - p->pred_ptr[v]); };
  // the Sum node's inputs: pool offsets of the H_t values, uploaded once per workspace
  {
    std::vector<long> h_offs(T, 0);
    for (int t = 0; t < T; ++t) h_offs[t] = p->tag_offset[p->node_tag[t * per_t + per_t - 1]];
    if (S.offs_ws != ws || S.offs_plan != (const void*)p) {
      CK(cudaMemcpy(offs, h_offs.data(), T * 8, cudaMemcpyHostToDevice));
      S.offs_ws = ws;
      S.offs_plan = p;
    }
  }
  const dim3 eg(592), eb(256);
  int64_t nl = 0;
  // gradients are overwritten by every step: zero the in-place accumulators first
  {
    size_t wsz = lstm_w_offset(d, L);
    CK(cudaMemsetAsync(d.dW, 0, wsz * 4, st));
    CK(cudaMemsetAsync(d.db, 0, (size_t)L * 4 * H * 4, st));
    CK(cudaMemsetAsync(d.dW_o, 0, (size_t)Cp * H * 4, st));
    CK(cudaMemsetAsync(d.db_o, 0, (size_t)Cp * 4, st));
  }

  for (int v : p->order) {
    const int kind = p->kind[v], opk = p->op[v], orig = p->orig[v];
    auto pp = preds_of(v);
    const LstmNode ni = info(orig);
    const int t = ni.t, l = ni.l;
    if (opk == SLM_OP_INPUT) continue;
    if (kind != SLM_KIND_GRAD) {
      if (opk == SLM_OP_LSTM_GATES) {
        const bool lower_state = l > 0;
        const float* x = V(pp.first[0]);
        const float* sprev = pp.second > 1 ? V(pp.first[1]) : nullptr;
        const int Kin = l == 0 ? K0 : H;
        CK(launch_k(lstm_pack_kernel, eg, eb, 0, st, pdl, x, lower_state ? H : I, lower_state ? 2 * H : I, Kin, sprev,
                    H, B, op));
        slmk::EpiLstmGates e{V(v), d.b + (size_t)l * 4 * H, H};
        if ((s = launch_tc_bn<slmk::EpiLstmGates, false, false, true>(B, 1, S.maps.wK[l], opK[l], 4 * H, B, Kin + H,
                                                                      0, 0, e, st, pdl, gdbg(SLM_K_GEMM_FWD))) != SLM_OK)
          return s;
        nl += 2;
      } else if (opk == SLM_OP_LSTM_CELL) {
        CK(launch_k(lstm_cell_fwd_kernel, eg, eb, 0, st, pdl, (const float*)V(pp.first[0]),
                    (const float*)(pp.second > 1 ? V(pp.first[1]) : nullptr), H, B, V(v)));
        ++nl;
      } else if (opk == SLM_OP_HEAD_CE) {
        CK(launch_k(lstm_hpack_kernel, eg, eb, 0, st, pdl, (const float*)V(pp.first[0]), H, B, hop));
        slmk::EpiStoreF32 e{logits, Cp};
        if ((s = launch_tc_bn<slmk::EpiStoreF32, false, false, true>(B, 1, S.maps.woK, S.maps.hopK, Cp, B, H, 0, 0, e,
                                                                     st, pdl, gdbg(SLM_K_GEMM_FWD))) != SLM_OK)
          return s;
        CK(launch_k(lstm_head_ce_kernel, dim3(B), eb, 0, st, pdl, logits, d.b_o, labels + (size_t)t * B,
                    C, Cp, scale, rowloss, (bf*)nullptr, (float*)nullptr));
        CK(launch_k(lstm_rowsum_kernel, dim3(1), eb, 0, st, pdl, (const float*)rowloss, B, scale, V(v)));
        nl += 4;
      } else if (opk == SLM_OP_SUM) {
        CK(launch_k(lstm_sum_kernel, dim3(1), dim3(32), 0, st, pdl, (const uint8_t*)pool, (const long*)offs, T, V(v)));
        ++nl;
      } else {
        set_error("unsupported op in lstm plan");
        return SLM_E_UNSUPPORTED;
      }
    } else {
      if (opk == SLM_OP_SUM) {
        CK(launch_k(fill_kernel, dim3(1), eb, 0, st, pdl, V(v), T, 1.0f));
        ++nl;
      } else if (opk == SLM_OP_HEAD_CE) {
        // preds = [g[Sum], a[S^{L-1}_t]]: recompute logits, dlogits, dh = dlog W_o, dW_o += ...
        const float* sL = V(pp.first[pp.second - 1]);
        CK(launch_k(lstm_hpack_kernel, eg, eb, 0, st, pdl, sL, H, B, hop));
        slmk::EpiStoreF32 e{logits, Cp};
        if ((s = launch_tc_bn<slmk::EpiStoreF32, false, false, true>(B, 1, S.maps.woK, S.maps.hopK, Cp, B, H, 0, 0, e,
                                                                     st, pdl, gdbg(SLM_K_GEMM_FWD))) != SLM_OK)
          return s;
        CK(launch_k(lstm_head_ce_kernel, dim3(B), eb, 0, st, pdl, logits, d.b_o, labels + (size_t)t * B,
                    C, Cp, scale, (float*)nullptr, dlog_bf, dlog_f));
        // dh[b][h] = sum_c dlog[b][c] W_o[c][h]  -> gx (fp32 [B][H]) then (dh | 0) into the node
        slmk::EpiStoreF32 e2{V(v), 2 * H};
        if ((s = launch_tc_bn<slmk::EpiStoreF32, true, false, true>(B, 1, S.maps.woMN, S.maps.dlK, H, B, Cp, 0, 0, e2,
                                                                    st, pdl, gdbg(SLM_K_GEMM_DX))) != SLM_OK)
          return s;
        // zero the dc half of (dh | dc)
        CK(cudaMemset2DAsync(V(v) + H, (size_t)2 * H * 4, 0, (size_t)H * 4, B, st));
        // dW_o[c][h] += sum_b dlog[b][c] h[b][h]   (D[m=h][n=c], K = B)
        slmk::EpiAccF32 e3{d.dW_o, H};
        if ((s = launch_tc_bn<slmk::EpiAccF32, true, true, false>(128, 1, S.maps.hopMN, S.maps.dlMN, H, Cp, B, 0, 0,
                                                                  e3, st, pdl, gdbg(SLM_K_GEMM_DW))) != SLM_OK)
          return s;
        CK(launch_k(colsum_acc_kernel, dim3((Cp + 255) / 256), eb, 0, st, pdl, (const float*)dlog_f, B, Cp, d.db_o));
        nl += 6;
      } else if (opk == SLM_OP_LSTM_CELL) {
        // successor slices (order: layer above / head, next-step gates, next-step cell)
        const float* sl[3] = {nullptr, nullptr, nullptr};
        int ld[3] = {0, 0, 0};
        int k = 0;
        auto slice = [&](int succ_fwd, int offset_floats, int row_width) {
          const int gs = p->gnode[succ_fwd];
          if (gs < 0) return;
          sl[k] = V(gs) + offset_floats;
          ld[k] = row_width;
          ++k;
        };
        const int sv = orig;
        const int above = l + 1 < L ? sv + 1 : t * per_t + per_t - 1;   // G^{l+1}_t or H_t
        {
          const int wa = (l + 1 < L) ? (2 * H + 2 * H * (t > 0)) : 2 * H;   // row width of g[above]
          slice(above, 0, wa);
        }
        if (t + 1 < T) {
          const int gn = sv + per_t - 1;      // G^l_{t+1}
          const int xw = l == 0 ? I : 2 * H;
          slice(gn, xw, xw + 2 * H);
          const int sn = sv + per_t;          // S^l_{t+1}
          slice(sn, 4 * H, 4 * H + 2 * H);
        }
        const float* act = V(pp.first[pp.second - (t > 0 ? 2 : 1)]);
        const float* sprev = t > 0 ? V(pp.first[pp.second - 1]) : nullptr;
        CK(launch_k(lstm_cell_bwd_kernel, eg, eb, 0, st, pdl, sl[0], ld[0], sl[1], ld[1], sl[2], ld[2], act, sprev, H,
                    B, V(v)));
        ++nl;
      } else if (opk == SLM_OP_LSTM_GATES) {
        // preds = [g[S^l_t], a[G], a[x], a[S_{t-1}]?]
        const bool has_prev = t > 0;
        const int nf = has_prev ? 2 : 1;
        const float* dact = V(pp.first[0]);   // slot 0 of g[S^l_t] = d(acts), row width 4H (+2H)
        const float* act = V(pp.first[pp.second - nf - 1]);
        const float* x = V(pp.first[pp.second - nf]);
        const float* sprev = has_prev ? V(pp.first[pp.second - 1]) : nullptr;
        const int Kin = l == 0 ? K0 : H;
        // d(acts) rows of g[S] are [4H | 2H] wide when the cell has a predecessor
        const int drow = 4 * H + (has_prev ? 2 * H : 0);
        CK(launch_k(lstm_dpre_kernel, eg, eb, 0, st, pdl, dact, drow, act, H, B, dpre_bf, dpre_f));
        CK(launch_k(lstm_pack_kernel, eg, eb, 0, st, pdl, x, l > 0 ? H : I, l > 0 ? 2 * H : I, Kin, sprev, H, B, op));
        // d[x | h] = d_pre W_l:  D[m = k_in][n = b], K = 4H
        slmk::EpiStoreF32 e{gx, Kin + H};
        if ((s = launch_tc_bn<slmk::EpiStoreF32, true, false, true>(B, 1, S.maps.wMN[l], S.maps.dpK, Kin + H, B, 4 * H,
                                                                    0, 0, e, st, pdl, gdbg(SLM_K_GEMM_DX))) != SLM_OK)
          return s;
        CK(launch_k(lstm_gate_scatter_kernel, eg, eb, 0, st, pdl, (const float*)gx, Kin, H, B, I, l > 0 ? 1 : 0,
                    has_prev ? 1 : 0, V(v)));
        // dW_l[n = gate][m = k_in] += sum_b op[b][k_in] d_pre[b][gate]
        slmk::EpiAccF32 e2{d.dW + lstm_w_offset(d, l), Kin + H};
        if ((s = launch_tc_bn<slmk::EpiAccF32, true, true, false>(128, 1, opMN[l], S.maps.dpMN, Kin + H, 4 * H, B, 0,
                                                                  0, e2, st, pdl, gdbg(SLM_K_GEMM_DW))) != SLM_OK)
          return s;
        CK(launch_k(colsum_acc_kernel, dim3((4 * H + 255) / 256), eb, 0, st, pdl, (const float*)dpre_f, B, 4 * H,
                    d.db + (size_t)l * 4 * H));
        nl += 6;
      } else {
        set_error("unsupported gradient op in lstm plan");
        return SLM_E_UNSUPPORTED;
      }
    }
  }
  CK(cudaGetLastError());
  m.ts_used = ts_slot;
  if (launches) *launches = nl;
  return SLM_OK;
}

// kernels enqueue_lstm launches for this plan (the memsets are not counted)
int64_t lstm_launches(const slm_plan* p) {
  int64_t nl = 0;
  for (int v : p->order) {
    const int opk = p->op[v];
    if (opk == SLM_OP_INPUT) continue;
    if (p->kind[v] != SLM_KIND_GRAD)
      nl += opk == SLM_OP_LSTM_GATES ? 2 : opk == SLM_OP_HEAD_CE ? 4 : 1;
    else
      nl += opk == SLM_OP_HEAD_CE ? 6 : opk == SLM_OP_LSTM_GATES ? 6 : 1;
  }
  return nl;
}

}  // namespace
