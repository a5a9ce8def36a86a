// Executor of V' for the unrolled LSTM (included by runtime.cu after executor.cuh).
//
// Node semantics (graph: oracle.graph.lstm_graph / slm_graph_lstm, time-major ids):
//   X_t      Input [B][n_in]                 bound to x + t*B*n_in (caller buffer)
//   G^l_t    gates  [B][4H] = act([x | h_{t-1}] W_l^T + b_l)
//   S^l_t    cell   [B][2H] = (h, c)
//   H_t      head   scalar  = sum_b CE(h W_o^T + b_o, y_t) / (T B)
//   Sum      loss   scalar  (caller buffer)
// and one gradient node per non-Input node holding d(inputs) concatenated in pred order (A17).
//
// Lowering:
//   gates (fwd/mirror)  pack [x | h] bf16 -> tcgen05 GEMM, split-K fp32 partials (N = B = 64
//                       would leave 32 of 148 SMs busy) -> lstm_gates_cell_kernel (partials +
//                       bias + activations -> G; fused with the cell S when S^l_t is the next
//                       node of V', which it is in forward and recompute order)
//   head  (fwd)         pack h -> logits GEMM (split-K) -> softmax-CE rows -> row sum
//   grad head           pack h -> logits GEMM -> CE + dlogits -> dh GEMM (split-K) -> (dh | 0)
//   grad cell           sum of successor slices -> d(acts) | (0 | dc_prev)
//   grad gates          d_pre (+ db) -> dX GEMM (split-K) -> scatter into d(inputs)
//   weight gradients    the GEMM operands of each step are kept in a per-layer ring of CH time
//                       steps; once per chunk (in time order, independent of the plan)
//                       dW_l += opᵀ d_pre runs as ONE GEMM with K = B * CH (PAPER.md:488-489
//                       "in-place accumulation"), instead of CH GEMMs with K = B.
// Re-computed (mirror) nodes run the same kernels with the same configuration and every
// reduction has a fixed order, so the checkpointed step is bit-identical to the plain one.

namespace {

constexpr int kLstmChunk = 32;   // time steps per weight-gradient GEMM

struct LstmWs {
  size_t logits, dlog_f, rowloss, offs, cnt, hopR, dlR, hf, logitsF, rowlossF, dhR, PH, total;
  std::vector<size_t> P;                     // split-K partials, one buffer per stream (layers, head)
  std::vector<size_t> opL, opR, dpR, dpF, PX;   // per layer: forward operand, backward rings, dX partials
};

inline int lstm_kin0(int n_in) { return (n_in + 127) / 128 * 128; }   // keeps K_0 = Kin0 + H a multiple of 128
inline int lstm_cpad(int C) { return (C + 127) / 128 * 128; }
inline int lstm_K(const slm_lstm_desc& d, int l) { return (l == 0 ? lstm_kin0(d.n_in) : d.hidden) + d.hidden; }

// split-K factor: the largest s dividing K/64 with mtiles * s <= 148 (one wave)
inline int lstm_sk(int mtiles, int K) {
  const int kb = K / 64;
  int best = 1;
  for (int s = 1; s <= kb; ++s)
    if (kb % s == 0 && mtiles * s <= 148) best = s;
  return best;
}
struct LstmSplits {
  int g0, g1, x0, x1, lg, hd;   // gates (layer 0 / l > 0), dX (layer 0 / l > 0), logits, head dX
};
LstmSplits lstm_splits(const slm_lstm_desc& d, int gates_sk = 0, int dx_sk = 0) {
  const int H = d.hidden, Cp = lstm_cpad(d.n_classes);
  const int K0 = lstm_K(d, 0), K1 = 2 * H;
  // head: logits without split-K, dh with at most 4 K slices -- the per-step and the batched
  // (32-step) head backward use the same K slicing, so their values are bit-identical
  auto upto = [](int K, int q) {
    int b = 1;
    for (int x = 1; x <= q; ++x)
      if ((K / 64) % x == 0) b = x;
    return b;
  };
  LstmSplits s{lstm_sk(4 * H / 128, K0), lstm_sk(4 * H / 128, K1), lstm_sk(K0 / 128, 4 * H), lstm_sk(K1 / 128, 4 * H),
               1, upto(Cp, 4)};
  if (gates_sk > 0) {   // the largest divisor of K/64 not above the request
    auto fit = [&](int K) {
      int b = 1;
      for (int q = 1; q <= gates_sk; ++q)
        if ((K / 64) % q == 0) b = q;
      return b;
    };
    s.g0 = fit(K0);
    s.g1 = fit(K1);
  }
  if (dx_sk > 0) {
    s.x0 = upto(4 * H, dx_sk);
    s.x1 = upto(4 * H, dx_sk);
  }
  return s;
}

LstmWs lstm_ws_layout(const slm_lstm_desc& d, int gates_sk = 0, int dx_sk = 0) {
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  const size_t B = d.batch, H = d.hidden, T = d.steps, CH = kLstmChunk;
  const size_t K0 = lstm_K(d, 0), Kmax = std::max<size_t>(K0, 2 * H), Cp = lstm_cpad(d.n_classes);
  const LstmSplits sp = lstm_splits(d, gates_sk, dx_sk);
  const size_t pbytes = std::max({(size_t)std::max(sp.g0, sp.g1) * B * 4 * H, (size_t)sp.x0 * B * K0,
                                  (size_t)sp.x1 * B * 2 * H, (size_t)sp.lg * B * Cp, (size_t)sp.hd * B * H}) * 4;
  LstmWs L{};
  size_t off = 0;
  for (int i = 0; i <= 2 * d.n_layers; ++i) {   // layers, head, mirror streams
    L.P.push_back(off);
    off += al(pbytes);
  }
  L.logits = off;   off += al(B * Cp * 4);
  L.dlog_f = off;   off += al(CH * B * Cp * 4);
  L.rowloss = off;  off += al(B * 4);
  L.offs = off;     off += al(T * 4);   // per-step losses (loss_t)
  L.cnt = off;      off += 256;
  L.hopR = off;     off += al(CH * B * H * 2);
  L.hf = off;       off += 2 * al(CH * B * H * 2);   // forward head operands, chunk-parity double buffer
  L.logitsF = off;  off += al(CH * B * Cp * 4);
  L.rowlossF = off; off += al(CH * B * 4);
  L.dhR = off;      off += 2 * al(CH * B * 2 * H * 4);          // (dh | 0) of batched head steps, chunk parity
  L.PH = off;       off += al((size_t)sp.hd * CH * B * H * 4);  // split-K partials of the batched dh GEMM
  L.dlR = off;      off += al(CH * B * Cp * 2);
  for (int l = 0; l < d.n_layers; ++l) {
    L.opL.push_back(off);
    off += 2 * al(B * lstm_K(d, l) * 2);   // time-parity double buffer
    L.opR.push_back(off);
    off += al(CH * B * lstm_K(d, l) * 2);
    L.dpR.push_back(off);
    off += al(CH * B * 4 * H * 2);
    L.dpF.push_back(off);
    off += al(CH * B * 4 * H * 4);
    L.PX.push_back(off);   // dX partials [sk][B][K_l], double-buffered by time parity
    off += 2 * al((size_t)(l == 0 ? sp.x0 : sp.x1) * B * lstm_K(d, l) * 4);
  }
  L.total = off;
  return L;
}

size_t lstm_w_offset(const slm_lstm_desc& d, int l) {   // elements
  const size_t H = d.hidden, k0 = lstm_K(d, 0);
  return l == 0 ? 0 : 4 * H * k0 + (size_t)(l - 1) * 4 * H * 2 * H;
}

slm_status lstm_bind_maps(const slm_lstm_desc& d, LstmMaps& M, void* ws, int gates_sk, int dx_sk) {
  if (M.ws == ws) return SLM_OK;
  const uint64_t B = d.batch, H = d.hidden, Cp = lstm_cpad(d.n_classes), CH = kLstmChunk;
  const LstmWs L = lstm_ws_layout(d, gates_sk, dx_sk);
  const LstmSplits sp = lstm_splits(d, gates_sk, dx_sk);
  uint8_t* w = (uint8_t*)ws;
  const __nv_bfloat16* W = (const __nv_bfloat16*)d.W;
  const int nl = d.n_layers;
  M.wK.resize(nl);
  M.wMN.resize(nl);
  M.wK32.resize(nl);
  M.opK.resize(2 * nl);
  M.opRMN.resize(nl);
  M.dpRK.resize(nl);
  M.dpRMN.resize(nl);
  M.pX.resize(nl);
  M.pG.resize(nl);
  M.pGm.resize(nl);
  M.pXd.resize(2 * nl);
  M.opRK.resize(nl);
  slm_status st;
  for (int l = 0; l < nl; ++l) {
    const uint64_t K = lstm_K(d, l);
    if ((st = make_map(&M.wK[l], W + lstm_w_offset(d, l), K, 4 * H, 128)) != SLM_OK) return st;
    if ((st = make_map(&M.wK32[l], W + lstm_w_offset(d, l), K, 4 * H, 32)) != SLM_OK) return st;
    if ((st = make_map(&M.wMN[l], W + lstm_w_offset(d, l), K, 4 * H, 64)) != SLM_OK) return st;
    for (int par = 0; par < 2; ++par)
      if ((st = make_map(&M.opK[2 * l + par], w + L.opL[l] + par * ((B * K * 2 + 255) / 256 * 256), K, B,
                         (uint32_t)B)) != SLM_OK)
        return st;
    if ((st = make_map(&M.opRK[l], w + L.opR[l], K, CH * B, (uint32_t)B)) != SLM_OK) return st;
    if ((st = make_map(&M.opRMN[l], w + L.opR[l], K, CH * B, 64)) != SLM_OK) return st;
    if ((st = make_map(&M.dpRK[l], w + L.dpR[l], 4 * H, CH * B, (uint32_t)B)) != SLM_OK) return st;
    if ((st = make_map(&M.dpRMN[l], w + L.dpR[l], 4 * H, CH * B, 64)) != SLM_OK) return st;
    if ((st = make_map_f32(&M.pX[l], w + L.P[l], K, (uint64_t)(l == 0 ? sp.x0 : sp.x1) * B)) != SLM_OK) return st;
    for (int par = 0; par < 2; ++par) {
      const size_t bytes = ((size_t)(l == 0 ? sp.x0 : sp.x1) * B * K * 4 + 255) / 256 * 256;
      if ((st = make_map_f32(&M.pXd[2 * l + par], w + L.PX[l] + par * bytes, K,
                             (uint64_t)(l == 0 ? sp.x0 : sp.x1) * B)) != SLM_OK)
        return st;
    }
    if ((st = make_map_f32(&M.pG[l], w + L.P[l], 4 * H, (uint64_t)std::max(sp.g0, sp.g1) * B)) != SLM_OK) return st;
    if ((st = make_map_f32(&M.pGm[l], w + L.P[nl + 1 + l], 4 * H, (uint64_t)std::max(sp.g0, sp.g1) * B)) != SLM_OK)
      return st;
  }
  if ((st = make_map(&M.woK, d.W_o, H, Cp, 128)) != SLM_OK) return st;
  if ((st = make_map(&M.woMN, d.W_o, H, Cp, 64)) != SLM_OK) return st;
  if ((st = make_map(&M.hopRK, w + L.hopR, H, CH * B, (uint32_t)B)) != SLM_OK) return st;
  for (int par = 0; par < 2; ++par)
    for (int bi = 0; bi < 2; ++bi)
      if ((st = make_map(&M.hfK[par][bi], w + L.hf + par * ((CH * B * H * 2 + 255) / 256 * 256), H, CH * B,
                         bi ? 256u : 64u)) != SLM_OK)
        return st;
  for (int bi = 0; bi < 3; ++bi) {   // batched head backward: N tiles 64 / 128 / 256
    if ((st = make_map(&M.hopRKb[bi], w + L.hopR, H, CH * B, 64u << bi)) != SLM_OK) return st;
    if ((st = make_map(&M.dlRKb[bi], w + L.dlR, Cp, CH * B, 64u << bi)) != SLM_OK) return st;
  }
  if ((st = make_map_f32(&M.pHB, w + L.PH, H, (uint64_t)sp.hd * CH * B)) != SLM_OK) return st;
  if ((st = make_map(&M.hopRMN, w + L.hopR, H, CH * B, 64)) != SLM_OK) return st;
  if ((st = make_map(&M.dlRK, w + L.dlR, Cp, CH * B, (uint32_t)B)) != SLM_OK) return st;
  if ((st = make_map(&M.dlRMN, w + L.dlR, Cp, CH * B, 64)) != SLM_OK) return st;
  if ((st = make_map_f32(&M.pL, w + L.P[nl], Cp, (uint64_t)sp.lg * B)) != SLM_OK) return st;
  if ((st = make_map_f32(&M.pH, w + L.P[nl], H, (uint64_t)sp.hd * B)) != SLM_OK) return st;
  M.ws = ws;
  return SLM_OK;
}

struct LstmNode {
  int t, l;     // time, layer (-1 for X_t, L for H_t / Sum)
};

// Which V' node's value currently sits (as bf16) in each forward GEMM operand: the x and h
// halves of layer l's operand [x | h_{t-1}] and the head operand.  Cell-state kernels write
// their h (and, at layer 0, the next input) straight into the operands of their consumers;
// a gates / head node re-packs only when its operand does not already hold its inputs.
// kZeros marks the all-zero h of t = 0.  Used identically by enqueue_lstm and lstm_launches.
// Operands are double-buffered by time parity (G^l_t reads buffer t % 2), so a producer for
// step t+1 never waits for the consumer of step t.
struct OperandTracker {
  static constexpr int kZeros = -2;
  std::vector<int> wx, wh;   // [2 l + parity]
  explicit OperandTracker(int L) : wx(2 * L, -1), wh(2 * L, -1) {}
  bool gates_needs_pack(int l, int t, int xnode, int hnode) const {
    return wx[2 * l + t % 2] != xnode || wh[2 * l + t % 2] != hnode;
  }
  void packed(int l, int t, int xnode, int hnode) {
    wx[2 * l + t % 2] = xnode;
    wh[2 * l + t % 2] = hnode;
  }
  // cell state node u = S^l_t produced: h -> layer l's h half for t+1, layer l+1's x half
  // (step t) or the head operand (step t); layer 0 also writes x_{t+1} (Input node xnext_node)
  void cell(int u, int l, int t, int L, int T, int xnext_node) {
    if (t + 1 < T) wh[2 * l + (t + 1) % 2] = u;
    if (l + 1 < L) wx[2 * (l + 1) + t % 2] = u;
    if (l == 0 && t + 1 < T) wx[(t + 1) % 2] = xnext_node;
  }
};

slm_status enqueue_lstm(const slm_plan* p, slm_model& m, const void* xin, const int32_t* labels, void* pool,
                        void* ws, float* loss, cudaStream_t st, int64_t* launches) {
  using namespace slmk;
  using bf = __nv_bfloat16;
  const slm_lstm_desc& d = m.ld;
  slm_lstm_state& S = m.lst;
  const bool pdl = m.pdl != 0;
  int ts_slot = 0;
  if (m.profile_ts > 0 && (int)m.ts_kind.size() < m.profile_ts) {
    m.ts_kind.resize(m.profile_ts);
    m.ts_aux.resize(m.profile_ts);
  }
  auto gdbg = [&](int kind) -> int {   // launch slot for the device-clock GEMM timing
    if (m.profile_ts <= 0 || m.ts_buf == nullptr || ts_slot >= m.profile_ts) return 0;
    m.ts_kind[ts_slot] = kind;
    m.ts_aux[ts_slot] = m.ts_cur_aux;
    return ((++ts_slot) << 8) | (m.profile_ts_dep ? 8 : 0);
  };
  const int L = d.n_layers, T = d.steps, B = d.batch, H = d.hidden, I = d.n_in, C = d.n_classes;
  const int Cp = lstm_cpad(C), K0 = lstm_kin0(I), CH = kLstmChunk;
  const LstmWs W = lstm_ws_layout(d, m.lstm_sk, m.lstm_skx);
  const LstmSplits sp = lstm_splits(d, m.lstm_sk, m.lstm_skx);
  uint8_t* w = (uint8_t*)ws;
  auto Pb = [&](int i) { return (const float*)(w + W.P[i]); };   // split-K partials of stream i
  float* logits = (float*)(w + W.logits);
  float* dlog_f = (float*)(w + W.dlog_f);
  float* loss_t = (float*)(w + W.offs);
  bf* hopR = (bf*)(w + W.hopR);
  bf* dlR = (bf*)(w + W.dlR);
  const float scale = 1.0f / ((float)T * (float)B);
  slm_status s;
  if ((s = lstm_bind_maps(d, S.maps, ws, m.lstm_sk, m.lstm_skx)) != SLM_OK) return s;
  const LstmMaps& M = S.maps;

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
  const dim3 eg(592), eb(256);
  // element-wise grids sized to the work (one element per thread, at most 4 CTAs per SM) so
  // the kernels of concurrent layer streams share the SMs (option lstm_grid = 0: 592 CTAs)
  auto gsz = [&](size_t n) {
    if (!m.lstm_grid) return eg;
    return dim3((unsigned)std::max<size_t>(1, std::min<size_t>(592, (n + 255) / 256)));
  };
  int64_t nl = 0;
  // gradients are overwritten by every step: zero the in-place accumulators first
  CK(cudaMemsetAsync(d.dW, 0, lstm_w_offset(d, L) * 4, st));
  CK(cudaMemsetAsync(d.db, 0, (size_t)L * 4 * H * 4, st));
  CK(cudaMemsetAsync(d.dW_o, 0, (size_t)Cp * H * 4, st));
  CK(cudaMemsetAsync(d.db_o, 0, (size_t)Cp * 4, st));
  // weight-gradient chunk of time t: slot in the ring and whether t closes the chunk (the
  // backward visits each layer's steps in descending t, so the chunk's lowest t comes last)
  auto chunk_rows = [&](int t) { return std::min(CH, T - (t / CH) * CH) * B; };

  OperandTracker trk(L);
  auto opl = [&](int l, int par) {
    return (bf*)(w + W.opL[l] + par * (((size_t)B * lstm_K(d, l) * 2 + 255) / 256 * 256));
  };
  // forward head operands: a ring of CH steps per chunk parity, consumed by one batched head
  auto hfb = [&](int t) {
    return (bf*)(w + W.hf + ((t / CH) % 2) * (((size_t)CH * B * H * 2 + 255) / 256 * 256)) + (size_t)(t % CH) * B * H;
  };
  // the operand side outputs of the kernel producing S^l_t (V' node u); the top layer's h
  // goes to the forward head ring only for forward (not re-computed) states
  auto op_out = [&](int u, int l, int t, int knd) {
    slmk::OpOut o{};
    if (t + 1 < T) {
      o.h_self = opl(l, (t + 1) % 2) + (l == 0 ? K0 : H);
      o.ld_self = lstm_K(d, l);
    }
    o.h_up = l + 1 < L ? opl(l + 1, t % 2) : (knd == SLM_KIND_FWD ? hfb(t) : nullptr);
    o.ld_up = l + 1 < L ? lstm_K(d, l + 1) : H;
    if (l == 0 && t + 1 < T) {
      o.xnext = (const float*)((const uint8_t*)xin + (size_t)(t + 1) * B * I * 4);
      o.I = I;
      o.Kin0 = K0;
      o.x0 = opl(0, (t + 1) % 2);
      o.ld0 = lstm_K(d, 0);
    }
    trk.cell(u, l, t, L, T, (t + 1) * per_t);
    return o;
  };

  // ---- layer wavefront (option lstm_streams): every launch unit runs on the stream of its
  // layer (the head and the loss on stream L); happens-before edges come from tracking, per
  // resource (pool tag, forward operand half), the last writer and the latest reader on each
  // stream, so concurrent units never touch a buffer out of V' order.  A dependency is a
  // (stream, unit sequence number); it is skipped when the waiting stream is already ordered
  // after that unit (same stream, or an earlier wait on a later unit of that stream).  Events
  // live in a per-stream ring large enough to hold a step's units; a re-recorded slot only
  // makes a (very old) wait more conservative, never wrong.
  const bool msm = m.lstm_streams != 0 && st != nullptr;
  // lstm_streams = 2: re-computed (mirror) units get streams of their own (L+1+l), so the
  // recompute of segment j-1 can overlap the backward of segment j
  const int NSTR = m.lstm_streams >= 2 ? 2 * L + 1 : L + 1;
  constexpr int kRing = 16384;
  const int ntag = (int)p->tag_size.size();
  auto OPX = [&](int l, int par) { return ntag + 4 * l + par; };
  auto OPH = [&](int l, int par) { return ntag + 4 * l + 2 + par; };
  auto HFR = [&](int par) { return ntag + 4 * L + par; };       // forward head ring, chunk parity
  auto DHR = [&](int par) { return ntag + 4 * L + 2 + par; };   // batched (dh | 0) ring, chunk parity
  auto PXR = [&](int l, int par) { return ntag + 4 * L + 4 + 2 * l + par; };   // dX partials of layer l
  const int HOP = ntag + 6 * L + 3;   // the highest resource id
  std::vector<int> rd, wr;
  // dependencies are unit ids u = seq * NSTR + stream (seq = per-stream unit counter)
  std::vector<long> res_w, res_r;   // [resource] last writer unit; [resource][stream] latest reader
  std::vector<long> seqn(NSTR, 0), waits;
  std::vector<long> known((size_t)NSTR * NSTR, -1);   // [a][s]: latest seq of s stream a is ordered after
  if (msm) {
    while ((int)S.streams.size() < NSTR) {
      cudaStream_t x;
      CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
      S.streams.push_back(x);
    }
    if ((int)S.ev.size() < NSTR * kRing) S.ev.resize((size_t)NSTR * kRing, nullptr);
    while ((int)S.join.size() < NSTR) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      S.join.push_back(e);
    }
    if (!S.fork) CK(cudaEventCreateWithFlags(&S.fork, cudaEventDisableTiming));
    res_w.assign(HOP + 1, -1);
    res_r.assign((size_t)(HOP + 1) * NSTR, -1);
    // events are created lazily up to the ring size
    CK(cudaEventRecord(S.fork, st));
    for (int i = 0; i < NSTR; ++i) CK(cudaStreamWaitEvent(S.streams[i], S.fork, 0));
  }
  auto evt = [&](long u) -> cudaEvent_t& { return S.ev[(size_t)(u % NSTR) * kRing + (size_t)((u / NSTR) % kRing)]; };
  auto unit_begin = [&](int sid, cudaStream_t* out) -> slm_status {
    waits.clear();
    for (int r : rd)
      if (res_w[r] >= 0) waits.push_back(res_w[r]);
    for (int r : wr) {
      if (res_w[r] >= 0) waits.push_back(res_w[r]);
      for (int i = 0; i < NSTR; ++i)
        if (res_r[(size_t)r * NSTR + i] >= 0) waits.push_back(res_r[(size_t)r * NSTR + i]);
    }
    // per source stream only the latest unit matters
    std::vector<long> need(NSTR, -1);
    for (long u : waits) need[u % NSTR] = std::max(need[u % NSTR], u / NSTR);
    for (int s2 = 0; s2 < NSTR; ++s2) {
      if (s2 == sid || need[s2] < 0 || known[(size_t)sid * NSTR + s2] >= need[s2]) continue;
      CK(cudaStreamWaitEvent(S.streams[sid], evt(need[s2] * NSTR + s2), 0));
      known[(size_t)sid * NSTR + s2] = need[s2];
    }
    *out = S.streams[sid];
    return SLM_OK;
  };
  auto unit_end = [&](int sid) -> slm_status {
    const long u = seqn[sid]++ * NSTR + sid;
    cudaEvent_t& e = evt(u);
    if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventRecord(e, S.streams[sid]));
    for (int r : rd) res_r[(size_t)r * NSTR + sid] = u;
    for (int r : wr) {
      res_w[r] = u;
      for (int i = 0; i < NSTR; ++i) res_r[(size_t)r * NSTR + i] = -1;
    }
    return SLM_OK;
  };

  // which V' node's value each pool tag holds (host view of V' order), for the batched head
  // backward: a chunk of g[H_t] runs as one unit when every a[S^{L-1}_t] it reads is resident
  std::vector<int> owner(p->tag_size.size(), -1);
  std::vector<char> hb_batched(T, 0);
  auto dh_ring = [&](int t) {
    return (float*)(w + W.dhR + ((t / CH) % 2) * (((size_t)CH * B * 2 * H * 4 + 255) / 256 * 256)) +
           (size_t)(t % CH) * B * 2 * H;
  };
  auto head_state = [&](int t) {   // the V' node a[S^{L-1}_t] the head gradient of step t reads
    const int gh = p->gnode[t * per_t + per_t - 1];
    if (gh < 0) return -1;
    return p->preds[p->pred_ptr[gh + 1] - 1];
  };
  // the lowest step t_lo >= the chunk start such that every head input of t_lo..t is resident
  auto ready_from = [&](int t) {
    int lo = t + 1;
    for (int t2 = t; t2 >= t - t % CH; --t2) {
      const int a = head_state(t2);
      if (a < 0 || owner[p->node_tag[a]] != a) break;
      lo = t2;
    }
    return lo;
  };

  const std::vector<int>& order = p->order;
  for (size_t oi = 0; oi < order.size(); ++oi) {
    const int v = order[oi];
    const int kind = p->kind[v], opk = p->op[v], orig = p->orig[v];
    auto pp = preds_of(v);
    const LstmNode ni = info(orig);
    const int t = ni.t, l = ni.l;
    if (opk == SLM_OP_INPUT) continue;
    // ---- the launch unit: this node, plus the next one when the two are fused
    const bool lay = opk == SLM_OP_LSTM_GATES || opk == SLM_OP_LSTM_CELL;
    const int sid = !lay ? L : (kind == SLM_KIND_MIRROR && NSTR > L + 1 ? L + 1 + l : l);
    int partner = -1;
    if (oi + 1 < order.size()) {
      const int u = order[oi + 1];
      const bool pu0 = p->pred_ptr[u + 1] > p->pred_ptr[u] && p->preds[p->pred_ptr[u]] == v;
      if (kind != SLM_KIND_GRAD && opk == SLM_OP_LSTM_GATES && p->op[u] == SLM_OP_LSTM_CELL && p->kind[u] == kind && pu0)
        partner = u;
      if (kind == SLM_KIND_GRAD && opk == SLM_OP_LSTM_CELL && p->op[u] == SLM_OP_LSTM_GATES &&
          p->kind[u] == SLM_KIND_GRAD && pu0)
        partner = u;
    }
    rd.clear();
    wr.clear();
    for (int node : {v, partner}) {
      if (node < 0) continue;
      auto pn = preds_of(node);
      for (int i = 0; i < pn.second; ++i)
        if (pn.first[i] != v) rd.push_back(p->node_tag[pn.first[i]]);
      wr.push_back(p->node_tag[node]);
    }
    auto cell_writes = [&]() {
      if (t + 1 < T) wr.push_back(OPH(l, (t + 1) % 2));
      if (l + 1 < L) wr.push_back(OPX(l + 1, t % 2));
      else if (kind == SLM_KIND_FWD) wr.push_back(HFR((t / CH) % 2));
      if (l == 0 && t + 1 < T) wr.push_back(OPX(0, (t + 1) % 2));
    };
    if (kind != SLM_KIND_GRAD) {
      if (opk == SLM_OP_LSTM_GATES) {
        const int hn = pp.second > 1 ? pp.first[1] : OperandTracker::kZeros;
        if (trk.gates_needs_pack(l, t, pp.first[0], hn)) {
          wr.push_back(OPX(l, t % 2));
          wr.push_back(OPH(l, t % 2));
        } else {
          rd.push_back(OPX(l, t % 2));
          rd.push_back(OPH(l, t % 2));
        }
        if (partner >= 0) cell_writes();
      } else if (opk == SLM_OP_LSTM_CELL) {
        cell_writes();
      } else if (opk == SLM_OP_HEAD_CE) {
        // one batched unit per chunk of forward heads, at the chunk's last step
        wr.clear();
        rd.clear();
        if (t % CH == CH - 1 || t == T - 1) {
          rd.push_back(HFR((t / CH) % 2));
          for (int t2 = t - t % CH; t2 <= t; ++t2) wr.push_back(p->node_tag[t2 * per_t + per_t - 1]);
        }
      }
    }
    bool hb_now = false;   // this g[H_t] runs the batched head backward of steps hb_lo..t
    int hb_lo = t;
    if (kind == SLM_KIND_GRAD && opk == SLM_OP_HEAD_CE && !hb_batched[t]) {
      hb_lo = ready_from(t);
      if (hb_lo < t) {
        hb_now = true;
        rd.clear();
        wr.clear();
        for (int t2 = hb_lo; t2 <= t; ++t2) rd.push_back(p->node_tag[head_state(t2)]);
        wr.push_back(DHR((t / CH) % 2));
      }
    }
    if (kind == SLM_KIND_GRAD && opk == SLM_OP_LSTM_CELL && l == L - 1 && hb_batched[t]) rd.push_back(DHR((t / CH) % 2));
    if (kind == SLM_KIND_GRAD && opk == SLM_OP_LSTM_CELL) {   // reads dX partials of its gates successors
      if (l + 1 < L) rd.push_back(PXR(l + 1, t % 2));
      if (t + 1 < T) rd.push_back(PXR(l, (t + 1) % 2));
    }
    if (kind == SLM_KIND_GRAD && (opk == SLM_OP_LSTM_GATES || (opk == SLM_OP_LSTM_CELL && partner >= 0)))
      wr.push_back(PXR(l, t % 2));
    const bool skip_unit = kind == SLM_KIND_GRAD && opk == SLM_OP_HEAD_CE && hb_batched[t];
    if (skip_unit) continue;
    cudaStream_t cs = st;
    if (msm && (s = unit_begin(sid, &cs)) != SLM_OK) return s;
    m.ts_cur_aux = sid * 4 + (kind == SLM_KIND_GRAD ? 2 : kind == SLM_KIND_MIRROR ? 1 : 0);
    if (kind != SLM_KIND_GRAD) {
      if (opk == SLM_OP_LSTM_GATES) {
        const bool lower_state = l > 0;
        const float* x = V(pp.first[0]);
        const float* sprev = pp.second > 1 ? V(pp.first[1]) : nullptr;
        const int Kin = l == 0 ? K0 : H, sk = l == 0 ? sp.g0 : sp.g1;
        const int xn = pp.first[0], hn = pp.second > 1 ? pp.first[1] : OperandTracker::kZeros;
        if (trk.gates_needs_pack(l, t, xn, hn)) {
          CK(launch_k(lstm_pack_kernel, gsz((size_t)B * (Kin + H)), eb, 0, cs, pdl, x, lower_state ? H : I, lower_state ? 2 * H : I, Kin, sprev,
                      H, B, opl(l, t % 2)));
          trk.packed(l, t, xn, hn);
          ++nl;
        }
        // fuse the cell when V' runs S^l_t (same kind) right after G^l_t
        float* s_out = nullptr;
        const float* s_prev = nullptr;
        slmk::OpOut oo{};
        if (oi + 1 < order.size()) {
          const int u = order[oi + 1];
          auto pu = preds_of(u);
          if (p->op[u] == SLM_OP_LSTM_CELL && p->kind[u] == kind && pu.first[0] == v) {
            s_out = V(u);
            s_prev = pu.second > 1 ? V(pu.first[1]) : nullptr;
            oo = op_out(u, l, t, kind);
            ++oi;
          }
        }
        if (sk == 1 && m.lstm_fuse_cell) {   // one kernel: GEMM with the activations and the cell in its epilogue
          slmk::EpiGatesCell e{V(v), s_out, s_prev, d.b + (size_t)l * 4 * H, H, B, oo};
          if ((s = launch_tc_bn<slmk::EpiGatesCell, false, false, true>(B, 1, M.wK32[l], M.opK[2 * l + t % 2], 4 * H, B,
                                                                        Kin + H, 0, 0, e, cs, pdl,
                                                                        gdbg(SLM_K_GEMM_FWD))) != SLM_OK)
            return s;
          nl += 1;
        } else {
          slmk::EpiPartialTma e{B};
          if ((s = launch_tc_bn<slmk::EpiPartialTma, false, false, true>(
                   B, sk, M.wK[l], M.opK[2 * l + t % 2], 4 * H, B, Kin + H, 0, 0, e, cs, pdl, gdbg(SLM_K_GEMM_FWD),
                   sid > L ? &M.pGm[l] : &M.pG[l])) != SLM_OK)
            return s;
          CK(launch_k(lstm_gates_cell_kernel, gsz((size_t)B * H), eb, 0, cs, pdl, Pb(sid), sk, d.b + (size_t)l * 4 * H,
                      H, B, V(v), s_prev, s_out, oo));
          nl += 2;
        }
      } else if (opk == SLM_OP_LSTM_CELL) {
        CK(launch_k(lstm_cell_fwd_kernel, gsz((size_t)B * H), eb, 0, cs, pdl, (const float*)V(pp.first[0]),
                    (const float*)(pp.second > 1 ? V(pp.first[1]) : nullptr), H, B, V(v), op_out(v, l, t, kind)));
        ++nl;
      } else if (opk == SLM_OP_HEAD_CE) {
        // batched forward heads of steps t0..t (the chunk ends here): logits for n*B rows in one
        // GEMM, the softmax-CE rows, then the per-step losses into the H_t tags
        if (t % CH == CH - 1 || t == T - 1) {
          const int t0 = t - t % CH, n = t - t0 + 1, N = n * B, bi = N % 256 == 0 ? 1 : 0;
          float* lgF = (float*)(w + W.logitsF);
          float* rlF = (float*)(w + W.rowlossF);
          slmk::EpiStoreF32 e{lgF, Cp};
          if ((s = launch_tc_bn<slmk::EpiStoreF32, false, false, true>(bi ? 256 : 64, 1, M.woK, M.hfK[(t / CH) % 2][bi],
                                                                       Cp, N, H, 0, 0, e, cs, pdl,
                                                                       gdbg(SLM_K_GEMM_FWD))) != SLM_OK)
            return s;
          CK(launch_k(lstm_head_ce_kernel, dim3(N), dim3(1024), 0, cs, pdl, (const float*)lgF, 1, lgF, d.b_o,
                      labels + (size_t)t0 * B, C, Cp, N, scale, rlF, (bf*)nullptr, (float*)nullptr, (unsigned*)nullptr,
                      (float*)nullptr));
          slmk::StepOut so{};
          for (int i = 0; i < n; ++i) so.p[i] = V((t0 + i) * per_t + per_t - 1);
          CK(launch_k(lstm_step_loss_kernel, dim3(n), dim3(1024), 0, cs, pdl, (const float*)rlF, B, scale, so,
                      loss_t + t0));
          nl += 3;
        }
      } else if (opk == SLM_OP_SUM) {
        CK(launch_k(lstm_sum_kernel, dim3(1), dim3(32), 0, cs, pdl, (const float*)loss_t, T, V(v)));
        ++nl;
      } else {
        set_error("unsupported op in lstm plan");
        return SLM_E_UNSUPPORTED;
      }
    } else {
      const int slot = t % CH;
      const bool flush = slot == 0;
      if (opk == SLM_OP_SUM) {
        CK(launch_k(fill_kernel, dim3(1), eb, 0, cs, pdl, V(v), T, 1.0f));
        ++nl;
      } else if (opk == SLM_OP_HEAD_CE && hb_now) {
        // batched head backward of steps t0..t: h operands, logits GEMM (N = n B), CE rows ->
        // d logits (bf16 ring + fp32), dh GEMM (same K slicing as the per-step path), (dh | 0)
        // into the chunk's dh ring + db_o (per step, descending), dW_o for the chunk
        const int t0 = hb_lo, n = t - t0 + 1, N = n * B, r0 = (t0 % CH) * B;   // ring rows of t0
        const int bi = N % 256 == 0 ? 2 : N % 128 == 0 ? 1 : 0, bnb = 64 << bi;
        slmk::StepIn in{};
        for (int i = 0; i < n; ++i) in.p[i] = V(head_state(t0 + i));
        CK(launch_k(lstm_hpack_multi_kernel, gsz((size_t)n * B * H), eb, 0, cs, pdl, in, n, H, B, hopR + (size_t)r0 * H));
        float* lgF = (float*)(w + W.logitsF);
        slmk::EpiStoreF32 e{lgF, Cp};
        if ((s = launch_tc_bn<slmk::EpiStoreF32, false, false, true>(bnb, 1, M.woK, M.hopRKb[bi], Cp, N, H, 0, r0, e, cs,
                                                                     pdl, gdbg(SLM_K_GEMM_FWD))) != SLM_OK)
          return s;
        CK(launch_k(lstm_head_ce_kernel, dim3(N), dim3(1024), 0, cs, pdl, (const float*)lgF, 1, lgF, d.b_o,
                    labels + (size_t)t0 * B, C, Cp, N, scale, (float*)nullptr, dlR + (size_t)r0 * Cp, dlog_f,
                    (unsigned*)nullptr, (float*)nullptr));
        slmk::EpiPartialTma e2{N};
        if ((s = launch_tc_bn<slmk::EpiPartialTma, true, false, true>(bnb, sp.hd, M.woMN, M.dlRKb[bi], H, N, Cp, 0, r0,
                                                                      e2, cs, pdl, gdbg(SLM_K_GEMM_DX), &M.pHB)) != SLM_OK)
          return s;
        CK(launch_k(lstm_head_bwd_finish_kernel, dim3(std::max((Cp + 31) / 32, 148)), dim3(512), 0, cs, pdl,
                    (const float*)(w + W.PH), sp.hd, H, N, dh_ring(t0), (const float*)dlog_f, Cp, B, n, d.db_o));
        nl += 5;
        if (t0 % CH == 0) {   // the chunk is complete: dW_o over all its rows
          slmk::EpiAccF32 e3{d.dW_o, H};
          if ((s = launch_tc_bn<slmk::EpiAccF32, true, true, false>(Cp % 256 ? 128 : 256, 1, M.hopRMN, M.dlRMN, H, Cp,
                                                                    chunk_rows(t0), 0, 0, e3, cs, pdl,
                                                                    gdbg(SLM_K_GEMM_DW))) != SLM_OK)
            return s;
          ++nl;
        }
        for (int t2 = t0; t2 <= t; ++t2) hb_batched[t2] = 1;
      } else if (opk == SLM_OP_HEAD_CE) {
        // preds = [g[Sum], a[S^{L-1}_t]]: recompute logits (the head reads only its input, A6)
        const float* sL = V(pp.first[pp.second - 1]);
        CK(launch_k(lstm_hpack_kernel, gsz((size_t)B * H), eb, 0, cs, pdl, sL, H, B, hopR + (size_t)slot * B * H));
        slmk::EpiPartialTma e{B};
        if ((s = launch_tc_bn<slmk::EpiPartialTma, false, false, true>(B, sp.lg, M.woK, M.hopRK, Cp, B, H, 0, slot * B,
                                                                       e, cs, pdl, gdbg(SLM_K_GEMM_FWD), &M.pL)) != SLM_OK)
          return s;
        CK(launch_k(lstm_head_ce_kernel, dim3(B), dim3(1024), 0, cs, pdl, Pb(sid), sp.lg, logits, d.b_o,
                    labels + (size_t)t * B, C, Cp, B, scale, (float*)nullptr, dlR + (size_t)slot * B * Cp, dlog_f,
                    (unsigned*)nullptr, (float*)nullptr));
        // dh[b][h] = sum_c dlog[b][c] W_o[c][h]  (split-K partials) -> (dh | 0)
        slmk::EpiPartialTma e2{B};
        if ((s = launch_tc_bn<slmk::EpiPartialTma, true, false, true>(B, sp.hd, M.woMN, M.dlRK, H, B, Cp, 0, slot * B,
                                                                      e2, cs, pdl, gdbg(SLM_K_GEMM_DX), &M.pH)) != SLM_OK)
          return s;
        CK(launch_k(lstm_head_bwd_finish_kernel, dim3(std::max((Cp + 31) / 32, 148)), dim3(512), 0, cs, pdl, Pb(sid),
                    sp.hd, H, B, V(v), (const float*)dlog_f, Cp, B, 1, d.db_o));
        nl += 5;
        if (flush) {   // dW_o[c][h] += sum over the chunk's rows of dlog[r][c] h[r][h]
          slmk::EpiAccF32 e3{d.dW_o, H};
          if ((s = launch_tc_bn<slmk::EpiAccF32, true, true, false>(Cp % 256 ? 128 : 256, 1, M.hopRMN, M.dlRMN, H, Cp, chunk_rows(t), 0,
                                                                    0, e3, cs, pdl, gdbg(SLM_K_GEMM_DW))) != SLM_OK)
            return s;
          ++nl;
        }
      } else if (opk == SLM_OP_LSTM_CELL || opk == SLM_OP_LSTM_GATES) {
        // g[S^l_t]: successor slices (order: layer above / head, next-step gates, next-step cell);
        // g[G^l_t]: preds = [g[S^l_t], a[G], a[x], a[S_{t-1}]?]
        const bool has_prev = t > 0;
        const int Kin = l == 0 ? K0 : H, K = Kin + H, skx = l == 0 ? sp.x0 : sp.x1;
        bf* opS = (bf*)(w + W.opR[l]) + (size_t)slot * B * K;
        bf* dpS = (bf*)(w + W.dpR[l]) + (size_t)slot * B * 4 * H;
        float* dpFS = (float*)(w + W.dpF[l]) + (size_t)slot * B * 4 * H;
        int vg = -1;   // the gates gradient node handled by this iteration
        if (opk == SLM_OP_LSTM_CELL) {
          // successor contributions, in ascending successor id (A17): the gates node above (its
          // dX partials, x columns) or the head, the next step's gates (dX partials, h
          // columns), the next step's cell (its gradient node, (0 | dc) slot)
          slmk::GradSrcs src{};
          int k = 0;
          auto pxs = [&](int ll, int tt, int col) {   // layer ll's dX partials of step tt
            const int sk2 = ll == 0 ? sp.x0 : sp.x1, K2 = lstm_K(d, ll);
            const size_t bytes = ((size_t)sk2 * B * K2 * 4 + 255) / 256 * 256;
            src.s[k++] = slmk::GradSrc{(const float*)(w + W.PX[ll] + (tt % 2) * bytes) + col, K2, sk2, -1,
                                       (long)B * K2};
          };
          const int sv = orig;
          if (l + 1 < L) {
            if (p->gnode[sv + 1] >= 0) pxs(l + 1, t, 0);                    // G^{l+1}_t
          } else if (hb_batched[t]) {
            src.s[k++] = slmk::GradSrc{dh_ring(t), 2 * H, 1, H, 0};          // batched head gradient
          } else {
            const int gs = p->gnode[t * per_t + per_t - 1];                  // H_t
            if (gs >= 0) src.s[k++] = slmk::GradSrc{V(gs), 2 * H, 1, H, 0};
          }
          if (t + 1 < T) {
            if (p->gnode[sv + per_t - 1] >= 0) pxs(l, t + 1, l == 0 ? K0 : H);   // G^l_{t+1}
            const int gs = p->gnode[sv + per_t];                                 // S^l_{t+1}
            if (gs >= 0) src.s[k++] = slmk::GradSrc{V(gs) + 4 * H, 6 * H, 1, H, 0};
          }
          const float* act = V(pp.first[pp.second - (t > 0 ? 2 : 1)]);
          const float* sprev = t > 0 ? V(pp.first[pp.second - 1]) : nullptr;
          // fuse with g[G^l_t]'s element-wise part when V' runs it next
          if (oi + 1 < order.size()) {
            const int u = order[oi + 1];
            auto pu = preds_of(u);
            if (p->op[u] == SLM_OP_LSTM_GATES && p->kind[u] == SLM_KIND_GRAD && pu.first[0] == v) {
              const int nf = has_prev ? 2 : 1;
              const float* x = V(pu.first[pu.second - nf]);
              CK(launch_k(lstm_cell_bwd_dpre_kernel, gsz((size_t)B * (Kin + H)), eb, 0, cs, pdl, src, act, sprev, H, B,
                          V(v), dpS, dpFS, x, l > 0 ? H : I, l > 0 ? 2 * H : I, Kin, opS));
              ++nl;
              vg = u;
              ++oi;
            }
          }
          if (vg < 0) {
            CK(launch_k(lstm_cell_bwd_kernel, gsz((size_t)B * H), eb, 0, cs, pdl, src, act, sprev, H, B, V(v)));
            ++nl;
          }
        } else {
          vg = v;
          const int nf = has_prev ? 2 : 1;
          const float* dact = V(pp.first[0]);   // slot 0 of g[S^l_t] = d(acts), row width 4H (+2H)
          const float* act = V(pp.first[pp.second - nf - 1]);
          const float* x = V(pp.first[pp.second - nf]);
          const float* sprev = has_prev ? V(pp.first[pp.second - 1]) : nullptr;
          const int drow = 4 * H + (has_prev ? 2 * H : 0);
          CK(launch_k(lstm_dpre_kernel, gsz((size_t)B * 4 * H), eb, 0, cs, pdl, dact, drow, act, H, B, dpS, dpFS, x, l > 0 ? H : I,
                      l > 0 ? 2 * H : I, Kin, sprev, opS));
          ++nl;
        }
        if (vg >= 0) {
          // d[x | h] = d_pre W_l:  D[m = k_in][n = b], K = 4H, split-K partials kept (time-parity
          // double buffer) and read in place by the two cell gradients that consume them
          slmk::EpiPartialTma e{B};
          if ((s = launch_tc_bn<slmk::EpiPartialTma, true, false, true>(B, skx, M.wMN[l], M.dpRK[l], K, B, 4 * H, 0,
                                                                        slot * B, e, cs, pdl, gdbg(SLM_K_GEMM_DX),
                                                                        &M.pXd[2 * l + t % 2])) != SLM_OK)
            return s;
          ++nl;
          if (flush) {   // dW_l[gate][k_in] += sum over the chunk's rows of op[r][k_in] d_pre[r][gate]
            slmk::EpiAccF32 e2{d.dW + lstm_w_offset(d, l), K};
            if ((s = launch_tc_bn<slmk::EpiAccF32, true, true, false>((4 * H) % 256 ? 128 : 256, 1, M.opRMN[l],
                                                                      M.dpRMN[l], K, 4 * H, chunk_rows(t), 0, 0, e2,
                                                                      cs, pdl, gdbg(SLM_K_GEMM_DW))) != SLM_OK)
              return s;
            // db_l += column sums of the chunk's fp32 d_pre rows (time order, plan-independent)
            CK(launch_k(colsum_acc_kernel, dim3(4 * H / 32), dim3(512), 0, cs, pdl, (const float*)(w + W.dpF[l]),
                        chunk_rows(t), 4 * H, d.db + (size_t)l * 4 * H));
            nl += 2;
          }
        }
      } else {
        set_error("unsupported gradient op in lstm plan");
        return SLM_E_UNSUPPORTED;
      }
    }
    if (msm && (s = unit_end(sid)) != SLM_OK) return s;
    for (int node : {v, partner})
      if (node >= 0) owner[p->node_tag[node]] = node;
    if (kind != SLM_KIND_GRAD && opk == SLM_OP_HEAD_CE && (t % CH == CH - 1 || t == T - 1))
      for (int t2 = t - t % CH; t2 <= t; ++t2) owner[p->node_tag[t2 * per_t + per_t - 1]] = t2 * per_t + per_t - 1;
  }
  if (msm) {   // join every stream back into the caller's
    for (int i = 0; i < NSTR; ++i) {
      CK(cudaEventRecord(S.join[i], S.streams[i]));
      CK(cudaStreamWaitEvent(st, S.join[i], 0));
    }
  }
  CK(cudaGetLastError());
  m.ts_used = ts_slot;
  if (launches) *launches = nl;
  return SLM_OK;
}

// kernels enqueue_lstm launches for this plan (the memsets are not counted); mirrors its
// fusion and operand-residency decisions
int64_t lstm_launches(const slm_plan* p, const slm_lstm_desc& d, int gates_sk, int fuse_cell) {
  int64_t nl = 0;
  const int L = d.n_layers, T = d.steps, per_t = 2 * L + 2, N = p->n_fwd, CH = kLstmChunk;
  OperandTracker trk(L);
  auto tl = [&](int o) {
    if (o == N - 1) return std::make_pair(T - 1, L);
    return std::make_pair(o / per_t, (o % per_t - 1) / 2);
  };
  std::vector<int> owner(p->tag_size.size(), -1);
  std::vector<char> hb_batched(T, 0);
  const LstmSplits sp = lstm_splits(d, gates_sk);
  auto head_state = [&](int t) {
    const int gh = p->gnode[t * per_t + per_t - 1];
    return gh < 0 ? -1 : p->preds[p->pred_ptr[gh + 1] - 1];
  };
  const std::vector<int>& order = p->order;
  for (size_t oi = 0; oi < order.size(); ++oi) {
    const int v = order[oi], opk = p->op[v], kind = p->kind[v];
    if (opk == SLM_OP_INPUT) continue;
    const auto [t, l] = tl(p->orig[v]);
    const int* pr = p->preds.data() + p->pred_ptr[v];
    const int np = p->pred_ptr[v + 1] - p->pred_ptr[v];
    int partner = -1;
    if (kind != SLM_KIND_GRAD) {
      if (opk == SLM_OP_LSTM_GATES) {
        const int xn = pr[0], hn = np > 1 ? pr[1] : OperandTracker::kZeros;
        if (trk.gates_needs_pack(l, t, xn, hn)) {
          ++nl;
          trk.packed(l, t, xn, hn);
        }
        nl += ((l == 0 ? sp.g0 : sp.g1) == 1 && fuse_cell) ? 1 : 2;   // GEMM with the cell epilogue, or + gates/cell kernel
        if (oi + 1 < order.size()) {
          const int u = order[oi + 1];
          if (p->op[u] == SLM_OP_LSTM_CELL && p->kind[u] == kind && p->preds[p->pred_ptr[u]] == v) {
            trk.cell(u, l, t, L, T, (t + 1) * per_t);
            partner = u;
            ++oi;
          }
        }
      } else if (opk == SLM_OP_LSTM_CELL) {
        trk.cell(v, l, t, L, T, (t + 1) * per_t);
        ++nl;
      } else if (opk == SLM_OP_HEAD_CE) {
        if (t % CH == CH - 1 || t == T - 1) {   // batched forward heads
          nl += 3;
          for (int t2 = t - t % CH; t2 <= t; ++t2) owner[p->node_tag[t2 * per_t + per_t - 1]] = t2 * per_t + per_t - 1;
        }
      } else {
        ++nl;
      }
    } else {
      const bool flush = t % CH == 0;
      if (opk == SLM_OP_HEAD_CE) {
        if (hb_batched[t]) continue;
        int lo = t + 1;
        for (int t2 = t; t2 >= t - t % CH; --t2) {
          const int a = head_state(t2);
          if (a < 0 || owner[p->node_tag[a]] != a) break;
          lo = t2;
        }
        if (lo < t) {   // batched head backward of steps lo..t
          nl += 5 + (lo % CH == 0);
          for (int t2 = lo; t2 <= t; ++t2) hb_batched[t2] = 1;
        } else {
          nl += 5 + flush;
        }
      } else if (opk == SLM_OP_LSTM_GATES) {
        nl += 2 + 2 * flush;   // d_pre/pack, dX GEMM (+ dW GEMM and db column sums)
      } else if (opk == SLM_OP_LSTM_CELL) {
        const int u = oi + 1 < order.size() ? order[oi + 1] : -1;
        if (u >= 0 && p->op[u] == SLM_OP_LSTM_GATES && p->kind[u] == SLM_KIND_GRAD && p->preds[p->pred_ptr[u]] == v) {
          nl += 2 + 2 * flush;   // fused cell/d_pre/pack + dX GEMM
          partner = u;
          ++oi;
        } else {
          nl += 1;
        }
      } else {
        nl += 1;
      }
    }
    for (int node : {v, partner})
      if (node >= 0) owner[p->node_tag[node]] = node;
  }
  return nl;
}

}  // namespace
