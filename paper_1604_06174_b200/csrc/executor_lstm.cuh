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
// Forward / re-computed (mirror) gates + cell nodes run as RUNS of up to
// kRunMax consecutive steps of one layer (lstm_run.cuh): the input projection of the run as one
// batched GEMM (N = n B), then ONE persistent launch for the n steps of the recurrence with the
// gates and the cell fused into its epilogue.  A run's recurrent state (bf16 h, fp32 c) stays in
// per-(layer, kind) side buffers, so consecutive runs of a layer continue without touching the
// pool; the bf16 h of every step also lands in the layer's chunk ring, which the next layer's
// input projection and the head read.  Only values some other unit reads through the pool are
// written to their tags ("materialised": kept checkpoints, mirrors, anything a gradient node
// reads); the dropped forward values of a segment never leave the chip.
//
// Scheduling: V' is split into phases (maximal ranges without gradient nodes).  In a phase whose
// gates/cell nodes all come in (G, S) pairs, the runs are issued chunk by chunk, layer by layer
// (a legal topological reorder of V': every value is produced before it is read, and the phase
// writes each of its tags once -- checked, else the phase runs node by node in V' order with runs
// of one step; both give the same bits).  Across streams, happens-before edges come from
// per-resource last-writer / reader tracking (option lstm_streams).
//
// The backward:
//   head  (fwd)         batched per 32-step chunk: logits GEMM over the chunk's ring rows ->
//                       softmax-CE rows -> per-step losses
//   grad head           pack h -> logits GEMM -> CE + dlogits -> dh GEMM (split-K) -> (dh | 0)
//   grad cell           sum of successor slices -> d(acts) | (0 | dc_prev)
//   grad gates          d_pre (+ db) -> dX GEMM (split-K) -> scatter into d(inputs)
//   weight gradients    the GEMM operands of each step are kept in a per-layer ring of CH time
//                       steps; once per chunk (in time order, independent of the plan)
//                       dW_l += opᵀ d_pre runs as ONE GEMM with K = B * CH (PAPER.md:488-489
//                       "in-place accumulation"), instead of CH GEMMs with K = B.
// Every reduction has a fixed order, so the checkpointed step is bit-identical to the plain one.

namespace {

constexpr int kLstmChunk = 32;   // time steps per weight-gradient GEMM

// split-K of a backward run's input-gradient GEMM d x = d_pre W_ih (M = H, N = 8 B, K = 4 H): without
// it 16 CTAs each run the whole K = 4H (35 us per run at C3); four K slices give 64 CTAs whose
// fp32 partials are summed in slice order (deterministic, the same in every plan)
constexpr int kDxSplit = 4;
struct LstmWs {
  size_t logits, dlog_f, rowloss, offs, cnt, hopR, dlR, logitsF, rowlossF, dhR, PH, bar, total;
  std::vector<size_t> P;                     // split-K partials, one buffer per stream (layers, head)
  std::vector<size_t> pdx;                   // per layer: split-K partials of the runs' input gradient
  std::vector<size_t> opR, dpR, dpF, PX;     // per layer: backward rings, dX partials
  // per lane (layer l, kind k: lane l + L k) of the forward runs: recurrent state hx [2][B][H]
  // bf16 and c [B][H] fp32, the chunk ring [2][CH B][H] bf16 of h, the packed input-projection
  // operand [kRunMax B][Kin] bf16 and the projection X [kRunMax B][4H] fp32
  std::vector<size_t> hx, cst, ring, xop, xp;
  // per layer, backward runs (batch 64): d_pre exchange [2][B][4H] bf16, dc state [B][H], the
  // partial exchange [H/128][4][4][B][32] fp32, the gradient from the layer above [2][CH B + 256][H]
  // fp32 (chunk parity; 256 rows of slack for the padded projection), step / exchange counters
  std::vector<size_t> dpx, dcst, xch, dxa;
  size_t bbar;
};
// the backward runs (lstm_run.cuh) serve batch 64; other batches keep the node-by-node backward
inline bool lstm_bwd_runs(const slm_lstm_desc& d) { return d.batch == 64; }

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
  L.logitsF = off;  off += al(CH * B * Cp * 4);
  L.rowlossF = off; off += al(CH * B * 4);
  L.dhR = off;      off += 2 * al(CH * B * 2 * H * 4);          // (dh | 0) of batched head steps, chunk parity
  L.PH = off;       off += al((size_t)sp.hd * CH * B * H * 4);  // split-K partials of the batched dh GEMM
  L.dlR = off;      off += al(CH * B * Cp * 2);
  L.bar = off;      off += al(2 * d.n_layers * 4);
  L.bbar = off;     off += al((size_t)d.n_layers * (1 + H / 128) * 4);
  if (lstm_bwd_runs(d))
    for (int l = 0; l < d.n_layers; ++l) {
      L.dpx.push_back(off);  off += al(2 * B * 4 * H * 2);
      L.dcst.push_back(off); off += al(B * H * 4);
      L.xch.push_back(off);  off += al((H / 128) * 16 * B * 32 * 4);
      L.dxa.push_back(off);  off += 2 * al((CH * B + 256) * H * 4);
      // split-K partials of the run's input-gradient GEMM (kDxSplit x [run rows padded to 256][H])
      L.pdx.push_back(off);  off += al((size_t)kDxSplit * ((slmk::kRunMax * B + 255) / 256 * 256) * H * 4);
    }
  const size_t RM = slmk::kRunMax;
  for (int ln = 0; ln < 2 * d.n_layers; ++ln) {
    const size_t kin = (ln % d.n_layers) == 0 ? (size_t)lstm_kin0(d.n_in) : H;
    L.hx.push_back(off);   off += al(2 * B * H * 2);
    L.cst.push_back(off);  off += al(B * H * 4);
    L.ring.push_back(off); off += al(2 * CH * B * H * 2);
    L.xop.push_back(off);  off += al(RM * B * kin * 2);
    L.xp.push_back(off);   off += 2 * al(RM * B * 4 * H * 4);   // double-buffered (run parity)
  }
  // backward rings of one chunk; with backward runs two of them (chunk parity), so the chunk's
  // weight-gradient GEMM can run on its own stream while the next chunk's runs fill the other
  const size_t nring = lstm_bwd_runs(d) ? 2 : 1;
  for (int l = 0; l < d.n_layers; ++l) {
    L.opR.push_back(off);
    off += nring * al(CH * B * lstm_K(d, l) * 2);
    L.dpR.push_back(off);
    off += nring * al(CH * B * 4 * H * 2);
    L.dpF.push_back(off);
    off += nring * al(CH * B * 4 * H * 4);
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
  M.opRMN.resize(nl);
  M.dpRK.resize(nl);
  M.dpRMN.resize(nl);
  M.dpR256.resize(nl);
  M.opRMN1.resize(nl);
  M.dpRMN1.resize(nl);
  M.dpR2561.resize(nl);
  M.dpxM.resize(nl);
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
    if ((st = make_map(&M.opRK[l], w + L.opR[l], K, CH * B, (uint32_t)B)) != SLM_OK) return st;
    if ((st = make_map(&M.opRMN[l], w + L.opR[l], K, CH * B, 64)) != SLM_OK) return st;
    if ((st = make_map(&M.dpRK[l], w + L.dpR[l], 4 * H, CH * B, (uint32_t)B)) != SLM_OK) return st;
    if ((st = make_map(&M.dpRMN[l], w + L.dpR[l], 4 * H, CH * B, 64)) != SLM_OK) return st;
    if ((st = make_map(&M.dpR256[l], w + L.dpR[l], 4 * H, CH * B, 256)) != SLM_OK) return st;
    if (lstm_bwd_runs(d)) {   // the odd-chunk halves
      const size_t ob = (CH * B * K * 2 + 255) / 256 * 256, db = (CH * B * 4 * H * 2 + 255) / 256 * 256;
      if ((st = make_map(&M.opRMN1[l], w + L.opR[l] + ob, K, CH * B, 64)) != SLM_OK) return st;
      if ((st = make_map(&M.dpRMN1[l], w + L.dpR[l] + db, 4 * H, CH * B, 64)) != SLM_OK) return st;
      if ((st = make_map(&M.dpR2561[l], w + L.dpR[l] + db, 4 * H, CH * B, 256)) != SLM_OK) return st;
    }
    if (lstm_bwd_runs(d) && (st = make_map(&M.dpxM[l], w + L.dpx[l], 4 * H, 2 * B, (uint32_t)B)) != SLM_OK) return st;
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
  const uint64_t RM = slmk::kRunMax;
  M.hxM.resize(2 * nl);
  M.xpM.resize(2 * nl);
  M.xpM1.resize(2 * nl);
  for (int bi = 0; bi < 2; ++bi) {
    M.ringM[bi].resize(2 * nl);
    M.xopM[bi].resize(2 * nl);
  }
  for (int ln = 0; ln < 2 * nl; ++ln) {
    const uint64_t kin = (ln % nl) == 0 ? (uint64_t)lstm_kin0(d.n_in) : H;
    if ((st = make_map(&M.hxM[ln], w + L.hx[ln], H, 2 * B, (uint32_t)B)) != SLM_OK) return st;
    if ((st = make_map_f32_box(&M.xpM[ln], w + L.xp[ln], 4 * H, RM * B, 32, 64)) != SLM_OK) return st;
    if ((st = make_map_f32_box(&M.xpM1[ln], w + L.xp[ln] + (RM * B * 4 * H * 4 + 255) / 256 * 256, 4 * H, RM * B, 32,
                               64)) != SLM_OK)
      return st;
    for (int bi = 0; bi < 2; ++bi) {
      if ((st = make_map(&M.ringM[bi][ln], w + L.ring[ln], H, 2 * CH * B, bi ? 256u : 64u)) != SLM_OK) return st;
      if ((st = make_map(&M.xopM[bi][ln], w + L.xop[ln], kin, RM * B, bi ? 256u : 64u)) != SLM_OK) return st;
    }
  }
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

// ---- schedule (see the header): launch units in issue order and the materialised set
struct LstmUnit {
  int type = 0;                       // 0 = the V' node at order index oi (+ fused successor), 1 = run,
                                      // 2 = backward run (steps t0, t0-1, .. t0-n+1; g = the g[S] nodes),
                                      // 3 = input gradient + weight-gradient flush of steps t0 .. t0+n-1
  int oi = -1;
  int l = 0, k = 0, t0 = 0, n = 0;    // run: layer, kind (0 forward, 1 mirror), first step, steps
  int g[slmk::kRunMax], s[slmk::kRunMax];   // the run's gates / cell nodes (s = -1: gates only)
};
struct LstmSched {
  std::vector<LstmUnit> units;
  std::vector<char> mat;   // per G' node: its value is written to its tag
  int fused = 0;           // phases issued chunk by chunk, layer by layer
};

LstmSched lstm_schedule(const slm_plan* p, const slm_lstm_desc& d, bool fuse, bool bwd_runs) {
  const int L = d.n_layers, T = d.steps, per_t = 2 * L + 2, CH = kLstmChunk, RM = slmk::kRunMax;
  const std::vector<int>& order = p->order;
  const int nn = (int)p->kind.size();
  LstmSched S;
  S.mat.assign(nn, 1);
  auto op = [&](int v) { return p->op[v]; };
  auto pred0 = [&](int v) { return p->preds[p->pred_ptr[v]]; };
  auto pred1 = [&](int v) { return p->pred_ptr[v + 1] - p->pred_ptr[v] > 1 ? p->preds[p->pred_ptr[v] + 1] : -1; };
  auto tof = [&](int v) { return p->orig[v] / per_t; };
  auto lof = [&](int v) { return (p->orig[v] % per_t - 1) / 2; };
  std::vector<std::vector<int>> readers(nn);
  for (int v : order)
    for (int i = p->pred_ptr[v]; i < p->pred_ptr[v + 1]; ++i) readers[p->preds[i]].push_back(v);
  struct Item {
    int oi, g, s;   // g >= 0: a forward / mirror gates node and its fused cell s (-1: none)
  };
  std::vector<Item> items;
  for (size_t oi = 0; oi < order.size(); ++oi) {
    const int v = order[oi];
    if (p->kind[v] != SLM_KIND_GRAD && op(v) == SLM_OP_LSTM_GATES) {
      int c = -1;
      if (oi + 1 < order.size()) {
        const int u = order[oi + 1];
        if (op(u) == SLM_OP_LSTM_CELL && p->kind[u] == p->kind[v] && pred0(u) == v) c = u;
      }
      items.push_back({(int)oi, v, c});
      if (c >= 0) ++oi;
    } else {
      items.push_back({(int)oi, -1, -1});
    }
  }
  auto node_unit = [&](int oi) {
    LstmUnit u;
    u.oi = oi;
    S.units.push_back(u);
  };
  auto kind01 = [&](int v) { return p->kind[v] == SLM_KIND_MIRROR ? 1 : 0; };
  std::vector<char> inph(nn, 0);
  auto is_grad = [&](const Item& it) { return it.g < 0 && p->kind[order[it.oi]] == SLM_KIND_GRAD; };
  auto grad_op = [&](const Item& it, int o) { return is_grad(it) && op(order[it.oi]) == o; };
  size_t a0 = 0;
  while (a0 < items.size()) {
    if (is_grad(items[a0]) && !bwd_runs) {
      node_unit(items[a0].oi);
      ++a0;
      continue;
    }
    if (is_grad(items[a0])) {
      // ---- gradient phase [a0, a1): g[S^l_t] -> backward runs, g[G^l_t] -> input gradient /
      // weight-gradient flush units.  Fused (chunk by chunk descending, layer by layer from the top)
      // when every g[S^l_t] of the phase has its g[G^l_t] in the phase and vice versa; else node by
      // node in V' order with runs of one step.
      size_t a1 = a0;
      while (a1 < items.size() && is_grad(items[a1])) ++a1;
      bool ok = fuse;
      for (size_t i = a0; i < a1; ++i) inph[order[items[i].oi]] = 1;
      auto gnode_of = [&](int gv, int dlt) { return p->gnode[p->orig[gv] + dlt]; };   // g[S^l_t] -> g[G^l_t]: orig - 1
      for (size_t i = a0; i < a1 && ok; ++i) {
        const int v = order[items[i].oi];
        if (op(v) == SLM_OP_LSTM_CELL) ok = gnode_of(v, -1) >= 0 && inph[gnode_of(v, -1)];
        else if (op(v) == SLM_OP_LSTM_GATES) ok = gnode_of(v, 1) >= 0 && inph[gnode_of(v, 1)];
      }
      auto bunit = [&](int type, int l, int t0, int n, const int* gs) {
        LstmUnit u;
        u.type = type;
        u.l = l;
        u.t0 = t0;
        u.n = n;
        for (int i = 0; i < n && gs; ++i) u.g[i] = gs[i];
        S.units.push_back(u);
      };
      if (!ok) {
        for (size_t i = a0; i < a1; ++i) {
          const int v = order[items[i].oi];
          if (op(v) == SLM_OP_LSTM_CELL) bunit(2, lof(v), tof(v), 1, &v);
          else if (op(v) == SLM_OP_LSTM_GATES) bunit(3, lof(v), tof(v), 1, nullptr);
          else node_unit(items[i].oi);
        }
      } else {
        ++S.fused;
        for (size_t i = a0; i < a1; ++i)   // g[Sum] and other non-step nodes first, in V' order
          if (!grad_op(items[i], SLM_OP_LSTM_CELL) && !grad_op(items[i], SLM_OP_LSTM_GATES) &&
              !grad_op(items[i], SLM_OP_HEAD_CE))
            node_unit(items[i].oi);
        // per chunk (descending): its head gradients in V' order, then per layer (top first) the
        // runs of its g[S] nodes, each followed by its input-gradient / flush unit
        std::vector<std::vector<int>> byc((T + CH - 1) / CH), lay((size_t)L * ((T + CH - 1) / CH));
        for (size_t i = a0; i < a1; ++i) {
          const int v = order[items[i].oi];
          if (op(v) == SLM_OP_HEAD_CE) byc[tof(v) / CH].push_back(items[i].oi);
          else if (op(v) == SLM_OP_LSTM_CELL) lay[(size_t)(tof(v) / CH) * L + lof(v)].push_back(v);
        }
        for (int c = (int)byc.size() - 1; c >= 0; --c) {
          for (int oi : byc[c]) node_unit(oi);
          // the chunk's runs: RM-step blocks descending, inside a block the layers from the top
          // (a wavefront with a lag of one block between neighbouring layers)
          std::vector<std::vector<LstmUnit>> blk((CH + RM - 1) / RM);
          for (int l = L - 1; l >= 0; --l) {
            std::vector<int>& gsv = lay[(size_t)c * L + l];
            std::sort(gsv.begin(), gsv.end(), [&](int x, int y) { return tof(x) > tof(y); });
            size_t k0 = 0;
            while (k0 < gsv.size()) {
              size_t k1 = k0 + 1;
              while (k1 < gsv.size() && tof(gsv[k1]) == tof(gsv[k1 - 1]) - 1 && tof(gsv[k1]) / RM == tof(gsv[k0]) / RM) ++k1;
              const int n = (int)(k1 - k0), th = tof(gsv[k0]);
              LstmUnit u2, u3;
              u2.type = 2;
              u2.l = u3.l = l;
              u2.t0 = th;
              u2.n = u3.n = n;
              for (int i = 0; i < n; ++i) u2.g[i] = gsv[k0 + i];
              u3.type = 3;
              u3.t0 = th - n + 1;
              blk[(th % CH) / RM].push_back(u2);
              blk[(th % CH) / RM].push_back(u3);
              k0 = k1;
            }
          }
          for (int b = (int)blk.size() - 1; b >= 0; --b)
            for (const LstmUnit& u : blk[b]) S.units.push_back(u);
        }
      }
      for (size_t i = a0; i < a1; ++i) inph[order[items[i].oi]] = 0;
      a0 = a1;
      continue;
    }
    size_t a1 = a0;
    while (a1 < items.size() && !is_grad(items[a1])) ++a1;
    // ---- phase [a0, a1): fusable when every gates / cell node is paired and the forward heads
    // come in whole chunks
    bool ok = fuse;
    std::vector<int> pn;
    for (size_t i = a0; i < a1; ++i) {
      const Item& it = items[i];
      if (it.g >= 0) {
        pn.push_back(it.g);
        if (it.s >= 0) pn.push_back(it.s);
        continue;
      }
      const int v = order[it.oi], o = op(v);
      pn.push_back(v);
      if (o == SLM_OP_LSTM_CELL || (o == SLM_OP_HEAD_CE && p->kind[v] != SLM_KIND_FWD) ||
          (o != SLM_OP_HEAD_CE && o != SLM_OP_INPUT && o != SLM_OP_SUM))
        ok = false;
    }
    for (int v : pn) inph[v] = 1;
    // a gates node without its cell must be the last step of its lane in the phase (the run computes
    // that step's cell into its side buffers only; e.g. the kept state closing a time segment)
    for (size_t i = a0; i < a1 && ok; ++i) {
      const Item& it = items[i];
      if (it.g < 0 || it.s >= 0) continue;
      for (size_t i2 = i + 1; i2 < a1; ++i2)
        if (items[i2].g >= 0 && lof(items[i2].g) == lof(it.g) && kind01(items[i2].g) == kind01(it.g)) ok = false;
    }
    if (ok)
      for (int v : pn)
        if (op(v) == SLM_OP_HEAD_CE) {
          const int t = tof(v), te = std::min(T - 1, t - t % CH + CH - 1);
          if (!inph[te * per_t + per_t - 1]) ok = false;   // forward nodes: G' id == forward id
        }
    if (ok) {
      // materialise a value iff some reader does not get it on chip / from a side buffer
      for (int v : pn) {
        const int o = op(v);
        if (o != SLM_OP_LSTM_GATES && o != SLM_OP_LSTM_CELL) continue;
        bool need = false;
        for (int r : readers[v]) {
          bool cov = false;
          if (o == SLM_OP_LSTM_GATES) {
            cov = inph[r] && op(r) == SLM_OP_LSTM_CELL && pred0(r) == v;
          } else if (inph[r] && p->kind[r] == p->kind[v]) {
            const int dr = p->orig[r] - p->orig[v];
            cov = (dr == per_t - 1 && op(r) == SLM_OP_LSTM_GATES) || (dr == per_t && op(r) == SLM_OP_LSTM_CELL) ||
                  (dr == 1 && op(r) == SLM_OP_LSTM_GATES) ||
                  (dr == 1 && op(r) == SLM_OP_HEAD_CE && p->kind[v] == SLM_KIND_FWD);
          }
          if (!cov) {
            need = true;
            break;
          }
        }
        S.mat[v] = need;
      }
      // the reordered phase must write each tag once and read no tag it writes
      std::vector<int> wt;
      for (int v : pn)
        if (((op(v) == SLM_OP_LSTM_GATES || op(v) == SLM_OP_LSTM_CELL) && S.mat[v]) || op(v) == SLM_OP_HEAD_CE)
          wt.push_back(p->node_tag[v]);
      std::sort(wt.begin(), wt.end());
      if (std::adjacent_find(wt.begin(), wt.end()) != wt.end()) ok = false;
      for (int v : pn) {
        if (!ok || op(v) != SLM_OP_LSTM_GATES) continue;
        const int sp = pred1(v), xn = pred0(v);
        for (int r : {sp, lof(v) > 0 ? xn : -1})
          if (r >= 0 && !(inph[r] && p->kind[r] == p->kind[v]) &&
              std::binary_search(wt.begin(), wt.end(), p->node_tag[r]))
            ok = false;
      }
      if (!ok)
        for (int v : pn) S.mat[v] = 1;
    }
    if (!ok) {   // node by node in V' order, runs of one step (a lone gates node: gates only)
      for (size_t i = a0; i < a1; ++i) {
        const Item& it = items[i];
        if (it.g < 0) {
          node_unit(it.oi);
          continue;
        }
        LstmUnit u;
        u.type = 1;
        u.l = lof(it.g);
        u.k = kind01(it.g);
        u.t0 = tof(it.g);
        u.n = 1;
        u.g[0] = it.g;
        u.s[0] = it.s;
        S.units.push_back(u);
      }
    } else {
      ++S.fused;
      // runs per lane (consecutive steps of one chunk, at most kRunMax), issued by (chunk, layer, kind)
      std::vector<LstmUnit> runs;
      std::vector<std::vector<std::pair<int, int>>> lane(2 * L);
      for (size_t i = a0; i < a1; ++i)
        if (items[i].g >= 0) lane[lof(items[i].g) + L * kind01(items[i].g)].push_back({items[i].g, items[i].s});
      for (int ln = 0; ln < 2 * L; ++ln) {
        LstmUnit u;
        u.type = 1;
        u.l = ln % L;
        u.k = ln / L;
        for (auto& gs : lane[ln]) {
          const int t = tof(gs.first);
          if (u.n > 0 && (t != u.t0 + u.n || t / RM != u.t0 / RM)) {   // runs stay inside an RM-step block
            runs.push_back(u);
            u.n = 0;
          }
          if (u.n == 0) u.t0 = t;
          u.g[u.n] = gs.first;
          u.s[u.n] = gs.second;
          ++u.n;
        }
        if (u.n > 0) runs.push_back(u);
      }
      // block by block, layer by layer inside a block: layer l's run of a block waits only for
      // layer l-1's run of the same block (a wavefront with a lag of one block)
      std::stable_sort(runs.begin(), runs.end(), [&](const LstmUnit& x, const LstmUnit& y) {
        return std::make_tuple(x.t0 / RM, x.l, x.k, x.t0) < std::make_tuple(y.t0 / RM, y.l, y.k, y.t0);
      });
      std::vector<int> head_oi(T / CH + 2, -1);   // V' index of each chunk's last forward head
      int sum_oi = -1;
      for (size_t i = a0; i < a1; ++i) {
        if (items[i].g >= 0) continue;
        const int v = order[items[i].oi];
        if (op(v) == SLM_OP_HEAD_CE) {
          const int t = tof(v);
          if (t % CH == CH - 1 || t == T - 1) head_oi[t / CH] = items[i].oi;
        } else if (op(v) == SLM_OP_SUM) {
          sum_oi = items[i].oi;
        }
      }
      for (size_t r = 0; r < runs.size(); ++r) {
        S.units.push_back(runs[r]);
        const int c = runs[r].t0 / CH;
        const bool last_top = r + 1 == runs.size() || runs[r + 1].t0 / CH != c;
        if (last_top && head_oi[c] >= 0) {
          node_unit(head_oi[c]);
          head_oi[c] = -1;
        }
      }
      for (int c = 0; c < (int)head_oi.size(); ++c)
        if (head_oi[c] >= 0) node_unit(head_oi[c]);
      if (sum_oi >= 0) node_unit(sum_oi);
    }
    for (int v : pn) inph[v] = 0;
    a0 = a1;
  }
  return S;
}

// Launch a persistent run kernel (its CTAs wait on each other every step, so all of them must be
// resident at once).  Not a cooperative launch: cooperative grids were measured to serialise
// across streams (the four layer runs of the wavefront ran one after the other).  Residency holds
// by construction instead: the runs that can be in flight together (one per forward or mirror
// lane: 2 L H / 32 <= 128 CTAs at C3 with one of the two kinds active) fit on the 148 SMs, every
// other kernel of the step finishes without waiting on a run, and a PDL successor of a run is
// only released by the run's final griddepcontrol.launch_dependents.
template <class... KArgs, class... Args>
cudaError_t launch_run(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                       Args... args) {
  return launch_kc(k, grid, block, smem, st, pdl, 1, args...);
}

slm_status launch_bwd_run(const CUtensorMap& w, const CUtensorMap& dpx, const slmk::BwdRun& a, cudaStream_t st,
                          bool pdl) {
  using C = slmk::BwdRunCfg;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(slmk::lstm_bwd_run_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  CK(launch_run(slmk::lstm_bwd_run_kernel, dim3(a.H / 32), dim3(slmk::kRunThreads), C::SMEM, st, pdl, w, dpx, a));
  return SLM_OK;
}

template <int B>
slm_status launch_fwd_run(const CUtensorMap& w, const CUtensorMap& h, const CUtensorMap& x, const slmk::FwdRun& a,
                          cudaStream_t st, bool pdl) {
  using C = slmk::FwdRunCfg<B>;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(slmk::lstm_fwd_run_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  CK(launch_run(slmk::lstm_fwd_run_kernel<B>, dim3(a.H / 32), dim3(slmk::kRunThreads), C::SMEM, st, pdl, w, h, x, a));
  return SLM_OK;
}

// dry = true: no CUDA call, only the launch count (slm_step_launches)
slm_status enqueue_lstm(const slm_plan* p, slm_model& m, const void* xin, const int32_t* labels, void* pool,
                        void* ws, float* loss, cudaStream_t st, int64_t* launches, bool dry = false) {
  using namespace slmk;
  using bf = __nv_bfloat16;
  const slm_lstm_desc& d = m.ld;
  slm_lstm_state& S = m.lst;
  const bool pdl = m.pdl != 0;
  int ts_slot = 0;
  if (!dry && m.profile_ts > 0 && (int)m.ts_kind.size() < m.profile_ts) {
    m.ts_kind.resize(m.profile_ts);
    m.ts_aux.resize(m.profile_ts);
  }
  auto gdbg = [&](int kind) -> int {   // launch slot for the device-clock GEMM timing
    if (dry || m.profile_ts <= 0 || m.ts_buf == nullptr || ts_slot >= m.profile_ts) return 0;
    m.ts_kind[ts_slot] = kind;
    m.ts_aux[ts_slot] = m.ts_cur_aux;
    return ((++ts_slot) << 8) | (m.profile_ts_dep ? 8 : 0);
  };
  // every CUDA call of the step goes through these (skipped in a dry run)
#define LK(call)      \
  do {                \
    if (!dry) CK(call); \
  } while (0)
#define LT(call)                                            \
  do {                                                      \
    if (!dry && (s = (call)) != SLM_OK) return s;           \
  } while (0)
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
  slm_status s = SLM_OK;
  if (!dry && (s = lstm_bind_maps(d, S.maps, ws, m.lstm_sk, m.lstm_skx)) != SLM_OK) return s;
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
  const dim3 eb(256);
  // element-wise grids sized to the work (one element per thread, at most 4 CTAs per SM) so
  // the kernels of concurrent layer streams share the SMs
  auto gsz = [&](size_t n) { return dim3((unsigned)std::max<size_t>(1, std::min<size_t>(592, (n + 255) / 256))); };
  int64_t nl = 0;
  // gradients are overwritten by every step: zero the in-place accumulators first
  LK(cudaMemsetAsync(d.dW, 0, lstm_w_offset(d, L) * 4, st));
  LK(cudaMemsetAsync(d.db, 0, (size_t)L * 4 * H * 4, st));
  LK(cudaMemsetAsync(d.dW_o, 0, (size_t)Cp * H * 4, st));
  LK(cudaMemsetAsync(d.db_o, 0, (size_t)Cp * 4, st));
  // the run kernels' step counters (monotone within a step; the host tracks each one's value)
  unsigned* bar = (unsigned*)(w + W.bar);
  LK(cudaMemsetAsync(bar, 0, (size_t)2 * L * 4, st));
  std::vector<unsigned> bar_val(2 * L, 0u);
  // weight-gradient chunk of time t: slot in the ring and whether t closes the chunk (the
  // backward visits each layer's steps in descending t, so the chunk's lowest t comes last)
  auto chunk_rows = [&](int t) { return std::min(CH, T - (t / CH) * CH) * B; };

  // backward runs: step / exchange counters, the lowest step each layer's state belongs to
  const bool bwdr = lstm_bwd_runs(d);
  unsigned* bbar = (unsigned*)(w + W.bbar);
  if (bwdr) LK(cudaMemsetAsync(bbar, 0, (size_t)L * (1 + H / 128) * 4, st));
  std::vector<unsigned> bbar_val(L, 0u), bxbar_val(L, 0u);
  std::vector<int> bstate(L, -1);
  auto dxa_ptr = [&](int l, int t) {   // rows of step t in the gradient layer l receives from layer l+1
    return (float*)(w + W.dxa[l] + ((t / CH) % 2) * (((size_t)(CH * B + 256) * H * 4 + 255) / 256 * 256)) +
           (size_t)(t % CH) * B * H;
  };
  // ---- forward lanes (layer l, kind k): side state and which V' node each holds
  auto lane_of = [&](int l, int k) { return l + L * k; };
  std::vector<int> hx_node(2 * L, -1), cs_node(2 * L, -1);
  std::vector<int> ring_node((size_t)2 * L * 2 * CH, -1);   // [lane][chunk parity][slot]
  auto rslot = [&](int t) { return ((t / CH) % 2) * CH + t % CH; };
  auto ring_ptr = [&](int ln, int t) { return (bf*)(w + W.ring[ln]) + (size_t)rslot(t) * B * H; };

  // ---- layer wavefront (option lstm_streams): every launch unit runs on the stream of its
  // layer (the head and the loss on stream L); happens-before edges come from tracking, per
  // resource (pool tag, ring buffer), the last writer and the latest reader on each
  // stream, so concurrent units never touch a buffer out of V' order.  A dependency is a
  // (stream, unit sequence number); it is skipped when the waiting stream is already ordered
  // after that unit (same stream, or an earlier wait on a later unit of that stream).  Events
  // live in a per-stream ring large enough to hold a step's units; a re-recorded slot only
  // makes a (very old) wait more conservative, never wrong.
  const bool msm = m.lstm_streams != 0 && (st != nullptr || dry);
  // lstm_streams = 2: re-computed (mirror) units get streams of their own (L+1+l), so the
  // recompute of segment j-1 can overlap the backward of segment j
  // + one stream for the weight-gradient GEMMs of the backward runs (WST)
  const int WST = m.lstm_streams >= 2 ? 2 * L + 1 : L + 1;
  // + one stream per layer for the input projections of the forward / recompute runs (PST + l)
  const int PST = WST + 1;
  const int NSTR = PST + L;
  constexpr int kRing = 16384;
  const int ntag = (int)p->tag_size.size();
  auto DHR = [&](int par) { return ntag + par; };                       // batched (dh | 0) ring, chunk parity
  auto PXR = [&](int l, int par) { return ntag + 2 + 2 * l + par; };    // dX partials of layer l
  // the chunk ring of a forward lane and the gradient layer l receives from layer l+1 are tracked
  // per RM-step block (rows of different blocks are disjoint): block id (t / RM) mod NBK
  constexpr int NBK = 2 * kLstmChunk / slmk::kRunMax;
  auto bk = [&](int t) { return (t / slmk::kRunMax) % NBK; };
  auto RNG = [&](int ln, int t) { return ntag + 2 + 2 * L + NBK * ln + bk(t); };            // forward ring
  auto DXA = [&](int l, int t) { return ntag + 2 + 2 * L + NBK * 2 * L + NBK * l + bk(t); };  // from layer l+1
  // the backward rings (op / d_pre) of layer l, chunk parity
  auto WGR = [&](int l, int par) { return ntag + 2 + 2 * L + 3 * NBK * L + 2 * l + par; };
  // the projection X of lane ln, run parity
  auto XPR = [&](int ln, int par) { return ntag + 2 + 2 * L + 3 * NBK * L + 2 * L + 2 * ln + par; };
  const int HOP = ntag + 2 + 2 * L + 3 * NBK * L + 2 * L + 4 * L;   // the number of resources
  std::vector<int> xp_cnt(2 * L, 0);   // runs issued per lane (parity of the X half)
  std::vector<int> rd, wr;
  // dependencies are unit ids u = seq * NSTR + stream (seq = per-stream unit counter)
  std::vector<long> res_w, res_r;   // [resource] last writer unit; [resource][stream] latest reader
  std::vector<long> seqn(NSTR, 0), waits;
  std::vector<long> known((size_t)NSTR * NSTR, -1);   // [a][s]: latest seq of s stream a is ordered after
  if (msm) {
    if (!dry) {
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
      CK(cudaEventRecord(S.fork, st));
      for (int i = 0; i < NSTR; ++i) CK(cudaStreamWaitEvent(S.streams[i], S.fork, 0));
    }
    res_w.assign(HOP, -1);
    res_r.assign((size_t)HOP * NSTR, -1);
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
      LK(cudaStreamWaitEvent(S.streams[sid], evt(need[s2] * NSTR + s2), 0));
      known[(size_t)sid * NSTR + s2] = need[s2];
    }
    if (!dry) *out = S.streams[sid];
    return SLM_OK;
  };
  auto unit_end = [&](int sid) -> slm_status {
    const long u = seqn[sid]++ * NSTR + sid;
    if (!dry) {
      cudaEvent_t& e = evt(u);
      if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CK(cudaEventRecord(e, S.streams[sid]));
    }
    for (int r : rd) res_r[(size_t)r * NSTR + sid] = u;
    for (int r : wr) {
      res_w[r] = u;
      for (int i = 0; i < NSTR; ++i) res_r[(size_t)r * NSTR + i] = -1;
    }
    return SLM_OK;
  };

  // which V' node's value each pool tag holds (host view of the issue order), for the batched
  // head backward: a chunk of g[H_t] runs as one unit when every a[S^{L-1}_t] it reads is resident
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

  const LstmSched sched = lstm_schedule(p, d, m.lstm_fuse_runs != 0, bwdr);
  int run_idx = 0;
  const std::vector<int>& order = p->order;
  int skip_oi = -1;
  for (const LstmUnit& U : sched.units) {
    if (U.type == 1) {
      // ===== forward / mirror run of layer l, steps t0 .. t0 + n - 1 (lstm_run.cuh)
      const int l = U.l, k = U.k, ln = lane_of(l, k), t0 = U.t0, n = U.n;
      // cell = false: a lone gates node (n = 1, node by node); a fused run may end with a gates
      // node whose cell is not in the phase: its cell goes to the side buffers only
      const bool cell = n > 1 || U.s[0] >= 0;
      // with backward runs, re-computed runs share the layer's stream: at most one persistent
      // kernel per layer stream (<= L H / 32 resident CTAs), so every run's CTAs can be resident
      const int sid = (k == 1 && WST > L + 1 && !bwdr) ? L + 1 + l : l;
      const int Kin = l == 0 ? K0 : H;
      const int sprev = t0 > 0 ? preds_of(U.g[0]).first[1] : -1;
      const int init = sprev < 0 ? 1 : (hx_node[ln] == sprev && cs_node[ln] == sprev ? 0 : 2);
      // x operand rows of the input projection: the lower layer's ring when it holds the inputs
      bool xring = l > 0;
      for (int i = 0; i < n && xring; ++i)
        xring = ring_node[(size_t)lane_of(l - 1, k) * 2 * CH + rslot(t0 + i)] == preds_of(U.g[i]).first[0];
      // unit 1: the input projection into the lane's X half (its own stream per layer, so it runs
      // while the layer's previous run is still stepping); unit 2: the run
      const int xpar = xp_cnt[ln]++ % 2;
      rd.clear();
      wr.clear();
      if (l > 0 && xring)
        for (int i = 0; i < n; ++i) rd.push_back(RNG(lane_of(l - 1, k), t0 + i));
      if (l > 0 && !xring)
        for (int i = 0; i < n; ++i) rd.push_back(p->node_tag[preds_of(U.g[i]).first[0]]);
      wr.push_back(XPR(ln, xpar));
      cudaStream_t cs = st;
      if (msm && (s = unit_begin(PST + l, &cs)) != SLM_OK) return s;
      m.ts_cur_aux = sid * 4 + k;
      bf* xop = (bf*)(w + W.xop[ln]);
      // the projection always runs with 256-column tiles over n B rows rounded up to 256 (the
      // extra rows read neighbouring ring / operand rows, or zeros past the end, and land in unread
      // rows of X): tcgen05 results are not invariant to the MMA's N, so one tile shape for every
      // run length keeps runs of different lengths -- forward vs re-computed segments -- bit-identical
      const int bi = 1, bn = 256, npad = (n * B + 255) / 256 * 256;
      const CUtensorMap* bmap = &M.xopM[bi][ln];
      int brow = 0;
      if (l == 0) {
        LK(launch_k(lstm_xpack_kernel, gsz((size_t)n * B * K0), eb, 0, cs, pdl,
                    (const float*)((const uint8_t*)xin + (size_t)t0 * B * I * 4), I, K0, B, n, xop));
        ++nl;
      } else if (xring) {
        bmap = &M.ringM[bi][lane_of(l - 1, k)];
        brow = rslot(t0) * B;
      } else {
        StepIn in{};
        for (int i = 0; i < n; ++i) in.p[i] = V(preds_of(U.g[i]).first[0]);
        LK(launch_k(lstm_hpack_multi_kernel, gsz((size_t)n * B * H), eb, 0, cs, pdl, in, n, H, B, xop));
        ++nl;
      }
      float* xp = (float*)(w + W.xp[ln] + xpar * (((size_t)slmk::kRunMax * B * 4 * H * 4 + 255) / 256 * 256));
      EpiBiasF32 e{xp, 4 * H, d.b + (size_t)l * 4 * H};
      LT((launch_tc_bn<EpiBiasF32, false, false, true>(bn, 1, M.wK[l], *bmap, 4 * H, npad, Kin, 0, brow, e, cs, pdl,
                                                        gdbg(SLM_K_GEMM_FWD))));
      if (msm) {
        if ((s = unit_end(PST + l)) != SLM_OK) return s;
        rd.clear();
        wr.clear();
        if (init == 2) rd.push_back(p->node_tag[sprev]);
        rd.push_back(XPR(ln, xpar));
        for (int i = 0; i < n; ++i) {
          if (sched.mat[U.g[i]]) wr.push_back(p->node_tag[U.g[i]]);
          if (U.s[i] >= 0 && sched.mat[U.s[i]]) wr.push_back(p->node_tag[U.s[i]]);
        }
        if (cell)
          for (int i = 0; i < n; ++i) wr.push_back(RNG(ln, t0 + i));
        if ((s = unit_begin(sid, &cs)) != SLM_OK) return s;
      }
      const CUtensorMap& xpm = xpar ? M.xpM1[ln] : M.xpM[ln];
      FwdRun a{};
      a.H = H;
      a.n = n;
      a.t0 = t0;
      a.Kin = Kin;
      a.init = init;
      a.cell = cell ? 1 : 0;
      a.s_init = init == 2 ? V(sprev) : nullptr;
      a.hx = (bf*)(w + W.hx[ln]);
      a.cstate = (float*)(w + W.cst[ln]);
      a.hring = cell ? ring_ptr(ln, t0) : nullptr;
      a.bar = bar + ln;
      a.dbg = gdbg(SLM_K_BN_ACT);   // profile_ts: forward runs counted under kind 0
      a.ts = (m.lstm_run_ts && run_idx < m.lstm_run_ts_n)
                 ? (unsigned long long*)m.lstm_run_ts + (size_t)run_idx * slmk::kRunMax * 16
                 : nullptr;
      ++run_idx;
      a.base = bar_val[ln];
      for (int i = 0; i < n; ++i) {
        a.g_out[i] = sched.mat[U.g[i]] ? V(U.g[i]) : nullptr;
        a.s_out[i] = U.s[i] >= 0 && sched.mat[U.s[i]] ? V(U.s[i]) : nullptr;
      }
      bar_val[ln] += (unsigned)(H / 32) * (unsigned)(n + 1);
      switch (B) {
        case 64: LT((launch_fwd_run<64>(M.wK32[l], M.hxM[ln], xpm, a, cs, pdl))); break;
        case 128: LT((launch_fwd_run<128>(M.wK32[l], M.hxM[ln], xpm, a, cs, pdl))); break;
        default: LT((launch_fwd_run<256>(M.wK32[l], M.hxM[ln], xpm, a, cs, pdl))); break;
      }
      nl += 2;
      if (msm && (s = unit_end(sid)) != SLM_OK) return s;
      // side state: -1 where the run computed a cell that is not a node of V' (or none)
      hx_node[ln] = cs_node[ln] = cell ? U.s[n - 1] : -1;
      for (int i = 0; i < n && cell; ++i) ring_node[(size_t)ln * 2 * CH + rslot(t0 + i)] = U.s[i];
      for (int i = 0; i < n; ++i) {
        if (sched.mat[U.g[i]]) owner[p->node_tag[U.g[i]]] = U.g[i];
        if (U.s[i] >= 0 && sched.mat[U.s[i]]) owner[p->node_tag[U.s[i]]] = U.s[i];
      }
      continue;
    }
    if (U.type == 2 || U.type == 3) {
      // ===== backward runs (lstm_run.cuh): type 2 = steps t0, t0-1, .., t0-n+1 of layer l; type 3 =
      // the input gradient of steps t0 .. t0+n-1 for the layer below (one GEMM over their d_pre
      // ring rows) and, when the chunk is complete, its weight-gradient GEMM and db column sums
      const int l = U.l, n = U.n, sid = l;
      const int K = lstm_K(d, l), Kin = l == 0 ? K0 : H;
      rd.clear();
      wr.clear();
      cudaStream_t cs = st;
      // chunk-parity halves of the backward rings (op / d_pre bf16 / d_pre fp32)
      const size_t ob = ((size_t)CH * B * K * 2 + 255) / 256 * 256;
      const size_t db2 = ((size_t)CH * B * 4 * H * 2 + 255) / 256 * 256;
      const size_t df4 = ((size_t)CH * B * 4 * H * 4 + 255) / 256 * 256;
      if (U.type == 2) {
        const int t1 = U.t0;
        BwdRun a{};
        a.H = H;
        a.n = n;
        a.t1 = t1;
        a.Kin = Kin;
        a.first = t1 == T - 1 ? 1 : 0;
        if (!a.first && bstate[l] != t1 + 1) {
          set_error("lstm: backward steps of a layer out of order");
          return SLM_E_UNSUPPORTED;
        }
        a.ldh = l == L - 1 ? 2 * H : H;
        a.dpx = (bf*)(w + W.dpx[l]);
        a.dcstate = (float*)(w + W.dcst[l]);
        a.xch = (float*)(w + W.xch[l]);
        a.bar = bbar + l;
        a.base = bbar_val[l];
        a.xbar = bbar + L + l * (H / 128);
        a.xbase = bxbar_val[l];
        a.ts = (m.lstm_run_ts && run_idx < m.lstm_run_ts_n)
                   ? (unsigned long long*)m.lstm_run_ts + (size_t)run_idx * slmk::kRunMax * 16
                   : nullptr;
        ++run_idx;
        for (int i = 0; i < n; ++i) {
          const int t = t1 - i, gs = U.g[i];
          auto pp2 = preds_of(gs);
          const int actn = pp2.first[pp2.second - (t > 0 ? 2 : 1)], spn = t > 0 ? pp2.first[pp2.second - 1] : -1;
          a.act[i] = V(actn);
          a.sprev[i] = spn >= 0 ? V(spn) : nullptr;
          rd.push_back(p->node_tag[actn]);
          if (spn >= 0) rd.push_back(p->node_tag[spn]);
          a.dh_in[i] = l == L - 1 ? dh_ring(t) : dxa_ptr(l, t);
          const int slot = t % CH, cp = (t / CH) % 2;
          a.dpr[i] = (bf*)(w + W.dpR[l] + cp * db2) + (size_t)slot * B * 4 * H;
          a.dpf[i] = (float*)(w + W.dpF[l] + cp * df4) + (size_t)slot * B * 4 * H;
        }
        for (int t = t1 - n + 1; t <= t1; ++t) rd.push_back(l == L - 1 ? DHR((t / CH) % 2) : DXA(l, t));
        wr.push_back(WGR(l, (t1 / CH) % 2));
        if (msm && (s = unit_begin(sid, &cs)) != SLM_OK) return s;
        m.ts_cur_aux = sid * 4 + 2;
        bbar_val[l] += (unsigned)(H / 32) * (unsigned)(n + 1);
        bxbar_val[l] += 4u * (unsigned)(n - a.first);
        a.dbg = gdbg(SLM_K_BN_BWD);   // profile_ts: backward runs counted under kind 4
        LT((launch_bwd_run(M.wMN[l], M.dpxM[l], a, cs, pdl)));
        ++nl;
        bstate[l] = t1 - n + 1;
      } else {
        const int t0 = U.t0, slot0 = t0 % CH;
        // the weight-gradient operand rows [x_t | h_{t-1}] of the steps, from the tags of a[x]
        // and a[S_{t-1}] (the preds of g[G^l_t]: [g[S], a[G], a[x], a[S_{t-1}]?])
        StepPtrs xsp{}, hsp{};
        for (int i = 0; i < n; ++i) {
          const int t = t0 + i, gg = p->gnode[t * per_t + 1 + 2 * l];
          auto pg = preds_of(gg);
          const int xn = pg.first[pg.second - (t > 0 ? 2 : 1)], hn = t > 0 ? pg.first[pg.second - 1] : -1;
          xsp.p[i] = V(xn);
          hsp.p[i] = hn >= 0 ? V(hn) : nullptr;
          rd.push_back(p->node_tag[xn]);
          if (hn >= 0) rd.push_back(p->node_tag[hn]);
        }
        const int cp = (t0 / CH) % 2;
        if (l > 0)
          for (int t = t0; t < t0 + n; ++t) wr.push_back(DXA(l - 1, t));
        wr.push_back(WGR(l, cp));
        if (msm && (s = unit_begin(sid, &cs)) != SLM_OK) return s;
        m.ts_cur_aux = sid * 4 + 2;
        LK(launch_k(lstm_oppack_kernel, gsz((size_t)n * B * K / 8), eb, 0, cs, pdl, xsp, hsp, n, B, l == 0 ? I : H,
                    l == 0 ? I : 2 * H, Kin, H, (bf*)(w + W.opR[l] + cp * ob) + (size_t)slot0 * B * K));
        ++nl;
        if (l > 0) {   // d x_t (the h of layer l-1) = d_pre W_ih over the run's ring rows (N padded to 256)
          const int npad = (n * B + 255) / 256 * 256;
          if ((4 * H) % (64 * kDxSplit) == 0 && npad <= (slmk::kRunMax * B + 255) / 256 * 256) {
            float* pdx = (float*)(w + W.pdx[l]);
            slmk::EpiPartial e{pdx, (long)H, (long)npad * H};
            LT((launch_tc_bn<slmk::EpiPartial, true, false, true>(256, kDxSplit, M.wMN[l], cp ? M.dpR2561[l] : M.dpR256[l], H, npad, 4 * H,
                                                                  0, slot0 * B, e, cs, pdl, gdbg(SLM_K_GEMM_DX))));
            LK(launch_k(splitk_sum_kernel, gsz((size_t)n * B * H / 4), eb, 0, cs, pdl, (const float4*)pdx, kDxSplit,
                        (size_t)npad * H / 4, (size_t)n * B * H / 4, (float4*)dxa_ptr(l - 1, t0)));
            nl += 2;
          } else {
            EpiStoreF32Lim e{dxa_ptr(l - 1, t0), H, n * B};
            LT((launch_tc_bn<EpiStoreF32Lim, true, false, true>(256, 1, M.wMN[l], cp ? M.dpR2561[l] : M.dpR256[l], H, npad,
                                                                4 * H, 0, slot0 * B, e, cs, pdl, gdbg(SLM_K_GEMM_DX))));
            ++nl;
          }
        }
        if (slot0 == 0) {   // the chunk is complete: dW_l += op^T d_pre over its rows, db_l += column sums
          // as a unit of its own on the weight-gradient stream (it reads the chunk's ring half; the
          // runs of the chunk after next, which refill that half, wait for it), in issue order, so
          // every layer's chunks still accumulate in descending time (reading A23)
          cudaStream_t ws_ = cs;
          if (msm) {
            if ((s = unit_end(sid)) != SLM_OK) return s;
            rd.clear();
            wr.clear();
            rd.push_back(WGR(l, cp));
            if ((s = unit_begin(WST, &ws_)) != SLM_OK) return s;
          }
          slmk::EpiAccF32 e2{d.dW + lstm_w_offset(d, l), K};
          LT((launch_tc_bn<slmk::EpiAccF32, true, true, false>((4 * H) % 256 ? 128 : 256, 1,
                                                               cp ? M.opRMN1[l] : M.opRMN[l],
                                                               cp ? M.dpRMN1[l] : M.dpRMN[l], K, 4 * H, chunk_rows(t0), 0,
                                                               0, e2, ws_, pdl && !msm, gdbg(SLM_K_GEMM_DW))));
          LK(launch_k(colsum_acc_kernel, dim3(4 * H / 32), dim3(512), 0, ws_, pdl && !msm,
                      (const float*)(w + W.dpF[l] + cp * df4), chunk_rows(t0), 4 * H, d.db + (size_t)l * 4 * H));
          nl += 2;
          if (msm) {
            if ((s = unit_end(WST)) != SLM_OK) return s;
            continue;
          }
        }
      }
      if (msm && (s = unit_end(sid)) != SLM_OK) return s;
      continue;
    }
    const int oi = U.oi;
    if (oi == skip_oi) continue;   // the gradient gates node fused into the previous unit
    const int v = order[oi];
    const int kind = p->kind[v], opk = p->op[v], orig = p->orig[v];
    auto pp = preds_of(v);
    const LstmNode ni = info(orig);
    const int t = ni.t, l = ni.l;
    if (opk == SLM_OP_INPUT) continue;
    // ---- the launch unit: this node, plus the next one when the two are fused
    const bool lay = opk == SLM_OP_LSTM_GATES || opk == SLM_OP_LSTM_CELL;
    const int sid = !lay ? L : (kind == SLM_KIND_MIRROR && WST > L + 1 ? L + 1 + l : l);
    int partner = -1;
    if (oi + 1 < (int)order.size()) {
      const int u = order[oi + 1];
      const bool pu0 = p->pred_ptr[u + 1] > p->pred_ptr[u] && p->preds[p->pred_ptr[u]] == v;
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
    const int lane_top = lane_of(L - 1, 0);
    if (kind != SLM_KIND_GRAD) {
      if (opk == SLM_OP_LSTM_CELL) {
        // an isolated cell node (its gates node not right before it in V'): h into the ring of
        // its lane, the lane's recurrent state becomes stale
        wr.push_back(RNG(lane_of(l, kind == SLM_KIND_MIRROR ? 1 : 0), t));
      } else if (opk == SLM_OP_HEAD_CE) {
        // one batched unit per chunk of forward heads, at the chunk's last step
        wr.clear();
        rd.clear();
        if (t % CH == CH - 1 || t == T - 1) {
          for (int t2 = t - t % CH; t2 <= t; ++t2) rd.push_back(RNG(lane_top, t2));
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
    if (bwdr && kind == SLM_KIND_GRAD && opk == SLM_OP_HEAD_CE && !hb_now) wr.push_back(DHR((t / CH) % 2));
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
      if (opk == SLM_OP_LSTM_CELL) {
        const int ln = lane_of(l, kind == SLM_KIND_MIRROR ? 1 : 0);
        LK(launch_k(lstm_cell_fwd_kernel, gsz((size_t)B * H), eb, 0, cs, pdl, (const float*)V(pp.first[0]),
                    (const float*)(pp.second > 1 ? V(pp.first[1]) : nullptr), H, B, V(v), ring_ptr(ln, t)));
        ++nl;
        hx_node[ln] = cs_node[ln] = -1;
        ring_node[(size_t)ln * 2 * CH + rslot(t)] = v;
      } else if (opk == SLM_OP_HEAD_CE) {
        // batched forward heads of steps t0..t (the chunk ends here): logits for n*B rows in one
        // GEMM over the top layer's ring, the softmax-CE rows, then the per-step losses into the H_t tags
        if (t % CH == CH - 1 || t == T - 1) {
          const int t0 = t - t % CH, n = t - t0 + 1, Nr = n * B, bi = Nr % 256 == 0 ? 1 : 0;
          for (int t2 = t0; t2 <= t; ++t2)
            if (ring_node[(size_t)lane_top * 2 * CH + rslot(t2)] != t2 * per_t + per_t - 2) {
              set_error("lstm: forward head inputs not in the top layer's ring (unsupported V' order)");
              return SLM_E_UNSUPPORTED;
            }
          float* lgF = (float*)(w + W.logitsF);
          float* rlF = (float*)(w + W.rowlossF);
          slmk::EpiStoreF32 e{lgF, Cp};
          LT((launch_tc_bn<slmk::EpiStoreF32, false, false, true>(bi ? 256 : 64, 1, M.woK, M.ringM[bi][lane_top], Cp,
                                                                  Nr, H, 0, rslot(t0) * B, e, cs, pdl,
                                                                  gdbg(SLM_K_GEMM_FWD))));
          LK(launch_k(lstm_head_ce_kernel, dim3(Nr), dim3(1024), 0, cs, pdl, (const float*)lgF, 1, lgF, d.b_o,
                      labels + (size_t)t0 * B, C, Cp, Nr, scale, rlF, (bf*)nullptr, (float*)nullptr, (unsigned*)nullptr,
                      (float*)nullptr));
          slmk::StepOut so{};
          for (int i = 0; i < n; ++i) so.p[i] = V((t0 + i) * per_t + per_t - 1);
          LK(launch_k(lstm_step_loss_kernel, dim3(n), dim3(1024), 0, cs, pdl, (const float*)rlF, B, scale, so,
                      loss_t + t0));
          nl += 3;
        }
      } else if (opk == SLM_OP_SUM) {
        LK(launch_k(lstm_sum_kernel, dim3(1), dim3(32), 0, cs, pdl, (const float*)loss_t, T, V(v)));
        ++nl;
      } else {
        set_error("unsupported op in lstm plan");
        return SLM_E_UNSUPPORTED;
      }
    } else {
      const int slot = t % CH;
      const bool flush = slot == 0;
      if (opk == SLM_OP_SUM) {
        LK(launch_k(fill_kernel, dim3(1), eb, 0, cs, pdl, V(v), T, 1.0f));
        ++nl;
      } else if (opk == SLM_OP_HEAD_CE && hb_now) {
        // batched head backward of steps t0..t: h operands, logits GEMM (N = n B), CE rows ->
        // d logits (bf16 ring + fp32), dh GEMM (same K slicing as the per-step path), (dh | 0)
        // into the chunk's dh ring + db_o (per step, descending), dW_o for the chunk
        const int t0 = hb_lo, n = t - t0 + 1, N = n * B, r0 = (t0 % CH) * B;   // ring rows of t0
        const int bi = N % 256 == 0 ? 2 : N % 128 == 0 ? 1 : 0, bnb = 64 << bi;
        slmk::StepIn in{};
        for (int i = 0; i < n; ++i) in.p[i] = V(head_state(t0 + i));
        LK(launch_k(lstm_hpack_multi_kernel, gsz((size_t)n * B * H), eb, 0, cs, pdl, in, n, H, B, hopR + (size_t)r0 * H));
        float* lgF = (float*)(w + W.logitsF);
        slmk::EpiStoreF32 e{lgF, Cp};
        LT((launch_tc_bn<slmk::EpiStoreF32, false, false, true>(bnb, 1, M.woK, M.hopRKb[bi], Cp, N, H, 0, r0, e, cs,
                                                                     pdl, gdbg(SLM_K_GEMM_FWD))));
        LK(launch_k(lstm_head_ce_kernel, dim3(N), dim3(1024), 0, cs, pdl, (const float*)lgF, 1, lgF, d.b_o,
                    labels + (size_t)t0 * B, C, Cp, N, scale, (float*)nullptr, dlR + (size_t)r0 * Cp, dlog_f,
                    (unsigned*)nullptr, (float*)nullptr));
        slmk::EpiPartialTma e2{N};
        LT((launch_tc_bn<slmk::EpiPartialTma, true, false, true>(bnb, sp.hd, M.woMN, M.dlRKb[bi], H, N, Cp, 0, r0,
                                                                      e2, cs, pdl, gdbg(SLM_K_GEMM_DX), &M.pHB)));
        LK(launch_k(lstm_head_bwd_finish_kernel, dim3(std::max((Cp + 31) / 32, 148)), dim3(512), 0, cs, pdl,
                    (const float*)(w + W.PH), sp.hd, H, N, dh_ring(t0), (const float*)dlog_f, Cp, B, n, d.db_o));
        nl += 5;
        if (t0 % CH == 0) {   // the chunk is complete: dW_o over all its rows
          slmk::EpiAccF32 e3{d.dW_o, H};
          LT((launch_tc_bn<slmk::EpiAccF32, true, true, false>(Cp % 256 ? 128 : 256, 1, M.hopRMN, M.dlRMN, H, Cp,
                                                                    chunk_rows(t0), 0, 0, e3, cs, pdl,
                                                                    gdbg(SLM_K_GEMM_DW))));
          ++nl;
        }
        for (int t2 = t0; t2 <= t; ++t2) hb_batched[t2] = 1;
      } else if (opk == SLM_OP_HEAD_CE) {
        // preds = [g[Sum], a[S^{L-1}_t]]: recompute logits (the head reads only its input, A6)
        const float* sL = V(pp.first[pp.second - 1]);
        LK(launch_k(lstm_hpack_kernel, gsz((size_t)B * H), eb, 0, cs, pdl, sL, H, B, hopR + (size_t)slot * B * H));
        slmk::EpiPartialTma e{B};
        LT((launch_tc_bn<slmk::EpiPartialTma, false, false, true>(B, sp.lg, M.woK, M.hopRK, Cp, B, H, 0, slot * B,
                                                                       e, cs, pdl, gdbg(SLM_K_GEMM_FWD), &M.pL)));
        LK(launch_k(lstm_head_ce_kernel, dim3(B), dim3(1024), 0, cs, pdl, Pb(sid), sp.lg, logits, d.b_o,
                    labels + (size_t)t * B, C, Cp, B, scale, (float*)nullptr, dlR + (size_t)slot * B * Cp, dlog_f,
                    (unsigned*)nullptr, (float*)nullptr));
        // dh[b][h] = sum_c dlog[b][c] W_o[c][h]  (split-K partials) -> (dh | 0)
        slmk::EpiPartialTma e2{B};
        LT((launch_tc_bn<slmk::EpiPartialTma, true, false, true>(B, sp.hd, M.woMN, M.dlRK, H, B, Cp, 0, slot * B,
                                                                      e2, cs, pdl, gdbg(SLM_K_GEMM_DX), &M.pH)));
        LK(launch_k(lstm_head_bwd_finish_kernel, dim3(std::max((Cp + 31) / 32, 148)), dim3(512), 0, cs, pdl, Pb(sid),
                    sp.hd, H, B, bwdr ? dh_ring(t) : V(v), (const float*)dlog_f, Cp, B, 1, d.db_o));
        nl += 5;
        if (flush) {   // dW_o[c][h] += sum over the chunk's rows of dlog[r][c] h[r][h]
          slmk::EpiAccF32 e3{d.dW_o, H};
          LT((launch_tc_bn<slmk::EpiAccF32, true, true, false>(Cp % 256 ? 128 : 256, 1, M.hopRMN, M.dlRMN, H, Cp, chunk_rows(t), 0,
                                                                    0, e3, cs, pdl, gdbg(SLM_K_GEMM_DW))));
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
              LK(launch_k(lstm_cell_bwd_dpre_kernel, gsz((size_t)B * (Kin + H)), eb, 0, cs, pdl, src, act, sprev, H, B,
                          V(v), dpS, dpFS, x, l > 0 ? H : I, l > 0 ? 2 * H : I, Kin, opS));
              ++nl;
              vg = u;
              skip_oi = oi + 1;
            }
          }
          if (vg < 0) {
            LK(launch_k(lstm_cell_bwd_kernel, gsz((size_t)B * H), eb, 0, cs, pdl, src, act, sprev, H, B, V(v)));
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
          LK(launch_k(lstm_dpre_kernel, gsz((size_t)B * 4 * H), eb, 0, cs, pdl, dact, drow, act, H, B, dpS, dpFS, x, l > 0 ? H : I,
                      l > 0 ? 2 * H : I, Kin, sprev, opS));
          ++nl;
        }
        if (vg >= 0) {
          // d[x | h] = d_pre W_l:  D[m = k_in][n = b], K = 4H, split-K partials kept (time-parity
          // double buffer) and read in place by the two cell gradients that consume them
          slmk::EpiPartialTma e{B};
          LT((launch_tc_bn<slmk::EpiPartialTma, true, false, true>(B, skx, M.wMN[l], M.dpRK[l], K, B, 4 * H, 0,
                                                                        slot * B, e, cs, pdl, gdbg(SLM_K_GEMM_DX),
                                                                        &M.pXd[2 * l + t % 2])));
          ++nl;
          if (flush) {   // dW_l[gate][k_in] += sum over the chunk's rows of op[r][k_in] d_pre[r][gate]
            slmk::EpiAccF32 e2{d.dW + lstm_w_offset(d, l), K};
            LT((launch_tc_bn<slmk::EpiAccF32, true, true, false>((4 * H) % 256 ? 128 : 256, 1, M.opRMN[l],
                                                                      M.dpRMN[l], K, 4 * H, chunk_rows(t), 0, 0, e2,
                                                                      cs, pdl, gdbg(SLM_K_GEMM_DW))));
            // db_l += column sums of the chunk's fp32 d_pre rows (time order, plan-independent)
            LK(launch_k(colsum_acc_kernel, dim3(4 * H / 32), dim3(512), 0, cs, pdl, (const float*)(w + W.dpF[l]),
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
      LK(cudaEventRecord(S.join[i], S.streams[i]));
      LK(cudaStreamWaitEvent(st, S.join[i], 0));
    }
  }
  LK(cudaGetLastError());
  if (!dry) m.ts_used = ts_slot;
  if (launches) *launches = nl;
  return SLM_OK;
}

#undef LK
#undef LT

// kernels enqueue_lstm launches for this plan (the memsets are not counted): a dry run
int64_t lstm_launches(const slm_plan* p, const slm_model& m) {
  int64_t n = 0;
  enqueue_lstm(p, const_cast<slm_model&>(m), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &n, true);
  return n;
}

}  // namespace
