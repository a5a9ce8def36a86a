// Executor of V' for op-granularity graphs (included by runtime.cu).
//
// The graph is any DAG of Input, BN, ReLU, FC, Add and SoftmaxCE nodes (e.g. oracle.graph.
// preact_resnet_graph: per layer BN(x) -> ReLU -> FC -> Add(x, .), FC projections between stages;
// PAPER.md:431-446 and "conv-bn-relu counted as one layer", :437), with per-node parameters
// (slm_ops_desc).  The step runs V' node by node on one stream: every node -- forward,
// re-computed (mirror) or gradient -- reads its inputs from and writes its value to its pool tag,
// exactly as the plan allocated them, so a "drop bn-relu" plan (Sec. 4.2)
// really re-computes BN and ReLU outputs from the kept FC / Add values.  Node semantics are
// oracle/opgraph.py's; FC operands (x, W, dy) are bf16 (reading A11), everything else fp32.
//
// Lowering per node (B = batch, w = width = out_bytes / (4 B)):
//   BN / ReLU / Add     ops_kernels.cuh (element-wise, fixed-order per-feature reductions)
//   FC forward          x -> bf16 operand, tcgen05 GEMM D[dout][B] = W x^T (+ bias epilogue)
//   FC backward         dy -> bf16, dx = dy W (GEMM, W read MN-major), dW = dy^T x (GEMM over
//                       K = B, bf16 output), db = column sums of dy
//   SoftmaxCE           kernels_simt.cuh ce_fwd / ce_reduce / ce_bwd (loss = mean over B_global)
//   gradient node g[v]  upstream dy = the sum of g[s]'s slice for v over v's successors s in
//                       successor order (reading A17) -- used in place when it is one whole slice
#pragma once
#include "ops_kernels.cuh"

namespace {

bool ops_supported(int op) {
  return op == SLM_OP_INPUT || op == SLM_OP_BN || op == SLM_OP_RELU || op == SLM_OP_FC || op == SLM_OP_ADD ||
         op == SLM_OP_SOFTMAX_CE || op == SLM_OP_CONV || op == SLM_OP_POOL;
}

// workspace: bf16 GEMM operands (x / im2col columns, dy), the summed upstream gradient, the conv
// column gradient dcol (fp32), the chunk partials of the many-row reductions, CE row losses
struct OpsWs {
  size_t xq, gq, dy, dcol, wt, parts, stat, rowloss, total;
};
// float offsets (after the 4 x max-width scratch) of each node's kept BN statistics (mean[C],
// rstd[C]); the last entry is the total.  Only the chunked (many-row) BNs keep them: their
// gradient reads them instead of re-reducing x (the values are the forward's bit for bit, as a
// re-computed BN produces the same statistics).  2 C floats per BN node -- workspace, not part of
// the plan's activation memory (like the saved mean / inverse std of library BN layers).
std::vector<size_t> bn_stat_slots(const slm_model& m) {
  const size_t n = m.od.rows.size();
  std::vector<size_t> off(n + 1, 0);
  for (size_t u = 0; u < n; ++u)
    off[u + 1] = off[u] + (m.od.op[u] == SLM_OP_BN && m.od.rows[u] > slmk::kSmallRows ? 2 * (size_t)m.od.shape[u][2] : 0);
  return off;
}
OpsWs ops_ws_layout(const slm_model& m) {
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  const size_t B = m.od.batch, E = (size_t)m.od.max_elems, Kc = (size_t)m.od.max_col;
  OpsWs L{};
  size_t off = 0;
  L.xq = off;      off += al(std::max(E, Kc) * 2);
  L.gq = off;      off += al(E * 2);
  L.dy = off;      off += al(E * 4);
  L.dcol = off;    off += al(std::max(Kc * 4, (size_t)m.od.max_colT * 2));   // or the bf16 im2col of dy
  L.wt = off;      off += al((size_t)m.od.max_wt * 2);                       // flipped kernel, bf16
  L.parts = off;   off += al((size_t)m.od.max_parts * 4 * 4);
  // per-channel mean, rstd, S1, S2 of the current BN, then every BN node's (mean, rstd) kept from
  // its forward for its gradient node (bn_stat_slots)
  L.stat = off;    off += al(((size_t)m.ops_maxw * 4 + bn_stat_slots(m).back()) * 4);
  L.rowloss = off; off += al(B * 4);
  L.total = off;
  return L;
}

slm_status enqueue_ops(const slm_plan* p, slm_model& m, const void* x0, const int32_t* labels, void* pool, void* ws,
                       float* loss, cudaStream_t st, int64_t* launches, bool dry = false) {
  using namespace slmk;
  using bf = __nv_bfloat16;
#define OK_(call)       \
  do {                  \
    if (!dry) CK(call); \
  } while (0)
#define OT_(call)                                  \
  do {                                             \
    if (!dry && (s = (call)) != SLM_OK) return s;  \
  } while (0)
  const slm_ops_model& d = m.od;
  const int B = d.batch, N = p->n_fwd;
  const float inv_bg = 1.0f / (float)(d.batch_global > 0 ? d.batch_global : B);
  const bool pdl = m.pdl != 0;
  const OpsWs W = ops_ws_layout(m);
  uint8_t* w8 = (uint8_t*)ws;
  bf* xq = (bf*)(w8 + W.xq);
  bf* gq = (bf*)(w8 + W.gq);
  float* dyw = (float*)(w8 + W.dy);
  float* rowloss = (float*)(w8 + W.rowloss);
  float* dcol = (float*)(w8 + W.dcol);
  float* parts = (float*)(w8 + W.parts);
  float* stat = (float*)(w8 + W.stat);
  const int MW = m.ops_maxw;
  float *ss1 = stat + 2 * MW, *ss2 = stat + 3 * MW;   // stat[0, 2 MW): spare
  const std::vector<size_t> bnslot = bn_stat_slots(m);
  auto bn_mu = [&](int u) { return stat + 4 * (size_t)MW + bnslot[u]; };   // then rstd at + C
  const size_t PS = (size_t)d.max_parts;   // one partial array: chunks x C floats
  slm_status s = SLM_OK;
  int64_t nl = 0;
  // rows (batch H W) and width (C) of a node's value; mirrors / gradient nodes use their forward node's
  auto rows = [&](int node) { return (int)d.rows[p->orig[node]]; };
  auto width = [&](int node) { return (int)(p->out_bytes[node] / (4 * (int64_t)rows(node))); };
  auto shp = [&](int node) { return d.shape[p->orig[node]]; };
  std::vector<void*> tp(p->tag_size.size(), nullptr);
  for (size_t t = 0; t < tp.size(); ++t)
    if (p->tag_offset[t] >= 0) tp[t] = (uint8_t*)pool + p->tag_offset[t];
  for (int v = 0; v < N; ++v) {
    const int t = p->node_tag[v];
    if (t < 0 || p->tag_offset[t] >= 0) continue;
    if (p->op[v] == SLM_OP_INPUT) tp[t] = const_cast<void*>(x0);
    else if (p->op[v] == SLM_OP_SOFTMAX_CE) tp[t] = loss;
  }
  auto V = [&](int node) -> float* { return (float*)tp[p->node_tag[node]]; };
  const int* pred = p->preds.data();
  auto ew = [&](size_t n) { return dim3((unsigned)std::max<size_t>(1, std::min<size_t>(1184, (n + 255) / 256))); };
  const dim3 eb(256), ebf(kFinThreads);
  // tensor maps of one GEMM operand (encoded per launch: host work only, captured into the graph)
  CUtensorMap ma, mb;
  auto kmap = [&](CUtensorMap* mp, const void* base, int inner, int rows, int box_rows) -> slm_status {
    return dry ? SLM_OK : make_map(mp, base, (uint64_t)inner, (uint64_t)rows, (uint32_t)box_rows);
  };
  // N tile over the batch of an FC GEMM with M output rows: the largest that still gives >= 64
  // CTAs (M = 2048, B = 256: 64-column tiles, 64 CTAs instead of 16; every output element's
  // K accumulation is the same whatever the tile, so the bits do not depend on it)
  auto fc_bn = [&](int M) {
    int bn = B % 256 == 0 ? 256 : B % 128 == 0 ? 128 : 64;
    while (bn > 64 && (int64_t)(M / 128) * (B / bn) < 64) bn /= 2;
    return bn;
  };
  auto ntile = [](int64_t R) { return R % 256 == 0 ? 256 : R % 128 == 0 ? 128 : 64; };
  // per-channel sums over R rows: the 8-feature few-row kernels up to kSmallRows rows, the
  // chunked kernels beyond
  auto nchunk = [](int64_t R) { return (int)((R + kRowChunk - 1) / kRowChunk); };
  auto colsum = [&](const float* x, int64_t R, int C, float* out) -> slm_status {
    if (R <= kSmallRows) {
      OK_(launch_k(op_colsum8_kernel, dim3(C / 8), eb, 0, st, pdl, x, (int)R, C, out));
      ++nl;
    } else {
      OK_(launch_k(op_colpart_kernel, dim3(C / 128, nchunk(R)), eb, 0, st, pdl, x, (int)R, C, parts));
      OK_(launch_k(op_colfin_kernel, dim3((C + 31) / 32), ebf, 0, st, pdl, (const float*)parts, nchunk(R), C, out));
      nl += 2;
    }
    return SLM_OK;
  };
  auto geom = [&](int v, int in_node) {
    const auto so = shp(v), si = shp(in_node);
    return ConvGeom{si[0], si[1], si[2], so[3], so[4], so[0], so[1]};
  };
  // Implicit GEMM (slmk::ConvB): a stride-1 convolution whose positions tile into whole image
  // rows reads its im2col operand as 4-D TMA boxes of the bf16 NHWC tensor -- the columns are
  // never written.  conv_tile: the largest N tile (positions) of whole image rows that also
  // divides an image, else 0 (explicit im2col).
  // (R = output positions; a box spans s wo x s rows input elements, each <= 256)
  // a tile of bn positions = whole output rows of one image, or whole images (small maps: 8 x 8 at
  // bn = 256 is 4 images, where row tiles would stop at bn = 64 and re-read the weights 4x as often)
  auto tiles_rows = [](const ConvGeom& g, int64_t R, int bn) {
    const int hw = g.Ho * g.Wo;
    if (R % bn || g.s * g.Wo > 256) return false;
    if (hw % bn == 0) return bn % g.Wo == 0 && g.s * (bn / g.Wo) <= 256;
    return bn % hw == 0 && g.s * g.Ho <= 256;
  };
  // N tile of an implicit conv GEMM with M output rows: the largest valid tile that still gives
  // >= 128 CTAs, else the smallest valid one (0: none, explicit im2col)
  auto conv_tile = [&](const ConvGeom& g, int64_t R, int M) {
    int pick = 0;
    for (int bn = 256; bn >= 64; bn /= 2)
      if (tiles_rows(g, R, bn)) {
        pick = bn;
        if ((int64_t)(M / 128) * (R / bn) >= 128) break;
      }
    return pick;
  };
  auto kmap4 = [&](CUtensorMap* mp, const void* base, const ConvGeom& g, int64_t R, int box_pos) -> slm_status {
    return dry ? SLM_OK
               : make_map4(mp, base, (uint64_t)g.Cin, (uint64_t)g.W, (uint64_t)g.H, (uint64_t)(R / (g.Ho * g.Wo)),
                           (uint32_t)g.Wo, (uint32_t)std::min(box_pos / g.Wo, g.Ho), (uint32_t)g.s,
                           (uint32_t)std::max(1, box_pos / (g.Ho * g.Wo)));
  };
  auto convb = [](int on, const ConvGeom& g) { return ConvB{on, g.Cin, g.k, g.Ho * g.Wo, g.Wo, g.s}; };
  auto cvt = [&](const float* x, int64_t n, bf* out) -> slm_status {
    OK_(launch_k(op_cvt_bf16_kernel, ew((size_t)n / 8), eb, 0, st, pdl, (const float4*)x, (size_t)n / 8, (uint4*)out));
    ++nl;
    return SLM_OK;
  };
  // Conv forward: col = im2col(x) (bf16), y = col W^T + b (tcgen05, M = C_out, N = rows, K = k k C_in)
  auto conv_fwd = [&](int v, int in_node, const float* x, float* y) -> slm_status {
    const ConvGeom g = geom(v, in_node);
    const int64_t R = rows(v);
    const int K = g.k * g.k * g.Cin, Cout = width(v);
    if (const int bn = conv_tile(g, R, Cout)) {   // implicit GEMM over bf16(x)
      if ((s = cvt(x, rows(in_node) * (int64_t)g.Cin, xq)) != SLM_OK) return s;
      if ((s = kmap(&ma, d.W[p->orig[v]], K, Cout, 128)) != SLM_OK) return s;
      if ((s = kmap4(&mb, xq, g, R, bn)) != SLM_OK) return s;
      EpiBiasF32 e{y, Cout, d.b[p->orig[v]]};
      OT_((launch_tc_bn<EpiBiasF32, false, false, true>(bn, 1, ma, mb, Cout, (int)R, K, 0, 0, e, st, pdl, 0, nullptr, 1,
                                                       -1, convb(1, g))));
      ++nl;
      return SLM_OK;
    }
    OK_(launch_k(op_im2col_kernel, ew((size_t)R * 32), eb, 0, st, pdl, x, g, (size_t)R, xq));
    if ((s = kmap(&ma, d.W[p->orig[v]], K, Cout, 128)) != SLM_OK) return s;
    if ((s = kmap(&mb, xq, K, (int)R, ntile(R))) != SLM_OK) return s;
    EpiBiasF32 e{y, Cout, d.b[p->orig[v]]};
    OT_((launch_tc_bn<EpiBiasF32, false, false, true>(ntile(R), 1, ma, mb, Cout, (int)R, K, 0, 0, e, st, pdl)));
    nl += 2;
    return SLM_OK;
  };
  // FC x -> y = x W^T + b   (W [dout][din] bf16)
  auto fc_fwd = [&](int v, const float* x, int din, int dout, float* y) -> slm_status {
    if ((s = cvt(x, (int64_t)B * din, xq)) != SLM_OK) return s;
    const int bn = fc_bn(dout);
    if ((s = kmap(&ma, d.W[p->orig[v]], din, dout, 128)) != SLM_OK) return s;
    if ((s = kmap(&mb, xq, din, B, bn)) != SLM_OK) return s;
    EpiBiasF32 e{y, dout, d.b[p->orig[v]]};
    OT_((launch_tc_bn<EpiBiasF32, false, false, true>(bn, 1, ma, mb, dout, B, din, 0, 0, e, st, pdl)));
    ++nl;
    return SLM_OK;
  };

  for (int v : p->order) {
    const int kind = p->kind[v], op = p->op[v], u = p->orig[v];
    const int* pv = pred + p->pred_ptr[v];
    const int np = p->pred_ptr[v + 1] - p->pred_ptr[v];
    if (kind != SLM_KIND_GRAD) {
      const int w = width(v);
      switch (op) {
        case SLM_OP_INPUT:
          break;
        case SLM_OP_BN: {
          const int R = rows(v);
          if (R <= kSmallRows) {
            OK_(launch_k(op_bn_fwd_kernel, dim3(w / 8), eb, 0, st, pdl, (const float*)V(pv[0]), d.gamma[u],
                         d.beta[u], R, w, V(v)));
            ++nl;
          } else {   // chunked two-pass statistics, then the affine map
            const dim3 gr(w / 128, nchunk(R)), gf((w + 31) / 32);
            float *mu = bn_mu(u), *rs = mu + w;
            OK_(launch_k(op_colpart_kernel, gr, eb, 0, st, pdl, (const float*)V(pv[0]), R, w, parts));
            OK_(launch_k(op_bn_fin_kernel, gf, ebf, 0, st, pdl, (const float*)parts, (const float*)nullptr, nchunk(R), R,
                         w, mu, rs));
            OK_(launch_k(op_bn_sq_kernel, gr, eb, 0, st, pdl, (const float*)V(pv[0]), R, w, (const float*)mu,
                         parts + PS));
            OK_(launch_k(op_bn_fin_kernel, gf, ebf, 0, st, pdl, (const float*)parts, (const float*)(parts + PS),
                         nchunk(R), R, w, (float*)nullptr, rs));
            OK_(launch_k(op_bn_apply_kernel, gr, eb, 0, st, pdl, (const float*)V(pv[0]), R, w, (const float*)mu,
                         (const float*)rs, d.gamma[u], d.beta[u], V(v)));
            nl += 5;
          }
          break;
        }
        case SLM_OP_RELU:
          OK_(launch_k(op_relu_fwd_kernel, ew((size_t)rows(v) * w / 4), eb, 0, st, pdl, (const float4*)V(pv[0]),
                       (size_t)rows(v) * w / 4, (float4*)V(v)));
          ++nl;
          break;
        case SLM_OP_ADD:
          OK_(launch_k(op_add_fwd_kernel, ew((size_t)rows(v) * w / 4), eb, 0, st, pdl, (const float4*)V(pv[0]),
                       (const float4*)V(pv[1]), (size_t)rows(v) * w / 4, (float4*)V(v)));
          ++nl;
          break;
        case SLM_OP_FC:
          if ((s = fc_fwd(v, V(pv[0]), width(pv[0]), w, V(v))) != SLM_OK) return s;
          break;
        case SLM_OP_CONV:
          if ((s = conv_fwd(v, pv[0], V(pv[0]), V(v))) != SLM_OK) return s;
          break;
        case SLM_OP_POOL: {
          const auto si = shp(pv[0]);
          OK_(launch_k(op_pool_fwd_kernel, ew((size_t)B * w), eb, 0, st, pdl, (const float*)V(pv[0]), B, si[0] * si[1],
                       w, V(v)));
          ++nl;
          break;
        }
        case SLM_OP_SOFTMAX_CE: {
          const int wi = width(pv[0]);
          OK_(launch_k(ce_fwd_kernel, dim3(B), eb, 0, st, pdl, (const float*)V(pv[0]), labels, wi, rowloss));
          OK_(launch_k(ce_reduce_kernel, dim3(1), eb, 0, st, pdl, (const float*)rowloss, B, inv_bg, V(v)));
          nl += 2;
          break;
        }
        default:
          set_error("op graph executor: unsupported op " + std::to_string(op));
          return SLM_E_UNSUPPORTED;
      }
      continue;
    }
    // ---- gradient node of u: preds = [successor gradient nodes (successor order)..., the forward
    // values its backward reads (op metadata, reading A6)]
    const int wu = width(u);
    int k = 0;
    GradSlices gs{};
    while (k < np && p->kind[pv[k]] == SLM_KIND_GRAD) {
      const int sg = pv[k], so = p->orig[sg];
      const int* sp = pred + p->pred_ptr[so];
      const int ns = p->pred_ptr[so + 1] - p->pred_ptr[so];
      int off = 0, ld = 0;
      for (int i = 0; i < ns; ++i) ld += width(sp[i]);
      for (int i = 0; i < ns; ++i) {
        if (sp[i] == u) {
          if (gs.n == 8) {
            set_error("op graph executor: more than 8 gradient slices");
            return SLM_E_UNSUPPORTED;
          }
          gs.p[gs.n] = V(sg) + off;
          gs.ld[gs.n] = ld;
          ++gs.n;
        }
        off += width(sp[i]);
      }
      ++k;
    }
    const int* rest = pv + k;
    const float* dy = nullptr;
    if (op != SLM_OP_SOFTMAX_CE) {
      if (gs.n == 0) {
        set_error("op graph executor: gradient node without an upstream gradient");
        return SLM_E_UNSUPPORTED;
      }
      if (gs.n == 1 && gs.ld[0] == wu) {
        dy = gs.p[0];   // one whole slice in the node's own layout (an in-place output aliases it element for element)
      } else {
        OK_(launch_k(op_gsum_kernel, ew((size_t)rows(u) * wu / 4), eb, 0, st, pdl, gs, rows(u), wu, dyw));
        ++nl;
        dy = dyw;
      }
    }
    const int Ru = rows(u);
    switch (op) {
      case SLM_OP_RELU:   // rest = [output]
        OK_(launch_k(op_relu_bwd_kernel, ew((size_t)Ru * wu / 4), eb, 0, st, pdl, (const float4*)dy,
                     (const float4*)V(rest[0]), (size_t)Ru * wu / 4, (float4*)V(v)));
        ++nl;
        break;
      case SLM_OP_BN:   // rest = [x]
        if (Ru <= kSmallRows) {
          OK_(launch_k(op_bn_bwd_kernel, dim3(wu / 8), eb, 0, st, pdl, dy, (const float*)V(rest[0]),
                       d.gamma[u], Ru, wu, V(v), d.dgamma[u], d.dbeta[u]));
          ++nl;
        } else {
          const dim3 gr(wu / 128, nchunk(Ru)), gf((wu + 31) / 32);
          const float* xr = V(rest[0]);
          const float *mu = bn_mu(u), *rs = mu + wu;   // the forward's statistics
          OK_(launch_k(op_bn_bpart_kernel, gr, eb, 0, st, pdl, dy, xr, Ru, wu, mu, rs, parts + 2 * PS, parts + 3 * PS));
          OK_(launch_k(op_parts2_kernel, gf, ebf, 0, st, pdl, (const float*)(parts + 2 * PS),
                       (const float*)(parts + 3 * PS), nchunk(Ru), wu, ss1, ss2));
          OK_(launch_k(op_bn_bapply_kernel, gr, eb, 0, st, pdl, dy, xr, Ru, wu, mu, rs, (const float*)ss1,
                       (const float*)ss2, d.gamma[u], V(v), d.dgamma[u], d.dbeta[u]));
          nl += 3;
        }
        break;
      case SLM_OP_ADD:   // [dy | dy]
        OK_(launch_k(op_add_bwd_kernel, ew((size_t)Ru * wu / 4), eb, 0, st, pdl, (const float4*)dy, Ru, wu / 4,
                     (float4*)V(v)));
        ++nl;
        break;
      case SLM_OP_POOL: {   // rest = []; dx[b][q][c] = dy[b][c] / HW
        const auto si = shp(pred[p->pred_ptr[u]]);
        OK_(launch_k(op_pool_bwd_kernel, ew((size_t)B * si[0] * si[1] * wu), eb, 0, st, pdl, dy, B, si[0] * si[1], wu,
                     V(v)));
        ++nl;
        break;
      }
      case SLM_OP_CONV: {   // rest = [x]
        const int xin = rest[0];
        const ConvGeom g = geom(u, xin);
        const int K = g.k * g.k * g.Cin, Cout = wu;
        const int64_t Rin = rows(xin);
        const bool flip = g.k == 3 && g.s == 1;   // dx by the flipped kernel (below)
        bf* wt = (bf*)(w8 + W.wt);
        if (flip)   // first: the dx GEMM prefetches Wt before its dependency wait (PREFETCH_A)
          OK_(launch_k(op_wflip_kernel, dim3(g.Cin / 32, Cout / 32, g.k * g.k), eb, 0, st, pdl, (const bf*)d.W[u], g.k,
                       g.Cin, Cout, wt));
        nl += flip;
        // bf16 dy and the im2col columns of x (the GEMM operands; implicit: bf16 x), db = column
        // sums of dy
        if ((s = cvt(dy, Ru * Cout, gq)) != SLM_OK) return s;
        const bool implicit_a = 64 % g.Wo == 0 && tiles_rows(g, Ru, 64);
        if (implicit_a) {
          if ((s = cvt(V(xin), Rin * g.Cin, xq)) != SLM_OK) return s;
        } else {
          OK_(launch_k(op_im2col_kernel, ew((size_t)Ru * 32), eb, 0, st, pdl, (const float*)V(xin), g, (size_t)Ru, xq));
          ++nl;
        }
        if ((s = colsum(dy, Ru, Cout, d.db[u])) != SLM_OK) return s;
        // dW[C_out][K] = sum_r dy[r][o] col[r][k]: D[m = K][n = C_out], both operands MN-major, K = rows.
        // Few output tiles and a long K (batch H W): split K over ~one wave of CTAs, fp32 partials in
        // the dcol workspace (not yet in use), summed in split order into the bf16 dW
        const ConvB cbw = implicit_a ? convb(2, g) : ConvB{};
        if ((s = implicit_a ? kmap4(&ma, xq, g, Ru, 64) : kmap(&ma, xq, K, Ru, 64)) != SLM_OK) return s;
        if ((s = kmap(&mb, gq, Cout, Ru, 64)) != SLM_OK) return s;
        const int bnw = Cout % 256 == 0 ? 256 : 128;
        const int tiles = (K / 128) * (Cout / bnw);
        int split = 1;
        while (split * 2 * tiles <= 148 && Ru % (64 * split * 2) == 0 && (int64_t)split * 2 * Cout <= Ru) split *= 2;
        if (split == 1) {
          EpiStoreBF16 e1{(bf*)d.dW[u], K};
          OT_((launch_tc_bn<EpiStoreBF16, true, true, false>(bnw, 1, ma, mb, K, Cout, Ru, 0, 0, e1, st, pdl, 0, nullptr,
                                                            1, -1, cbw)));
        } else {
          EpiPartial e1{dcol, (long)K, (long)K * Cout};
          OT_((launch_tc_bn<EpiPartial, true, true, false>(bnw, split, ma, mb, K, Cout, Ru, 0, 0, e1, st, pdl, 0, nullptr,
                                                          1, -1, cbw)));
          OK_(launch_k(op_splitk_bf16_kernel, ew((size_t)K * Cout / 4), eb, 0, st, pdl, (const float*)dcol, split,
                       (size_t)K * Cout, (bf*)d.dW[u]));
          ++nl;
        }
        ++nl;   // the dW GEMM
        if (flip) {
          // dx = im2col(dy) Wt^T with Wt the flipped, transposed kernel (op_wflip_kernel, launched
          // first -- the GEMM requests its A (Wt) tiles before griddepcontrol.wait, so Wt's producer
          // must not be the immediately preceding kernel): one GEMM of the forward's shape (M = C_in,
          // N = rows, K = k k C_out) instead of the fp32 column gradient and its col2im gather;
          // implicit over bf16(dy) when the positions tile into whole image rows
          const ConvGeom gt{g.Ho, g.Wo, Cout, g.k, 1, g.Ho, g.Wo};
          const int Kt = g.k * g.k * Cout;
          const int bn = conv_tile(gt, Rin, g.Cin);
          bf* colT = (bf*)dcol;
          if (bn) {
            if ((s = kmap4(&mb, gq, gt, Rin, bn)) != SLM_OK) return s;
          } else {
            OK_(launch_k(op_im2col_kernel, ew((size_t)Rin * 32), eb, 0, st, pdl, dy, gt, (size_t)Rin, colT));
            ++nl;
            if ((s = kmap(&mb, colT, Kt, (int)Rin, ntile(Rin))) != SLM_OK) return s;
          }
          if ((s = kmap(&ma, wt, Kt, g.Cin, 128)) != SLM_OK) return s;
          EpiStoreF32 e3{V(v), g.Cin};
          const int bnx = bn ? bn : ntile(Rin);
          OT_((launch_tc_bn<EpiStoreF32, false, false, true>(bnx, 1, ma, mb, g.Cin, (int)Rin, Kt, 0, 0, e3, st, pdl, 0,
                                                            nullptr, 1, -1,
                                                            bn ? convb(1, gt) : ConvB{})));
          ++nl;
          break;
        }
        // dcol[r][k] = sum_o dy[r][o] W[o][k]: D[m = K][n = r], W MN-major (K = C_out rows)
        if ((s = kmap(&ma, d.W[u], K, Cout, 64)) != SLM_OK) return s;
        if ((s = kmap(&mb, gq, Cout, Ru, ntile(Ru))) != SLM_OK) return s;
        EpiStoreF32 e2{dcol, K};
        OT_((launch_tc_bn<EpiStoreF32, true, false, true>(ntile(Ru), 1, ma, mb, K, Ru, Cout, 0, 0, e2, st, pdl)));
        // dx = col2im(dcol) (gather over the taps in order)
        OK_(launch_k(op_col2im_kernel, ew((size_t)Rin * 32), eb, 0, st, pdl, (const float*)dcol, g,
                     (size_t)Rin, V(v)));
        nl += 2;
        break;
      }
      case SLM_OP_SOFTMAX_CE:   // rest = [x]; dx may alias x
        OK_(launch_k(ce_bwd_kernel<bf>, dim3(B), eb, 0, st, pdl, (const float*)V(rest[0]), labels, width(rest[0]),
                     inv_bg, V(v), (bf*)nullptr));
        ++nl;
        break;
      case SLM_OP_FC: {   // rest = [x]
        const int din = width(rest[0]), dout = wu;
        // bf16 dy and x (the GEMM operands), db = column sums of dy -- all before dx may overwrite dy
        if ((s = cvt(dy, (int64_t)B * dout, gq)) != SLM_OK) return s;
        if ((s = cvt(V(rest[0]), (int64_t)B * din, xq)) != SLM_OK) return s;
        OK_(launch_k(op_colsum8_kernel, dim3(dout / 8), eb, 0, st, pdl, dy, B, dout, d.db[u]));
        // dW[dout][din] = sum_b dy[b][dout] x[b][din]: D[m = din][n = dout], both operands MN-major, K = B
        if ((s = kmap(&ma, xq, din, B, 64)) != SLM_OK) return s;
        if ((s = kmap(&mb, gq, dout, B, 64)) != SLM_OK) return s;
        EpiStoreBF16 e1{(bf*)d.dW[u], din};
        OT_((launch_tc_bn<EpiStoreBF16, true, true, false>(dout % 256 == 0 ? 256 : 128, 1, ma, mb, din, dout, B, 0, 0,
                                                          e1, st, pdl)));
        // dx[b][din] = sum_o dy[b][o] W[o][din]: D[m = din][n = b], W MN-major (K = dout rows)
        if ((s = kmap(&ma, d.W[u], din, dout, 64)) != SLM_OK) return s;
        const int bnx = fc_bn(din);
        if ((s = kmap(&mb, gq, dout, B, bnx)) != SLM_OK) return s;
        EpiStoreF32 e2{V(v), din};
        OT_((launch_tc_bn<EpiStoreF32, true, false, true>(bnx, 1, ma, mb, din, B, dout, 0, 0, e2, st, pdl)));
        nl += 3;   // colsum, dW, dx (the converts count themselves)
        break;
      }
      default:
        set_error("op graph executor: unsupported gradient op " + std::to_string(op));
        return SLM_E_UNSUPPORTED;
    }
  }
  OK_(cudaGetLastError());
  if (launches) *launches = nl;
  return SLM_OK;
#undef OK_
#undef OT_
}

}  // namespace
