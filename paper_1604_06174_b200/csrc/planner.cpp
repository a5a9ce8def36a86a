// Host planner of arXiv 1604.06174 in plain C++ (no CUDA).
//
//   validate / topological order        PAPER.md:261, 266 (Kahn, lowest id first)
//   strategies -> mirror counts m       Sec. 4.2-4.4, Alg. 3, App. A
//   Alg. 2 mirrored gradient graph
//   Fig. 2 liveness-counter allocator
//
// Readings of silent / ambiguous points are DESIGN.md A1-A20; they are chosen so that every
// tie has a total order and every budget is an integer, so plans are reproducible bit for
// bit (tests/test_planner_parity.py compares them against the independent Python oracle).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>
#include <new>
#include <queue>
#include <map>
#include <set>
#include <string>
#include <unordered_set>
#include <vector>

#include "slm_internal.h"

namespace slm {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

static const OpMeta kOps[] = {
    //  amin amax fwd_ip out    in_mask grad_inplace low
    {0, 0, -1, false, 0x0, GI_NONE, false},          // INPUT
    {1, 1, 0, false, 0x1, GI_SUCC0, false},          // BLOCK       (A10: bwd reads input)
    {1, 1, -1, false, 0x1, GI_IN0, false},           // SOFTMAX_CE  (bwd reads input, in place on it)
    {1, 1, -1, false, 0x1, GI_NONE, false},          // FC          (bwd reads input)
    {1, 1, 0, true, 0x0, GI_OUT, true},              // SIGMOID     (bwd reads output)
    {1, 1, 0, true, 0x0, GI_OUT, true},              // RELU
    {1, 1, 0, false, 0x1, GI_SUCC0, true},           // BN
    {2, 2, 0, false, 0x0, GI_NONE, false},           // ADD
    {2, 2, 0, false, 0x3, GI_NONE, false},           // MUL
    {1, 1, 0, false, 0x0, GI_SUCC0, true},           // IDENTITY
    {1, 2, -1, true, 0x3, GI_NONE, false},           // LSTM_GATES  (A6/A13)
    {1, 2, -1, false, 0x3, GI_NONE, false},          // LSTM_CELL
    {1, 1, -1, false, 0x1, GI_NONE, false},          // HEAD_CE
    {1, 1 << 30, -1, false, 0x0, GI_NONE, false},    // SUM
    {1, 1, -1, false, 0x1, GI_NONE, false},          // CONV        (bwd reads input, as FC)
    {1, 1, -1, false, 0x0, GI_NONE, false},          // POOL        (bwd needs the shapes only)
};

const OpMeta* op_meta(int op) {
  if (op < 0 || op >= (int)(sizeof(kOps) / sizeof(kOps[0]))) return nullptr;
  return &kOps[op];
}

namespace {

// Kahn's algorithm over the vertex set `verts`, lowest id first among ready vertices;
// predecessors outside the set are ignored (they are already available).
template <class PredFn>
std::vector<int> kahn(std::vector<int> verts, PredFn preds_of) {
  std::sort(verts.begin(), verts.end());
  auto local = [&](int v) -> int {
    auto it = std::lower_bound(verts.begin(), verts.end(), v);
    return (it != verts.end() && *it == v) ? (int)(it - verts.begin()) : -1;
  };
  std::vector<int> indeg(verts.size(), 0);
  std::vector<std::vector<int>> succ(verts.size());
  for (size_t i = 0; i < verts.size(); ++i)
    for (int p : preds_of(verts[i])) {
      int lp = local(p);
      if (lp >= 0) {
        indeg[i]++;
        succ[lp].push_back((int)i);
      }
    }
  std::priority_queue<int, std::vector<int>, std::greater<int>> heap;
  for (size_t i = 0; i < verts.size(); ++i)
    if (indeg[i] == 0) heap.push((int)i);
  std::vector<int> out;
  out.reserve(verts.size());
  while (!heap.empty()) {
    int i = heap.top();
    heap.pop();
    out.push_back(verts[i]);
    for (int s : succ[i])
      if (--indeg[s] == 0) heap.push(s);
  }
  return out;
}

std::vector<int> topo_order(const slm_graph& g) {
  std::vector<int> all(g.nodes.size());
  for (size_t i = 0; i < all.size(); ++i) all[i] = (int)i;
  return kahn(all, [&](int v) -> const std::vector<int>& { return g.nodes[v].preds; });
}

std::vector<std::vector<int>> successors(const slm_graph& g) {
  std::vector<std::vector<int>> succ(g.nodes.size());
  for (int v = 0; v < (int)g.nodes.size(); ++v)
    for (int p : g.nodes[v].preds)
      if (std::find(succ[p].begin(), succ[p].end(), v) == succ[p].end()) succ[p].push_back(v);
  for (auto& s : succ) std::sort(s.begin(), s.end());
  return succ;
}

struct Diag {
  int code, node;
};

std::vector<Diag> validate(const slm_graph& g) {
  std::vector<Diag> d;
  int n = (int)g.nodes.size();
  bool dangling = false;
  for (int i = 0; i < n; ++i) {
    const Node& nd = g.nodes[i];
    const OpMeta* m = op_meta(nd.op);
    if (!m) {
      d.push_back({SLM_DIAG_BAD_OP, i});
      continue;
    }
    if ((int)nd.preds.size() < m->arity_min || (int)nd.preds.size() > m->arity_max)
      d.push_back({SLM_DIAG_ARITY, i});
    for (int p : nd.preds)
      if (p < 0 || p >= n) {
        d.push_back({SLM_DIAG_DANGLING, i});
        dangling = true;
        break;
      }
    if (nd.out_bytes <= 0) d.push_back({SLM_DIAG_ZERO_SIZE, i});
  }
  if (g.outputs.empty()) d.push_back({SLM_DIAG_BAD_OUTPUT, -1});
  for (int o : g.outputs)
    if (o < 0 || o >= n) d.push_back({SLM_DIAG_BAD_OUTPUT, o});
  if (!dangling) {
    std::vector<int> ord = topo_order(g);
    if ((int)ord.size() != n) {
      std::vector<char> placed(n, 0);
      for (int v : ord) placed[v] = 1;
      for (int i = 0; i < n; ++i)
        if (!placed[i]) d.push_back({SLM_DIAG_CYCLE, i});
    }
  }
  return d;
}

// ---------------------------------------------------------------- strategies -> m
std::vector<char> candidates(const slm_graph& g) {
  // Alg. 3's C, reading A19: every non-Input node not flagged NOT_CANDIDATE
  std::vector<char> c(g.nodes.size());
  for (size_t v = 0; v < g.nodes.size(); ++v)
    c[v] = g.nodes[v].op != SLM_OP_INPUT && !(g.nodes[v].flags & SLM_NODE_NOT_CANDIDATE);
  return c;
}

// Alg. 3 with readings A1 (Input adds 0) and A2 (final y).
void alg3(const slm_graph& g, const std::vector<int>& topo, int64_t B, int64_t* x_out,
          int64_t* y_out, std::vector<int>* m) {
  std::vector<char> C = candidates(g);
  int64_t temp = 0, x = 0, y = 0;
  m->assign(g.nodes.size(), 0);
  for (int v : topo) {
    if (g.nodes[v].op == SLM_OP_INPUT) {                // A1
      (*m)[v] = 0;
      continue;
    }
    temp += g.nodes[v].out_bytes;
    if (C[v] && temp > B) {
      x += g.nodes[v].out_bytes;
      y = std::max(y, temp);
      (*m)[v] = 0;
      temp = 0;
    } else {
      (*m)[v] = 1;
    }
  }
  y = std::max(y, temp);                                // A2
  *x_out = x;
  *y_out = y;
}

int64_t isqrt64(unsigned __int128 v) {
  // floor(sqrt(v)) exactly (v may exceed 2^64: x0*y0 in bytes^2, reading A3)
  if (v == 0) return 0;
  long double s = sqrtl((long double)v);
  unsigned __int128 r = (unsigned __int128)s;
  while (r * r > v) --r;
  while ((r + 1) * (r + 1) <= v) ++r;
  return (int64_t)r;
}

// Sec. 4.3, reading A4
std::vector<int> sqrt_plan(const slm_graph& g, const std::vector<int>& topo) {
  std::vector<char> C = candidates(g);
  std::vector<int> S;
  for (int v : topo)
    if (C[v]) S.push_back(v);
  std::vector<int> m(g.nodes.size(), 0);
  int64_t n = (int64_t)S.size();
  if (n == 0) return m;
  int64_t k = isqrt64((unsigned __int128)(n - 1)) + 1;
  std::vector<char> kept(n + 1, 0);
  for (int64_t j = 1; j <= k; ++j) kept[(j * n) / k] = 1;
  for (int64_t i = 1; i <= n; ++i) m[S[i - 1]] = kept[i] ? 0 : 1;
  return m;
}

// Chain path for the recursive plan: [X_0 .. X_n] or NotAChain.
bool chain_positions(const slm_graph& g, const std::vector<int>& topo, std::vector<int>* path) {
  auto succ = successors(g);
  if (topo.empty() || g.nodes[topo[0]].op != SLM_OP_INPUT) return false;
  for (size_t i = 0; i < topo.size(); ++i) {
    const Node& nd = g.nodes[topo[i]];
    if (i > 0 && !(nd.preds.size() == 1 && nd.preds[0] == topo[i - 1])) return false;
    if (succ[topo[i]].size() > 1) return false;
  }
  std::vector<char> C = candidates(g);
  size_t last = 0;
  for (size_t i = 0; i < topo.size(); ++i)
    if (C[topo[i]]) last = i;
  path->assign(topo.begin(), topo.begin() + last + 1);
  return true;
}

// Sec. 4.4, reading A5
void recursive_fill(const std::vector<int>& path, int64_t k, int64_t lo, int64_t hi, int level,
                    std::vector<int>* m) {
  if (hi - lo < 2) return;
  std::vector<int64_t> splits;
  for (int64_t j = 1; j <= k; ++j) {
    int64_t s = lo + (j * (hi - lo)) / (k + 1);
    if (s > lo && s < hi) splits.push_back(s);
  }
  std::sort(splits.begin(), splits.end());
  splits.erase(std::unique(splits.begin(), splits.end()), splits.end());
  for (int64_t s : splits) (*m)[path[s]] = level;
  int64_t prev = lo;
  for (int64_t s : splits) {
    recursive_fill(path, k, prev, s, level + 1, m);
    prev = s;
  }
  recursive_fill(path, k, prev, hi, level + 1, m);
}

// Sec. 4.2
std::vector<int> drop_cheap_plan(const slm_graph& g) {
  std::vector<int> m(g.nodes.size(), 0);
  for (size_t v = 0; v < g.nodes.size(); ++v) {
    bool is_out = std::find(g.outputs.begin(), g.outputs.end(), (int)v) != g.outputs.end();
    if (op_meta(g.nodes[v].op)->low_cost && !is_out && g.nodes[v].op != SLM_OP_INPUT) m[v] = 1;
  }
  return m;
}

// ---------------------------------------------------------------- Alg. 2 + Fig. 2
struct GN {
  int kind, op, orig, level, inplace_slot;
  int64_t out_bytes;
  std::vector<int> preds;
};

struct Built {
  std::vector<GN> nodes;
  std::vector<int> order, a, gnode;
  std::vector<char> pinned, external;
  int extra = 0;
};

slm_status build_mirrored(const slm_graph& g, const std::vector<int>& m,
                          const std::vector<int>& topo, Built* out) {
  const int N = (int)g.nodes.size();
  if (g.outputs.size() != 1) {
    set_error("gradient graph needs exactly one loss output (MultipleRoots)");
    return SLM_E_MULTIPLE_ROOTS;
  }
  if ((int)m.size() != N) {
    set_error("mirror plan length != number of nodes");
    return SLM_E_INVALID_PLAN;
  }
  int maxm = 0;
  for (int v = 0; v < N; ++v) {
    if (m[v] < 0 || (g.nodes[v].op == SLM_OP_INPUT && m[v] != 0)) {
      set_error("InvalidPlan: negative mirror count or m > 0 on an Input node");
      return SLM_E_INVALID_PLAN;
    }
    maxm = std::max(maxm, m[v]);
  }
  auto& nodes = out->nodes;
  nodes.clear();
  nodes.reserve(3 * N);
  for (int v = 0; v < N; ++v) {
    const Node& nd = g.nodes[v];
    nodes.push_back({SLM_KIND_FWD, nd.op, v, 0, op_meta(nd.op)->fwd_inplace, nd.out_bytes, nd.preds});
  }
  auto& a = out->a;
  a.resize(N);
  for (int v = 0; v < N; ++v) a[v] = v;
  for (int k = 1; k <= maxm; ++k)
    for (int v : topo)
      if (k <= m[v]) {
        const Node& nd = g.nodes[v];
        GN mn{SLM_KIND_MIRROR, nd.op, v, k, op_meta(nd.op)->fwd_inplace, nd.out_bytes, {}};
        for (int u : nd.preds) mn.preds.push_back(a[u]);
        a[v] = (int)nodes.size();
        nodes.push_back(std::move(mn));
      }
  auto succ = successors(g);
  std::vector<char> reaches(N, 0);
  for (auto it = topo.rbegin(); it != topo.rend(); ++it) {
    int v = *it;
    bool r = std::find(g.outputs.begin(), g.outputs.end(), v) != g.outputs.end();
    for (int s : succ[v]) r = r || reaches[s];
    reaches[v] = r;
  }
  auto& order = out->order;
  order = topo;
  std::vector<char> in_order(nodes.size() + N + 16, 0);
  for (int v : topo) in_order[v] = 1;
  auto& gnode = out->gnode;
  gnode.assign(N, -1);
  for (auto it = topo.rbegin(); it != topo.rend(); ++it) {
    int v = *it;
    const Node& nd = g.nodes[v];
    if (nd.op == SLM_OP_INPUT || !reaches[v]) continue;
    const OpMeta* meta = op_meta(nd.op);
    GN gn{SLM_KIND_GRAD, nd.op, v, 0, -1, 0, {}};
    for (int s : succ[v])
      if (gnode[s] >= 0) gn.preds.push_back(gnode[s]);          // successor gradients
    if (meta->grad_inplace == GI_SUCC0 && !gn.preds.empty()) gn.inplace_slot = 0;
    if (meta->grad_needs_out) {
      if (meta->grad_inplace == GI_OUT) gn.inplace_slot = (int)gn.preds.size();
      gn.preds.push_back(a[v]);                                  // a[v]
    }
    bool first_in = true;
    for (size_t i = 0; i < nd.preds.size(); ++i)
      if ((meta->grad_needs_in >> i) & 1) {                      // a[u], u in pred[v]
        if (meta->grad_inplace == GI_IN0 && first_in) gn.inplace_slot = (int)gn.preds.size();
        first_in = false;
        gn.preds.push_back(a[nd.preds[i]]);
      }
    for (int u : nd.preds) gn.out_bytes += g.nodes[u].out_bytes;  // A17
    int gid = (int)nodes.size();
    nodes.push_back(std::move(gn));
    gnode[v] = gid;
    if ((int)in_order.size() < (int)nodes.size()) in_order.resize(nodes.size() * 2, 0);
    // V' <- append(V', topological-order(ancestors(g[v])) - V')
    std::vector<int> fresh, stack{gid};
    std::unordered_set<int> seen;
    while (!stack.empty()) {
      int w = stack.back();
      stack.pop_back();
      if (in_order[w] || seen.count(w)) continue;
      seen.insert(w);
      fresh.push_back(w);
      for (int p : nodes[w].preds) stack.push_back(p);
    }
    std::vector<int> app =
        kahn(fresh, [&](int w) -> const std::vector<int>& { return nodes[w].preds; });
    for (int w : app) {
      order.push_back(w);
      in_order[w] = 1;
    }
  }
  // pinned / external (readings A8, A9)
  out->pinned.assign(nodes.size(), 0);
  out->external.assign(nodes.size(), 0);
  for (int v = 0; v < N; ++v) {
    const Node& nd = g.nodes[v];
    if (nd.op == SLM_OP_INPUT) {
      out->pinned[v] = out->external[v] = 1;
      if (nd.flags & SLM_NODE_REQUEST_GRAD)
        for (int s : succ[v])
          if (gnode[s] >= 0) out->pinned[gnode[s]] = 1;
    }
    if (nd.flags & SLM_NODE_PIN) out->pinned[v] = 1;
  }
  for (int o : g.outputs) out->pinned[o] = out->external[o] = 1;
  out->extra = 0;
  for (int v : order)
    if (nodes[v].kind == SLM_KIND_MIRROR) out->extra++;           // A7
  return SLM_OK;
}

struct Alloc {
  std::vector<int> tag_of;
  std::vector<int64_t> tag_size, tag_offset;
  std::vector<char> tag_ext;
  int64_t pool_bytes = 0, exact_peak = 0;
};

// Fig. 2, reading A8; offsets reading A9.
void allocate(const Built& b, int flags, int64_t align, Alloc* out, const std::vector<int>& group) {
  const auto& nodes = b.nodes;
  const bool grouped = (flags & SLM_ALLOC_GROUPED) != 0, by_kind = (flags & SLM_ALLOC_GROUP_MIRRORS) != 0;
  const bool parity = (flags & SLM_ALLOC_MIRROR_PARITY) != 0;
  // MIRROR_PARITY (reading A24): recompute phase of each mirror.  A maximal run of consecutive
  // mirrors in V' joins the latest phase one of its mirrors reads a mirror of (it continues that
  // segment's re-computation); a run that reads no earlier mirror starts a new phase.  The tag
  // group of a mirror is the parity of its phase.
  std::vector<int> mpar(nodes.size(), 0);
  if (parity) {
    std::vector<int> phase(nodes.size(), -1);
    int n_phase = 0;
    const auto& ord = b.order;
    for (size_t i = 0; i < ord.size();) {
      if (nodes[ord[i]].kind != SLM_KIND_MIRROR) {
        ++i;
        continue;
      }
      size_t j = i;
      while (j < ord.size() && nodes[ord[j]].kind == SLM_KIND_MIRROR) ++j;
      int ph = -1;
      for (size_t k = i; k < j; ++k)
        for (int u : nodes[ord[k]].preds)
          if (nodes[u].kind == SLM_KIND_MIRROR && phase[u] >= 0) ph = std::max(ph, phase[u]);
      if (ph < 0) ph = n_phase++;
      for (size_t k = i; k < j; ++k) {
        phase[ord[k]] = ph;
        mpar[ord[k]] = ph & 1;
      }
      i = j;
    }
  }
  auto grp = [&](int v) {
    const int g = grouped ? group[nodes[v].orig] : 0;
    const bool im = nodes[v].kind == SLM_KIND_MIRROR;
    if (parity) return 3 * g + (im ? 1 + mpar[v] : 0);
    return by_kind ? 2 * g + (im ? 1 : 0) : g;
  };
  std::vector<int> tag_group;
  std::vector<int> cnt(nodes.size(), 0);
  for (int v : b.order)
    for (int p : nodes[v].preds) cnt[p]++;
  out->tag_of.assign(nodes.size(), -1);
  auto& tag_of = out->tag_of;
  auto& tag_size = out->tag_size;
  auto& tag_ext = out->tag_ext;
  tag_size.clear();
  tag_ext.clear();
  // free tags per allocation group: (size, id) -> smallest fit, lowest id
  std::map<int, std::set<std::pair<int64_t, int>>> free_by_group;
  auto release = [&](int tag) { free_by_group[tag_group[tag]].insert({tag_size[tag], tag}); };
  for (int v : b.order) {
    const GN& nd = nodes[v];
    int t = -1;
    if (b.external[v]) {
      t = (int)tag_size.size();
      tag_size.push_back(nd.out_bytes);
      tag_ext.push_back(1);
      tag_group.push_back(grp(v));
    } else {
      int s = nd.inplace_slot;
      if ((flags & SLM_ALLOC_INPLACE) && s >= 0 && s < (int)nd.preds.size()) {
        int u = nd.preds[s];
        if (cnt[u] == 1 && nodes[u].out_bytes == nd.out_bytes && !b.pinned[u]) t = tag_of[u];
      }
      if (t < 0 && (flags & SLM_ALLOC_SHARING)) {
        auto& free_tags = free_by_group[grp(v)];
        auto it = free_tags.lower_bound({nd.out_bytes, -1});
        if (it != free_tags.end()) {
          t = it->second;
          free_tags.erase(it);
        }
      }
      if (t < 0) {
        t = (int)tag_size.size();
        tag_size.push_back(nd.out_bytes);
        tag_ext.push_back(0);
        tag_group.push_back(grp(v));
      }
    }
    tag_of[v] = t;
    for (int u : nd.preds) {
      if (--cnt[u] == 0 && !b.pinned[u] && tag_of[u] != t) release(tag_of[u]);
    }
    if (cnt[v] == 0 && !b.pinned[v]) release(t);
  }
  out->tag_offset.assign(tag_size.size(), -1);
  int64_t run = 0, peak = 0;
  for (size_t t = 0; t < tag_size.size(); ++t) {
    peak += tag_size[t];
    if (tag_ext[t]) continue;
    int64_t off = (run + align - 1) / align * align;
    out->tag_offset[t] = off;
    run = off + tag_size[t];
  }
  out->pool_bytes = run;
  out->exact_peak = peak;
}

// App. A grid, reading A3
const double kGrid[6] = {0.7071067811865476, 0.8122523963562356, 0.9330329915368074,
                         1.0717734625362931, 1.2311444133449163, 1.4142135623730951};

struct Evaluated {
  std::vector<int> m;
  Built b;
  Alloc al;
  int64_t x = 0, y = 0, B = 0;
};

slm_status evaluate(const slm_graph& g, const std::vector<int>& topo, std::vector<int> m,
                    int flags, int64_t align, Evaluated* e) {
  e->m = std::move(m);
  slm_status st = build_mirrored(g, e->m, topo, &e->b);
  if (st != SLM_OK) return st;
  std::vector<int> group(g.nodes.size());
  for (size_t v = 0; v < g.nodes.size(); ++v) group[v] = g.nodes[v].group;
  allocate(e->b, flags, align, &e->al, group);
  return SLM_OK;
}

void export_plan(const slm_graph& g, Evaluated& e, slm_plan* p) {
  p->graph_kind = g.kind;
  std::memcpy(p->dims, g.dims, sizeof(p->dims));
  p->n_fwd = (int)g.nodes.size();
  p->m = e.m;
  p->max_m = 0;
  for (int x : e.m) p->max_m = std::max(p->max_m, x);
  const auto& nodes = e.b.nodes;
  size_t nn = nodes.size();
  p->kind.resize(nn);
  p->op.resize(nn);
  p->orig.resize(nn);
  p->level.resize(nn);
  p->inplace_slot.resize(nn);
  p->out_bytes.resize(nn);
  p->pred_ptr.assign(nn + 1, 0);
  p->preds.clear();
  for (size_t i = 0; i < nn; ++i) {
    p->kind[i] = nodes[i].kind;
    p->op[i] = nodes[i].op;
    p->orig[i] = nodes[i].orig;
    p->level[i] = nodes[i].level;
    p->inplace_slot[i] = nodes[i].inplace_slot;
    p->out_bytes[i] = nodes[i].out_bytes;
    p->pred_ptr[i] = (int)p->preds.size();
    p->preds.insert(p->preds.end(), nodes[i].preds.begin(), nodes[i].preds.end());
  }
  p->pred_ptr[nn] = (int)p->preds.size();
  p->order = e.b.order;
  p->a = e.b.a;
  p->gnode = e.b.gnode;
  p->node_tag = e.al.tag_of;
  p->tag_size = e.al.tag_size;
  p->tag_offset = e.al.tag_offset;
  p->extra_forward = e.b.extra;
  p->exact_peak = e.al.exact_peak;
  p->pool_bytes = e.al.pool_bytes;
  p->x = e.x;
  p->y = e.y;
  p->budget = e.B;
}

slm_status make_plan(const slm_graph& g, const slm_plan_opts& o, slm_plan* p) {
  int flags = o.alloc_flags;
  int64_t align = o.align > 0 ? o.align : 256;
  if (align & (align - 1)) {
    set_error("align must be a power of two");
    return SLM_E_ARG;
  }
  std::vector<int> topo = topo_order(g);
  Evaluated e;
  slm_status st = SLM_OK;
  switch (o.strategy) {
    case SLM_PLAN_NONE:
      st = evaluate(g, topo, std::vector<int>(g.nodes.size(), 0), flags, align, &e);
      break;
    case SLM_PLAN_SQRT:
      st = evaluate(g, topo, sqrt_plan(g, topo), flags, align, &e);
      break;
    case SLM_PLAN_BUDGET: {
      if (o.budget_bytes < 0) {
        set_error("negative budget");
        return SLM_E_ARG;
      }
      std::vector<int> m;
      int64_t x, y;
      alg3(g, topo, o.budget_bytes, &x, &y, &m);
      st = evaluate(g, topo, m, flags, align, &e);
      e.x = x;
      e.y = y;
      e.B = o.budget_bytes;
      break;
    }
    case SLM_PLAN_SEARCH: {
      // App. A, reading A3
      std::vector<Evaluated> evs;
      evs.reserve(8);
      std::vector<int64_t> budgets;
      auto run = [&](int64_t B) -> slm_status {
        std::vector<int> m;
        int64_t x, y;
        alg3(g, topo, B, &x, &y, &m);
        evs.emplace_back();
        slm_status s2 = evaluate(g, topo, m, flags, align, &evs.back());
        evs.back().x = x;
        evs.back().y = y;
        evs.back().B = B;
        return s2;
      };
      if ((st = run(0)) != SLM_OK) return st;                    // "first ... with B = 0"
      unsigned __int128 xy = (unsigned __int128)evs[0].x * (unsigned __int128)evs[0].y;
      int64_t B1 = isqrt64(xy);                                  // "B = sqrt(x y)"
      if ((st = run(B1)) != SLM_OK) return st;
      for (double f : kGrid)                                     // "size 6 grid"
        if ((st = run((int64_t)std::floor((double)B1 * f))) != SLM_OK) return st;
      size_t best = 0;
      for (size_t i = 1; i < evs.size(); ++i) {
        auto key = [&](size_t j) {
          return std::make_tuple(evs[j].al.exact_peak, evs[j].b.extra, evs[j].B);
        };
        if (key(i) < key(best)) best = i;
      }
      for (auto& ev : evs) {
        p->trace.push_back(ev.B);
        p->trace.push_back(ev.x);
        p->trace.push_back(ev.y);
        p->trace.push_back(ev.al.exact_peak);
        p->trace.push_back(ev.b.extra);
      }
      e = std::move(evs[best]);
      break;
    }
    case SLM_PLAN_RECURSIVE: {
      if (o.k < 1) {
        set_error("recursive plan needs k >= 1");
        return SLM_E_DOMAIN;
      }
      std::vector<int> path;
      if (!chain_positions(g, topo, &path)) {
        set_error("NotAChain: the recursive plan is defined on linear chains");
        return SLM_E_NOT_A_CHAIN;
      }
      std::vector<int> m(g.nodes.size(), 0);
      recursive_fill(path, o.k, 0, (int64_t)path.size() - 1, 0, &m);
      st = evaluate(g, topo, m, flags, align, &e);
      break;
    }
    case SLM_PLAN_EXPLICIT: {
      if (!o.m || o.n_m != (int)g.nodes.size()) {
        set_error("explicit plan needs m with one entry per node");
        return SLM_E_INVALID_PLAN;
      }
      st = evaluate(g, topo, std::vector<int>(o.m, o.m + o.n_m), flags, align, &e);
      break;
    }
    case SLM_PLAN_DROP_CHEAP:
      st = evaluate(g, topo, drop_cheap_plan(g), flags, align, &e);
      break;
    default:
      set_error("unknown strategy");
      return SLM_E_ARG;
  }
  if (st != SLM_OK) return st;
  export_plan(g, e, p);
  return SLM_OK;
}

slm_status too_small(int32_t need, int32_t* n) {
  if (n) *n = need;
  set_error("buffer too small");
  return SLM_E_BUFFER_TOO_SMALL;
}

}  // namespace
}  // namespace slm

using namespace slm;

// ====================================================================== C ABI
extern "C" {

const char* slm_last_error(void) { return slm::g_err.c_str(); }

slm_status slm_graph_validate(const slm_node_desc* nodes, int32_t n, const int32_t* outputs,
                              int32_t n_out, slm_diag* diags, int32_t cap, int32_t* n_diags) {
  if ((n > 0 && !nodes) || n < 0 || n_out < 0 || (n_out > 0 && !outputs)) {
    set_error("null/negative argument");
    return SLM_E_ARG;
  }
  slm_graph g;
  g.nodes.resize(n);
  for (int i = 0; i < n; ++i) {
    if (nodes[i].n_preds < 0 || (nodes[i].n_preds > 0 && !nodes[i].preds)) {
      set_error("bad preds");
      return SLM_E_ARG;
    }
    g.nodes[i] = {nodes[i].op, std::vector<int>(nodes[i].preds, nodes[i].preds + nodes[i].n_preds),
                  nodes[i].out_bytes, nodes[i].flags};
  }
  g.outputs.assign(outputs, outputs + n_out);
  auto d = validate(g);
  if (n_diags) *n_diags = (int32_t)d.size();
  if ((int32_t)d.size() > cap) return too_small((int32_t)d.size(), n_diags);
  for (size_t i = 0; i < d.size(); ++i) diags[i] = {d[i].code, d[i].node};
  return SLM_OK;
}

slm_status slm_graph_create(const slm_node_desc* nodes, int32_t n, const int32_t* outputs,
                            int32_t n_out, slm_graph** out) {
  if (!out) {
    set_error("null out");
    return SLM_E_ARG;
  }
  *out = nullptr;
  int32_t nd = 0;
  slm_status st = slm_graph_validate(nodes, n, outputs, n_out, nullptr, 0, &nd);
  if (st != SLM_OK && st != SLM_E_BUFFER_TOO_SMALL) return st;
  if (nd > 0) {
    set_error("invalid graph (" + std::to_string(nd) + " diagnostics)");
    return SLM_E_GRAPH_INVALID;
  }
  auto* g = new (std::nothrow) slm_graph();
  if (!g) return SLM_E_ARG;
  g->nodes.resize(n);
  for (int i = 0; i < n; ++i)
    g->nodes[i] = {nodes[i].op, std::vector<int>(nodes[i].preds, nodes[i].preds + nodes[i].n_preds),
                   nodes[i].out_bytes, nodes[i].flags};
  g->outputs.assign(outputs, outputs + n_out);
  *out = g;
  return SLM_OK;
}

slm_status slm_graph_chain(int32_t n_layers, int32_t batch, int32_t width, slm_graph** out) {
  if (!out || n_layers < 0 || batch <= 0 || width <= 0) {
    set_error("bad chain dims");
    return SLM_E_ARG;
  }
  auto* g = new slm_graph();
  int64_t u = (int64_t)batch * width * 4;
  g->nodes.push_back({SLM_OP_INPUT, {}, u, 0});
  for (int l = 0; l < n_layers; ++l) g->nodes.push_back({SLM_OP_BLOCK, {l}, u, 0});
  g->nodes.push_back({SLM_OP_SOFTMAX_CE, {n_layers}, 4, SLM_NODE_NOT_CANDIDATE});
  g->outputs = {n_layers + 1};
  g->kind = SLM_MODEL_CHAIN;
  g->dims[0] = n_layers;
  g->dims[1] = batch;
  g->dims[2] = width;
  *out = g;
  return SLM_OK;
}

slm_status slm_graph_lstm(int32_t L, int32_t T, int32_t B, int32_t H, int32_t I, slm_graph** out) {
  if (!out || L <= 0 || T <= 0 || B <= 0 || H <= 0 || I <= 0) {
    set_error("bad lstm dims");
    return SLM_E_ARG;
  }
  auto* g = new slm_graph();
  std::vector<int> s_prev(L, -1), heads;
  for (int t = 0; t < T; ++t) {
    int x = (int)g->nodes.size();
    g->nodes.push_back({SLM_OP_INPUT, {}, (int64_t)B * I * 4, 0});
    int below = x;
    for (int l = 0; l < L; ++l) {
      int gid = (int)g->nodes.size();
      std::vector<int> pg{below};
      if (s_prev[l] >= 0) pg.push_back(s_prev[l]);
      g->nodes.push_back({SLM_OP_LSTM_GATES, pg, (int64_t)B * 4 * H * 4, 0, l});
      int sid = (int)g->nodes.size();
      std::vector<int> ps{gid};
      if (s_prev[l] >= 0) ps.push_back(s_prev[l]);
      g->nodes.push_back({SLM_OP_LSTM_CELL, ps, (int64_t)B * 2 * H * 4, 0, l});
      s_prev[l] = sid;
      below = sid;
    }
    heads.push_back((int)g->nodes.size());
    g->nodes.push_back({SLM_OP_HEAD_CE, {below}, 4, SLM_NODE_NOT_CANDIDATE, L});
  }
  g->nodes.push_back({SLM_OP_SUM, heads, 4, SLM_NODE_NOT_CANDIDATE, L});
  g->outputs = {(int)g->nodes.size() - 1};
  g->kind = SLM_MODEL_LSTM;
  int d[5] = {L, T, B, H, I};
  std::memcpy(g->dims, d, sizeof(d));
  *out = g;
  return SLM_OK;
}

slm_status slm_lstm_segment_mirrors(const slm_graph* g, int32_t seg, int32_t* m, int32_t n_nodes) {
  if (!g || !m || seg < 1 || g->kind != SLM_MODEL_LSTM || n_nodes < (int32_t)g->nodes.size()) {
    set_error("slm_lstm_segment_mirrors: bad arguments");
    return SLM_E_ARG;
  }
  int t = -1;
  for (size_t v = 0; v < g->nodes.size(); ++v) {
    const int op = g->nodes[v].op;
    if (op == SLM_OP_INPUT) ++t;
    int mv = 0;
    if (op == SLM_OP_LSTM_GATES) mv = 1;
    else if (op == SLM_OP_LSTM_CELL) mv = (t % seg == seg - 1) ? 0 : 1;
    m[v] = mv;
  }
  return SLM_OK;
}

slm_status slm_graph_size(const slm_graph* g, int32_t* n) {
  if (!g || !n) {
    set_error("null argument");
    return SLM_E_ARG;
  }
  *n = (int32_t)g->nodes.size();
  return SLM_OK;
}

slm_status slm_graph_topo(const slm_graph* g, int32_t* order, int32_t cap, int32_t* n) {
  if (!g) {
    set_error("null graph");
    return SLM_E_ARG;
  }
  auto t = topo_order(*g);
  if (n) *n = (int32_t)t.size();
  if ((int32_t)t.size() > cap || !order) return too_small((int32_t)t.size(), n);
  std::copy(t.begin(), t.end(), order);
  return SLM_OK;
}

void slm_graph_destroy(slm_graph* g) { delete g; }

slm_status slm_graph_mark_not_candidate(slm_graph* g, int32_t op, int32_t* n_marked) {
  if (!g || !op_meta(op)) {
    set_error("slm_graph_mark_not_candidate: null graph or unknown op");
    return SLM_E_ARG;
  }
  int32_t c = 0;
  for (auto& nd : g->nodes)
    if (nd.op == op && !(nd.flags & SLM_NODE_NOT_CANDIDATE)) {
      nd.flags |= SLM_NODE_NOT_CANDIDATE;
      ++c;
    }
  if (n_marked) *n_marked = c;
  return SLM_OK;
}

slm_status slm_plan_create(const slm_graph* g, const slm_plan_opts* opts, slm_plan** out) {
  if (!g || !opts || !out) {
    set_error("null argument");
    return SLM_E_ARG;
  }
  *out = nullptr;
  int64_t total = 0;
  for (auto& nd : g->nodes) total += nd.out_bytes;
  if (total == 0) {
    set_error("degenerate graph (sum of sizes is 0)");
    return SLM_E_DEGENERATE;
  }
  auto* p = new (std::nothrow) slm_plan();
  static std::atomic<uint64_t> next_uid{1};
  if (p) p->uid = next_uid.fetch_add(1);
  if (!p) return SLM_E_ARG;
  slm_status st;
  try {
    st = make_plan(*g, *opts, p);
  } catch (const std::exception& e) {
    set_error(std::string("planner exception: ") + e.what());
    st = SLM_E_ARG;
  }
  if (st != SLM_OK) {
    delete p;
    return st;
  }
  *out = p;
  return SLM_OK;
}

slm_status slm_plan_get_info(const slm_plan* p, slm_plan_info* info) {
  if (!p || !info) {
    set_error("null argument");
    return SLM_E_ARG;
  }
  info->n_nodes = (int32_t)p->kind.size();
  info->n_order = (int32_t)p->order.size();
  info->n_tags = (int32_t)p->tag_size.size();
  info->n_trace = (int32_t)(p->trace.size() / 5);
  info->extra_forward = p->extra_forward;
  info->max_m = p->max_m;
  info->exact_peak = p->exact_peak;
  info->pool_bytes = p->pool_bytes;
  info->x = p->x;
  info->y = p->y;
  info->budget = p->budget;
  return SLM_OK;
}

slm_status slm_plan_mirror(const slm_plan* p, int32_t* m, int32_t cap, int32_t* n) {
  if (!p) {
    set_error("null plan");
    return SLM_E_ARG;
  }
  if (n) *n = (int32_t)p->m.size();
  if ((int32_t)p->m.size() > cap || !m) return too_small((int32_t)p->m.size(), n);
  std::copy(p->m.begin(), p->m.end(), m);
  return SLM_OK;
}

slm_status slm_plan_nodes(const slm_plan* p, int32_t* kind, int32_t* op, int32_t* orig,
                          int32_t* level, int64_t* out_bytes, int32_t* inplace_slot,
                          int32_t* pred_ptr, int32_t cap_nodes, int32_t* preds,
                          int32_t cap_preds, int32_t* n_preds_total) {
  if (!p) {
    set_error("null plan");
    return SLM_E_ARG;
  }
  int32_t nn = (int32_t)p->kind.size(), np = (int32_t)p->preds.size();
  if (n_preds_total) *n_preds_total = np;
  if (cap_nodes < nn || cap_preds < np || !kind || !op || !orig || !level || !out_bytes ||
      !inplace_slot || !pred_ptr || (np > 0 && !preds)) {
    set_error("buffer too small");
    return SLM_E_BUFFER_TOO_SMALL;
  }
  for (int i = 0; i < nn; ++i) {
    kind[i] = p->kind[i];
    op[i] = p->op[i];
    orig[i] = p->orig[i];
    level[i] = p->level[i];
    out_bytes[i] = p->out_bytes[i];
    inplace_slot[i] = p->inplace_slot[i];
    pred_ptr[i] = p->pred_ptr[i];
  }
  pred_ptr[nn] = p->pred_ptr[nn];
  std::copy(p->preds.begin(), p->preds.end(), preds);
  return SLM_OK;
}

slm_status slm_plan_order(const slm_plan* p, int32_t* order, int32_t cap, int32_t* n) {
  if (!p) {
    set_error("null plan");
    return SLM_E_ARG;
  }
  if (n) *n = (int32_t)p->order.size();
  if ((int32_t)p->order.size() > cap || !order) return too_small((int32_t)p->order.size(), n);
  std::copy(p->order.begin(), p->order.end(), order);
  return SLM_OK;
}

slm_status slm_plan_tags(const slm_plan* p, int32_t* node_tag, int32_t cap_nodes,
                         int64_t* tag_size, int64_t* tag_offset, int32_t cap_tags) {
  if (!p) {
    set_error("null plan");
    return SLM_E_ARG;
  }
  if (cap_nodes < (int32_t)p->node_tag.size() || cap_tags < (int32_t)p->tag_size.size() ||
      !node_tag || !tag_size || !tag_offset) {
    set_error("buffer too small");
    return SLM_E_BUFFER_TOO_SMALL;
  }
  std::copy(p->node_tag.begin(), p->node_tag.end(), node_tag);
  std::copy(p->tag_size.begin(), p->tag_size.end(), tag_size);
  std::copy(p->tag_offset.begin(), p->tag_offset.end(), tag_offset);
  return SLM_OK;
}

slm_status slm_plan_trace(const slm_plan* p, int64_t* rows, int32_t cap_rows, int32_t* n) {
  if (!p) {
    set_error("null plan");
    return SLM_E_ARG;
  }
  int32_t nr = (int32_t)(p->trace.size() / 5);
  if (n) *n = nr;
  if (nr > cap_rows || (nr > 0 && !rows)) return too_small(nr, n);
  std::copy(p->trace.begin(), p->trace.end(), rows);
  return SLM_OK;
}

void slm_plan_destroy(slm_plan* p) { delete p; }

slm_status slm_recursion_estimate(int64_t n, int64_t k, int64_t* units, int64_t* depth) {
  // Eq. 2 iterated with ceiling division while n > 1
  if (n < 1 || k < 1) {
    set_error("DomainError: n and k must be >= 1");
    return SLM_E_DOMAIN;
  }
  if (!units || !depth) {
    set_error("null output");
    return SLM_E_ARG;
  }
  int64_t u = 0, d = 0;
  while (n > 1) {
    u += k;
    n = (n + k) / (k + 1);
    ++d;
  }
  *units = u;
  *depth = d;
  return SLM_OK;
}

}  // extern "C"
