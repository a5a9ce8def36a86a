// Internal structures shared by the host planner (planner.cpp) and the device runtime
// (runtime.cu).  Not part of the ABI.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "slm.h"

namespace slm {

// Per-op metadata (readings A6, A18): the minimum backward dependencies the paper
// asks frameworks to declare and the in-place slots.
enum GradInplace { GI_NONE = -1, GI_SUCC0 = 0, GI_OUT = 1, GI_IN0 = 2 };
struct OpMeta {
  int arity_min, arity_max;
  int fwd_inplace;       // predecessor slot the forward may overwrite, -1 none
  bool grad_needs_out;   // backward reads the op's output
  int grad_needs_in;     // bitmask of predecessor slots the backward reads
  int grad_inplace;      // GradInplace
  bool low_cost;         // Sec. 4.2 "low cost operations"
};
const OpMeta* op_meta(int op);  // nullptr for an unknown op

struct Node {
  int op;
  std::vector<int> preds;
  int64_t out_bytes;
  int flags;
  int group = 0;   // allocation group (SLM_ALLOC_GROUPED): the LSTM builder uses the layer
};

void set_error(const std::string& msg);

}  // namespace slm

struct slm_graph {
  std::vector<slm::Node> nodes;
  std::vector<int> outputs;
  int kind = -1;           // -1 generic, SLM_MODEL_CHAIN, SLM_MODEL_LSTM
  int dims[5] = {0, 0, 0, 0, 0};  // chain: n, batch, width; lstm: L, T, B, H, I
};

struct slm_plan {
  // process-unique id (never reused): the device runtime keys its captured CUDA graphs on it, so a
  // new plan that lands at a freed plan's address can never replay that plan's graph
  uint64_t uid = 0;
  // the forward graph it was planned for
  int graph_kind = -1;
  int dims[5] = {0, 0, 0, 0, 0};
  int n_fwd = 0;
  std::vector<int> m;
  // G' = forward nodes, mirrors, gradient nodes (Alg. 2)
  std::vector<int> kind, op, orig, level, inplace_slot;
  std::vector<int64_t> out_bytes;
  std::vector<int> pred_ptr, preds;
  std::vector<int> order;        // V'
  std::vector<int> a;            // deepest mirror of each forward node
  std::vector<int> gnode;        // forward node -> gradient node (-1 none)
  // allocation (Fig. 2)
  std::vector<int> node_tag;     // -1 if not in V'
  std::vector<int64_t> tag_size, tag_offset;
  int extra_forward = 0;
  int max_m = 0;
  int64_t exact_peak = 0, pool_bytes = 0, x = 0, y = 0, budget = 0;
  std::vector<int64_t> trace;    // 5 per row
};
