/*
 * slm.h — C ABI of the B200-native implementation of arXiv 1604.06174,
 *         "Training Deep Nets with Sublinear Memory Cost" (Chen, Xu, Zhang, Guestrin 2016).
 *
 * The library solves the paper's problem statement: given a computation
 * graph G=(V, pred) and either a mirror plan m or a memory budget B, produce the memory-
 * optimised gradient graph, its execution order V' and a static memory plan
 * ("plan(graph, budget)"), then train with it on the GPU ("step(plan, params, batch)").
 *
 *   host planner (plain C++, no CUDA):     slm_graph_*, slm_plan_*, slm_recursion_estimate
 *   device step (sm_100a, hand-written):   slm_model_*, slm_workspace_bytes, slm_step*
 *   data parallel (NCCL over NVLink):      slm_comm_*
 *
 * Conventions (all functions):
 *   - Every function returns slm_status: SLM_OK (0) or a negative error code; nothing throws
 *     across the ABI.  slm_last_error() returns a thread-local description of the last error
 *     (valid until the next call on the same thread).
 *   - Host objects (graph, plan, model, comm) are owned by the library through create/destroy
 *     pairs; input arrays are copied, never retained.
 *   - Array outputs are caller-allocated.  Passing a capacity smaller than needed returns
 *     SLM_E_BUFFER_TOO_SMALL and writes the needed count to the *n output (cap = 0 queries).
 *   - Device memory (params, grads, batch, pool, workspace, loss) is always caller-owned.
 *     slm_step never allocates device memory: the plan is static ("to
 *     allocate the memory to each node before the execution starts").
 *   - slm_step is asynchronous on the caller's stream; argument, shape and size errors are
 *     reported synchronously, device faults surface at the caller's next synchronisation.
 *   - Plans are immutable and may be shared between threads; a model or comm object is used
 *     by one thread at a time.
 */
#ifndef SLM_H_
#define SLM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t slm_status;
enum {
  SLM_OK = 0,
  SLM_E_ARG = -1,              /* null pointer, bad enum, negative budget, ...            */
  SLM_E_GRAPH_INVALID = -2,    /* cycle | arity | dangling pred | zero size   */
  SLM_E_MULTIPLE_ROOTS = -3,   /* gradient graph needs exactly one loss output     */
  SLM_E_INVALID_PLAN = -4,     /* m(v) > 0 on an Input node, bad length           */
  SLM_E_NOT_A_CHAIN = -5,      /* recursive plan on a non-chain graph             */
  SLM_E_DOMAIN = -6,           /* recursion_estimate / recursive plan with n < 1 or k < 1  */
  SLM_E_DEGENERATE = -7,       /* sum of node sizes is 0                                  */
  SLM_E_ORDER = -8,            /* internal: execution order is not a permutation           */
  SLM_E_SHAPE = -9,            /* model dims do not match the graph / plan                */
  SLM_E_BUFFER_TOO_SMALL = -10,
  SLM_E_UNSUPPORTED = -11,     /* configuration outside what the sm_100a kernels implement */
  SLM_E_CUDA = -20,            /* CUDA runtime/driver error (message in slm_last_error)   */
  SLM_E_NCCL = -21             /* NCCL error or libnccl.so.2 not loadable                  */
};

const char* slm_last_error(void);
/* Library version, e.g. "slm 0.1 sm_100a". */
const char* slm_version(void);

/* ====================================================================== graph
 * G = (V, pred) of Alg. 2.  Nodes are dense ids 0..n-1, each producing ONE
 * output of out_bytes bytes ("each node represents an operation").  Weights
 * and their gradients are not nodes.  Op kinds carry the metadata the paper
 * asks frameworks to declare: which inputs/outputs the backward reads
 * (minimum dependencies) and which input an op may overwrite in place.
 */
enum {
  SLM_OP_INPUT = 0,       /* external input (bound to a caller buffer)                       */
  SLM_OP_BLOCK = 1,       /* residual block x + ReLU(BN(x)) W^T + b; bwd reads its input      */
  SLM_OP_SOFTMAX_CE = 2,  /* mean softmax cross-entropy loss; bwd reads its input            */
  SLM_OP_FC = 3,          /* fully connected; bwd reads its input                            */
  SLM_OP_SIGMOID = 4,     /* bwd reads its output (Fig. 1 sigmoid)         */
  SLM_OP_RELU = 5,        /* bwd reads its output                                            */
  SLM_OP_BN = 6,          /* batch-norm (no running stats); bwd reads its input              */
  SLM_OP_ADD = 7,         /* 2 inputs                                                        */
  SLM_OP_MUL = 8,         /* 2 inputs; bwd reads both                                        */
  SLM_OP_IDENTITY = 9,
  SLM_OP_LSTM_GATES = 10, /* (x_or_lower_state[, prev_state]); bwd reads output and inputs    */
  SLM_OP_LSTM_CELL = 11,  /* (gates[, prev_state]); bwd reads both inputs                     */
  SLM_OP_HEAD_CE = 12,    /* per-step softmax head + CE; bwd reads its input                  */
  SLM_OP_SUM = 13,        /* scalar sum of any number of inputs                               */
  SLM_OP_CONV = 14,       /* convolution (NHWC, "same" padding); bwd reads its input          */
  SLM_OP_POOL = 15        /* global average pool over the spatial positions; bwd reads nothing */
};
enum {
  SLM_NODE_NOT_CANDIDATE = 1, /* exclude from Alg. 3's candidate set C         */
  SLM_NODE_PIN = 2,           /* never recycle this node's storage                          */
  SLM_NODE_REQUEST_GRAD = 4   /* (Input) keep the gradient flowing into this input          */
};

typedef struct {
  int32_t op;             /* SLM_OP_*                                                      */
  int32_t n_preds;
  const int32_t* preds;   /* n_preds node ids (copied)                                      */
  int64_t out_bytes;      /* > 0                                                            */
  int32_t flags;          /* SLM_NODE_*                                                     */
} slm_node_desc;

enum { SLM_DIAG_CYCLE = 1, SLM_DIAG_ARITY = 2, SLM_DIAG_DANGLING = 3, SLM_DIAG_ZERO_SIZE = 4,
       SLM_DIAG_BAD_OUTPUT = 5, SLM_DIAG_BAD_OP = 6 };
typedef struct { int32_t code; int32_t node; } slm_diag;

typedef struct slm_graph slm_graph;

/* Diagnostics are data, not errors: returns SLM_OK with *n_diags = 0 for a valid graph. */
slm_status slm_graph_validate(const slm_node_desc* nodes, int32_t n, const int32_t* outputs,
                              int32_t n_out, slm_diag* diags, int32_t cap, int32_t* n_diags);
/* Validates and copies; SLM_E_GRAPH_INVALID if any diagnostic. */
slm_status slm_graph_create(const slm_node_desc* nodes, int32_t n, const int32_t* outputs,
                            int32_t n_out, slm_graph** out);
/* Residual chain X_0 -> Block_0..Block_{n-1} -> SoftmaxCE (node 0 = Input, node l+1 =
 * Block_l, node n+1 = loss, 4 bytes, NOT_CANDIDATE).  Node sizes batch*width*4 (fp32 x). */
slm_status slm_graph_chain(int32_t n_layers, int32_t batch, int32_t width, slm_graph** out);
/* Unrolled LSTM: per step t an Input X_t (batch*n_in*4), per layer
 * G^l_t (batch*4H*4) and S^l_t (batch*2H*4), a head H_t (4 bytes); final Sum (the loss). */
slm_status slm_graph_lstm(int32_t n_layers, int32_t steps, int32_t batch, int32_t hidden,
                          int32_t n_in, slm_graph** out);
/* Restricts Alg. 3's candidate set C (reading A19) on an existing graph: every
 * node whose op is `op` (SLM_OP_*) gets SLM_NODE_NOT_CANDIDATE, so the budget / App. A search
 * plans only split elsewhere — e.g. op = SLM_OP_LSTM_GATES leaves the LSTM's cell states as the
 * only split points (reading A25).  *n_marked = nodes changed (may be NULL).
 * SLM_E_ARG for a null graph or an unknown op. */
slm_status slm_graph_mark_not_candidate(slm_graph* g, int32_t op, int32_t* n_marked);
/* Time-segment mirror counts for a graph built by slm_graph_lstm (the LSTM
 * is checkpointed along time): m[v] = 1 for every gates/cell node except the cell states
 * S^l_t at segment ends (t % seg == seg - 1), which are kept; 0 elsewhere.  Feed the result
 * to slm_plan_create with strategy SLM_STRATEGY_EXPLICIT.  m has room for n_nodes entries;
 * SLM_E_ARG when seg < 1 or the graph is not an LSTM graph. */
slm_status slm_lstm_segment_mirrors(const slm_graph* g, int32_t seg, int32_t* m, int32_t n_nodes);
slm_status slm_graph_size(const slm_graph* g, int32_t* n_nodes);
/* topological-order(V) of Alg. 2: Kahn, lowest id first among ready nodes. */
slm_status slm_graph_topo(const slm_graph* g, int32_t* order, int32_t cap, int32_t* n);
void slm_graph_destroy(slm_graph* g);

/* ====================================================================== plan
 * Strategies choose the mirror-count function m: V -> N:
 *   NONE        m = 0 everywhere (ordinary gradient graph)
 *   SQRT        Sec. 4.3: k = ceil(sqrt n) segments over the candidates
 *   BUDGET      Alg. 3 with budget_bytes
 *   SEARCH      App. A grid search over B; trace of 8 evaluated budgets
 *   RECURSIVE   Sec. 4.4 recursion with k kept results per level; chains
 *   EXPLICIT    user-set mirror counts ("set the mirror attribute")
 *   DROP_CHEAP  Sec. 4.2 drop results of low-cost ops
 * then Alg. 2 builds G' and V' and the Fig. 2 allocator assigns temporal
 * tags with in-place and sharing.  Readings of silent points: DESIGN.md
 * A1-A20.  Tags of Input nodes and of the loss are bound to caller buffers (offset -1); all
 * other tags get 256-byte-aligned offsets in one pool of pool_bytes.  exact_peak = sum of
 * all tag sizes (unaligned, external tags included) = the paper's "exact memory cost"
 * (PAPER.md:334, 397).
 */
enum { SLM_PLAN_NONE = 0, SLM_PLAN_SQRT = 1, SLM_PLAN_BUDGET = 2, SLM_PLAN_SEARCH = 3,
       SLM_PLAN_RECURSIVE = 4, SLM_PLAN_EXPLICIT = 5, SLM_PLAN_DROP_CHEAP = 6 };
/* SLM_ALLOC_GROUPED (with SHARING): a freed tag is reused only by a node of the same allocation
 * group (slm_graph_lstm: the layer of a gates/cell node, L for the head and the loss; every
 * other builder: one group), so the plan never makes work of two layers share memory and the
 * layer wavefront keeps its concurrency (reading A22; an extension, not the paper). */
/* SLM_ALLOC_GROUP_MIRRORS: re-computed (mirror) nodes and the other nodes never share a tag, so
 * the recompute of one segment does not wait for the backward of the next (A22). */
/* SLM_ALLOC_MIRROR_PARITY: like GROUP_MIRRORS, and a mirror reuses only tags of mirrors whose
 * recompute phase has the same parity (a maximal run of consecutive mirrors in V' continues the
 * latest phase it reads a mirror of, else starts a new one), so the recompute of segment
 * j-1 writes memory disjoint from everything the backward of segment j reads or writes: the
 * executor runs the two concurrently (reading A24; an extension, not the paper).
 * Costs one more segment of mirrors (still O(sqrt n) for the sqrt plan). */
enum { SLM_ALLOC_INPLACE = 1, SLM_ALLOC_SHARING = 2, SLM_ALLOC_GROUPED = 4, SLM_ALLOC_GROUP_MIRRORS = 8,
       SLM_ALLOC_MIRROR_PARITY = 16 };

typedef struct {
  int32_t strategy;       /* SLM_PLAN_*                                                    */
  int32_t k;              /* RECURSIVE: results kept per level (>= 1)                       */
  int64_t budget_bytes;   /* BUDGET: B >= 0                                                 */
  const int32_t* m;       /* EXPLICIT: n_nodes mirror counts (copied)                       */
  int32_t n_m;
  int32_t alloc_flags;    /* SLM_ALLOC_INPLACE | SLM_ALLOC_SHARING (0 = "no optimization")  */
  int32_t align;          /* pool offset alignment in bytes, power of two; 0 -> 256         */
} slm_plan_opts;

typedef struct slm_plan slm_plan;
slm_status slm_plan_create(const slm_graph* g, const slm_plan_opts* opts, slm_plan** out);

typedef struct {
  int32_t n_nodes;        /* nodes of G' (forward + all mirrors + gradient nodes)           */
  int32_t n_order;        /* |V'| (dead mirrors are not in V', reading A7)                  */
  int32_t n_tags;
  int32_t n_trace;        /* SEARCH: 8; else 0                                              */
  int32_t extra_forward;  /* mirror nodes in V' = re-computed forward ops                   */
  int32_t max_m;
  int64_t exact_peak;     /* bytes                                                          */
  int64_t pool_bytes;     /* bytes the caller must provide to slm_step                      */
  int64_t x, y, budget;   /* Alg. 3 outputs for BUDGET / SEARCH          */
} slm_plan_info;
slm_status slm_plan_get_info(const slm_plan* p, slm_plan_info* info);
/* m over the forward nodes (checkpoint set = {v : m(v) = 0}); cap >= n forward nodes. */
slm_status slm_plan_mirror(const slm_plan* p, int32_t* m, int32_t cap, int32_t* n);

enum { SLM_KIND_FWD = 0, SLM_KIND_MIRROR = 1, SLM_KIND_GRAD = 2 };
/* Nodes of G' in CSR form: per node kind, op, orig (forward node it mirrors/differentiates),
 * level (mirror level), out_bytes, inplace_slot; preds in pred_ptr[i]..pred_ptr[i+1].
 * cap_nodes >= n_nodes, cap_preds >= total preds (query with cap 0). */
slm_status slm_plan_nodes(const slm_plan* p, int32_t* kind, int32_t* op, int32_t* orig,
                          int32_t* level, int64_t* out_bytes, int32_t* inplace_slot,
                          int32_t* pred_ptr, int32_t cap_nodes, int32_t* preds,
                          int32_t cap_preds, int32_t* n_preds_total);
/* V'. */
slm_status slm_plan_order(const slm_plan* p, int32_t* order, int32_t cap, int32_t* n);
/* node_tag[n_nodes] (-1 for nodes not in V'); tag_size/tag_offset[n_tags] (offset -1 =
 * external: bound to an Input buffer or the loss). */
slm_status slm_plan_tags(const slm_plan* p, int32_t* node_tag, int32_t cap_nodes,
                         int64_t* tag_size, int64_t* tag_offset, int32_t cap_tags);
/* App. A trace rows (B, x, y, exact_peak, extra_forward), 5 int64 per row. */
slm_status slm_plan_trace(const slm_plan* p, int64_t* rows, int32_t cap_rows, int32_t* n);
void slm_plan_destroy(slm_plan* p);

/* Eq. 2 g(n) = k + g(n/(k+1)) iterated with ceiling division. */
slm_status slm_recursion_estimate(int64_t n, int64_t k, int64_t* units, int64_t* depth);

/* ====================================================================== device step
 * The training step of the chain: executes V' on the GPU, writing
 * every node into its planned pool slot; forward, re-computation (mirrors) and backward
 * run hand-written sm_100a kernels (tcgen05/TMEM GEMMs fed by TMA in bf16 mode, fp32 FFMA
 * kernels in f32 mode).  There is no CPU fallback: without an sm_100a device every step
 * call returns SLM_E_CUDA / SLM_E_UNSUPPORTED.
 */
enum { SLM_F32 = 0, SLM_BF16 = 1 };
enum { SLM_MODEL_CHAIN = 0, SLM_MODEL_LSTM = 1, SLM_MODEL_OPS = 2 };

/* Chain parameters, all device pointers, row-major, caller-owned:
 *   W      [n][d][d]  (out, in)  fp32 (SLM_F32) or bf16 (SLM_BF16)
 *   b, gamma, beta    [n][d] fp32
 *   dW     [n][d][d]  same dtype as W (bf16 grads are rounded from fp32 accumulators)
 *   db, dgamma, dbeta [n][d] fp32
 * Gradients are overwritten by every step, not accumulated.  batch_global = total batch
 * over all data-parallel ranks (the loss is the mean over it); 0 means batch. */
typedef struct {
  int32_t dtype;
  int32_t n_layers, batch, width, batch_global;
  const void* W; const float* b; const float* gamma; const float* beta;
  void* dW; float* db; float* dgamma; float* dbeta;
} slm_chain_desc;

typedef struct slm_model slm_model;
slm_status slm_model_chain(const slm_chain_desc* desc, slm_model** out);

/* Unrolled multi-layer LSTM (reading A13: gate order i, f, g, o; h_0 = c_0 = 0;
 * a softmax head after the top layer at every step; loss = sum_t sum_b CE / (T B)).
 * All device pointers, caller-owned; bf16 GEMM operands only (reading A11):
 *   W     bf16, layer 0 [4H][Kin0 + H] then layers 1.. [4H][2H], each = [W_ih | W_hh] (out, in);
 *         Kin0 = round_up(n_in, 128), the padding columns are ignored (they multiply zeros)
 *   b     fp32 [L][4H] (= b_ih + b_hh)
 *   W_o   bf16 [Cp][H], Cp = round_up(n_classes, 128); rows >= n_classes are never read
 *         into the loss (their logits are masked) but must be finite
 *   b_o   fp32 [Cp]
 *   dW, db, dW_o, db_o   fp32, same layouts; overwritten by every step (the per-step weight
 *         gradients are summed over time inside the step).
 * Constraints of the tcgen05 path: batch in {64, 128, 256}, hidden % 128 == 0.
 * Step inputs: x0 = x fp32 [T][B][n_in], labels int32 [T][B] in [0, n_classes).
 * The LSTM runs replicas-only across GPUs (comm must be NULL). */
typedef struct {
  int32_t n_layers, steps, batch, hidden, n_in, n_classes;
  const void* W; const float* b; const void* W_o; const float* b_o;
  float* dW; float* db; float* dW_o; float* db_o;
} slm_lstm_desc;
slm_status slm_model_lstm(const slm_lstm_desc* desc, slm_model** out);
/* Op-granularity graphs: any DAG built with
 * slm_graph_create from Input, BN, ReLU, FC, Add and SoftmaxCE nodes (e.g. the pre-activation
 * network of oracle.graph.preact_resnet_graph: per layer BN(x) -> ReLU -> FC -> Add(x, .)), so
 * that the DROP_CHEAP plan ("drop bn-relu") really re-computes BN and ReLU outputs.  Every node's
 * value is [batch][w] fp32 with w = out_bytes / (4 batch) (the loss: 4 bytes).  Node semantics
 * (oracle/opgraph.py): BN with batch statistics (biased variance, eps 1e-5), ReLU'(0) = 0,
 * FC y = x W^T + b, Add, SoftmaxCE = mean CE over batch_global (0 = batch) with labels in [0, w).
 * Per-node parameter arrays of n_nodes entries (host arrays of DEVICE pointers, copied; entries of
 * other ops ignored):
 *   FC  W bf16 [dout][din], b fp32 [dout]; grads dW bf16 (rounded from fp32), db fp32
 *   BN  gamma, beta fp32 [w]; grads dgamma, dbeta fp32
 * Gradients are overwritten by every step.  Constraints of the tcgen05 path: batch % 64 == 0,
 * every width % 128 == 0.  Step inputs: x0 [batch][w_input] fp32, labels int32 [batch].
 * Runs replicas-only (comm must be NULL).  SLM_E_ARG / SLM_E_UNSUPPORTED (message in
 * slm_last_error) for an unsupported op, a bad width or a missing parameter.
 * Convolutional graphs (oracle.graph.preact_resnet_conv_graph):
 * `shape` = 5 int32 per node (H, W, C, k, s); a node's value is then the NHWC tensor
 * [batch][H][W][C] fp32 (rows = batch H W of width C; out_bytes must equal 4 batch H W C), BN
 * normalises each channel over all rows, and two more ops are available:
 *   Conv (SLM_OP_CONV)  k x k ("same" zero padding k / 2), stride s, k in {1, 3}, s in {1, 2}:
 *       W bf16 [C_out][k k C_in] (K index (u k + v) C_in + c), b fp32 [C_out]; the output H, W
 *       must be (H_in - 1) / s + 1; C_in % 128 == 0.  Lowered as im2col + tcgen05 GEMM (forward:
 *       y = col W^T + b; backward: dW = dy^T col, dcol = dy W, col2im gather), db = sum dy.
 *   Pool (SLM_OP_POOL)  global average over the H W positions -> [batch][C] (H = W = 1).
 * FC nodes then need an input with H = W = 1.  shape = NULL: H = W = 1, C = out_bytes / (4 batch). */
typedef struct {
  int32_t batch, batch_global, n_nodes;
  const void* const* W; const float* const* b; const float* const* gamma; const float* const* beta;
  void* const* dW; float* const* db; float* const* dgamma; float* const* dbeta;
  const int32_t* shape;   /* n_nodes x (H, W, C, k, s), or NULL (copied) */
} slm_ops_desc;
slm_status slm_model_ops(const slm_graph* g, const slm_ops_desc* desc, slm_model** out);
void slm_model_destroy(slm_model* m);
/* Options (int64 values):
 *   use_graph       capture the whole step in a CUDA graph per buffer set (default 1)
 *   gemm_impl       0 = tcgen05/TMA tensor-core GEMMs (bf16, default), 1 = SIMT FFMA GEMMs
 *   fused           1 (default) = chain: one fused Block kernel per node of V' (blk_fused.cuh:
 *                   split-K tcgen05 GEMM over a cluster + batch norm in the epilogue);
 *                   0 = the basic lowering (separate BN kernels)
 *   block_cfg       fused Block shape: 0 = default for the batch, 1..4 = explicit (BM, S)
 *   overlap         1 (default) = chain: each segment's recompute on its own stream, concurrent
 *                   with the backward of the next segment, when the plan makes that sound
 *                   (SLM_ALLOC_MIRROR_PARITY plans); other plans run sequentially
 *   pdl             1 (default) = programmatic dependent launch between the step's kernels
 *   poison          debug: 1 = fill a pool tag with NaN once its value is dead (forces the
 *                   sequential schedule); a plan that clobbers a live value then yields NaN
 *   lstm_streams    1 = LSTM layer wavefront: one stream per layer + one for the head, ordered
 *                   by per-buffer last-writer / reader events (0 = the caller's stream);
 *                   2 (default) = plus one stream per layer for re-computed (mirror) units, so
 *                   with a SLM_ALLOC_MIRROR_PARITY plan the recompute of a time segment runs
 *                   concurrently with the backward of the next one
 *   lstm_fuse_runs  1 (default) = LSTM forward / recompute phases as persistent chunk x layer
 *                   runs (lstm_run.cuh); 0 = node by node in V' order
 *   profile_events  1 = record a CUDA event pair around every kernel of the step, by kind
 *                   (read with slm_model_kernel_times after the stream is synchronised)
 *   profile_ts      N > 0: the first N tcgen05 GEMM launches of a step record the device clock
 *                   (%globaltimer) at start and end of every CTA into profile_ts_buffer
 *                   (caller-owned, zeroed device buffer of N*1024*2 uint64, passed as an int64
 *                   pointer value); slm_model_kernel_times then adds each launch's span
 *                   (latest end - earliest start) to its GEMM kind.  Works inside the CUDA graph.
 *   profile_ts_dep  1 = a CTA's span starts when it returns from its dependency wait
 *   lstm_run_ts, lstm_run_ts_n   debug: per-step device clocks of the first persistent LSTM runs
 * Every change drops the captured CUDA graphs.  SLM_E_ARG for an unknown key. */
slm_status slm_model_set_option(slm_model* m, const char* key, int64_t value);
/* Reads an option back, or the read-only state "last_overlap" (1 = the last enqueued chain step
 * ran its segment recomputes on the recompute stream, concurrently with the backward; option
 * overlap + a plan that allows it).  SLM_E_ARG for unknown keys. */
slm_status slm_model_get_option(const slm_model* m, const char* key, int64_t* value);
/* Kernel kinds for slm_model_kernel_times. */
enum { SLM_K_BN_ACT = 0, SLM_K_GEMM_FWD = 1, SLM_K_GEMM_DX = 2, SLM_K_GEMM_DW = 3, SLM_K_BN_BWD = 4,
       SLM_K_CE = 5, SLM_K_COUNT = 6 };
/* Sum of event-timed durations (ms) and launch counts per kind since the last reset,
 * accumulated over every step run with profile_events = 1; reset = 1 clears them. */
slm_status slm_model_kernel_times(slm_model* m, float* ms, int64_t* count, int32_t n_kinds,
                                  int32_t reset);
/* Per-kernel scratch (bf16 operand copies, BN statistics, loss partials): the paper's
 * "temporal memory", not part of the feature-map plan. */
slm_status slm_workspace_bytes(const slm_plan* p, const slm_model* m, size_t* bytes);
/* Kernels launched by one slm_step of this (plan, model) — for launch accounting. */
slm_status slm_step_launches(const slm_plan* p, const slm_model* m, int64_t* launches);

typedef struct slm_comm slm_comm;

/* step(plan, params, batch) -> loss, grads.
 *   x0      device [batch][d] fp32 (bound to the Input node's tag); LSTM: [T][B][n_in]
 *   labels  device [batch] int32 in [0, d); LSTM: [T][B] in [0, n_classes)
 *   pool    device, >= plan pool_bytes, 256-byte aligned
 *   ws      device, >= slm_workspace_bytes, 256-byte aligned
 *   loss    device, 1 float (bound to the loss node's tag)
 *   stream  cudaStream_t (NULL = legacy default stream)
 *   comm    NULL for one GPU; else gradients are all-reduced (sum) over the ranks in
 *           buckets overlapped with the rest of the backward, and loss is the global mean. */
slm_status slm_step(const slm_plan* p, slm_model* m, const void* x0, const int32_t* labels,
                    void* pool, size_t pool_bytes, void* ws, size_t ws_bytes, float* loss,
                    void* stream, slm_comm* comm);
/* The same step with HOST inputs/outputs (the end-to-end path): copies x0_host/labels_host
 * (pinned host memory recommended) into x0_dev/labels_dev on the stream, runs slm_step and
 * copies the loss back into *loss_host; synchronises the stream before returning. */
slm_status slm_step_host(const slm_plan* p, slm_model* m, const float* x0_host,
                         const int32_t* labels_host, void* x0_dev, int32_t* labels_dev,
                         void* pool, size_t pool_bytes, void* ws, size_t ws_bytes,
                         float* loss_dev, float* loss_host, void* stream, slm_comm* comm);

/* ====================================================================== data parallel
 * One process per GPU.  The caller distributes a 128-byte unique id (e.g. broadcast over a
 * torch.distributed process group) and each rank calls slm_comm_init.  NCCL is loaded at
 * run time (libnccl.so.2); bucket_bytes groups per-layer gradients into all-reduce buckets. */
slm_status slm_comm_unique_id(void* id128);
slm_status slm_comm_init(int32_t rank, int32_t world, const void* id128, int64_t bucket_bytes,
                         slm_comm** out);
void slm_comm_destroy(slm_comm* c);

#ifdef __cplusplus
}
#endif
#endif /* SLM_H_ */
