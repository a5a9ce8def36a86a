"""B200-native sublinear-memory training (arXiv 1604.06174) — Python binding of libslm.

Thin wrappers over the C ABI (include/slm.h), same names, argument marshalling only:

    g    = Graph.chain(n_layers, batch, width)            # slm_graph_chain
    plan = Plan(g, "sqrt")                                # slm_plan_create  (plan(graph, budget))
    mdl  = ChainModel(params, grads, dtype="bf16")        # slm_model_chain
    loss = mdl.step(plan, x0, labels)                     # slm_step         (step(plan, params, batch))

PyTorch is used only for device memory, streams and process groups.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib

__all__ = ["Graph", "Plan", "ChainModel", "LstmModel", "Comm", "recursion_estimate", "STRATEGY", "OP", "lib"]

STRATEGY = {"none": 0, "sqrt": 1, "budget": 2, "search": 3, "recursive": 4, "explicit": 5,
            "drop_cheap": 6}
OP = dict(input=0, block=1, softmax_ce=2, fc=3, sigmoid=4, relu=5, bn=6, add=7, mul=8,
          identity=9, lstm_gates=10, lstm_cell=11, head_ce=12, sum=13, conv=14, pool=15)
ALLOC_INPLACE, ALLOC_SHARING, ALLOC_GROUPED, ALLOC_GROUP_MIRRORS, ALLOC_MIRROR_PARITY = 1, 2, 4, 8, 16
NODE_NOT_CANDIDATE, NODE_PIN, NODE_REQUEST_GRAD = 1, 2, 4


def _i32arr(xs):
    return (C.c_int32 * max(1, len(xs)))(*xs)


class Graph:
    """slm_graph: G = (V, pred)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def chain(cls, n_layers, batch, width):
        h = C.c_void_p()
        check(lib.slm_graph_chain(n_layers, batch, width, C.byref(h)), "slm_graph_chain")
        return cls(h)

    @classmethod
    def lstm(cls, n_layers, steps, batch, hidden, n_in):
        h = C.c_void_p()
        check(lib.slm_graph_lstm(n_layers, steps, batch, hidden, n_in, C.byref(h)), "slm_graph_lstm")
        return cls(h)

    def mark_not_candidate(self, op):
        """Removes every node of op `op` from Alg. 3's candidate set (slm_graph_mark_not_candidate);
        returns the number of nodes changed."""
        n = C.c_int32()
        check(lib.slm_graph_mark_not_candidate(self._h, int(op), C.byref(n)), "slm_graph_mark_not_candidate")
        return n.value

    def lstm_segment_mirrors(self, seg):
        """Time-segment mirror counts (slm_lstm_segment_mirrors) for Plan(..., 'explicit', m=...)."""
        n = len(self)
        arr = (C.c_int32 * max(1, n))()
        check(lib.slm_lstm_segment_mirrors(self._h, seg, arr, n), "slm_lstm_segment_mirrors")
        return list(arr)[:n]

    @staticmethod
    def _descs(nodes):
        keep = []
        arr = (_lib.NodeDesc * max(1, len(nodes)))()
        for i, (op, preds, size, flags) in enumerate(nodes):
            p = _i32arr(list(preds))
            keep.append(p)
            arr[i] = _lib.NodeDesc(op, len(preds), C.cast(p, _lib.i32p), size, flags)
        return arr, keep

    @classmethod
    def from_nodes(cls, nodes, outputs):
        """nodes: list of (op, preds, out_bytes, flags)."""
        arr, keep = cls._descs(nodes)
        outs = _i32arr(outputs)
        h = C.c_void_p()
        check(lib.slm_graph_create(arr, len(nodes), outs, len(outputs), C.byref(h)), "slm_graph_create")
        return cls(h)

    @classmethod
    def validate(cls, nodes, outputs):
        arr, keep = cls._descs(nodes)
        outs = _i32arr(outputs)
        n = C.c_int32()
        cap = 4 * len(nodes) + 8
        diags = (_lib.Diag * cap)()
        check(lib.slm_graph_validate(arr, len(nodes), outs, len(outputs), diags, cap, C.byref(n)),
              "slm_graph_validate")
        return [(diags[i].code, diags[i].node) for i in range(n.value)]

    def __len__(self):
        n = C.c_int32()
        check(lib.slm_graph_size(self._h, C.byref(n)))
        return n.value

    def topo(self):
        n = len(self)
        out = (C.c_int32 * max(1, n))()
        cnt = C.c_int32()
        check(lib.slm_graph_topo(self._h, out, n, C.byref(cnt)), "slm_graph_topo")
        return list(out[: cnt.value])

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.slm_graph_destroy(self._h)
            self._h = None


class Plan:
    """slm_plan: mirror plan m, gradient graph G', V' and the Fig. 2 memory plan."""

    def __init__(self, graph, strategy="sqrt", budget=0, k=1, m=None,
                 alloc_flags=ALLOC_INPLACE | ALLOC_SHARING, align=256):
        s = STRATEGY[strategy] if isinstance(strategy, str) else int(strategy)
        marr = _i32arr(list(m)) if m is not None else None
        opts = _lib.PlanOpts(s, k, budget, C.cast(marr, _lib.i32p) if marr is not None else None,
                             len(m) if m is not None else 0, alloc_flags, align)
        h = C.c_void_p()
        check(lib.slm_plan_create(graph._h, C.byref(opts), C.byref(h)), "slm_plan_create")
        self._h = h
        self.graph = graph
        info = _lib.PlanInfo()
        check(lib.slm_plan_get_info(h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in _lib.PlanInfo._fields_}

    def __getattr__(self, k):
        info = self.__dict__.get("info")
        if info is not None and k in info:
            return info[k]
        raise AttributeError(k)

    @property
    def m(self):
        n = len(self.graph)
        out = (C.c_int32 * max(1, n))()
        cnt = C.c_int32()
        check(lib.slm_plan_mirror(self._h, out, n, C.byref(cnt)))
        return list(out[: cnt.value])

    @property
    def order(self):
        n = self.info["n_order"]
        out = (C.c_int32 * max(1, n))()
        cnt = C.c_int32()
        check(lib.slm_plan_order(self._h, out, n, C.byref(cnt)))
        return list(out[: cnt.value])

    @property
    def nodes(self):
        nn = self.info["n_nodes"]
        tot = C.c_int32()
        lib.slm_plan_nodes(self._h, None, None, None, None, None, None, None, 0, None, 0, C.byref(tot))
        arrs = [(C.c_int32 * max(1, nn))() for _ in range(4)]
        ob = (C.c_int64 * max(1, nn))()
        ip = (C.c_int32 * max(1, nn))()
        pp = (C.c_int32 * (nn + 1))()
        preds = (C.c_int32 * max(1, tot.value))()
        check(lib.slm_plan_nodes(self._h, *arrs, ob, ip, pp, nn, preds, tot.value, C.byref(tot)))
        out = []
        for i in range(nn):
            out.append(dict(kind=arrs[0][i], op=arrs[1][i], orig=arrs[2][i], level=arrs[3][i],
                            out_bytes=ob[i], inplace_slot=ip[i], preds=list(preds[pp[i]:pp[i + 1]])))
        return out

    @property
    def tags(self):
        nn, nt = self.info["n_nodes"], self.info["n_tags"]
        nt_ = (C.c_int32 * max(1, nn))()
        ts = (C.c_int64 * max(1, nt))()
        to = (C.c_int64 * max(1, nt))()
        check(lib.slm_plan_tags(self._h, nt_, nn, ts, to, nt))
        return list(nt_[:nn]), list(ts[:nt]), list(to[:nt])

    @property
    def trace(self):
        n = self.info["n_trace"]
        rows = (C.c_int64 * max(1, 5 * n))()
        cnt = C.c_int32()
        check(lib.slm_plan_trace(self._h, rows, n, C.byref(cnt)))
        return [tuple(rows[5 * i:5 * i + 5]) for i in range(cnt.value)]

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.slm_plan_destroy(self._h)
            self._h = None


def recursion_estimate(n, k):
    u, d = C.c_int64(), C.c_int64()
    check(lib.slm_recursion_estimate(n, k, C.byref(u), C.byref(d)), "slm_recursion_estimate")
    return u.value, d.value


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


class Comm:
    """slm_comm: NCCL communicator built from a unique id broadcast over torch.distributed."""

    def __init__(self, rank, world, pg=None, bucket_bytes=256 << 20):
        uid = self.broadcast_unique_id(rank, world, pg)
        h = C.c_void_p()
        check(lib.slm_comm_init(rank, world, uid, bucket_bytes, C.byref(h)), "slm_comm_init")
        self._h, self.rank, self.world = h, rank, world

    @staticmethod
    def broadcast_unique_id(rank, world, pg=None):
        """Rank 0 draws the 128-byte NCCL unique id (slm_comm_unique_id); it is broadcast over
        the torch.distributed group (any backend, e.g. gloo) to every rank."""
        import torch
        import torch.distributed as dist
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            check(lib.slm_comm_unique_id(uid), "slm_comm_unique_id")
        t = torch.tensor(list(uid), dtype=torch.uint8)
        if world > 1:
            obj = [t]
            dist.broadcast_object_list(obj, src=0, group=pg)
            t = obj[0]
        for i in range(128):
            uid[i] = int(t[i])
        return uid

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.slm_comm_destroy(self._h)
            self._h = None


class _Model:
    """Common slm_model methods (include/slm.h "device step")."""

    def _init(self, h, options):
        self._h = h
        for k, v in options.items():
            self.set_option(k, v)
        self._bufs = {}

    def set_option(self, key, value):
        check(lib.slm_model_set_option(self._h, key.encode(), int(value)), "slm_model_set_option")

    def get_option(self, key):
        v = C.c_int64()
        check(lib.slm_model_get_option(self._h, key.encode(), C.byref(v)), "slm_model_get_option")
        return v.value

    def workspace_bytes(self, plan):
        n = C.c_size_t()
        check(lib.slm_workspace_bytes(plan._h, self._h, C.byref(n)), "slm_workspace_bytes")
        return n.value

    def kernel_times(self, reset=True):
        """{kind: (total_ms, count)} of the event-timed kernels (option profile_events=1)."""
        n = len(_lib.K_KINDS)
        ms = (C.c_float * n)()
        cnt = (C.c_int64 * n)()
        check(lib.slm_model_kernel_times(self._h, ms, cnt, n, int(reset)), "slm_model_kernel_times")
        return {k: (ms[i], cnt[i]) for i, k in enumerate(_lib.K_KINDS)}

    def launches(self, plan):
        n = C.c_int64()
        check(lib.slm_step_launches(plan._h, self._h, C.byref(n)))
        return n.value

    def buffers(self, plan, device="cuda"):
        """Caller-owned pool (plan.pool_bytes) + workspace + loss scalar, cached for the two most
        recently used plans (older entries are released; pass `bufs` to manage them yourself)."""
        import torch
        key = id(plan)
        if key in self._bufs:
            self._bufs[key] = self._bufs.pop(key)   # most recent last
        else:
            while len(self._bufs) >= 2:
                self._bufs.pop(next(iter(self._bufs)))
            pool = torch.empty(max(256, plan.pool_bytes), dtype=torch.uint8, device=device)
            ws = torch.empty(self.workspace_bytes(plan), dtype=torch.uint8, device=device)
            loss = torch.zeros(1, dtype=torch.float32, device=device)
            self._bufs[key] = (plan, pool, ws, loss)
        return self._bufs[key][1:]

    def step(self, plan, x0, labels, stream=None, comm=None, bufs=None):
        """step(plan, params, batch) -> loss (device tensor); grads written into `grads`."""
        import torch
        pool, ws, loss = bufs if bufs is not None else self.buffers(plan, x0.device)
        st = stream if stream is not None else torch.cuda.current_stream(x0.device)
        check(lib.slm_step(plan._h, self._h, _ptr(x0), _ptr(labels), _ptr(pool), pool.numel(), _ptr(ws),
                           ws.numel(), _ptr(loss), C.c_void_p(st.cuda_stream),
                           comm._h if comm is not None else None), "slm_step")
        return loss

    def step_host(self, plan, x0_host, labels_host, x0_dev, labels_dev, loss_host, stream=None,
                  comm=None, bufs=None):
        """End-to-end step from (pinned) host tensors; returns the host loss value."""
        import torch
        pool, ws, loss = bufs if bufs is not None else self.buffers(plan, x0_dev.device)
        st = stream if stream is not None else torch.cuda.current_stream(x0_dev.device)
        check(lib.slm_step_host(plan._h, self._h, _ptr(x0_host), _ptr(labels_host), _ptr(x0_dev),
                                _ptr(labels_dev), _ptr(pool), pool.numel(), _ptr(ws), ws.numel(),
                                _ptr(loss), _ptr(loss_host), C.c_void_p(st.cuda_stream),
                                comm._h if comm is not None else None), "slm_step_host")
        return float(loss_host[0])

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.slm_model_destroy(self._h)
            self._h = None


class ChainModel(_Model):
    """slm_model for the residual chain.  params/grads: dicts of CUDA tensors
    W [n,d,d] (bf16 or f32), b/gamma/beta [n,d] f32; dW like W; db/dgamma/dbeta f32."""

    def __init__(self, params, grads, dtype="bf16", batch=None, batch_global=0, **options):
        W = params["W"]
        n, d = W.shape[0], W.shape[1]
        self.params, self.grads = params, grads
        self.dtype = dtype
        self.n, self.d = n, d
        self.batch = batch
        desc = _lib.ChainDesc(1 if dtype == "bf16" else 0, n, batch, d, batch_global,
                              _ptr(W), _ptr(params["b"]), _ptr(params["gamma"]), _ptr(params["beta"]),
                              _ptr(grads["W"]), _ptr(grads["b"]), _ptr(grads["gamma"]), _ptr(grads["beta"]))
        h = C.c_void_p()
        check(lib.slm_model_chain(C.byref(desc), C.byref(h)), "slm_model_chain")
        self._init(h, options)


class LstmModel(_Model):
    """slm_model for the unrolled LSTM (include/slm.h slm_lstm_desc).  params: dict of CUDA
    tensors W (flat bf16: layer 0 [4H, Kin0+H] then [4H, 2H] per layer), b [L, 4H] f32,
    W_o bf16 [Cp, H], b_o f32 [Cp]; grads: the same keys in fp32."""

    def __init__(self, params, grads, n_layers, steps, batch, hidden, n_in, n_classes, **options):
        self.params, self.grads = params, grads
        self.L, self.T, self.B, self.H, self.I, self.C = n_layers, steps, batch, hidden, n_in, n_classes
        desc = _lib.LstmDesc(n_layers, steps, batch, hidden, n_in, n_classes,
                             _ptr(params["W"]), _ptr(params["b"]), _ptr(params["W_o"]), _ptr(params["b_o"]),
                             _ptr(grads["W"]), _ptr(grads["b"]), _ptr(grads["W_o"]), _ptr(grads["b_o"]))
        h = C.c_void_p()
        check(lib.slm_model_lstm(C.byref(desc), C.byref(h)), "slm_model_lstm")
        self._init(h, options)

    @staticmethod
    def kin0(n_in):
        return -(-n_in // 128) * 128

    @staticmethod
    def cpad(n_classes):
        return -(-n_classes // 128) * 128

    @staticmethod
    def pack_w(W, n_in):
        """Per-layer [W_ih | W_hh] at the true widths ([4H, I + H], then [4H, 2H]) -> the flat C-ABI
        layout, layer 0 zero-padded to Kin0 = round_up(I, 128) input columns (reading A21: the
        GEMM's K tiles by 64).  W: list of tensors / arrays; returns a flat torch tensor (CPU)."""
        import torch
        out = []
        for l, w in enumerate(W):
            w = torch.as_tensor(w)
            if l == 0:
                H4 = w.shape[0]
                H = H4 // 4
                k0 = LstmModel.kin0(n_in)
                wp = torch.zeros(H4, k0 + H, dtype=w.dtype)
                wp[:, :n_in] = w[:, :n_in]
                wp[:, k0:] = w[:, n_in:]
                w = wp
            out.append(w.reshape(-1))
        return torch.cat(out)

    @staticmethod
    def unpack_w(flat, n_layers, hidden, n_in):
        """Inverse of pack_w for a flat gradient (or weight) buffer: per-layer arrays at the true
        widths (the padding columns dropped)."""
        H = hidden
        k0 = LstmModel.kin0(n_in)
        out, o = [], 0
        for l in range(n_layers):
            kin = k0 if l == 0 else H
            w = flat[o:o + 4 * H * (kin + H)].reshape(4 * H, kin + H)
            o += 4 * H * (kin + H)
            if l == 0:
                w = np.concatenate([w[:, :n_in], w[:, k0:]], axis=1) if isinstance(w, np.ndarray) else \
                    __import__("torch").cat([w[:, :n_in], w[:, k0:]], dim=1)
            out.append(w)
        return out


class OpsModel(_Model):
    """slm_model for an op-granularity graph (slm_model_ops).  graph: a Graph built
    with Graph.from_nodes from Input / BN / ReLU / FC / Add / SoftmaxCE nodes; params / grads:
    {node id: {"W": bf16 [dout, din], "b": f32 [dout]}} for FC nodes and {"gamma", "beta"} (f32)
    for BN nodes (grads: the same keys, W bf16)."""

    def __init__(self, graph, params, grads, batch, batch_global=0, shapes=None, **options):
        """shapes: per node (H, W, C, k, s) for convolutional graphs (Conv params
        {"W": bf16 [C_out, k*k*C_in], "b": f32 [C_out]}), None for [batch][w] graphs."""
        n = len(graph)
        self.params, self.grads, self.graph = params, grads, graph
        arrs = {k: (C.c_void_p * max(1, n))() for k in ("W", "b", "gamma", "beta", "dW", "db", "dgamma", "dbeta")}
        for v in range(n):
            pv, gv = params.get(v, {}), grads.get(v, {})
            for k in ("W", "b", "gamma", "beta"):
                if k in pv:
                    arrs[k][v] = _ptr(pv[k]).value
            for k in ("W", "b", "gamma", "beta"):
                if k in gv:
                    arrs["d" + k][v] = _ptr(gv[k]).value
        self._arrs = arrs
        vpp = C.POINTER(C.c_void_p)
        self._shape = None
        if shapes is not None:
            flat = [int(x) for sh in shapes for x in sh]
            self._shape = (C.c_int32 * len(flat))(*flat)
        desc = _lib.OpsDesc(batch, batch_global, n, *(C.cast(arrs[k], vpp) for k in
                                                       ("W", "b", "gamma", "beta", "dW", "db", "dgamma", "dbeta")),
                            C.cast(self._shape, C.POINTER(C.c_int32)) if self._shape is not None else None)
        h = C.c_void_p()
        check(lib.slm_model_ops(graph._h, C.byref(desc), C.byref(h)), "slm_model_ops")
        self._init(h, options)

    @staticmethod
    def preact_nodes(depths, widths, batch):
        """Node list (op, preds, out_bytes, flags) of the pre-activation network of SURVEY 8(f) f1:
        per layer BN(x) -> ReLU -> FC -> Add(x, .), an FC projection where the width changes, a
        SoftmaxCE loss (the same graph as oracle.graph.preact_resnet_graph)."""
        nodes = [(OP["input"], [], batch * widths[0] * 4, 0)]
        x = 0
        for dep, w in zip(depths, widths):
            if nodes[x][2] != batch * w * 4:
                nodes.append((OP["fc"], [x], batch * w * 4, 0))
                x = len(nodes) - 1
            for _ in range(dep):
                nodes.append((OP["bn"], [x], batch * w * 4, 0))
                nodes.append((OP["relu"], [len(nodes) - 1], batch * w * 4, 0))
                nodes.append((OP["fc"], [len(nodes) - 1], batch * w * 4, 0))
                nodes.append((OP["add"], [x, len(nodes) - 1], batch * w * 4, 0))
                x = len(nodes) - 1
        nodes.append((OP["softmax_ce"], [x], 4, 1))
        return nodes

    @staticmethod
    def preact_conv_nodes(batch, hw, stages, classes):
        """(nodes, shapes) of the convolutional pre-activation ResNet of SURVEY 8(f) f4 (the graph of
        oracle.graph.preact_resnet_conv_graph): stages [(C, depth)], basic blocks
        BN -> ReLU -> Conv3x3_s -> BN -> ReLU -> Conv3x3 -> Add, the first block of every later stage
        with stride 2 and a Conv1x1_s2 projection shortcut of the pre-activated input; head
        BN -> ReLU -> Pool -> FC(classes) -> SoftmaxCE.  shapes[v] = (H, W, C, k, s)."""
        c0 = stages[0][0]
        nodes, shapes = [(OP["input"], [], batch * hw * hw * c0 * 4, 0)], [(hw, hw, c0, 0, 0)]

        def add(op, preds, H, C, k=0, s=0, flags=0):
            nodes.append((OP[op], list(preds), batch * H * H * C * 4 if op != "softmax_ce" else 4, flags))
            shapes.append((H, H, C, k, s))
            return len(nodes) - 1

        x, H = 0, hw
        for i, (C_, depth) in enumerate(stages):
            for j in range(depth):
                s = 2 if (i > 0 and j == 0) else 1
                cin = shapes[x][2]
                Ho = (H - 1) // s + 1
                r = add("relu", [add("bn", [x], H, cin)], H, cin)
                c1 = add("conv", [r], Ho, C_, 3, s)
                c2 = add("conv", [add("relu", [add("bn", [c1], Ho, C_)], Ho, C_)], Ho, C_, 3, 1)
                short = add("conv", [r], Ho, C_, 1, s) if (s != 1 or cin != C_) else x
                x = add("add", [c2, short], Ho, C_)
                H = Ho
        C_ = shapes[x][2]
        r = add("relu", [add("bn", [x], H, C_)], H, C_)
        fc = add("fc", [add("pool", [r], 1, C_)], 1, classes)
        add("softmax_ce", [fc], 1, 1, flags=1)
        return nodes, shapes


def debug_gemm(kind, impl, bn, M, N, K, A, B, out, resid=None, bias=None, stream=None, split=1):
    """Test hook (include/slm_debug.h)."""
    import torch
    st = stream if stream is not None else torch.cuda.current_stream(A.device)
    check(lib.slm_debug_gemm(kind, impl, bn, split, M, N, K, _ptr(A), _ptr(B), _ptr(out), _ptr(resid),
                             _ptr(bias), C.c_void_p(st.cuda_stream)), "slm_debug_gemm")
