"""ctypes binding of libslm.so (include/slm.h).  Argument marshalling only: every step of
the path runs in the library (host planner in C++, device step in sm_100a kernels).

There is no fallback: if the in-tree libslm.so is missing this module raises at import."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SLM_LIB: an alternative in-tree build of the same library (compile-time kernel experiments, e.g.
# scripts that A/B two builds); default libslm.so
LIB_PATH = os.path.join(_HERE, os.environ.get("SLM_LIB", "libslm.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python paper_1604_06174_b200/build.py` "
                      "(or __graft_entry__.build()); there is no non-native fallback")
lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

i32, i64, f32p, vp = C.c_int32, C.c_int64, C.POINTER(C.c_float), C.c_void_p
i32p, i64p = C.POINTER(C.c_int32), C.POINTER(C.c_int64)


class NodeDesc(C.Structure):
    _fields_ = [("op", i32), ("n_preds", i32), ("preds", i32p), ("out_bytes", i64), ("flags", i32)]


class Diag(C.Structure):
    _fields_ = [("code", i32), ("node", i32)]


class PlanOpts(C.Structure):
    _fields_ = [("strategy", i32), ("k", i32), ("budget_bytes", i64), ("m", i32p), ("n_m", i32),
                ("alloc_flags", i32), ("align", i32)]


class PlanInfo(C.Structure):
    _fields_ = [("n_nodes", i32), ("n_order", i32), ("n_tags", i32), ("n_trace", i32),
                ("extra_forward", i32), ("max_m", i32), ("exact_peak", i64), ("pool_bytes", i64),
                ("x", i64), ("y", i64), ("budget", i64)]


class ChainDesc(C.Structure):
    _fields_ = [("dtype", i32), ("n_layers", i32), ("batch", i32), ("width", i32),
                ("batch_global", i32), ("W", vp), ("b", vp), ("gamma", vp), ("beta", vp),
                ("dW", vp), ("db", vp), ("dgamma", vp), ("dbeta", vp)]


class LstmDesc(C.Structure):
    _fields_ = [("n_layers", i32), ("steps", i32), ("batch", i32), ("hidden", i32), ("n_in", i32),
                ("n_classes", i32), ("W", vp), ("b", vp), ("W_o", vp), ("b_o", vp),
                ("dW", vp), ("db", vp), ("dW_o", vp), ("db_o", vp)]


class OpsDesc(C.Structure):
    _fields_ = [("batch", i32), ("batch_global", i32), ("n_nodes", i32),
                ("W", C.POINTER(vp)), ("b", C.POINTER(vp)), ("gamma", C.POINTER(vp)), ("beta", C.POINTER(vp)),
                ("dW", C.POINTER(vp)), ("db", C.POINTER(vp)), ("dgamma", C.POINTER(vp)), ("dbeta", C.POINTER(vp)),
                ("shape", C.POINTER(i32))]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("slm_last_error", C.c_char_p)
_sig("slm_version", C.c_char_p)
_sig("slm_graph_validate", i32, C.POINTER(NodeDesc), i32, i32p, i32, C.POINTER(Diag), i32, i32p)
_sig("slm_graph_create", i32, C.POINTER(NodeDesc), i32, i32p, i32, C.POINTER(vp))
_sig("slm_graph_chain", i32, i32, i32, i32, C.POINTER(vp))
_sig("slm_graph_lstm", i32, i32, i32, i32, i32, i32, C.POINTER(vp))
_sig("slm_graph_size", i32, vp, i32p)
_sig("slm_graph_topo", i32, vp, i32p, i32, i32p)
_sig("slm_graph_destroy", None, vp)
_sig("slm_plan_create", i32, vp, C.POINTER(PlanOpts), C.POINTER(vp))
_sig("slm_plan_get_info", i32, vp, C.POINTER(PlanInfo))
_sig("slm_plan_mirror", i32, vp, i32p, i32, i32p)
_sig("slm_plan_nodes", i32, vp, i32p, i32p, i32p, i32p, i64p, i32p, i32p, i32, i32p, i32, i32p)
_sig("slm_plan_order", i32, vp, i32p, i32, i32p)
_sig("slm_plan_tags", i32, vp, i32p, i32, i64p, i64p, i32)
_sig("slm_plan_trace", i32, vp, i64p, i32, i32p)
_sig("slm_plan_destroy", None, vp)
_sig("slm_recursion_estimate", i32, i64, i64, i64p, i64p)
_sig("slm_model_chain", i32, C.POINTER(ChainDesc), C.POINTER(vp))
_sig("slm_model_lstm", i32, C.POINTER(LstmDesc), C.POINTER(vp))
_sig("slm_model_ops", i32, vp, C.POINTER(OpsDesc), C.POINTER(vp))
_sig("slm_debug_ts_meta", i32, vp, i32p, i32p, i32, i32p)
_sig("slm_lstm_segment_mirrors", i32, vp, i32, i32p, i32)
_sig("slm_model_destroy", None, vp)
_sig("slm_model_set_option", i32, vp, C.c_char_p, i64)
_sig("slm_model_get_option", i32, vp, C.c_char_p, i64p)
_sig("slm_graph_mark_not_candidate", i32, vp, i32, i32p)
_sig("slm_workspace_bytes", i32, vp, vp, C.POINTER(C.c_size_t))
_sig("slm_step_launches", i32, vp, vp, i64p)
_sig("slm_step", i32, vp, vp, vp, vp, vp, C.c_size_t, vp, C.c_size_t, vp, vp, vp)
_sig("slm_step_host", i32, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp, C.c_size_t, vp, vp, vp, vp)
_sig("slm_comm_unique_id", i32, vp)
_sig("slm_comm_init", i32, i32, i32, vp, i64, C.POINTER(vp))
_sig("slm_comm_destroy", None, vp)
_sig("slm_debug_gemm", i32, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp)

# names declared in include/slm.h + include/slm_debug.h (checked by tests/test_abi.py)
EXPORTS = [n for n in dir(lib) if n.startswith("slm_")]

STATUS = {0: "OK", -1: "E_ARG", -2: "E_GRAPH_INVALID", -3: "E_MULTIPLE_ROOTS", -4: "E_INVALID_PLAN",
          -5: "E_NOT_A_CHAIN", -6: "E_DOMAIN", -7: "E_DEGENERATE", -8: "E_ORDER", -9: "E_SHAPE",
          -10: "E_BUFFER_TOO_SMALL", -11: "E_UNSUPPORTED", -20: "E_CUDA", -21: "E_NCCL"}


class SlmError(RuntimeError):
    def __init__(self, code, where):
        msg = (lib.slm_last_error() or b"").decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(code, code)} ({msg})")
        self.code = code


def check(code, where=""):
    if code != 0:
        raise SlmError(code, where)
    return code

_sig("slm_model_kernel_times", i32, vp, f32p, i64p, i32, i32)
K_KINDS = ["bn_act", "gemm_fwd", "gemm_dx", "gemm_dw", "bn_bwd", "ce"]
_sig("slm_debug_timestamps", i32, vp)
_sig("slm_debug_plan_alias", i32, vp, i32, i32)
_sig("slm_debug_block", i32, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
     C.c_int, vp)
