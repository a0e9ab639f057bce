"""ctypes binding of libpropd.so (the C ABI declared in include/propd.h).

The product path has no fallback: if the shared library is missing or fails
to load, every backend constructor raises.  Build it with
`python -c "import __graft_entry__ as g; g.build()"` (or `make`).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_int, c_int64, c_void_p

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpropd.so")
ABI_VERSION = 5

F32 = 0
BF16 = 1

P = c_void_p
I = c_int
L = c_int64

# name -> argument types (all return int unless listed in _RESTYPES)
SIGNATURES = {
    "propd_last_error": [],
    "propd_abi_version": [],
    "propd_num_sms": [],
    "propd_prepare": [],
    "propd_gemm_ws_barrier_ctas": [],
    "propd_debug_timeline": [P],
    "propd_pad_rows": [I, I, I, P, P, P, P, P, P],
    "propd_tree_embed": [I, I, I, I, I, I, P, P, P, P, P, P, P, P, P, P, P, P, P, P],
    "propd_embed_rows": [I, I, I, P, P, P, P, P, P],
    "propd_bonus_embed": [I, I, I, P, P, P, P, P, P, P, P, P, P, P],
    "propd_add_ln": [I, I, P, I, P, P, P, P, P, P],
    "propd_gelu": [I, L, P, P],
    "propd_residual_add": [I, L, P, P, P],
    "propd_gather_rows": [I, I, I, P, P, P, P],
    "propd_argmax_rows": [I, P, I, I, P, P, P],
    "propd_topk_rows": [I, I, I, I, P, P, P, P],
    "propd_kv_append": [I, I, I, I, I, P, I, P, P, P, P, P, P, P],
    "propd_attn_workspace_bytes": [I, I, I, I],
    "propd_tree_attention": [I, I, I, I, I, I, I, I, I, I, P, I, P, P, P, P, P, P, P, I, I, P, I, P, L, P],
    "propd_gemm_ws": [I, P, I, I, P, I, P, I, P, I, I, I, P],
    "propd_gemm_ws_ph": [I, P, I, I, P, I, P, I, P, I, I, I, "phases", P],
    "propd_ws_split_count": [I, I],
    "propd_gemm": [I, I, P, I, I, P, I, P, I, "epi", P],
    "propd_qkv_finish": [I, P, I, I, I, P, I, P, I, P, P, P, P, P, P, P],
    "propd_gelu_finish": [I, P, I, P, I, P, I, P],
    "propd_early_member": [I, I, I, I, I, P, P, P, P, P, P],
    "propd_row_lse": [I, P, I, I, P, P, c_double, P, P],
    "propd_early_prob_member": [I, I, I, I, c_double, P, P, P, P, P, P, P],
    "propd_verify_commit_ex": [I, I, I, I, I, I, I, I, I, L, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P,
                               "typical", P],
    "propd_prune_compact": [I, I, P, P, P, P, P, P, P, P, P, P, P],
    "propd_verify_commit": [I, I, I, I, I, I, I, I, I, L, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P],
    "propd_kv_compact": [I, I, I, I, I, I, I, L, P, P, P, P, P, P, P],
    "propd_seq_advance": [I, P, P, P, I, P],
    "propd_scatter_i32": [I, P, P, P, P],
    "propd_stats_replay_select": [I, I, I, P, c_double, P, P, P, P, P],
}
_RESTYPES = {"propd_last_error": ctypes.c_char_p, "propd_attn_workspace_bytes": c_int64}


PRO_NONE, PRO_LN, PRO_GELU, PRO_XGELU, PRO_XATTN = 0, 1, 2, 4, 5
ATTN_SCRATCH_LAST = 0x100  # propd_tree_attention impl flag (include/propd.h)
ATTN_QKV_F32 = 0x200  # propd_tree_attention: Q / tree K/V from the fp32 QKV accumulator
TAIL_NONE, TAIL_QKV = 0, 1


class WsPhases(ctypes.Structure):
    """propd_ws_phases (include/propd.h): in-kernel prologue / tail phases of a weight-streaming GEMM."""

    _fields_ = [("pro_mode", c_int), ("pro_src", P), ("pro_ld", c_int), ("pro_dst", P), ("pro_ldd", c_int),
                ("pro_cols", c_int), ("tail_mode", c_int), ("tail_q", P), ("tail_ldq", c_int), ("A", c_int),
                ("dh", c_int), ("Lmax", c_int), ("row_seq", P), ("row_node", P), ("seq_slot", P), ("seq_len", P),
                ("kcache", P), ("vcache", P), ("bar", P), ("zero_buf", P), ("zero_ld", c_int), ("zero_cols", c_int),
                ("attn_splits", c_int), ("attn_part", P)]


EPI_STORE, EPI_STORE_F32, EPI_ADD_F32, EPI_GELU, EPI_QKV = 0, 1, 2, 3, 4


class GemmEpi(ctypes.Structure):
    """propd_gemm_epi (include/propd.h): epilogue of a many-row projection."""

    _fields_ = [("mode", c_int), ("Y", P), ("ldy", c_int), ("A", c_int), ("dh", c_int), ("Lmax", c_int),
                ("row_seq", P), ("row_node", P), ("seq_slot", P), ("seq_len", P), ("kcache", P), ("vcache", P)]


class Typical(ctypes.Structure):
    """propd_typical (include/propd.h): typical-acceptance inputs of propd_verify_commit_ex."""

    _fields_ = [("row_logits", P), ("ld", c_int), ("row_stats", P), ("root_logits", P), ("root_ld", c_int),
                ("root_stats", P), ("log_eps", c_double), ("log_alpha", c_double), ("temperature", c_double),
                ("depth", P)]


class PropdError(RuntimeError):
    """A libpropd call returned a nonzero status."""


_lib = None


def load():
    """Load libpropd.so once; raise loudly when it is absent or stale."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the B200 kernels are not built "
            "(run __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        structs = {"phases": WsPhases, "typical": Typical, "epi": GemmEpi}
        fn.argtypes = [ctypes.POINTER(structs[a]) if isinstance(a, str) else a for a in argtypes]
        fn.restype = _RESTYPES.get(name, c_int)
    if lib.propd_abi_version() != ABI_VERSION:
        raise ImportError(f"libpropd ABI {lib.propd_abi_version()} != expected {ABI_VERSION}; rebuild")
    _lib = lib
    return lib


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point and raise on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise PropdError(f"{name}: {lib.propd_last_error().decode()}")
