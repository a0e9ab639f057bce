"""B200Backend: the reference's ModelBackend plugin API on sm_100a kernels.

Drop-in boundary (paths relative to /root/reference/pkg/src/treedecode/):
`ModelBackend` (backends.py:53-95) — vocab_size / num_layers /
draft_head_count, prefill, draft, next_argmax, forward_tree (with the
mid-stack prune callback), commit — with the reference's argument meaning and
ValueError messages (backends.py:98-108, 239-348).  A reference
`DecodeEngine(B200Backend(cfg), ...)` runs unchanged on it.

On top of that per-sequence API the backend offers the batched step used by
`paper_2402_13485_b200.engine.DecodeEngine`: one call runs draft (K4a),
tree materialisation (K1), the tree pass with on-device early pruning (K3),
greedy accept + KV compaction (K5) and the bonus pass for the whole batch.

Device state per sequence slot: KV cache [layer][slot][head][Lmax][dh],
committed length, root token (argmax of the last committed row's logits),
final LN'd hidden of that row (the draft heads' input).
"""

from __future__ import annotations

import math
import os
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import call, ptr
from .config import TinyTransformerConfig
from .planning import HeadPredictions
from .tree import TreeTemplate, mask_to_bits
from .weights import DeviceWeights, seeded_weights

MAX_TREE = 256  # ancestor bitsets of <= 4 x 64 bits per row


@dataclass
class DecodeState:
    """Per-sequence committed context + the last verified tree (backends.py:31-40)."""

    committed: list = field(default_factory=list)
    last_tree: tuple | None = None
    slot: int = -1
    _tree: dict | None = field(default=None, repr=False)
    _fin: object = field(default=None, repr=False, compare=False)

    @property
    def length(self) -> int:
        return len(self.committed)


@dataclass(frozen=True)
class TreeForward:
    """Survivor indices into the drafted tree, their argmax and logits (backends.py:43-50)."""

    survivors: tuple
    argmax: np.ndarray
    logits: np.ndarray | None


def validate_commit_path(mask: np.ndarray, accepted) -> None:
    """Each accepted node must see exactly the earlier accepted nodes (backends.py:98-108)."""
    seen: set = set()
    for idx in accepted:
        if not 0 <= idx < mask.shape[0]:
            raise ValueError(f"accepted index {idx} outside the verified tree")
        if set(np.nonzero(mask[idx])[0].tolist()) != seen | {idx}:
            raise ValueError("accepted path is not a contiguous root chain")
        seen.add(idx)


def subsample_mask(mask: np.ndarray, survivors) -> np.ndarray:
    """Ancestor-closed row/column gather with the reference's checks (token_tree.py:188-207)."""
    n = mask.shape[0]
    s = np.asarray(survivors, dtype=np.int64)
    if s.ndim != 1:
        raise ValueError("survivors must be a flat index list")
    if s.size and (s[0] < 0 or s[-1] >= n):
        raise ValueError("survivor index out of range")
    if np.any(np.diff(s) <= 0):
        raise ValueError("survivors must be strictly increasing")
    kept = np.zeros(n, dtype=bool)
    kept[s] = True
    for i in s:
        if not kept[mask[i]].all():
            raise ValueError(f"survivor {i}: an ancestor was dropped (set is not ancestor-closed)")
    return mask[np.ix_(s, s)].copy()


@dataclass
class Rows:
    """Device row tables of one pass: rows [row_off[b], row_off[b+1]) belong
    to batch entry b (sequence slot seq_slot[b]); row_node = tree node index."""

    M: int
    B: int
    seq_slot: object
    row_seq: object
    row_node: object
    row_off: object
    max_keys: int
    max_rows: int
    kv_keys: int = 0  # host count of K/V rows the pass streams (roofline accounting)
    live: object = None  # device int32 [1]: live row count when M is a padded capacity
    scratch_last: bool = False  # entry B-1 is the scratch slot holding the pad rows


@dataclass
class StepOutput:
    """Host copies of one batched tree step (engine bookkeeping)."""

    committed: np.ndarray  # [B, D+1] accepted tokens + bonus, -1 padded
    acc_len: np.ndarray  # [B]
    acc_surv: np.ndarray  # [B, D] accepted indices into the pruned tree
    surv_cnt: np.ndarray  # [B]
    ranks_dev: object  # device int8 [B, D] acceptance records
    ranks: np.ndarray | None = None  # host copy of the records (multi-rank step table)
    trace: dict | None = None
    order: np.ndarray | None = None  # selection order after this step's stats replay (single process)
    lcurve: np.ndarray | None = None


class B200Backend:
    """ModelBackend on B200 kernels.  dtype "fp32" is the parity mode (all
    GEMMs in true fp32, TF32 off); "bf16" is the performance mode."""

    def __init__(self, config: TinyTransformerConfig = TinyTransformerConfig(), *, dtype: str = "fp32",
                 device=None, weights: dict | None = None, random_device_init: bool = False,
                 max_slots: int = 16, max_tree: int = MAX_TREE, kv_len: int | None = None,
                 attn_impl: int = 0, use_graphs: bool = False, use_gws: bool = True) -> None:
        import torch

        self.lib = _lib.load()
        if not torch.cuda.is_available():
            raise RuntimeError("B200Backend needs a CUDA device; there is no CPU fallback")
        self.torch = torch
        self.config = config
        self.device = torch.device(device if device is not None else "cuda")
        if dtype not in ("fp32", "bf16"):
            raise ValueError("dtype must be 'fp32' or 'bf16'")
        self.dtype_name = dtype
        self.tdtype = torch.float32 if dtype == "fp32" else torch.bfloat16
        self.code = _lib.F32 if dtype == "fp32" else _lib.BF16
        if dtype == "fp32":
            torch.backends.cuda.matmul.allow_tf32 = False  # true fp32 GEMMs for parity
        self.attn_impl = attn_impl
        self.max_tree = int(max_tree)
        if self.max_tree > MAX_TREE:
            raise ValueError(f"max_tree must be <= {MAX_TREE}")
        cfg = config
        if random_device_init:
            self.w = DeviceWeights(cfg, self.tdtype, self.device)
        else:
            self.w = DeviceWeights(cfg, self.tdtype, self.device,
                                   host=weights if weights is not None else seeded_weights(cfg))
        self.A, self.dh, self.H, self.V = cfg.heads, cfg.head_dim, cfg.hidden, cfg.vocab
        # cache slots hold committed rows (< max_positions) plus one tree
        self.Lmax = (kv_len if kv_len is not None else cfg.max_positions) + self.max_tree
        self.max_slots = int(max_slots)
        self.scratch_slot = self.max_slots  # extra cache slot: pad rows of graph-captured passes
        dev, T = self.device, self.tdtype
        shape = (cfg.layers, self.max_slots + 1, self.A, self.Lmax, self.dh)
        # zero-filled: key blocks streamed by the tensor-core kernel may extend
        # past the live keys; masked keys get p = 0, and 0 * garbage-NaN would
        # poison the P.V product, so every cache row must hold a finite value
        self.kcache = torch.zeros(shape, device=dev, dtype=T)
        self.vcache = torch.zeros(shape, device=dev, dtype=T)
        self.n_slots = self.max_slots + 1
        self.layer_stride = self.n_slots * self.A * self.Lmax * self.dh
        self.seq_len = torch.zeros(self.n_slots, device=dev, dtype=torch.int32)
        self.root = torch.zeros(self.n_slots, device=dev, dtype=torch.int32)
        self.hidden = torch.zeros(self.n_slots, self.H, device=dev, dtype=T)
        self.last_logits = torch.zeros(self.n_slots, self.V, device=dev, dtype=torch.float32)
        self.use_graphs = bool(use_graphs)
        # weight-streaming tcgen05 projections for <= 128 rows (bf16 mode);
        # fp32 accumulator for QKV / W1 partial sums (kept zero between uses)
        self.use_gws = (dtype == "bf16") and use_gws and cfg.hidden % 128 == 0
        self._acc = torch.zeros(128, 4 * cfg.hidden, device=dev, dtype=torch.float32) if self.use_gws else None
        # in-kernel prologue/tail phases (LN, GELU, QKV finish) between the
        # weight-streaming projections: five launches per layer
        call("propd_prepare")
        # the phases meet at grid barriers: only when the split-K grids (<= 2
        # CTAs per SM) are confirmed co-resident on this device
        self.ws_phases = (self.use_gws and cfg.hidden <= 4096 and os.environ.get("PROPD_WS_PHASES", "1") != "0" and
                          self.lib.propd_gemm_ws_barrier_ctas() >= 2 * self.lib.propd_num_sms())
        if self.ws_phases:
            self._acc2 = torch.zeros(128, 4 * cfg.hidden, device=dev, dtype=torch.float32)
            self._bar = torch.zeros(32, device=dev, dtype=torch.int32)
        # W_2's GELU operand is converted per ring stage inside every CTA at
        # <= 20 live rows (measured: 2-3 us per launch faster than the
        # grid-barrier GELU phase at B=1); QKV then zeroes the W_1 accumulator
        # rows ahead (include/propd.h PROPD_PRO_XGELU)
        self.ws_conv = (self.ws_phases and os.environ.get("PROPD_WS_CONV", "1") != "0")  # "0": barrier GELU (A/B)
        # one-row passes (bonus / AR) at small batch: the attention runs inside
        # the QKV launch (one (row, head, key split) per CTA) and W_o combines
        # the partials (propd_ws_phases.attn_splits, PRO_XATTN)
        self.ws_fuse_attn = (self.ws_phases and self.dh == 128 and os.environ.get("PROPD_FUSE_ATTN", "1") != "0")
        # tree passes: the QKV tail folded into the transposed attention kernel (PROPD_ATTN_QKV_F32)
        self.ws_qkv_fold = (self.ws_phases and self.dh == 128 and os.environ.get("PROPD_QKV_FOLD", "1") != "0")
        if self.ws_fuse_attn:
            H = cfg.hidden
            self._qkv_ctas = (3 * H // 128) * self.lib.propd_ws_split_count(3 * H, H)
            self._attn_part = torch.empty(self._qkv_ctas * (4 + self.dh), device=dev, dtype=torch.float32)
        self.device_rows = os.environ.get("PROPD_DEVICE_ROWS", "1") != "0"  # sync-free post-prune pass ("0": host sync, A/B)
        # trees of > 128 rows: one survivor-count read per step selects the <= 128-row part B
        self.ws_split_sync = os.environ.get("PROPD_SPLIT_SYNC", "1") != "0"
        self._graphs: dict = {}
        self._templates: dict = {}
        self._host: dict = {}
        self._slot_static: dict = {}
        self._pool = torch.cuda.graph_pool_handle() if self.use_graphs else None
        self._cap_stream = None
        self._len = [0] * self.max_slots  # host mirror of seq_len
        self._free = list(range(self.max_slots - 1, -1, -1))
        self._ws = torch.empty(0, device=dev, dtype=torch.uint8)
        self._one_mask = torch.ones(1, device=dev, dtype=torch.int64)  # single-node template {0}
        self._keepalive: list = []
        self.launches = 0  # libpropd kernel launches issued (bench accounting)
        self.attn_timer = None  # list -> per-launch {ms, bytes, role, kind} of K2 / GEMM launches (bench)
        self.timeline = None  # device trace buffer while kernels record per-CTA timelines (bench)
        self.mark_only = False  # with attn_timer: record only the verify-pass markers
        self._capturing = False
        self._capture_events: list = []
        self._pending_events: list = []
        self._role = "eager"

    def plant_draft_head(self, d: int = 0) -> None:
        """Planted-acceptance harness: draft head d := the LM
        head, so its top-1 is the model's own next-token argmax.  With random
        weights acceptance is otherwise ~0 (out/run_tiny/summary.csv:2); with
        head 0 planted every step accepts the depth-1 node, which exercises
        the accept walk, the KV compaction and multi-token commits at scale."""
        V = self.V
        if not 0 <= d < self.config.draft_heads:
            raise ValueError("draft head index out of range")
        self.w.w_draft[:, d * V:(d + 1) * V].copy_(self.w.w_lm)

    # ------------------------------------------------------------------ API
    @property
    def vocab_size(self) -> int:
        return self.config.vocab

    @property
    def num_layers(self) -> int:
        return self.config.layers

    @property
    def draft_head_count(self) -> int:
        return self.config.draft_heads

    def stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def _call(self, name, *args):
        self.launches += 1
        call(name, *args)
        # temporaries created for this launch may be recycled only after it
        # has been issued (their blocks are then reused in stream order)
        self._keepalive.clear()

    # ------------------------------------------------------------- slots
    def _alloc_slot(self, state: DecodeState) -> int:
        if not self._free:
            raise RuntimeError(f"no free sequence slots (max_slots={self.max_slots})")
        slot = self._free.pop()
        state.slot = slot
        self._len[slot] = 0
        self.seq_len[slot] = 0
        state._fin = weakref.finalize(state, self._release, slot)
        return slot

    def _release(self, slot: int) -> None:
        self._free.append(slot)

    def release(self, state: DecodeState) -> None:
        """Return a finished sequence's cache slot to the pool."""
        fin = getattr(state, "_fin", None)
        if fin is not None and fin.alive:
            fin()
        state.slot = -1

    def _i32(self, values):
        """Device int32 copy of host values, kept alive until the next launch
        is issued (an inline `ptr(self._i32(a))` would otherwise free the
        block before the kernel reads it and alias the next temporary)."""
        t = self.torch.tensor(np.asarray(values, dtype=np.int32), device=self.device)
        self._keepalive.append(t)
        return t

    def _workspace(self, M: int, B: int) -> object:
        """Split-KV partials for one attention launch of the CUDA-core kernel
        (fp32 parity mode, head dims != 128).  The bf16 dh = 128 kernels
        combine their key splits through DSMEM and need none.  Under graph
        capture a fresh (graph-owned) buffer per launch; eagerly a grown
        shared one."""
        if self.tdtype == self.torch.bfloat16 and self.dh == 128:
            return None
        splits = min(64, -(-(4 * 148) // max(1, B * self.A)))
        if splits <= 1:
            return None
        need = int(self.lib.propd_attn_workspace_bytes(M, self.A, self.dh, splits))
        if self.use_graphs:
            return self.torch.empty(need, device=self.device, dtype=self.torch.uint8)
        if self._ws.numel() < need:
            self._ws = self.torch.empty(need, device=self.device, dtype=self.torch.uint8)
        return self._ws

    # ----------------------------------------------------------- layers
    def _run_layers(self, x, rt: Rows, l0: int, l1: int, mask, n_tmpl: int, W: int, pending=None):
        """Blocks l0..l1-1 over the rows of `rt` (backends.py:202-237).  Returns
        the last MLP output not yet added to the residual stream x."""
        if self.use_gws and rt.M <= 128:
            if self.ws_phases:
                return self._run_layers_phased(x, rt, l0, l1, mask, n_tmpl, W, pending)
            return self._run_layers_ws(x, rt, l0, l1, mask, n_tmpl, W, pending)
        torch, T, H, st = self.torch, self.tdtype, self.H, self.stream()
        M = rt.M
        ws = self._workspace(M, rt.B)
        live = ptr(rt.live)
        h = torch.empty(M, H, device=self.device, dtype=T)
        ctx = torch.empty(M, H, device=self.device, dtype=T)
        q = torch.empty(M, H, device=self.device, dtype=T)  # Q operand (K/V go straight to the cache)
        g = torch.empty(M, 4 * H, device=self.device, dtype=T)
        for l in range(l0, l1):
            self._call("propd_add_ln", self.code, M, live, H, ptr(x), ptr(pending), ptr(h), None, None, st)
            pending = None
            qkv_epi = _lib.GemmEpi(mode=_lib.EPI_QKV, Y=ptr(q), ldy=H, A=self.A, dh=self.dh, Lmax=self.Lmax,
                                   row_seq=ptr(rt.row_seq), row_node=ptr(rt.row_node), seq_slot=ptr(rt.seq_slot),
                                   seq_len=ptr(self.seq_len), kcache=ptr(self.kcache[l]), vcache=ptr(self.vcache[l]))
            self._gemm(M, live, 3 * H, H, h, self.w.wqkv[l], qkv_epi)
            self._attention(rt, q, l, mask, n_tmpl, W, ctx, ws)
            self._gemm(M, live, H, H, ctx, self.w.wo[l], _lib.GemmEpi(mode=_lib.EPI_ADD_F32, Y=ptr(x), ldy=H))
            self._call("propd_add_ln", self.code, M, live, H, ptr(x), None, ptr(h), None, None, st)
            self._gemm(M, live, 4 * H, H, h, self.w.w1[l], _lib.GemmEpi(mode=_lib.EPI_GELU, Y=ptr(g), ldy=4 * H))
            self._gemm(M, live, H, 4 * H, g, self.w.w2[l], _lib.GemmEpi(mode=_lib.EPI_ADD_F32, Y=ptr(x), ldy=H))
        return None

    def _gemm(self, M, live, N, K, X, W, epi) -> None:
        """Many-row projection epilogue(X[M,K] W[K,N]) (propd_gemm: tcgen05 in bf16,
        the CUDA-core SGEMM in the fp32 parity mode)."""
        st = self.stream()
        self._keepalive.append(epi)
        self._timed("gemm_tc", lambda: self._call("propd_gemm", self.code, M, live, N, K, ptr(X), K, ptr(W), N, epi,
                                                  st), M, K, N, epi.mode == _lib.EPI_ADD_F32)

    # ------------------------------------------------- per-launch timing (bench)
    def _timed(self, kind: str, launch, M: int = 0, K: int = 0, N: int = 0, acc: bool = False, shapes=None):
        """Run `launch` bracketed by CUDA events when the bench's kernel timer
        is on (kind "attn": K2; "gemm": weight-streaming projections [M,K] x
        [K,N], one or a chain given as `shapes` = [(K, N, accumulate), ...];
        "gemm_tc": the many-row tcgen05 / fp32 projections)."""
        if self.attn_timer is None or self.mark_only:
            return launch()
        ev0 = self._timing_event()
        ev0.record()
        out = launch()
        ev1 = self._timing_event()
        ev1.record()
        self._events_sink().append((ev0, ev1, self._role, M, kind, shapes or [(K, N, acc)]))
        return out

    def _mark(self, name: str) -> None:
        """Marker (an event node when captured) bracketing the verify pass:
        tree embed .. verify/commit, without draft and bonus.  Recorded in the
        per-launch timing region and in the marks-only region (`mark_only`:
        two event nodes per step, the PDL chain otherwise intact)."""
        if self.attn_timer is None:
            return
        ev = self._timing_event()
        ev.record()
        self._events_sink().append((ev, None, name, 0, "mark", None))

    def _timing_event(self):
        torch = self.torch
        if self._capturing:  # event-record nodes inside the graph
            return torch.cuda.Event(enable_timing=True, external=True)
        return torch.cuda.Event(enable_timing=True)

    def _events_sink(self) -> list:
        return self._capture_events if self._capturing else self._pending_events

    def _harvest(self, keys: dict) -> None:
        """After a step's synchronisation: per-launch time + algorithmic bytes.
        K2: K/V rows streamed + Q read + O written.  GEMM: weights + X read +
        fp32 Y written (read too when accumulating), for the live rows."""
        if self.attn_timer is None:
            self._pending_events.clear()
            return
        elt = 2 if self.tdtype != self.torch.float32 else 4
        begin = None
        for e0, e1, role, M, kind, shapes in self._pending_events:
            if kind == "mark":  # verify-pass markers: K1 .. K5 of the tree pass
                if role == "verify_begin":
                    begin = e0
                elif begin is not None:
                    self.attn_timer.append({"ms": begin.elapsed_time(e0), "role": "tree", "kind": "verify",
                                            "bytes": 0})
                    begin = None
                continue
            kv, rows = keys.get(role, (0, M))
            flops = 0
            if kind == "attn":
                nbytes = kv * 2 * self.H * elt + 2 * rows * self.H * elt
            else:
                rows = min(rows, M) if M else rows
                nbytes = sum(K * N * elt + rows * K * elt + rows * N * 4 * (2 if acc else 1) for K, N, acc in shapes)
                flops = sum(2 * rows * K * N for K, N, _ in shapes)
            self.attn_timer.append({"ms": e0.elapsed_time(e1), "role": role, "kind": kind, "bytes": nbytes,
                                    "flops": flops})
        self._pending_events.clear()

    def _gemm_ws(self, M, live, N, K, X, W, Y, ldy, acc: int, phases=None) -> None:
        """One weight-streaming projection Y (+)= X[M,K] W[K,N] (X, W row-major,
        contiguous), optionally with in-kernel prologue/tail phases."""
        st = self.stream()
        if phases is None:
            launch = lambda: self._call("propd_gemm_ws", M, live, N, K, ptr(X), K, ptr(W), N, ptr(Y), ldy, acc, 0, st)
        else:
            launch = lambda: self._call("propd_gemm_ws_ph", M, live, N, K, ptr(X), K, ptr(W), N, ptr(Y), ldy, acc, 0,
                                        phases, st)
        self._timed("gemm", launch, M, K, N, bool(acc))

    def _attention(self, rt: Rows, qkv, l: int, mask, n_tmpl: int, W: int, ctx, ws, acc=None) -> None:
        """K2 over the rows of `rt` for layer l (Q = columns [0, H) of qkv; with
        `acc`, Q and the tree rows' K/V come from the fp32 QKV accumulator and
        the kernel writes the tree rows into the cache: PROPD_ATTN_QKV_F32)."""
        H, M = self.H, rt.M
        ws_bytes = 0 if ws is None else ws.numel()
        impl = self.attn_impl | (_lib.ATTN_SCRATCH_LAST if rt.scratch_last else 0)
        if acc is not None:
            impl |= _lib.ATTN_QKV_F32
            qkv = acc
        self._timed("attn", lambda: self._call(
            "propd_tree_attention", self.code, impl, rt.B, M, self.A, self.dh, self.Lmax, self.n_slots,
            rt.max_rows, rt.max_keys, ptr(qkv), 3 * H if acc is not None else qkv.shape[1], ptr(self.kcache[l]), ptr(self.vcache[l]),
            ptr(rt.seq_slot), ptr(self.seq_len), ptr(rt.row_off), ptr(rt.row_node), ptr(mask), n_tmpl, W, ptr(ctx),
            H, ptr(ws), ws_bytes, self.stream()), M)

    def _run_layers_phased(self, x, rt: Rows, l0: int, l1: int, mask, n_tmpl: int, W: int, pending=None):
        """Blocks l0..l1-1 as five launches per layer (bf16, <= 128 rows):
        QKV GEMM [prologue LN(x), tail Q -> qkv, K/V -> cache] -> K2 -> W_o
        GEMM (adds into x) -> W_1 GEMM [prologue LN(x)] -> W_2 GEMM [prologue
        GELU(acc), adds into x].  The prologues/tails meet at in-kernel grid
        barriers while the weight ring keeps streaming (propd_ws_phases)."""
        torch, T, H = self.torch, self.tdtype, self.H
        self._flush(x, pending)
        M = rt.M
        ws = self._workspace(M, rt.B)
        acc1, acc2, live, bar = self._acc, self._acc2, ptr(rt.live), ptr(self._bar)
        h = torch.empty(M, H, device=self.device, dtype=T)
        ctx = torch.empty(M, H, device=self.device, dtype=T)
        qkv = torch.empty(M, 3 * H, device=self.device, dtype=T)
        g = torch.empty(M, 4 * H, device=self.device, dtype=T)
        ln = dict(pro_mode=_lib.PRO_LN, pro_src=ptr(x), pro_ld=H, pro_dst=ptr(h), pro_ldd=H, pro_cols=H, bar=bar)
        gelu = _lib.WsPhases(pro_mode=_lib.PRO_GELU, pro_src=ptr(acc2), pro_ld=4 * H, pro_dst=ptr(g), pro_ldd=4 * H,
                             pro_cols=4 * H, bar=bar)
        if self.ws_conv:  # converted per stage at <= 20 live rows, the barrier GELU phase into g above
            gelu = _lib.WsPhases(pro_mode=_lib.PRO_XGELU, pro_src=ptr(acc2), pro_ld=4 * H, pro_dst=ptr(g),
                                 pro_ldd=4 * H, pro_cols=4 * H, bar=bar)
        zero_acc2 = dict(zero_buf=ptr(acc2), zero_ld=4 * H, zero_cols=4 * H) if self.ws_conv else {}
        splits = 0  # fused one-row attention: key splits per (row, head)
        if rt.max_rows == 1 and mask is self._one_mask and rt.live is None:
            splits = self.fused_one_row_splits(M)
        fused = dict(attn_splits=splits, attn_part=ptr(self._attn_part)) if splits else {}
        if splits:
            wo_phases = _lib.WsPhases(pro_mode=_lib.PRO_XATTN, pro_src=ptr(self._attn_part), pro_cols=H, A=self.A,
                                      dh=self.dh, bar=bar, zero_buf=ptr(acc1), zero_ld=3 * H, zero_cols=3 * H,
                                      **fused)
        # tree passes on the transposed attention kernel: QKV has no tail (no
        # grid barrier, no bf16 Q / K/V pass); the attention reads Q and the tree
        # rows' K/V from the fp32 accumulator and writes those K/V rows into the
        # cache itself; W_o re-zeroes the accumulator (PROPD_ATTN_QKV_F32)
        fold = (not splits and self.ws_qkv_fold and mask is not None and self.dh == 128 and rt.max_rows <= 64
                and W <= 4 and (mask is not self._one_mask or rt.max_rows <= 4))
        wo_zero = _lib.WsPhases(bar=bar, zero_buf=ptr(acc1), zero_ld=3 * H, zero_cols=3 * H) if fold else None
        for l in range(l0, l1):
            # with the converting GELU, QKV zeroes the W_1 accumulator rows ahead (W_2 read them last)
            pro_qkv, pro_w1 = dict(ln, **zero_acc2), _lib.WsPhases(**ln)
            if fold:
                qkv_phases = _lib.WsPhases(**pro_qkv)
            else:
                qkv_phases = _lib.WsPhases(tail_mode=_lib.TAIL_QKV, tail_q=ptr(qkv), tail_ldq=3 * H, A=self.A,
                                           dh=self.dh, Lmax=self.Lmax, row_seq=ptr(rt.row_seq),
                                           row_node=ptr(rt.row_node), seq_slot=ptr(rt.seq_slot),
                                           seq_len=ptr(self.seq_len), kcache=ptr(self.kcache[l]),
                                           vcache=ptr(self.vcache[l]), **pro_qkv, **fused)
            self._gemm_ws(M, live, 3 * H, H, h, self.w.wqkv[l], acc1, 3 * H, 1, qkv_phases)
            if splits:  # attention inside the QKV launch, partials combined by W_o (which re-zeroes acc1)
                self._gemm_ws(M, live, H, H, ctx, self.w.wo[l], x, H, 1, wo_phases)
            elif fold:
                self._attention(rt, qkv, l, mask, n_tmpl, W, ctx, ws, acc=acc1)
                self._gemm_ws(M, live, H, H, ctx, self.w.wo[l], x, H, 1, wo_zero)
            else:
                self._attention(rt, qkv, l, mask, n_tmpl, W, ctx, ws)
                self._gemm_ws(M, live, H, H, ctx, self.w.wo[l], x, H, 1)
            self._gemm_ws(M, live, 4 * H, H, h, self.w.w1[l], acc2, 4 * H, 1, pro_w1)
            self._gemm_ws(M, live, H, 4 * H, g, self.w.w2[l], x, H, 1, gelu)
        return None

    def fused_one_row_splits(self, M: int) -> int:
        """Key splits of the attention fused into the QKV launch for a one-row
        pass (bonus / AR) over M sequences (0: the separate attention kernel)."""
        if not (self.ws_fuse_attn and 1 <= M <= 128):
            return 0
        splits = min(16, self._qkv_ctas // (M * self.A))
        return splits if splits >= 2 else 0

    def _run_layers_ws(self, x, rt: Rows, l0: int, l1: int, mask, n_tmpl: int, W: int, pending=None):
        """Same blocks with separate LN / finish kernels between the
        weight-streaming projections (H > 4096, or ws_phases off): QKV / W1
        accumulate into an fp32 scratch that the finish kernels turn into bf16
        operands (K/V straight into the cache, GELU on the way); W_o and W_2
        accumulate into the residual stream x."""
        torch, T, H, st = self.torch, self.tdtype, self.H, self.stream()
        M = rt.M
        ws = self._workspace(M, rt.B)
        acc, live = self._acc, ptr(rt.live)
        h = torch.empty(M, H, device=self.device, dtype=T)
        ctx = torch.empty(M, H, device=self.device, dtype=T)
        qkv = torch.empty(M, 3 * H, device=self.device, dtype=T)
        g = torch.empty(M, 4 * H, device=self.device, dtype=T)
        for l in range(l0, l1):
            self._call("propd_add_ln", self.code, M, live, H, ptr(x), ptr(pending), ptr(h), None, None, st)
            pending = None
            kc, vc = self.kcache[l], self.vcache[l]
            self._gemm_ws(M, live, 3 * H, H, h, self.w.wqkv[l], acc, 3 * H, 1)
            self._call("propd_qkv_finish", M, live, self.A, self.dh, self.Lmax, ptr(acc), 3 * H, ptr(qkv), 3 * H,
                       ptr(rt.row_seq), ptr(rt.row_node), ptr(rt.seq_slot), ptr(self.seq_len), ptr(kc), ptr(vc), st)
            self._attention(rt, qkv, l, mask, n_tmpl, W, ctx, ws)
            self._gemm_ws(M, live, H, H, ctx, self.w.wo[l], x, H, 1)
            self._call("propd_add_ln", self.code, M, live, H, ptr(x), None, ptr(h), None, None, st)
            self._gemm_ws(M, live, 4 * H, H, h, self.w.w1[l], acc, 4 * H, 1)
            self._call("propd_gelu_finish", M, live, 4 * H, ptr(acc), 4 * H, ptr(g), 4 * H, st)
            self._gemm_ws(M, live, H, 4 * H, g, self.w.w2[l], x, H, 1)
        return None

    def _proj_f32(self, X, Wt, N, live=None):
        """fp32 logits X @ Wt ([M,H] x [H,N]) for the LM / early / draft heads
        (rows >= *live, when given, are left unwritten)."""
        torch = self.torch
        M = X.shape[0]
        out = torch.empty(M, N, device=self.device, dtype=torch.float32)
        if self.use_gws and M <= 128 and N % 128 == 0 and X.dtype == torch.bfloat16:
            self._gemm_ws(M, ptr(live), N, self.H, X, Wt, out, N, 0)
        else:
            self._gemm(M, ptr(live), N, self.H, X, Wt, _lib.GemmEpi(mode=_lib.EPI_STORE_F32, Y=ptr(out), ldy=N))
        return out

    def _flush(self, x, pending):
        if pending is not None:
            self._call("propd_residual_add", self.code, x.numel(), ptr(x), ptr(pending), self.stream())

    def _lm_argmax(self, hfin, live=None):
        logits = self._proj_f32(hfin, self.w.w_lm, self.V, live)
        am = self.torch.empty(hfin.shape[0], device=self.device, dtype=self.torch.int32)
        self._call("propd_argmax_rows", hfin.shape[0], ptr(live), self.V, self.V, ptr(logits), ptr(am), self.stream())
        return logits, am

    # ------------------------------------------------- causal append (prefill/extend)
    def _extend(self, slots, token_lists, keep_logits: bool = True) -> None:
        """Causal forward of new committed rows for each slot; appends K/V,
        updates hidden/root/last_logits/seq_len (backends.py:239-259)."""
        torch, st = self.torch, self.stream()
        B = len(slots)
        lens = [len(t) for t in token_lists]
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        M = int(offs[-1])
        toks = np.concatenate([np.asarray(t, dtype=np.int32) for t in token_lists])
        pos = np.concatenate([np.arange(self._len[s], self._len[s] + n, dtype=np.int32) for s, n in zip(slots, lens)])
        node = np.concatenate([np.arange(n, dtype=np.int32) for n in lens])
        seq = np.repeat(np.arange(B, dtype=np.int32), lens)
        x = torch.empty(M, self.H, device=self.device, dtype=torch.float32)
        d_tok, d_pos = self._i32(toks), self._i32(pos)
        self._call("propd_embed_rows", self.code, M, self.H, ptr(d_tok), ptr(d_pos), ptr(self.w.emb),
                   ptr(self.w.pos), ptr(x), st)
        seq_slot = self._i32(slots)
        rt = Rows(M, B, seq_slot, self._i32(seq), self._i32(node), self._i32(offs),
                  max_keys=max(self._len[s] + n for s, n in zip(slots, lens)), max_rows=max(lens),
                  kv_keys=sum(self._len[s] + n for s, n in zip(slots, lens)))
        pending = self._run_layers(x, rt, 0, self.num_layers, None, max(lens), 0)
        last = self._i32(offs[1:] - 1)
        hfin = torch.empty(B, self.H, device=self.device, dtype=self.tdtype)
        self._call("propd_add_ln", self.code, B, None, self.H, ptr(x), ptr(pending), ptr(hfin), ptr(last), None, st)
        logits, am = self._lm_argmax(hfin)
        idx = seq_slot.long()
        self.hidden.index_copy_(0, idx, hfin)
        if keep_logits:
            self.last_logits.index_copy_(0, idx, logits)
        self._call("propd_scatter_i32", B, ptr(seq_slot), ptr(am), ptr(self.root), st)
        self._call("propd_seq_advance", B, ptr(seq_slot), ptr(self.seq_len), ptr(self._i32(lens)), 0, st)
        for s, n in zip(slots, lens):
            self._len[s] += n

    def _check_tokens(self, toks) -> None:
        a = np.asarray(toks, dtype=np.int64)
        if a.size == 0:
            raise ValueError("cannot extend with zero tokens")
        if np.any((a < 0) | (a >= self.config.vocab)):
            raise ValueError("token id outside the vocabulary")

    # ------------------------------------------------- ModelBackend methods
    def prefill(self, prompt) -> DecodeState:
        if len(prompt) == 0:
            raise ValueError("prompt must be non-empty")
        return self.prefill_batch([prompt])[0]

    def prefill_batch(self, prompts) -> list:
        """Ingest several prompts in one causal pass (engine.py:209 batched)."""
        for p in prompts:
            if len(p) == 0:
                raise ValueError("prompt must be non-empty")
            self._check_tokens(p)
            if len(p) > self.config.max_positions:
                raise ValueError("sequence exceeds max_positions")
        states = [DecodeState() for _ in prompts]
        slots = [self._alloc_slot(s) for s in states]
        self._extend(slots, [list(map(int, p)) for p in prompts])
        for s, p in zip(states, prompts):
            s.committed.extend(int(t) for t in p)
        return states

    def synthetic_states(self, B: int, L: int, seed: int = 0) -> list:
        """B sequences whose committed context is L random tokens and whose
        device state (K/V cache rows, last hidden, root token) is random
        synthetic data of the right shape — the bench's stand-in for a
        prefill of L tokens (decode-step cost does not depend on the values)."""
        torch = self.torch
        if L + 1 > self.config.max_positions:
            raise ValueError("sequence exceeds max_positions")
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        rng = np.random.default_rng(seed)
        states = []
        for _ in range(B):
            st = DecodeState(committed=rng.integers(0, self.V, size=L).tolist())
            slot = self._alloc_slot(st)
            for l in range(self.num_layers):
                for cache in (self.kcache, self.vcache):
                    blk = cache[l, slot, :, :L]
                    blk.copy_(torch.randn(blk.shape, device=self.device, generator=g, dtype=torch.float32))
            self.hidden[slot].copy_(torch.randn(self.H, device=self.device, generator=g))
            self.root[slot] = int(rng.integers(0, self.V))
            self.seq_len[slot] = L
            self._len[slot] = L
            states.append(st)
        return states

    def draft(self, state: DecodeState, k: int) -> HeadPredictions:
        """D draft heads on the last committed row, stable top-k (backends.py:274-285)."""
        if not 1 <= k <= self.config.vocab:
            raise ValueError("k outside 1..vocab")
        tok, val = self._draft_dev(self._i32([state.slot]), 1, k)
        return HeadPredictions(tok[0].cpu().numpy().astype(np.int64), val[0].cpu().numpy().astype(np.float64))

    def _draft_dev(self, seq_slot, B: int, k: int):
        if k > 1024:
            raise ValueError("draft top-k above 1024 is not supported by the device top-k")
        torch, D, V = self.torch, self.config.draft_heads, self.V
        hid = self.hidden.index_select(0, seq_slot.long())
        logits = self._proj_f32(hid, self.w.w_draft, D * V)
        tok = torch.empty(B, D, k, device=self.device, dtype=torch.int32)
        val = torch.empty(B, D, k, device=self.device, dtype=torch.float32)
        self._call("propd_topk_rows", B * D, V, V, k, ptr(logits), ptr(tok), ptr(val), self.stream())
        return tok, val

    def next_argmax(self, state: DecodeState) -> int:
        return int(self.root[state.slot].item())

    def last_logits_of(self, state: DecodeState) -> np.ndarray:
        """Logits of the last committed row (the reference's state.last_logits)."""
        return self.last_logits[state.slot].double().cpu().numpy()

    def forward_tree(self, state: DecodeState, tokens, positions, mask, *, prune_layer=None, early_topk=0,
                     prune_callback=None) -> TreeForward:
        """One masked pass over all tree nodes, optional mid-stack prune (backends.py:290-335)."""
        torch, st, cfg = self.torch, self.stream(), self.config
        toks = np.asarray(tokens, dtype=np.int64)
        pos = np.asarray(positions, dtype=np.int64)
        n = toks.size
        mask = np.asarray(mask)
        if mask.shape != (n, n) or pos.shape != (n,):
            raise ValueError("tokens, positions, and mask sizes disagree")
        if np.any((toks < 0) | (toks >= cfg.vocab)):
            raise ValueError("token id outside the vocabulary")
        if np.any(pos < state.length) or np.any(pos >= cfg.max_positions):
            raise ValueError("tree positions must follow the committed context")
        if prune_callback is not None:
            if prune_layer is None or not 1 <= prune_layer < cfg.layers:
                raise ValueError("prune layer must lie strictly inside the stack")
            if early_topk < 1:
                raise ValueError("early_topk must be positive when pruning")
        if n > self.max_tree:
            raise ValueError(f"tree of {n} nodes exceeds the backend's max_tree={self.max_tree}")
        vis = mask.astype(bool)
        slot, L = state.slot, self._len[state.slot]
        bits = torch.from_numpy(mask_to_bits(vis).view(np.int64)).to(self.device)
        W = bits.shape[1]
        x = torch.empty(n, self.H, device=self.device, dtype=torch.float32)
        self._call("propd_embed_rows", self.code, n, self.H, ptr(self._i32(toks)), ptr(self._i32(pos)),
                   ptr(self.w.emb), ptr(self.w.pos), ptr(x), st)
        seq_slot = self._i32([slot])
        rt = Rows(n, 1, seq_slot, self._i32(np.zeros(n)), self._i32(np.arange(n)), self._i32([0, n]),
                  max_keys=L + n, max_rows=n)
        keep = np.arange(n)
        if prune_callback is not None:
            pending = self._run_layers(x, rt, 0, prune_layer, bits, n, W)
            self._flush(x, pending)
            xe = x.to(self.tdtype)
            early = self._proj_f32(xe, self.w.w_early, self.V)
            kk = min(early_topk, cfg.vocab)
            if kk > 1024:
                raise ValueError("early top-K above 1024 is not supported by the device top-k")
            idx = torch.empty(n, kk, device=self.device, dtype=torch.int32)
            self._call("propd_topk_rows", n, self.V, self.V, kk, ptr(early), ptr(idx), None, st)
            lists = [list(map(int, r)) for r in idx.cpu().numpy()]
            surv = [int(s) for s in prune_callback(lists)]
            vis = subsample_mask(vis, surv)
            keep = np.asarray(surv, dtype=np.int64)
            S = keep.size
            x2 = torch.empty(S, self.H, device=self.device, dtype=torch.float32)
            self._call("propd_gather_rows", _lib.F32, S, self.H, ptr(x), ptr(self._i32(keep)), ptr(x2), st)
            x = x2
            rt = Rows(S, 1, seq_slot, self._i32(np.zeros(S)), self._i32(keep), self._i32([0, S]),
                      max_keys=L + n, max_rows=S)
            pending = self._run_layers(x, rt, prune_layer, cfg.layers, bits, n, W)
        else:
            pending = self._run_layers(x, rt, 0, cfg.layers, bits, n, W)
        S = rt.M
        hfin = torch.empty(S, self.H, device=self.device, dtype=self.tdtype)
        self._call("propd_add_ln", self.code, S, None, self.H, ptr(x), ptr(pending), ptr(hfin), None, None, st)
        logits, am = self._lm_argmax(hfin)
        state.last_tree = (toks[keep].copy(), vis.copy())
        state._tree = {"keep": keep, "positions": pos, "L": L}
        return TreeForward(tuple(int(i) for i in keep), am.cpu().numpy().astype(np.int64),
                           logits.double().cpu().numpy())

    def commit(self, state: DecodeState, accepted, bonus) -> None:
        """Append the accepted root chain + bonus (backends.py:337-348).  The
        accepted rows' K/V are moved into place from the tree pass (no
        recompute) whenever the chain sat at its commit positions."""
        acc = [int(a) for a in accepted]
        if acc:
            if state.last_tree is None:
                raise ValueError("commit with accepted nodes needs a preceding tree forward")
            ttoks, tmask = state.last_tree
            validate_commit_path(tmask, acc)
            new = [int(ttoks[i]) for i in acc] + [int(bonus)]
        else:
            new = [int(bonus)]
        self._check_tokens(new)
        slot, L = state.slot, self._len[state.slot]
        if L + len(new) > self.config.max_positions:
            raise ValueError("sequence exceeds max_positions")
        info = state._tree
        nodes = [int(info["keep"][a]) for a in acc] if (acc and info) else []
        fast = bool(acc) and info is not None and info["L"] == L and all(
            int(info["positions"][nd]) == L + j for j, nd in enumerate(nodes)) and all(
            b > a for a, b in zip(nodes, nodes[1:]))
        if fast:
            D = len(nodes)
            self._call("propd_kv_compact", self.code, 1, D, self.num_layers, self.A, self.dh, self.Lmax,
                       self.layer_stride, ptr(self._i32([slot])), ptr(self.seq_len), ptr(self._i32(nodes)),
                       ptr(self._i32([D])), ptr(self.kcache), ptr(self.vcache), self.stream())
            self._len[slot] += D
            self._extend([slot], [[int(bonus)]])
        else:
            self._extend([slot], [new])
        state.committed.extend(new)
        state.last_tree = None
        state._tree = None

    # ------------------------------------------------- batched steps
    # The batched step is organised as two device programs so that each can
    # be captured once in a CUDA graph and replayed (the per-step host cost
    # is then a few copies and two graph launches):
    #   part A  (B, tree)                    draft -> K1 -> layers 1..p
    #           [-> early head -> K3 membership + closure/compaction]
    #   part B  (B, tree, S_pad)             layers p+1..Ly on the S
    #           surviving rows padded to S_pad (pad rows form one extra
    #           scratch "sequence"), LM argmax, K5 accept + KV compaction,
    #           bonus pass.
    # Between them the host reads the survivor count S (the one mid-step sync).
    # Without pruning part A runs all layers and part B starts at the LM head.

    def _key_bound(self, need: int) -> int:
        """Key bound of an attention launch.  The kernels place their key-split
        boundaries from each sequence's device length, so a captured graph
        stays valid as sequences grow: graphs are launched with the cache
        capacity (no KV-length term in the graph keys), eager passes with the
        exact bound."""
        return self.Lmax if self.use_graphs else min(self.Lmax, need)

    def _slot_buf(self, B: int, slots):
        """Device int32 [B+1] = active slots + the scratch slot (pad rows)."""
        torch = self.torch
        host = np.asarray(list(slots) + [self.scratch_slot], dtype=np.int32)
        if not self.use_graphs:
            t = torch.from_numpy(host).to(self.device)
            self._keepalive.append(t)
            return t
        ent = self._slot_static.get(B)
        if ent is None:
            ent = self._slot_static[B] = [torch.empty(B + 1, device=self.device, dtype=torch.int32),
                                          torch.empty(B + 1, dtype=torch.int32).pin_memory(), None]
        buf, pin, last = ent
        key = host.tobytes()
        if key != last:  # the active set changed: stage it (graphs read the device buffer)
            self.torch.cuda.current_stream(self.device).synchronize()  # the pinned buffer may still be in flight
            pin.numpy()[:] = host
            buf.copy_(pin, non_blocking=True)
            ent[2] = key
        return buf

    def _graph_key(self, key) -> tuple:
        # graphs with K2 timing event nodes are kept apart from clean ones
        # (an event node between two kernels also breaks their PDL overlap)
        return key + (self.attn_timer is not None, self.mark_only, self.timeline is not None)

    def _capture(self, full_key, fn):
        """Capture fn into a CUDA graph under full_key (nothing is launched)."""
        torch = self.torch
        n0 = self.launches
        if self._cap_stream is None:
            self._cap_stream = torch.cuda.Stream(self.device)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        self._capturing, self._capture_events = True, []
        try:
            with torch.cuda.graph(g, pool=self._pool, stream=self._cap_stream):
                outs = fn()
        finally:
            self._capturing = False
        ent = self._graphs[full_key] = (g, outs, self.launches - n0, self._capture_events)
        self.launches = n0  # counted when replayed
        return ent

    def _run(self, key, fn):
        """Eager: run fn.  Graph mode: capture fn once per key, then replay."""
        if not self.use_graphs:
            return fn()
        full = self._graph_key(key)
        ent = self._graphs.get(full)
        if ent is None:
            ent = self._capture(full, fn)
        self.launches += ent[2]
        ent[0].replay()
        self._pending_events.extend(ent[3])
        return ent[1]

    def _precapture(self, key, fn) -> None:
        """Graph mode: capture fn for key now (not replayed), so a variant the
        step may switch to later is not captured inside a timed region."""
        if self.use_graphs and self._graph_key(key) not in self._graphs:
            self._capture(self._graph_key(key), fn)

    def _bonus_program(self, seq_slot, bonus, B: int, max_keys: int, keep_logits: bool = False):
        """One committed row per sequence at position seq_len (backends.py:239-259
        for the bonus token): K/V append, hidden/root update, seq_len += 1."""
        torch, st = self.torch, self.stream()
        dev = self.device
        x = torch.empty(B, self.H, device=dev, dtype=torch.float32)
        positions = torch.empty(B, device=dev, dtype=torch.int32)
        row_seq = torch.empty(B, device=dev, dtype=torch.int32)
        row_node = torch.empty(B, device=dev, dtype=torch.int32)
        row_off = torch.empty(B + 1, device=dev, dtype=torch.int32)
        self._call("propd_bonus_embed", self.code, B, self.H, ptr(bonus), ptr(seq_slot), ptr(self.seq_len),
                   ptr(self.w.emb), ptr(self.w.pos), ptr(x), ptr(positions), ptr(row_seq), ptr(row_node),
                   ptr(row_off), st)
        rt = Rows(B, B, seq_slot, row_seq, row_node, row_off, max_keys=max_keys, max_rows=1)
        role, self._role = self._role, "bonus"
        pending = self._run_layers(x, rt, 0, self.num_layers, self._one_mask, 1, 1)
        self._role = role
        hfin = torch.empty(B, self.H, device=dev, dtype=self.tdtype)
        self._call("propd_add_ln", self.code, B, None, self.H, ptr(x), ptr(pending), ptr(hfin), None, None, st)
        logits, am = self._lm_argmax(hfin)
        self.hidden.index_copy_(0, seq_slot.long(), hfin)
        if keep_logits:  # the next step's root row (typical acceptance)
            self.last_logits.index_copy_(0, seq_slot.long(), logits)
        self._call("propd_scatter_i32", B, ptr(seq_slot), ptr(am), ptr(self.root), st)
        self._call("propd_seq_advance", B, ptr(seq_slot), ptr(self.seq_len), None, 1, st)

    def step_autoregressive(self, states) -> np.ndarray:
        """AR iteration for a batch: commit each sequence's root argmax (engine.py:231-241)."""
        B = len(states)
        lens = [self._len[s.slot] for s in states]
        if max(lens) + 1 > self.config.max_positions:
            raise ValueError("sequence exceeds max_positions")
        slot_buf = self._slot_buf(B, [s.slot for s in states])
        kb = self._key_bound(max(lens) + 1)

        def program():
            seq_slot = slot_buf[:B]
            bonus = self.root.index_select(0, seq_slot.long())
            self._bonus_program(seq_slot, bonus, B, kb)
            return bonus

        self._role = "bonus"
        bonus = self._run(("ar", B), program)
        out = bonus.cpu().numpy()
        self._harvest({"bonus": (sum(lens) + B, B)})
        for s, t in zip(states, out):
            s.committed.append(int(t))
            self._len[s.slot] += 1
        return out

    def _part_a(self, B, tmpl, k, prune, slot_buf, kb):
        torch, st, cfg = self.torch, self.stream(), self.config
        n, D, H, V = len(tmpl), cfg.draft_heads, self.H, self.V
        dev = self.device
        td = tmpl.device(dev)
        seq_slot = slot_buf[:B]
        o = {}
        o["draft_tok"], o["draft_val"] = self._draft_dev(seq_slot, B, k)
        self._mark("verify_begin")
        M = B * n
        i32 = lambda m: torch.empty(m, device=dev, dtype=torch.int32)
        o["tokens"], o["positions"] = i32(M), i32(M)
        row_seq, row_node, row_off = i32(M), i32(M), i32(B + 1)
        x = torch.empty(M, H, device=dev, dtype=torch.float32)
        self._call("propd_tree_embed", self.code, B, n, D, k, H, ptr(td["depth"]), ptr(td["rank"]),
                   ptr(o["draft_tok"]), ptr(seq_slot), ptr(self.seq_len), ptr(self.w.emb), ptr(self.w.pos),
                   ptr(o["tokens"]), ptr(o["positions"]), ptr(x), ptr(row_seq), ptr(row_node), ptr(row_off), st)
        rt = Rows(M, B, seq_slot, row_seq, row_node, row_off, max_keys=kb, max_rows=n)
        p = prune.layer if prune is not None else cfg.layers
        pending = self._run_layers(x, rt, 0, p, td["mask"], n, tmpl.words)
        o["x"], o["rt"] = x, rt
        if prune is None:
            o["pending"] = pending
            return o
        self._flush(x, pending)
        Pn = len(tmpl.parent_nodes)
        member = torch.ones(M, device=dev, dtype=torch.uint8)
        if Pn > 0:
            par = td[("par_rows", B)]
            xp = torch.empty(B * Pn, H, device=dev, dtype=self.tdtype)
            self._call("propd_gather_rows", self.code, B * Pn, H, ptr(x), ptr(par), ptr(xp), st)
            early = self._proj_f32(xp, self.w.w_early, V)
            o["early"] = early
            if getattr(prune, "threshold", None) is not None:  # probability-based (marginal path probability)
                est = torch.empty(B * Pn, 2, device=dev, dtype=torch.float64)
                self._call("propd_row_lse", B * Pn, None, V, V, ptr(early), None, 1.0, ptr(est), st)
                self._call("propd_early_prob_member", B, n, Pn, V, math.log(prune.threshold), ptr(early), ptr(est),
                           ptr(td["parent"]), ptr(td["parent_slot"]), ptr(o["tokens"]), ptr(member), st)
            else:
                self._call("propd_early_member", B, n, Pn, V, min(prune.topk, V), ptr(early), ptr(td["parent"]),
                           ptr(td["parent_slot"]), ptr(o["tokens"]), ptr(member), st)
        o["alive"] = torch.empty(M, device=dev, dtype=torch.uint8)
        # compacted row tables sized for the worst case + pad entry
        cap = max(M, self._s_bucket(M))
        o["nrs"], o["nrn"], o["nsrc"], o["node_row"] = i32(cap), i32(cap), i32(cap), i32(M)
        o["noff"], o["surv_cnt"], o["total"] = i32(B + 2), i32(B), i32(1)
        self._call("propd_prune_compact", B, n, ptr(td["parent"]), ptr(member), ptr(o["alive"]), ptr(o["nrs"]),
                   ptr(o["nrn"]), ptr(o["nsrc"]), ptr(o["noff"]), ptr(o["node_row"]), ptr(o["surv_cnt"]),
                   ptr(o["total"]), st)
        return o

    def _part_b(self, B, tmpl, k, prune, slot_buf, kb, a, S_pad, device_rows=False, accept=None, row_cap=None):
        """Layers p+1..Ly over the survivors (row capacity S_pad; at most
        row_cap survivors per sequence, default the tree size), LM argmax, K5
        accept + KV compaction, bonus pass."""
        torch, st, cfg = self.torch, self.stream(), self.config
        n, D, H = len(tmpl), cfg.draft_heads, self.H
        dev = self.device
        td = tmpl.device(dev)
        seq_slot = slot_buf[:B]
        if prune is not None:
            # rows [S, S_pad) become the scratch sequence (batch entry B)
            self._call("propd_pad_rows", B, S_pad, 0 if device_rows else 1, ptr(a["total"]), ptr(a["nrs"]), ptr(a["nrn"]), ptr(a["nsrc"]),
                       ptr(a["noff"]), st)
            x = torch.empty(S_pad, H, device=dev, dtype=torch.float32)
            self._call("propd_gather_rows", 0, S_pad, H, ptr(a["x"]), ptr(a["nsrc"]), ptr(x), st)
            rt = Rows(S_pad, B + 1, slot_buf, a["nrs"], a["nrn"], a["noff"], max_keys=kb,
                      max_rows=min(n, row_cap) if row_cap else n, live=a["total"] if device_rows else None,
                      scratch_last=True)
            pending = self._run_layers(x, rt, prune.layer, cfg.layers, td["mask"], n, tmpl.words)
            alive, node_row = a["alive"], a["node_row"]
        else:
            x, pending, alive, node_row = a["x"], a["pending"], None, None
        S = x.shape[0]
        live = a["total"] if (prune is not None and device_rows) else None
        hfin = torch.empty(S, H, device=dev, dtype=self.tdtype)
        self._call("propd_add_ln", self.code, S, ptr(live), H, ptr(x), ptr(pending), ptr(hfin), None, None, st)
        row_logits, row_argmax = self._lm_argmax(hfin, live)
        i32 = lambda m: torch.empty(m, device=dev, dtype=torch.int32)
        o = {"acc_node": i32(B * D), "acc_surv": i32(B * D), "acc_len": i32(B), "bonus": i32(B),
             "committed": i32(B * (D + 1)), "ranks": torch.empty(B, D, device=dev, dtype=torch.int8),
             "row_argmax": row_argmax, "row_logits": row_logits,
             "root_before": self.root.index_select(0, seq_slot.long())}
        typ = None
        if accept is not None:  # typical acceptance: softmax statistics of the tree rows and the root rows
            eps, alpha, temp = accept
            V = self.V
            rst = torch.empty(S, 2, device=dev, dtype=torch.float64)
            self._call("propd_row_lse", S, ptr(live), V, V, ptr(row_logits), None, float(temp), ptr(rst), st)
            o["root_stats"] = torch.empty(B, 2, device=dev, dtype=torch.float64)
            self._call("propd_row_lse", B, None, V, V, ptr(self.last_logits), ptr(seq_slot), float(temp),
                       ptr(o["root_stats"]), st)
            o["row_stats"] = rst
            typ = _lib.Typical(row_logits=ptr(row_logits), ld=V, row_stats=ptr(rst), root_logits=ptr(self.last_logits),
                               root_ld=V, root_stats=ptr(o["root_stats"]), log_eps=math.log(eps),
                               log_alpha=math.log(alpha), temperature=float(temp), depth=ptr(td["depth"]))
        self._call("propd_verify_commit_ex", self.code, B, n, D, k, cfg.layers, self.A, self.dh, self.Lmax,
                   self.layer_stride, ptr(td["parent"]), ptr(a["tokens"]), ptr(alive), ptr(node_row),
                   ptr(row_argmax), ptr(self.root), ptr(a["draft_tok"]), ptr(seq_slot), ptr(self.seq_len),
                   ptr(self.kcache), ptr(self.vcache), ptr(o["acc_node"]), ptr(o["acc_surv"]), ptr(o["acc_len"]),
                   ptr(o["bonus"]), ptr(o["committed"]), ptr(o["ranks"]), typ, st)
        self._mark("verify_end")
        self._bonus_program(seq_slot, o["bonus"], B, kb, keep_logits=accept is not None)
        return o

    @staticmethod
    def _s_bucket(S: int) -> int:
        """Post-prune row counts padded to few distinct values (graph reuse):
        multiples of 8 up to 64, of 32 up to 512, then of 128."""
        step = 8 if S <= 64 else (32 if S <= 512 else 128)
        return ((S + step - 1) // step) * step

    def _host_bufs(self, B: int, D: int, G: int) -> dict:
        """Pinned host staging buffers for the per-step readback (per shape)."""
        key = (B, D, G)
        hb = self._host.get(key)
        if hb is None:
            torch = self.torch
            pin = lambda n, dt: torch.empty(n, dtype=dt).pin_memory()
            hb = self._host[key] = {"committed": pin(B * (D + 1), torch.int32), "acc_len": pin(B, torch.int32),
                                    "acc_surv": pin(B * D, torch.int32), "surv_cnt": pin(B, torch.int32),
                                    "ranks": pin(B * D, torch.int8),
                                    "order": pin(G, torch.int32), "lcurve": pin(G, torch.float64)}
        return hb

    def step_tree(self, states, tmpl: TreeTemplate, k: int, prune=None, trace: bool = False,
                  stats=None, accept=None) -> StepOutput:
        """One batched ProPD tree iteration on the device (engine.py:243-303):
        K4a draft -> K1 tree embed -> layers 1..p -> K3 early prune + row
        compaction -> layers p+1..Ly on survivors -> LM argmax -> K5 accept +
        KV compaction -> bonus pass.  One mid-step sync (survivor count)."""
        cfg = self.config
        B, n, D = len(states), len(tmpl), cfg.draft_heads
        if n > self.max_tree:
            raise ValueError(f"tree of {n} nodes exceeds the backend's max_tree={self.max_tree}")
        if tmpl.max_depth > D:
            raise ValueError("tree deeper than the draft heads")
        lens = [self._len[s.slot] for s in states]
        # forward_tree's bound (backends.py:308-309): positions L + depth - 1 < max_positions
        if max(lens) + tmpl.max_depth > cfg.max_positions:
            raise ValueError("tree positions must follow the committed context")
        if max(lens) + n > self.Lmax:  # tree rows live at cache slots L + node
            raise ValueError(f"KV cache capacity {self.Lmax} exceeded (kv_len too small for this tree)")
        # captured graphs hold the template's device pointers: the backend owns
        # one canonical template per tree shape for its whole lifetime
        tmpl = self._templates.setdefault(tmpl.paths, tmpl)
        slot_buf = self._slot_buf(B, [s.slot for s in states])
        kb = self._key_bound(max(lens) + n + D + 1)
        td = tmpl.device(self.device)  # host->device uploads happen outside any capture
        if ("par_rows", B) not in td:
            rows = (np.arange(B, dtype=np.int32)[:, None] * n + tmpl.parent_nodes[None, :]).reshape(-1)
            td[("par_rows", B)] = self.torch.from_numpy(np.ascontiguousarray(rows)).to(self.device)
        pkey = (prune.layer, prune.topk, getattr(prune, "threshold", None), accept) if prune is not None else (
            None, accept)
        self._role = "tree"
        a = self._run(("A", B, tmpl.paths, k, pkey), lambda: self._part_a(B, tmpl, k, prune, slot_buf, kb))
        # Layers > p run on the survivors.  Part B is launched for the padded
        # capacity and every kernel of it reads the live row count on the
        # device (weight-streaming GEMMs up to 128 rows, the many-row GEMM
        # above; rows past it are never written back), so a step has no
        # mid-step sync; device_rows=False sizes it on the host instead.
        cap = self._s_bucket(B * n)
        device_rows = prune is not None and self.device_rows
        row_cap = None  # survivors per sequence bound of part B (None: the tree size)
        if prune is None:
            S_pad = B * n
        elif device_rows:
            S_pad = cap
            if cap > 128 and self.use_gws and self.ws_split_sync:  # (at cap <= 128 the read costs what a tier gains)
                # survivors that fit the weight-streaming GEMMs (<= 128 rows: HBM-bound, ~1.5x the
                # many-row GEMM there; <= 64 rows: a deeper weight ring) get a smaller part-B
                # variant; one host read of the survivor count picks among the variants, all
                # captured up front
                # the same read gives the largest survivor count of a sequence: <= 32 lets the
                # tree attention run 32-row tiles (two CTAs per SM where one would need two waves)
                tiers = [t for t in (64, 128) if t < cap] + [cap]
                caps = [32, n] if n > 32 else [n]
                live, most = (int(v) for v in self.torch.stack([a["total"][0], a["surv_cnt"].max()]).cpu())
                S_pad = next(t for t in tiers if live <= t)
                row_cap = next(c for c in caps if most <= c)
                self._role = "tree_pruned"  # (role of the timing events the variants record)
                for other in tiers:
                    for oc in caps:
                        if (other, oc) != (S_pad, row_cap):
                            self._precapture(("B", B, tmpl.paths, k, pkey, other, device_rows, oc),
                                             lambda o=other, c=oc: self._part_b(B, tmpl, k, prune, slot_buf, kb, a,
                                                                                o, device_rows, accept, c))
        else:
            S = int(a["total"].item())  # mid-step sync: row count of layers > p
            S_pad = self._s_bucket(S) if self.use_graphs else S
        self._role = "tree_pruned"
        b = self._run(("B", B, tmpl.paths, k, pkey, S_pad, device_rows, row_cap),
                      lambda: self._part_b(B, tmpl, k, prune, slot_buf, kb, a, S_pad, device_rows, accept, row_cap))
        if stats is not None:  # single process: replay this batch's records right away (K4)
            P, counts, alpha, order_dev, lcurve_dev = stats
            self.stats_replay_select(b["ranks"], B, P, counts, alpha, order_dev, lcurve_dev)
        # one synchronisation for every host-visible result of the step
        hb = self._host_bufs(B, D, order_dev.numel() if stats is not None else 0)
        hb["committed"].copy_(b["committed"], non_blocking=True)
        hb["acc_len"].copy_(b["acc_len"], non_blocking=True)
        hb["acc_surv"].copy_(b["acc_surv"], non_blocking=True)
        hb["ranks"].copy_(b["ranks"].view(-1), non_blocking=True)
        if prune is not None:
            hb["surv_cnt"].copy_(a["surv_cnt"], non_blocking=True)
        if stats is not None:
            hb["order"].copy_(order_dev, non_blocking=True)
            hb["lcurve"].copy_(lcurve_dev, non_blocking=True)
        self.torch.cuda.current_stream(self.device).synchronize()
        out = StepOutput(hb["committed"].numpy().reshape(B, D + 1).copy(), hb["acc_len"].numpy().copy(),
                         hb["acc_surv"].numpy().reshape(B, D).copy(),
                         hb["surv_cnt"].numpy().copy() if prune is not None else np.full(B, n, dtype=np.int32),
                         b["ranks"], hb["ranks"].numpy().reshape(B, D).copy())
        if stats is not None:
            out.order = hb["order"].numpy().copy()
            out.lcurve = hb["lcurve"].numpy().copy()
        L0 = sum(lens)
        S_real = int(out.surv_cnt.sum())
        self._harvest({"tree": (L0 + B * n, B * n), "tree_pruned": (L0 + B * n, S_real),
                       "bonus": (L0 + int(out.acc_len.sum()) + B, B)})
        for L, acc in zip(lens, out.acc_len):
            # commit's bound (backends.py:247-248): the accepted chain + bonus
            # must fit; the reference raises from commit, so does this step
            if L + int(acc) + 1 > cfg.max_positions:
                raise ValueError("sequence exceeds max_positions")
        for s, row, acc in zip(states, out.committed, out.acc_len):
            new = [int(t) for t in row[: acc + 1]]
            s.committed.extend(new)
            self._len[s.slot] += len(new)
        if trace:
            alive = a["alive"].view(B, n).cpu().numpy() if prune is not None else np.ones((B, n), np.uint8)
            node_row = a["node_row"].view(B, n).cpu().numpy() if prune is not None else np.arange(B * n).reshape(B, n)
            out.trace = {"tokens": a["tokens"].view(B, n).cpu().numpy(),
                         "positions": a["positions"].view(B, n).cpu().numpy(),
                         "draft_tokens": a["draft_tok"].cpu().numpy(), "root": b["root_before"].cpu().numpy(),
                         "alive": alive, "node_row": node_row, "row_argmax": b["row_argmax"].cpu().numpy(),
                         # values behind the decisions (parity checks against the fp64 oracle)
                         "draft_val": a["draft_val"].cpu().numpy(),
                         "row_logits": b["row_logits"][:S_real].cpu().numpy(),
                         "early": a["early"].cpu().numpy() if "early" in a else None}
        return out

    def stats_replay_select(self, ranks_dev, S: int, P, counts, alpha, order, lcurve) -> None:
        """K4 on device: ordered fp64 replay of acceptance records + grid
        selection (acceptance.py:96-113, 186-206)."""
        D, k = P.shape
        self._call("propd_stats_replay_select", S, D, k, ptr(ranks_dev), float(alpha) if alpha is not None else -1.0,
                   ptr(P), ptr(counts), ptr(order), ptr(lcurve), self.stream())
