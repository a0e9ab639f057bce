"""Kernel-level parity of libpropd against numpy / torch fp32 references.

Integer and selection kernels must be bit-exact; attention is compared with
a plain torch fp32 implementation of the reference's masked softmax
attention (backends.py:216-233) at a stated tolerance:
  fp32 KV:  max |err| <= 2e-5 * max(1, |ref|_inf)
  bf16 KV:  max |err| <= 2e-2 * max(1, |ref|_inf)   (inputs rounded to bf16 first)
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import treedecode_port as op  # noqa: E402
from paper_2402_13485_b200 import _lib  # noqa: E402
from paper_2402_13485_b200._lib import call, ptr  # noqa: E402
from paper_2402_13485_b200.tree import TreeTemplate  # noqa: E402

DEV = torch.device("cuda:0")


def st():
    return torch.cuda.current_stream().cuda_stream


_KEEP = []  # inline temporaries must outlive the launch that reads them


def i32(a):
    t = torch.tensor(np.asarray(a, dtype=np.int32), device=DEV)
    _KEEP.append(t)
    return t


def keep(t):
    _KEEP.append(t)
    return t


# --------------------------------------------------------------- top-k / argmax
@pytest.mark.parametrize("V,k", [(256, 3), (256, 24), (32000, 64), (32000, 1), (1000, 1000), (64, 64), (50001, 7)])
def test_topk_matches_stable_argsort(V, k):
    rng = np.random.default_rng(V + k)
    x = rng.normal(size=(7, V)).astype(np.float32)
    x[1, : V // 2] = 0.0  # massive ties
    x[2] = np.round(x[2] * 4) / 4  # coarse ties
    x[3, 5] = -0.0
    x[3, 6] = 0.0
    dx = torch.from_numpy(x).to(DEV)
    idx = torch.empty(7, k, dtype=torch.int32, device=DEV)
    val = torch.empty(7, k, dtype=torch.float32, device=DEV)
    call("propd_topk_rows", 7, V, V, k, ptr(dx), ptr(idx), ptr(val), st())
    ref = np.argsort(-x, axis=1, kind="stable")[:, :k]
    assert np.array_equal(idx.cpu().numpy(), ref)
    assert np.array_equal(val.cpu().numpy(), np.take_along_axis(x, ref, axis=1))


@pytest.mark.parametrize("V,ld", [(32000, 32000), (32001, 32001), (5000, 5003), (3, 4)])
def test_argmax_first_max(V, ld):
    """First maximum (lowest index on ties), vectorised rows (ld % 4 == 0) and scalar ones."""
    rng = np.random.default_rng(V)
    x = rng.normal(size=(9, ld)).astype(np.float32)
    x[0, [min(5, V - 1), min(77, V - 1), V - 1]] = 100.0
    x[1] = 0.0
    x[2, V - 1] = 50.0
    x[3, :V] = np.round(x[3, :V])  # coarse ties
    x[:, V:] = 1e9  # padding past V is never a candidate
    dx = torch.from_numpy(x).to(DEV)
    out = torch.empty(9, dtype=torch.int32, device=DEV)
    call("propd_argmax_rows", 9, None, V, ld, ptr(dx), ptr(out), st())
    assert np.array_equal(out.cpu().numpy(), np.argmax(x[:, :V], axis=1))


def test_rows_dev_skips_padded_rows():
    """add_ln / argmax_rows with a device row count: rows < *rows_dev equal the
    unpadded result bit for bit, rows past it are not touched."""
    M, H, live = 8, 4096, 3
    torch.manual_seed(0)
    x0 = torch.randn(M, H, device=DEV)
    d = torch.randn(M, H, device=DEV).bfloat16()
    xa, xb = x0.clone(), x0.clone()
    oa = torch.full((M, H), 7.0, device=DEV).bfloat16()
    ob = oa.clone()
    call("propd_add_ln", 1, M, None, H, ptr(xa), ptr(d), ptr(oa), None, None, st())
    call("propd_add_ln", 1, M, ptr(i32([live])), H, ptr(xb), ptr(d), ptr(ob), None, None, st())
    assert torch.equal(xb[:live], xa[:live]) and torch.equal(ob[:live], oa[:live])
    assert torch.equal(xb[live:], x0[live:]) and bool((ob[live:] == 7.0).all())
    am = torch.full((M,), -5, dtype=torch.int32, device=DEV)
    call("propd_argmax_rows", M, ptr(i32([live])), H, H, ptr(xa), ptr(am), st())
    assert am[:live].tolist() == xa[:live].argmax(1).tolist() and am[live:].eq(-5).all()


# --------------------------------------------------------------- attention
def torch_tree_attention(q, kc, vc, slots, lens, row_off, row_node, mask_bool, A, dh):
    """Plain fp32 reference: for each row, softmax over cache keys [0,L) and
    visible tree keys L+j, scaled by 1/sqrt(dh) (backends.py:227-233)."""
    M = q.shape[0]
    out = torch.zeros(M, A * dh, dtype=torch.float32, device=q.device)
    B = len(slots)
    for b in range(B):
        L = lens[b]
        for m in range(row_off[b], row_off[b + 1]):
            node = row_node[m]
            if mask_bool is None:
                tree_vis = np.arange(node + 1)
            else:
                tree_vis = np.flatnonzero(mask_bool[node])
            keys = np.concatenate([np.arange(L), L + tree_vis])
            kk = torch.from_numpy(keys).to(q.device)
            for a in range(A):
                K = kc[slots[b], a, kk].float()
                Vv = vc[slots[b], a, kk].float()
                s = (K @ q[m, a * dh:(a + 1) * dh].float()) / np.sqrt(dh)
                p = torch.softmax(s, dim=0)
                out[m, a * dh:(a + 1) * dh] = p @ Vv
    return out


@pytest.mark.parametrize("dtype,dh,A,lens,paths,impl", [
    ("fp32", 16, 4, [6, 40, 1], "grid43", 1),
    ("fp32", 16, 2, [300], "full33", 1),
    ("fp32", 64, 2, [33, 129], "grid43", 1),
    ("bf16", 128, 4, [512, 77, 1000], "grid43", 1),
    ("bf16", 128, 2, [1500, 64], "full33", 1),
    ("bf16", 128, 4, [512, 77, 1000], "grid43", 0),
    ("bf16", 128, 3, [4096, 200], "full44", 0),
    ("bf16", 128, 2, [130, 2000, 7, 900], "chain", 0),
    # transposed kernel (<= 32 rows per sequence): cluster splits at B=1, ragged lengths, 32-node tree
    ("bf16", 128, 4, [512, 77, 1000], "grid43", 5),
    ("bf16", 128, 2, [130, 2000, 7, 900], "chain", 5),
    ("bf16", 128, 32, [1030], "grid43", 5),
    ("bf16", 128, 8, [1, 64, 4096], "grid48", 5),
    ("bf16", 128, 32, [3000], "grid48", 0),
    ("bf16", 128, 2, [1500, 64], "full33", 5),
    ("bf16", 128, 8, [1, 64, 4096], "grid416", 5),
    ("bf16", 128, 32, [1030], "grid416", 0),
])
def test_tree_attention_vs_torch(dtype, dh, A, lens, paths, impl):
    rng = np.random.default_rng(dh * 7 + len(lens))
    universe = {"grid43": op.grid_candidates(4, 3), "grid48": op.grid_candidates(4, 8),
                "grid416": op.grid_candidates(4, 16),
                "full33": op.complete_tree_paths(3, 3),
                "full44": op.complete_tree_paths(4, 4)[:200], "chain": [(1,) * d for d in range(1, 5)]}[paths]
    tmpl = TreeTemplate.from_paths(universe)
    n = len(tmpl)
    B = len(lens)
    slots = list(range(B))[::-1]
    H = A * dh
    Lmax = max(lens) + n + 8
    T = torch.float32 if dtype == "fp32" else torch.bfloat16
    code = _lib.F32 if dtype == "fp32" else _lib.BF16
    kc = torch.randn(B, A, Lmax, dh, device=DEV).to(T)
    vc = torch.randn(B, A, Lmax, dh, device=DEV).to(T)
    M = B * n
    qkv = torch.randn(M, 3 * H, device=DEV).to(T)
    row_off = [b * n for b in range(B + 1)]
    row_node = [i for b in range(B) for i in range(n)]
    seq_len = torch.zeros(B, dtype=torch.int32, device=DEV)
    for b, s in enumerate(slots):
        seq_len[s] = lens[b]
    out = torch.zeros(M, H, device=DEV, dtype=T)
    ws_bytes = _lib.load().propd_attn_workspace_bytes(M, A, dh, 0)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=DEV)
    mask = torch.from_numpy(tmpl.mask_bits.view(np.int64)).to(DEV)
    call("propd_tree_attention", code, impl, B, M, A, dh, Lmax, B, n, max(lens) + n, ptr(qkv), 3 * H, ptr(kc), ptr(vc),
         ptr(i32(slots)), ptr(seq_len), ptr(i32(row_off)), ptr(i32(row_node)), ptr(mask), n, tmpl.words, ptr(out), H,
         ptr(ws), ws_bytes, st())
    torch.cuda.synchronize()
    ref = torch_tree_attention(qkv[:, :H], kc, vc, slots, lens, row_off, row_node, tmpl.mask(), A, dh)
    err = (out.float() - ref).abs().max().item()
    tol = (2e-5 if dtype == "fp32" else 2e-2) * max(1.0, ref.abs().max().item())
    assert err <= tol, (err, tol)


@pytest.mark.parametrize("A,lens,rows", [(32, [1030], 1), (32, [5, 700, 64, 4096], 1), (8, [63, 65, 2000], 2),
                                          (32, [1], 1), (4, [300, 129], 3)])
def test_decode_attention_cluster_combine(A, lens, rows):
    """Streaming decode kernel (impl 3: <= 4 rows per sequence, key splits of one (sequence, head) reduced in a
    thread-block cluster) vs the torch fp32 reference; causal rows = the last `rows` tree nodes."""
    dh, B = 128, len(lens)
    H = A * dh
    n = rows
    Lmax = max(lens) + n + 8
    rng = np.random.default_rng(A + B)
    kc = torch.randn(B, A, Lmax, dh, device=DEV).bfloat16()
    vc = torch.randn(B, A, Lmax, dh, device=DEV).bfloat16()
    M = B * n
    qkv = (torch.randn(M, 3 * H, device=DEV) * 2).bfloat16()
    slots = list(range(B))
    row_off = [b * n for b in range(B + 1)]
    row_node = [i for b in range(B) for i in range(n)]
    out = torch.zeros(M, H, device=DEV, dtype=torch.bfloat16)
    call("propd_tree_attention", _lib.BF16, 3, B, M, A, dh, Lmax, B, n, max(lens) + n, ptr(qkv), 3 * H, ptr(kc),
         ptr(vc), ptr(i32(slots)), ptr(i32(lens)), ptr(i32(row_off)), ptr(i32(row_node)), None, n, 0, ptr(out), H,
         None, 0, st())
    torch.cuda.synchronize()
    ref = torch_tree_attention(qkv[:, :H], kc, vc, slots, lens, row_off, row_node, None, A, dh)
    err = (out.float() - ref).abs().max().item()
    assert err <= 2e-2 * max(1.0, ref.abs().max().item()), err
    del rng


@pytest.mark.parametrize("causal,big", [(False, False), (True, False), (False, True), (True, True)])
def test_tree_attention_tct_pruned_rows(causal, big):
    """Transposed kernel (impl 5) on a compacted survivor subset of a tree (rows = surviving nodes, row_node =
    their template indices), with the tree mask or causal (mask = NULL); big: a 200-node template (4 mask words)
    with up to 64 surviving rows (the 64-row variant)."""
    dh, A = 128, 4
    H = A * dh
    lens = [700, 3, 1500]
    B = len(lens)
    if big:
        tmpl = TreeTemplate.from_paths(op.complete_tree_paths(4, 4)[:200])
        keep = [list(range(0, 200, 4))[:50], [0, 3, 150, 199], list(range(5, 69))]
    else:
        tmpl = TreeTemplate.from_paths(op.grid_candidates(4, 8))
        keep = [[0, 1, 2, 8, 9, 20, 31], [0, 5], list(range(0, 32, 3))]
    n = len(tmpl)
    Lmax = max(lens) + n + 8
    kc = torch.randn(B, A, Lmax, dh, device=DEV).bfloat16()
    vc = torch.randn(B, A, Lmax, dh, device=DEV).bfloat16()
    row_off = [0]
    for k in keep:
        row_off.append(row_off[-1] + len(k))
    row_node = [i for k in keep for i in k]
    M = row_off[-1]
    qkv = torch.randn(M, 3 * H, device=DEV).bfloat16()
    slots = [2, 0, 1]
    seq_len = torch.zeros(B, dtype=torch.int32, device=DEV)
    for b, s_ in enumerate(slots):
        seq_len[s_] = lens[b]
    mask = None if causal else torch.from_numpy(tmpl.mask_bits.view(np.int64)).to(DEV)
    out = torch.zeros(M, H, device=DEV, dtype=torch.bfloat16)
    call("propd_tree_attention", _lib.BF16, 5, B, M, A, dh, Lmax, B, max(len(k) for k in keep), max(lens) + n,
         ptr(qkv), 3 * H, ptr(kc), ptr(vc), ptr(i32(slots)), ptr(seq_len), ptr(i32(row_off)), ptr(i32(row_node)),
         None if causal else ptr(mask), n, tmpl.words, ptr(out), H, None, 0, st())
    torch.cuda.synchronize()
    ref = torch_tree_attention(qkv[:, :H], kc, vc, slots, lens, row_off, row_node, None if causal else tmpl.mask(),
                               A, dh)
    err = (out.float() - ref).abs().max().item()
    assert err <= 2e-2 * max(1.0, ref.abs().max().item()), err


def test_tree_attention_causal_and_pruned_rows():
    """Causal new rows (mask=NULL) and a compacted subset of tree rows."""
    dh, A, B = 16, 2, 2
    H = A * dh
    lens = [5, 9]
    n = 10
    Lmax = 32
    kc = torch.randn(B, A, Lmax, dh, device=DEV)
    vc = torch.randn(B, A, Lmax, dh, device=DEV)
    # causal: rows = nodes 0..n-1 of each seq
    M = B * n
    qkv = torch.randn(M, 3 * H, device=DEV)
    row_off = [0, n, 2 * n]
    row_node = list(range(n)) * 2
    seq_len = i32(lens)
    out = torch.zeros(M, H, device=DEV)
    call("propd_tree_attention", _lib.F32, 1, B, M, A, dh, Lmax, B, n, max(lens) + n, ptr(qkv), 3 * H, ptr(kc), ptr(vc),
         ptr(i32([0, 1])), ptr(seq_len), ptr(i32(row_off)), ptr(i32(row_node)), None, n, 0, ptr(out), H, None, 0, st())
    ref = torch_tree_attention(qkv[:, :H], kc, vc, [0, 1], lens, row_off, row_node, None, A, dh)
    assert (out - ref).abs().max().item() <= 2e-5 * max(1.0, ref.abs().max().item())
    # pruned: keep an ancestor-closed subset of the grid tree rows
    tmpl = TreeTemplate.from_paths(op.grid_candidates(4, 3))
    keep = [0, 1, 2, 3, 5, 6]
    M = B * len(keep)
    qkv = torch.randn(M, 3 * H, device=DEV)
    row_off = [0, len(keep), 2 * len(keep)]
    row_node = keep * 2
    out = torch.zeros(M, H, device=DEV)
    mask = torch.from_numpy(tmpl.mask_bits.view(np.int64)).to(DEV)
    call("propd_tree_attention", _lib.F32, 1, B, M, A, dh, Lmax, B, 12, max(lens) + 12, ptr(qkv), 3 * H, ptr(kc), ptr(vc),
         ptr(i32([0, 1])), ptr(seq_len), ptr(i32(row_off)), ptr(i32(row_node)), ptr(mask), 12, 1, ptr(out), H, None, 0,
         st())
    ref = torch_tree_attention(qkv[:, :H], kc, vc, [0, 1], lens, row_off, row_node, tmpl.mask(), A, dh)
    assert (out - ref).abs().max().item() <= 2e-5 * max(1.0, ref.abs().max().item())


# --------------------------------------------------------------- K3 prune
def test_early_member_and_compaction_match_prune():
    rng = np.random.default_rng(5)
    V, topk = 300, 7
    paths = op.complete_tree_paths(3, 3)
    sel = op.grid_candidates(3, 3) + ((1, 2), (2,), (2, 1), (2, 1, 3), (1, 2, 2))
    sel = tuple(dict.fromkeys(p for p in sel if p in set(paths)))
    tmpl = TreeTemplate.from_paths(sel)
    n = len(tmpl)
    B = 5
    Pn = len(tmpl.parent_nodes)
    early = np.round(rng.normal(size=(B * Pn, V)).astype(np.float32) * 3) / 3  # ties
    tokens = rng.integers(0, V, size=(B, n)).astype(np.int32)
    # make some children land inside their parent's top-K
    for b in range(B):
        for i in range(n):
            par = tmpl.parent[i]
            if par >= 0 and rng.random() < 0.6:
                row = early[b * Pn + tmpl.parent_slot[par]]
                order = np.argsort(-row, kind="stable")
                tokens[b, i] = order[rng.integers(0, topk + 2)]
    td = tmpl.device(DEV)
    member = torch.empty(B * n, dtype=torch.uint8, device=DEV)
    d_early = torch.from_numpy(early).to(DEV)
    d_tok = torch.from_numpy(tokens.reshape(-1)).to(DEV)
    call("propd_early_member", B, n, Pn, V, topk, ptr(d_early), ptr(td["parent"]), ptr(td["parent_slot"]),
         ptr(d_tok), ptr(member), st())
    alive = torch.empty(B * n, dtype=torch.uint8, device=DEV)
    z = lambda m: torch.empty(m, dtype=torch.int32, device=DEV)
    nrs, nrn, nsrc, node_row, noff, cnt, total = z(B * n), z(B * n), z(B * n), z(B * n), z(B + 1), z(B), z(1)
    call("propd_prune_compact", B, n, ptr(td["parent"]), ptr(member), ptr(alive), ptr(nrs), ptr(nrn), ptr(nsrc),
         ptr(noff), ptr(node_row), ptr(cnt), ptr(total), st())
    alive = alive.cpu().numpy().reshape(B, n)
    off = 0
    for b in range(B):
        lists = []
        for i in range(n):
            if i in set(tmpl.parent_nodes.tolist()):
                row = early[b * Pn + tmpl.parent_slot[i]]
                lists.append(np.argsort(-row, kind="stable")[:topk].tolist())
            else:
                lists.append([])
        preds = op.Preds(np.arange(100, 100 + 9).reshape(3, 3), -np.tile(np.arange(3.0), (3, 1)))
        tree = op.build_tree(preds, sel, root_token=0)
        tree = op.Tree(tuple(op.Node(int(tokens[b, i]), nd.parent, nd.depth, nd.rank) for i, nd in
                             enumerate(tree.nodes)), 0)
        surv, _ = op.prune(tree, lists, op.PruneCfg(layer=1, topk=topk))
        assert np.flatnonzero(alive[b]).tolist() == list(surv)
        assert cnt[b].item() == len(surv)
        assert nrn[off: off + len(surv)].cpu().tolist() == list(surv)
        off += len(surv)
    assert total.item() == off


# --------------------------------------------------------------- K4 stats
@pytest.mark.parametrize("D,k,alpha", [(4, 3, 0.05), (4, 3, None), (3, 16, 0.05), (4, 64, None)])
def test_stats_replay_select_bit_exact(D, k, alpha):
    rng = np.random.default_rng(D * k)
    stats = op.Stats(D, k, alpha=alpha)
    P = torch.tensor(stats.P, dtype=torch.float64, device=DEV)
    counts = torch.zeros(D, dtype=torch.int64, device=DEV)
    order = torch.empty(D * k, dtype=torch.int32, device=DEV)
    lcurve = torch.empty(D * k, dtype=torch.float64, device=DEV)
    for step in range(6):
        S = int(rng.integers(1, 9))
        ranks = np.zeros((S, D), dtype=np.int8)
        for s in range(S):
            known = int(rng.integers(1, D + 1))
            toks = np.arange(D * k).reshape(D, k) + 1000
            preds = op.Preds(toks, -np.tile(np.arange(float(k)), (D, 1)))
            realized = {}
            for d in range(1, known + 1):
                r = int(rng.integers(0, k + 2))  # 0 or >k means miss
                tok = int(toks[d - 1, r - 1]) if 1 <= r <= k else 7
                realized[d] = tok
                ranks[s, d - 1] = r if 1 <= r <= k else -1
            stats.update(realized, preds)
        call("propd_stats_replay_select", S, D, k, ptr(keep(torch.from_numpy(ranks).to(DEV))),
             float(alpha) if alpha is not None else -1.0, ptr(P), ptr(counts), ptr(order), ptr(lcurve), st())
        assert np.array_equal(P.cpu().numpy(), stats.P)  # bit-exact fp64
        sel = op.select_best_nodes(stats, list(range(1, D * k + 1)))
        universe = op.grid_candidates(D, k)
        got = [universe[c] for c in order.cpu().numpy()]
        assert tuple(got) == sel[D * k][0]
        assert lcurve.cpu().numpy().tolist() == [sel[s][1] for s in range(1, D * k + 1)]


# --------------------------------------------------------------- K5 verify + compaction
def test_verify_commit_walk_and_compaction():
    rng = np.random.default_rng(11)
    D, k = 3, 3
    sel = op.complete_tree_paths(3, 3)[:20]
    sel = [p for p in sel if len(p) == 1 or p[:-1] in set(sel)]
    tmpl = TreeTemplate.from_paths(sel)
    n, B = len(tmpl), 6
    layers, A, dh, Lmax = 2, 2, 16, 64
    lens = rng.integers(3, 20, size=B)
    draft = rng.permutation(50)[: D * k].reshape(D, k)
    draft_tok = np.stack([rng.permutation(60)[: D * k].reshape(D, k) for _ in range(B)]).astype(np.int32)
    tokens = np.stack([[draft_tok[b, tmpl.depth[i] - 1, tmpl.rank[i] - 1] for i in range(n)] for b in range(B)])
    alive = (rng.random((B, n)) < 0.8)
    for b in range(B):
        for i in range(n):
            if tmpl.parent[i] >= 0 and not alive[b, tmpl.parent[i]]:
                alive[b, i] = False
    node_row = np.full((B, n), -1, dtype=np.int32)
    r = 0
    for b in range(B):
        for i in range(n):
            if alive[b, i]:
                node_row[b, i] = r
                r += 1
    # argmax per surviving row: often follow a chain so that something is accepted
    row_argmax = rng.integers(0, 60, size=r).astype(np.int32)
    root = np.zeros(B, dtype=np.int32)
    for b in range(B):
        root[b] = tokens[b, 0] if rng.random() < 0.8 else 59
        for i in range(n):
            if alive[b, i] and rng.random() < 0.5:
                kids = [c for c in range(n) if tmpl.parent[c] == i and alive[b, c]]
                if kids:
                    row_argmax[node_row[b, i]] = tokens[b, kids[-1]]
    kc = torch.randn(layers, B, A, Lmax, dh, device=DEV)
    vc = torch.randn(layers, B, A, Lmax, dh, device=DEV)
    kc0, vc0 = kc.clone(), vc.clone()
    td = tmpl.device(DEV)
    seq_len = i32(lens)
    z = lambda m: torch.empty(m, dtype=torch.int32, device=DEV)
    acc_node, acc_surv, acc_len, bonus, committed = z(B * D), z(B * D), z(B), z(B), z(B * (D + 1))
    ranks = torch.empty(B, D, dtype=torch.int8, device=DEV)
    call("propd_verify_commit", _lib.F32, B, n, D, k, layers, A, dh, Lmax, B * A * Lmax * dh, ptr(td["parent"]),
         ptr(i32(tokens.reshape(-1))), ptr(keep(torch.from_numpy(alive.astype(np.uint8).reshape(-1)).to(DEV))),
         ptr(i32(node_row.reshape(-1))), ptr(i32(row_argmax)), ptr(i32(root)), ptr(i32(draft_tok.reshape(-1))),
         ptr(i32(np.arange(B))), ptr(seq_len), ptr(kc), ptr(vc), ptr(acc_node), ptr(acc_surv), ptr(acc_len),
         ptr(bonus), ptr(committed), ptr(ranks), st())
    acc_node, acc_surv = acc_node.cpu().numpy().reshape(B, D), acc_surv.cpu().numpy().reshape(B, D)
    acc_len, bonus = acc_len.cpu().numpy(), bonus.cpu().numpy()
    committed, ranks = committed.cpu().numpy().reshape(B, D + 1), ranks.cpu().numpy()
    for b in range(B):
        preds = op.Preds(draft_tok[b], -np.tile(np.arange(float(k)), (D, 1)))
        tree = op.build_tree(preds, sel, root_token=0)
        surv = np.flatnonzero(alive[b]).tolist()
        vtree = op.restrict(tree, surv)
        am = [row_argmax[node_row[b, i]] for i in surv]
        acc, bon = op.verify(vtree, am, int(root[b]))
        assert acc_len[b] == len(acc) and bonus[b] == bon
        assert acc_surv[b, : len(acc)].tolist() == list(acc)
        nodes = [surv[a] for a in acc]
        assert acc_node[b, : len(acc)].tolist() == nodes
        newly = [int(tokens[b, nd]) for nd in nodes] + [bon]
        assert committed[b, : len(newly)].tolist() == newly
        for d in range(D):
            exp = 0
            if d < min(len(newly), D):
                rk = preds.rank_of(d + 1, newly[d])
                exp = rk if rk is not None else -1
            assert ranks[b, d] == exp
        assert seq_len[b].item() == lens[b] + len(acc)
        L = int(lens[b])
        for j, nd in enumerate(nodes):
            assert torch.equal(kc[:, b, :, L + j], kc0[:, b, :, L + nd])
            assert torch.equal(vc[:, b, :, L + j], vc0[:, b, :, L + nd])
        assert torch.equal(kc[:, b, :, :L], kc0[:, b, :, :L])


# --------------------------------------------------------------- weight-streaming GEMM
@pytest.mark.parametrize("M,N,K,acc", [(1, 128, 64, 0), (16, 12288, 4096, 1), (37, 4096, 4096, 1),
                                       (64, 4096, 16384, 1), (100, 32000, 4096, 0), (128, 16384, 4096, 1),
                                       (5, 256, 1024, 1)])
def test_gemm_ws_matches_fp32_reference(M, N, K, acc):
    """bf16 inputs, fp32 accumulation: |err| <= 2e-3 * sqrt(K) * max|x| * max|w| scale (fp32 rounding of
    the split-K reduction order); checked as relative to the reference's magnitude."""
    torch.manual_seed(M + N)
    X = torch.randn(M, K, device=DEV).bfloat16()
    Wt = (torch.randn(K, N, device=DEV) / K ** 0.5).bfloat16()
    ref = X.float() @ Wt.float()
    base = torch.randn(M, N, device=DEV) if acc else torch.full((M, N), float("nan"), device=DEV)
    Y = base.clone()
    call("propd_gemm_ws", M, None, N, K, ptr(X), K, ptr(Wt), N, ptr(Y), N, acc, 0, st())
    torch.cuda.synchronize()
    want = ref + (base if acc else 0)
    err = (Y - want).abs().max().item()
    assert err <= 1e-3 * max(1.0, want.abs().max().item()), err


@pytest.mark.parametrize("live", [0, 1, 13, 37, 64])
def test_gemm_ws_device_row_count(live):
    """rows_dev: rows < min(M, *rows_dev) are computed, the rest of Y is left untouched (bit-exact)."""
    M, N, K = 37, 4096, 1024
    torch.manual_seed(live)
    X = torch.randn(M, K, device=DEV).bfloat16()
    Wt = (torch.randn(K, N, device=DEV) / K ** 0.5).bfloat16()
    ref = X.float() @ Wt.float()
    for acc in (0, 1):
        base = torch.randn(M, N, device=DEV)
        Y = base.clone()
        call("propd_gemm_ws", M, ptr(i32([live])), N, K, ptr(X), K, ptr(Wt), N, ptr(Y), N, acc, 0, st())
        torch.cuda.synchronize()
        r = min(M, live)
        want = ref[:r] + (base[:r] if acc else 0)
        assert (Y[:r] - want).abs().max().item() <= 1e-3 * max(1.0, want.abs().max().item()) if r else True
        assert torch.equal(Y[r:], base[r:])


def test_qkv_and_gelu_finish():
    A, dh, M, Lmax = 4, 128, 7, 64
    H = A * dh
    acc = torch.randn(M, 3 * H, device=DEV)
    acc0 = acc.clone()
    qkv = torch.empty(M, 3 * H, device=DEV, dtype=torch.bfloat16)
    kc = torch.zeros(2, A, Lmax, dh, device=DEV, dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    row_seq, row_node = i32([0] * 3 + [1] * 4), i32([0, 1, 2, 0, 1, 2, 3])
    seq_slot, seq_len = i32([1, 0]), i32([5, 9])
    call("propd_qkv_finish", M, None, A, dh, Lmax, ptr(acc), 3 * H, ptr(qkv), 3 * H, ptr(row_seq), ptr(row_node),
         ptr(seq_slot), ptr(seq_len), ptr(kc), ptr(vc), st())
    torch.cuda.synchronize()
    assert torch.equal(qkv, acc0.bfloat16()) and acc.abs().max().item() == 0.0
    lens = {0: 5, 1: 9}  # seq_len is indexed by slot
    for m, (b, nd) in enumerate(zip([0] * 3 + [1] * 4, [0, 1, 2, 0, 1, 2, 3])):
        slot = [1, 0][b]
        t = lens[slot] + nd
        assert torch.equal(kc[slot, :, t].reshape(-1), acc0[m, H:2 * H].bfloat16())
        assert torch.equal(vc[slot, :, t].reshape(-1), acc0[m, 2 * H:].bfloat16())
    g_acc = torch.randn(M, 4 * H, device=DEV)
    g0 = g_acc.clone()
    out = torch.empty(M, 4 * H, device=DEV, dtype=torch.bfloat16)
    call("propd_gelu_finish", M, None, 4 * H, ptr(g_acc), 4 * H, ptr(out), 4 * H, st())
    torch.cuda.synchronize()
    ref = torch.nn.functional.gelu(g0, approximate="tanh")
    assert (out.float() - ref).abs().max().item() <= 1e-2 * max(1.0, ref.abs().max().item())
    assert g_acc.abs().max().item() == 0.0


# --------------------------------------------------------------- in-kernel GEMM phases
@pytest.mark.parametrize("rows,live,offset", [(1, None, 0.0), (16, None, 0.0), (40, 23, 0.0), (128, None, 0.0),
                                              (20, None, 2.0), (128, 32, 0.0), (128, 17, 0.0), (96, 30, 0.0)])
def test_phased_layers_match_separate_kernels(rows, live, offset):
    """Layer stack with the LN / GELU prologues and the QKV tail inside the weight-streaming GEMMs
    (propd_gemm_ws_ph: grid-barrier prologues, and the GELU operand converted per ring stage inside every
    CTA) == the same stack with separate add_ln / finish kernels: residual
    stream and the K/V rows written to the cache within bf16 rounding (the paths differ only in where the
    bf16 conversions happen; `offset` shifts every row mean)."""
    from paper_2402_13485_b200 import B200Backend, TinyTransformerConfig
    from paper_2402_13485_b200.backend import Rows

    cfg = TinyTransformerConfig(layers=3, hidden=1024, heads=8, vocab=1024, draft_heads=2, max_positions=600, seed=1)
    be = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=3, max_tree=rows)
    states = be.synthetic_states(2, 300, seed=3)
    n = rows
    tmpl_mask = None
    half = (n + 1) // 2
    rt = Rows(n, 2, i32([states[0].slot, states[1].slot]), i32([0] * half + [1] * (n - half)),
              i32(list(range(half)) + list(range(n - half))), i32([0, half, n]), max_keys=300 + n, max_rows=half,
              live=i32([live]) if live is not None else None)
    torch.manual_seed(rows)
    x0 = torch.randn(n, 1024, device=DEV) + offset
    outs = []
    assert be.ws_conv, "the converting prologues should be on for H = 1024"
    for phased, be.ws_conv in ((False, False), (True, False), (True, True)):
        be.ws_phases = phased
        be.kcache.zero_()
        be.vcache.zero_()
        x = x0.clone()
        be._run_layers(x, rt, 0, 3, tmpl_mask, n, 0)
        torch.cuda.synchronize()
        outs.append((x.clone(), be.kcache[:, :2, :, 300:300 + half].float().clone(),
                     be.vcache[:, :2, :, 300:300 + half].float().clone()))
    r = n if live is None else live
    xa, ka, va = outs[0]
    for xb, kb, vb in outs[1:]:  # phases in the GEMM launches
        scale = max(1.0, xa[:r].abs().max().item())
        assert (xa[:r] - xb[:r]).abs().max().item() <= 3e-2 * scale
        assert (ka - kb).abs().max().item() <= 3e-2 * max(1.0, ka.abs().max().item())
        assert (va - vb).abs().max().item() <= 3e-2 * max(1.0, va.abs().max().item())
    # the barrier path leaves its scratch zeroed; the converting GELU path zeroes the W_1 accumulator
    # ahead (in the next QKV launch), so only the barrier counters and the QKV accumulator are checked
    assert be._bar.abs().max().item() == 0 and be._acc.abs().max().item() == 0


# --------------------------------------------------------------- probability pruning / typical acceptance
def test_row_lse_matches_oracle():
    rng = np.random.default_rng(5)
    x = (rng.normal(size=(6, 3000)) * 3).astype(np.float32)
    x[2, :] = 0.0
    d = torch.from_numpy(x).to(DEV)
    for temp in (1.0, 0.7):
        st_ = torch.empty(6, 2, device=DEV, dtype=torch.float64)
        call("propd_row_lse", 6, None, 3000, 3000, ptr(d), None, temp, ptr(st_), st())
        lse, H = op.row_lse_entropy(x.astype(np.float64), temp)
        got = st_.cpu().numpy()
        assert np.allclose(got[:, 0], lse, rtol=1e-13, atol=1e-12)
        assert np.allclose(got[:, 1], H, rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("tau", [0.5, 0.02, 1e-4])
def test_probability_prune_matches_oracle(tau):
    """Survivor sets of probability-based pruning == oracle probability_prune on the same fp32 early logits."""
    rng = np.random.default_rng(int(1 / tau))
    tmpl = TreeTemplate.from_paths(op.grid_candidates(4, 8))
    n, B, V = len(tmpl), 3, 300
    Pn = len(tmpl.parent_nodes)
    tok = rng.integers(0, V, size=(B, n)).astype(np.int32)
    early = (rng.normal(size=(B, Pn, V)) * 2.5).astype(np.float32)
    for b in range(B):  # make some candidates likely so deep nodes survive
        for i in range(n):
            par = int(tmpl.parent[i])
            if par >= 0 and rng.random() < 0.5:
                early[b, tmpl.parent_slot[par], tok[b, i]] += 6.0
    d_early = torch.from_numpy(early.reshape(B * Pn, V)).to(DEV)
    est = torch.empty(B * Pn, 2, device=DEV, dtype=torch.float64)
    call("propd_row_lse", B * Pn, None, V, V, ptr(d_early), None, 1.0, ptr(est), st())
    member = torch.empty(B * n, device=DEV, dtype=torch.uint8)
    td = tmpl.device(DEV)
    d_tok = torch.from_numpy(tok.reshape(-1)).to(DEV)
    call("propd_early_prob_member", B, n, Pn, V, float(np.log(tau)), ptr(d_early), ptr(est), ptr(td["parent"]),
         ptr(td["parent_slot"]), ptr(d_tok), ptr(member), st())
    mem = member.view(B, n).cpu().numpy().astype(bool)
    for b in range(B):
        tree = op.Tree(tuple(op.Node(int(tok[b, i]), int(tmpl.parent[i]), int(tmpl.depth[i]), int(tmpl.rank[i]),
                                     1.0) for i in range(n)), 0)
        rows = np.zeros((n, V))
        for i in tmpl.parent_nodes:
            rows[i] = early[b, tmpl.parent_slot[i]]
        surv, _ = op.probability_prune(tree, rows, tau)
        alive = np.zeros(n, dtype=bool)
        for i in range(n):  # device closure: member and parent alive
            par = int(tmpl.parent[i])
            alive[i] = mem[b, i] and (par < 0 or alive[par])
        assert tuple(np.flatnonzero(alive)) == surv


@pytest.mark.parametrize("eps,alpha,temp", [(0.09, 0.3, 1.0), (0.3, 0.5, 0.7), (1e-3, 0.01, 1.0)])
def test_typical_acceptance_matches_oracle(eps, alpha, temp):
    """Typical-acceptance walk of verify_commit_ex (accepted path, bonus, committed tokens, KV compaction
    source slots) == oracle typical_verify on the same fp32 logits, over pruned trees."""
    rng = np.random.default_rng(int(eps * 1000) + 7)
    tmpl = TreeTemplate.from_paths(op.grid_candidates(4, 6))
    n, B, V, D, k = len(tmpl), 4, 200, 4, 6
    A, dh, layers, Lmax = 2, 16, 2, 64
    tok = rng.integers(0, V, size=(B, n)).astype(np.int32)
    alive = np.ones((B, n), dtype=np.uint8)
    alive[1, 7:] = 0
    alive[2, 3:] = 0
    for b in range(B):
        for i in range(n):
            par = int(tmpl.parent[i])
            if par >= 0 and not alive[b, par]:
                alive[b, i] = 0
    node_row = -np.ones((B, n), dtype=np.int32)
    S = 0
    for b in range(B):
        for i in range(n):
            if alive[b, i]:
                node_row[b, i] = S
                S += 1
    row_logits = (rng.normal(size=(S, V)) * 1.5).astype(np.float32)
    root_logits = (rng.normal(size=(B, V)) * 1.5).astype(np.float32)
    for b in range(B):  # boost some children so acceptance goes deep
        root_logits[b, tok[b, 0]] += 5.0
        for i in range(n):
            par = int(tmpl.parent[i])
            if par >= 0 and alive[b, i] and rng.random() < 0.6:
                row_logits[node_row[b, par], tok[b, i]] += 5.0
    dl = lambda a: keep(torch.from_numpy(np.ascontiguousarray(a)).to(DEV))  # inline temporaries stay alive
    d_rows, d_root = dl(row_logits), dl(root_logits)
    slots = np.arange(B, dtype=np.int32)
    rst = torch.empty(S, 2, device=DEV, dtype=torch.float64)
    call("propd_row_lse", S, None, V, V, ptr(d_rows), None, temp, ptr(rst), st())
    rootst = torch.empty(B, 2, device=DEV, dtype=torch.float64)
    call("propd_row_lse", B, None, V, V, ptr(d_root), ptr(i32(slots)), temp, ptr(rootst), st())
    row_argmax = dl(row_logits.argmax(1).astype(np.int32))
    root = dl(root_logits.argmax(1).astype(np.int32))
    draft = dl(rng.integers(0, V, size=(B, D, k)).astype(np.int32))
    seq_len = dl(np.full(B, 10, dtype=np.int32))
    kc = torch.randn(layers, B, A, Lmax, dh, device=DEV)
    vc = torch.randn_like(kc)
    outs = {name: torch.empty(sz, device=DEV, dtype=torch.int32)
            for name, sz in (("acc_node", B * D), ("acc_surv", B * D), ("acc_len", B), ("bonus", B),
                             ("committed", B * (D + 1)))}
    ranks = torch.empty(B, D, device=DEV, dtype=torch.int8)
    td = tmpl.device(DEV)
    typ = _lib.Typical(row_logits=ptr(d_rows), ld=V, row_stats=ptr(rst), root_logits=ptr(d_root), root_ld=V,
                       root_stats=ptr(rootst), log_eps=float(np.log(eps)), log_alpha=float(np.log(alpha)),
                       temperature=temp, depth=ptr(td["depth"]))
    call("propd_verify_commit_ex", _lib.F32, B, n, D, k, layers, A, dh, Lmax, B * A * Lmax * dh, ptr(td["parent"]),
         ptr(dl(tok.reshape(-1))), ptr(dl(alive.reshape(-1))), ptr(dl(node_row.reshape(-1))), ptr(row_argmax),
         ptr(root), ptr(draft), ptr(i32(slots)), ptr(seq_len), ptr(kc), ptr(vc), ptr(outs["acc_node"]),
         ptr(outs["acc_surv"]), ptr(outs["acc_len"]), ptr(outs["bonus"]), ptr(outs["committed"]), ptr(ranks), typ,
         st())
    torch.cuda.synchronize()
    got = {k_: v.cpu().numpy() for k_, v in outs.items()}
    deep = 0
    for b in range(B):
        surv = [i for i in range(n) if alive[b, i]]
        full = op.Tree(tuple(op.Node(int(tok[b, i]), int(tmpl.parent[i]), int(tmpl.depth[i]), int(tmpl.rank[i]),
                                     1.0) for i in range(n)), 0)
        vtree = op.restrict(full, surv)
        acc, bonus = op.typical_verify(vtree, row_logits[[node_row[b, i] for i in surv]], root_logits[b], eps,
                                       alpha, temp)
        L = int(got["acc_len"][b])
        assert L == len(acc)
        assert list(got["acc_surv"][b * D: b * D + L]) == list(acc)
        assert list(got["acc_node"][b * D: b * D + L]) == [surv[a] for a in acc]
        assert int(got["bonus"][b]) == bonus
        assert list(got["committed"][b * (D + 1): b * (D + 1) + L + 1]) == [vtree.nodes[a].token for a in acc] + [
            bonus]
        deep = max(deep, L)
    assert deep >= 2  # the cases exercise multi-node paths


# --------------------------------------------------------------- many-row projections (propd_gemm)
def _epi(mode, Y, ldy, **kw):
    e = _lib.GemmEpi(mode=mode, Y=ptr(Y), ldy=ldy)
    for k, v in kw.items():
        setattr(e, k, v)
    return e


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("M,N,K,mode", [(129, 4096, 4096, "store"), (300, 12288, 4096, "qkv"),
                                         (1000, 16384, 4096, "gelu"), (4096, 4096, 16384, "add"),
                                         (257, 32000, 4096, "f32"), (700, 4128, 1024, "add"), (1, 256, 64, "f32"),
                                         (160, 12288, 4096, "qkv"), (200, 16384, 4096, "gelu"),
                                         (512, 12288, 4096, "qkv"), (130, 4096, 1024, "store")])
def test_gemm_matches_fp32_reference(dtype, M, N, K, mode):
    """Y = epilogue(X . W): tcgen05 (bf16 operands, fp32 accumulation) and the fp32 CUDA-core path vs torch
    fp32 on the same (bf16-rounded) operands.  bf16: |err| <= 1e-3 * max(1, |ref|) on fp32 outputs
    (+ bf16 output rounding 8e-3 relative); fp32: 1e-5 relative."""
    if dtype == "fp32" and M * N * K > 2e10:
        pytest.skip("large shape: tensor-core path only")
    torch.manual_seed(M + N + K)
    T = torch.bfloat16 if dtype == "bf16" else torch.float32
    code = _lib.BF16 if dtype == "bf16" else _lib.F32
    X = torch.randn(M, K, device=DEV).to(T)
    W = (torch.randn(K, N, device=DEV) / K ** 0.5).to(T)
    ref = X.float() @ W.float()
    tol = (1e-3 if dtype == "bf16" else 1e-5) * max(1.0, ref.abs().max().item())
    otol = 8e-3 if dtype == "bf16" else 1e-5  # rounding of a dtype output
    wkw = {}
    if mode in ("f32", "add"):
        base = torch.randn(M, N, device=DEV) if mode == "add" else torch.full((M, N), float("nan"), device=DEV)
        Y = base.clone()
        epi = _epi(_lib.EPI_ADD_F32 if mode == "add" else _lib.EPI_STORE_F32, Y, N, **wkw)
        call("propd_gemm", code, M, None, N, K, ptr(X), K, ptr(W), N, epi, st())
        torch.cuda.synchronize()
        want = ref + (base if mode == "add" else 0)
        assert (Y - want).abs().max().item() <= tol
    elif mode in ("store", "gelu"):
        Y = torch.full((M, N), float("nan"), device=DEV).to(T)
        epi = _epi(_lib.EPI_GELU if mode == "gelu" else _lib.EPI_STORE, Y, N, **wkw)
        call("propd_gemm", code, M, None, N, K, ptr(X), K, ptr(W), N, epi, st())
        torch.cuda.synchronize()
        want = torch.nn.functional.gelu(ref, approximate="tanh") if mode == "gelu" else ref
        assert (Y.float() - want).abs().max().item() <= tol + otol * want.abs().max().item()
    else:  # QKV: Q -> Y, K/V -> cache slots seq_len[slot] + node
        A, dh, Lmax = 32, 128, 480
        H = A * dh
        assert N == 3 * H
        nseq = 3
        per = [M // 3, M // 3 + M % 3, M // 3]  # rows of three sequences
        assert max(per) + 250 <= Lmax
        row_seq = i32(np.repeat(np.arange(nseq), per))
        row_node = i32(np.concatenate([np.arange(p) for p in per]))
        seq_slot, seq_len = i32([2, 0, 1]), i32([7, 250, 31])
        kc = torch.zeros(3, A, Lmax, dh, device=DEV, dtype=T)
        vc = torch.zeros_like(kc)
        Y = torch.zeros(M, 3 * H, device=DEV, dtype=T)
        epi = _epi(_lib.EPI_QKV, Y, 3 * H, A=A, dh=dh, Lmax=Lmax, row_seq=ptr(row_seq), row_node=ptr(row_node),
                   seq_slot=ptr(seq_slot), seq_len=ptr(seq_len), kcache=ptr(kc), vcache=ptr(vc), **wkw)
        call("propd_gemm", code, M, None, N, K, ptr(X), K, ptr(W), N, epi, st())
        torch.cuda.synchronize()
        lim = tol + otol * ref.abs().max().item()
        assert (Y[:, :H].float() - ref[:, :H]).abs().max().item() <= lim
        rs, rn = row_seq.cpu().numpy(), row_node.cpu().numpy()
        slots, lens = seq_slot.cpu().numpy(), seq_len.cpu().numpy()
        for m in range(M):
            s = slots[rs[m]]
            pos = lens[s] + rn[m]
            assert (kc[s, :, pos].float().reshape(-1) - ref[m, H:2 * H]).abs().max().item() <= lim
            assert (vc[s, :, pos].float().reshape(-1) - ref[m, 2 * H:]).abs().max().item() <= lim


@pytest.mark.parametrize("live", [0, 129, 255, 1000])
def test_gemm_device_row_count(live):
    """rows_dev: rows < min(M, *rows_dev) are computed, the rest of Y is untouched (bit-exact)."""
    M, N, K = 700, 4096, 1024
    torch.manual_seed(live)
    X = torch.randn(M, K, device=DEV).bfloat16()
    W = (torch.randn(K, N, device=DEV) / K ** 0.5).bfloat16()
    ref = X.float() @ W.float()
    base = torch.randn(M, N, device=DEV)
    Y = base.clone()
    call("propd_gemm", _lib.BF16, M, ptr(i32([live])), N, K, ptr(X), K, ptr(W), N, _epi(_lib.EPI_ADD_F32, Y, N), st())
    torch.cuda.synchronize()
    r = min(M, live)
    if r:
        assert (Y[:r] - ref[:r] - base[:r]).abs().max().item() <= 1e-3 * max(1.0, ref.abs().max().item())
    assert torch.equal(Y[r:], base[r:])


# --------------------------------------------------------------- fused one-row attention
@pytest.mark.parametrize("B,L,hidden,heads", [(1, 300, 1024, 8), (3, 517, 1024, 8), (4, 70, 1024, 8),
                                              (2, 1024, 1024, 8), (1, 1030, 1024, 8), (1, 1024, 4096, 32)])
def test_fused_bonus_attention_matches_decode_kernel(B, L, hidden, heads):
    """Bonus pass with the attention inside the QKV launch (key-split partials, combined in W_o's
    converting prologue) == the same pass with the decode attention kernel: final hidden rows, the
    root argmax and the appended K/V rows within bf16 rounding (backends.py:239-259)."""
    from paper_2402_13485_b200 import B200Backend, TinyTransformerConfig

    cfg = TinyTransformerConfig(layers=3 if hidden <= 1024 else 2, hidden=hidden, heads=heads, vocab=1024,
                                draft_heads=2, max_positions=1100, seed=2)
    be = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=4, max_tree=16)
    assert be.ws_fuse_attn
    states = be.synthetic_states(B, L, seed=B)
    slots = i32([s.slot for s in states])
    lens0 = be.seq_len.clone()
    bonus = i32([(7 * b + 3) % 1024 for b in range(B)])
    outs = []
    for fuse in (False, True):
        be.ws_fuse_attn = fuse
        be.seq_len.copy_(lens0)
        be._bonus_program(slots, bonus, B, L + 2)
        torch.cuda.synchronize()
        hid = be.hidden[slots.long()].float().clone()
        kv = torch.stack([be.kcache[:, s.slot, :, L].float() for s in states]).clone()
        vv = torch.stack([be.vcache[:, s.slot, :, L].float() for s in states]).clone()
        outs.append((hid, kv, vv, be.seq_len.clone()))
    (h0, k0, v0, n0), (h1, k1, v1, n1) = outs
    assert torch.equal(n0, n1)
    for a, b in ((h0, h1), (k0, k1), (v0, v1)):
        assert (a - b).abs().max().item() <= 3e-2 * max(1.0, a.abs().max().item()), (a - b).abs().max().item()
    assert be._acc.abs().max().item() == 0  # the W_o launches re-zeroed the QKV accumulator


@pytest.mark.parametrize("cap,live", [(16, 1), (32, 20), (64, 32), (96, 32), (128, 30), (128, 1)])
def test_gemm_ws_gelu_prologue_7b_shape(cap, live):
    """W_2-shaped weight-streaming launch (K = 16384: ~29 k-blocks per CTA, so the converting warps cycle
    the ring many times) with the GELU prologue at every row capacity: equals GELU(src) @ W in fp32 on the
    live rows (regression: with 3 ring slots and 4 converting warps the slot barriers' parity aliased)."""
    N, K = 4096, 16384
    torch.manual_seed(cap + live)
    W = (torch.randn(K, N, device=DEV) / K ** 0.5).bfloat16()
    src = torch.randn(cap, K, device=DEV)
    ref = torch.nn.functional.gelu(src[:live], approximate="tanh").bfloat16().float() @ W.float()
    g = torch.empty(cap, K, device=DEV, dtype=torch.bfloat16)
    Y = torch.zeros(cap, N, device=DEV)
    bar = torch.zeros(32, device=DEV, dtype=torch.int32)
    ph = _lib.WsPhases(pro_mode=_lib.PRO_XGELU, pro_src=ptr(src), pro_ld=K, pro_dst=ptr(g), pro_ldd=K, pro_cols=K,
                       bar=ptr(bar))
    call("propd_gemm_ws_ph", cap, ptr(i32([live])), N, K, ptr(g), K, ptr(W), N, ptr(Y), N, 1, 0, ph, st())
    torch.cuda.synchronize()
    assert (Y[:live] - ref).abs().max().item() <= 1e-3 * max(1.0, ref.abs().max().item())
    assert Y[live:].abs().max().item() == 0.0
    assert bar.abs().max().item() == 0
