"""Teacher-forced step parity of the benchmarked bf16 path against the fp64
oracle at the 7B width (reference step engine.py:243-303,
forward_tree backends.py:290-335, verify verification.py:30-53, commit
backends.py:337-348).

`B200Backend(dtype="bf16", use_graphs=True).step_tree` — the batched step the
bench times (CUDA graphs, device row counts, transposed tcgen05 attention,
weight-streaming tcgen05 projections, K3 early prune, K5 accept + KV
compaction, the bonus pass with its attention fused into the QKV launches) — runs next to
`oracle.TinyModel` on the same reference-initialised weights at hidden 4096,
32 heads x 128, the prune layer strictly inside the stack.  The oracle
follows the device's drafts, survivors and commits (oracle/parity.py), and
every decision is compared where the oracle's margin exceeds twice the
measured error:

  logits        max |err| <= 5e-2 * max(1, |ref|_inf)   (bf16 weights/activations vs fp64)
  draft ranks, early membership, survivors, root / row argmax, accepted chain + bonus:
                identical wherever decidable; >= half of the rows decidable.
  draft picks   each device rank-r token scores >= the oracle's r-th best - 2 err (near-ties at V = 32000
                make rank identities decidable only where the gaps allow; measured 135/768 on the first run).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import parity  # noqa: E402
from oracle import treedecode_port as op  # noqa: E402
from paper_2402_13485_b200 import B200Backend, PruneConfig, TinyTransformerConfig, grid_candidates  # noqa: E402
from paper_2402_13485_b200.tree import TreeTemplate  # noqa: E402


def _vocab() -> int:
    """Vicuna's 32000 when the host has room for the fp64 oracle weights (~16 GB), else 8192."""
    try:
        import psutil

        return 32000 if psutil.virtual_memory().available > 96e9 else 8192
    except Exception:  # pragma: no cover
        return 8192


@pytest.mark.parametrize("B,kv,k,layers,p", [(4, 1024, 16, 5, 3), (1, 1024, 16, 5, 3)])
def test_bf16_batched_step_teacher_forced_at_7b_width(B, kv, k, layers, p):
    V = _vocab()
    mc = op.TinyCfg(layers=layers, hidden=4096, heads=32, vocab=V, draft_heads=4, max_positions=kv + 64, seed=11)
    w = op.init_weights(mc)
    w["w_draft"][0] = w["w_lm"]  # planted acceptance: every step accepts its depth-1 rank-1 node
    ref = op.TinyModel(mc, weights=w)
    be = B200Backend(TinyTransformerConfig(**mc.__dict__), dtype="bf16", weights=w, max_slots=B, max_tree=4 * k,
                     use_graphs=True)
    rng = np.random.default_rng(5)
    prompts = [rng.integers(0, V, size=kv - 7 * b).tolist() for b in range(B)]  # ragged KV lengths
    states = be.prefill_batch(prompts)
    ref_states = [ref.prefill(pr) for pr in prompts]
    tmpl = TreeTemplate.from_paths(grid_candidates(4, k), 4, k)
    prune = PruneConfig(layer=p, topk=50)
    rep = None
    for _ in range(3):
        rep = parity.teacher_forced_step(be, ref, states, ref_states, tmpl, k, prune, rep=rep)
    print("bf16 step parity (7B width):", rep.summary())
    assert rep.accepted >= 3 * B  # the planted head accepts every step: the commit / compaction path ran
    assert rep.frac("argmax") >= 0.5, rep.summary()  # the decision checks are not vacuous
    # (draft ranks are often closer than the bf16 error at V = 32000: every device pick is checked against the
    # oracle's r-th score within the error bound, identities where the gaps allow)
    assert rep.frac("member") >= 0.5 and rep.n["draft"][0] > 0, rep.summary()
    for st, sr in zip(states, ref_states):
        assert st.committed == sr.committed  # teacher forcing kept both sides on the same context
