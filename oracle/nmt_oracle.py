"""Float64 CPU oracle for the batched DL4MT/Nematus cGRU scorer of arXiv 1605.04809.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
module.  The product library (``paper_1605_04809_b200``) never imports it and
shares no code with it; both are fed by ``synth`` (random draws only).

What it computes.  PAPER.md gives no model equations; it names the model
("Bahdanau et al. ... more exactly the DL4MT variant also present in Nematus",
PAPER.md:13, §1; "attentional encoder-decoder ... trained with Nematus",
PAPER.md:30, §3; "word embeddings of size 500, and hidden layers of size 1024",
PAPER.md:32, §3).  The equations below are therefore the DL4MT/Nematus ones as
written out in SURVEY.md §8(c) (readings A1-A24 in DESIGN.md §2), evaluated in
float64, one plain formula per line, no blocking, fusion or reordering.

Batching semantics are the paper's ScoreBatch (§5.1, Alg. 1):
one forward step over a set of (state, word) rows, with states cached at the
target nodes and "reused ... as initial states when scoring another batch of
hypotheses at later time".  Rows are parent-indexed (reading A13):
row = unique parent, the candidate words are gathered from that row's
distribution, child = (s2, w).  Numbers are identical to the paper's eager rows.

Pins (tests/test_oracle.py): torch float64 GRUCell / bidirectional GRU after a
weight re-pack, scipy log_softmax, closed forms for zero weights, saturation
cases for attention, brute-force enumeration over a tiny vocabulary, prefix
additivity, cache reuse == recomputation, Fig. 1 structure (tests/golden/).
Oracle-vs-the-authors'-trained-implementation: PARITY UNPINNED (no weights or
printed model outputs exist in PAPER.md) - see DESIGN.md §2.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

BOS = -1  # y_prev of the root node: zero embedding (reading A9)


def sigmoid(x: np.ndarray) -> np.ndarray:
    return 1.0 / (1.0 + np.exp(-x))


def log_softmax(z: np.ndarray, axis: int = -1) -> np.ndarray:
    """log p = z - logsumexp(z), max-shifted (reading A6)."""
    m = np.max(z, axis=axis, keepdims=True)
    return z - (m + np.log(np.sum(np.exp(z - m), axis=axis, keepdims=True)))


def logsumexp(z: np.ndarray, axis: int = -1) -> np.ndarray:
    m = np.max(z, axis=axis, keepdims=True)
    return (m + np.log(np.sum(np.exp(z - m), axis=axis, keepdims=True))).squeeze(axis)


def gru(x: np.ndarray, h: np.ndarray, W, b, U, Wx, bx, Ux) -> np.ndarray:
    """DL4MT ``gru_layer`` step (reading A2): [r|u] = sigm(xW + b + hU) (first H cols = r);
    h~ = tanh(r*(hUx) + xWx + bx); h' = u*h + (1-u)*h~."""
    H = h.shape[-1]
    preact = x @ W + b + h @ U
    r = sigmoid(preact[..., :H])
    u = sigmoid(preact[..., H:])
    htilde = np.tanh(r * (h @ Ux) + x @ Wx + bx)
    return u * h + (1.0 - u) * htilde


def gru_nl(h1: np.ndarray, c: np.ndarray, U_nl, b_nl, Ux_nl, bx_nl, Wc, Wcx) -> np.ndarray:
    """Second GRU of DL4MT ``gru_cond_layer`` (reading A3): context c is the input, s1 the state;
    [r2|u2] = sigm(s1 U_nl + b_nl + c Wc); h~ = tanh(r2*(s1 Ux_nl + bx_nl) + c Wcx)."""
    H = h1.shape[-1]
    preact = h1 @ U_nl + b_nl + c @ Wc
    r2 = sigmoid(preact[..., :H])
    u2 = sigmoid(preact[..., H:])
    htilde = np.tanh(r2 * (h1 @ Ux_nl + bx_nl) + c @ Wcx)
    return u2 * h1 + (1.0 - u2) * htilde


class Model:
    """Float64 copy of a Nematus-named parameter set (arrays from ``synth.make_model``)."""

    def __init__(self, dims, params: Dict[str, np.ndarray]):
        self.dims = dims
        self.p = {k: np.asarray(v, dtype=np.float64) for k, v in params.items()}
        for k in list(self.p):
            if self.p[k].shape[0] == 1 and k not in ("decoder_c_tt",):
                self.p[k] = self.p[k][0]  # biases as vectors
        self.p["decoder_c_tt"] = float(self.p["decoder_c_tt"].reshape(-1)[0])
        self.p["decoder_U_att"] = self.p["decoder_U_att"].reshape(-1)
        self.V = self.p["ff_logit_W"].shape[1]
        self.H = self.p["decoder_Ux"].shape[0]
        self.E = self.p["Wemb_dec"].shape[1]


@dataclasses.dataclass
class Context:
    """Per-sentence source context, "available at all time" (§5.1)."""
    ctx: np.ndarray   # [Tx, 2H]  annotations [fwd_j ; bwd_j]
    pctx: np.ndarray  # [Tx, 2H]  attention keys ctx Wc_att + b_att
    s0: np.ndarray    # [H]       initial decoder state


def encode(m: Model, src: Sequence[int]) -> Context:
    """Bidirectional GRU encoder over the BPE source (caller appends EOS, reading A11)."""
    p = m.p
    src = np.asarray(src, dtype=np.int64)
    if src.size == 0:
        raise ValueError("empty source")
    x = p["Wemb"][src]                                   # [Tx, E]
    Tx, H = x.shape[0], m.H
    fwd = np.zeros((Tx, H))
    bwd = np.zeros((Tx, H))
    h = np.zeros(H)
    for j in range(Tx):                                  # ->h_j = GRU(x_j, ->h_{j-1}), ->h_{-1} = 0
        h = gru(x[j], h, p["encoder_W"], p["encoder_b"], p["encoder_U"],
                p["encoder_Wx"], p["encoder_bx"], p["encoder_Ux"])
        fwd[j] = h
    h = np.zeros(H)
    for j in reversed(range(Tx)):                        # <-h_j = GRU(x_j, <-h_{j+1}), <-h_{Tx} = 0
        h = gru(x[j], h, p["encoder_r_W"], p["encoder_r_b"], p["encoder_r_U"],
                p["encoder_r_Wx"], p["encoder_r_bx"], p["encoder_r_Ux"])
        bwd[j] = h
    ctx = np.concatenate([fwd, bwd], axis=1)
    s0 = np.tanh(ctx.mean(axis=0) @ p["ff_state_W"] + p["ff_state_b"])
    pctx = ctx @ p["decoder_Wc_att"] + p["decoder_b_att"]
    return Context(ctx=ctx, pctx=pctx, s0=s0)


def step(m: Model, c: Context, s: np.ndarray, y_prev: Sequence[int]) -> Dict[str, np.ndarray]:
    """One decoder forward step for R rows (Alg. 1 line 5, "(H_i, P_i) <- NMT(H_{i-1}, E_i)").

    s: [R, H] input states, y_prev: [R] previous words (BOS = -1 -> zero embedding).
    Returns the intermediates s1, alpha, c, s2, t, z (logits), logZ, argmax.
    """
    p = m.p
    s = np.atleast_2d(np.asarray(s, dtype=np.float64))
    y = np.asarray(y_prev, dtype=np.int64).reshape(-1)
    e = np.where((y >= 0)[:, None], p["Wemb_dec"][np.maximum(y, 0)], 0.0)      # [R, E]
    # GRU1 (cGRU first transition)
    s1 = gru(e, s, p["decoder_W"], p["decoder_b"], p["decoder_U"],
             p["decoder_Wx"], p["decoder_bx"], p["decoder_Ux"])                 # [R, H]
    # MLP attention (Bahdanau): a_j = tanh(pctx_j + s1 W_comb_att) . U_att + c_tt
    q = s1 @ p["decoder_W_comb_att"]                                            # [R, C]
    a = np.tanh(c.pctx[None, :, :] + q[:, None, :]) @ p["decoder_U_att"] + p["decoder_c_tt"]  # [R, Tx]
    alpha = np.exp(a - a.max(axis=1, keepdims=True))
    alpha = alpha / alpha.sum(axis=1, keepdims=True)
    ctx_r = alpha @ c.ctx                                                       # [R, C]
    # GRU2 (context as input, s1 as state)
    s2 = gru_nl(s1, ctx_r, p["decoder_U_nl"], p["decoder_b_nl"], p["decoder_Ux_nl"],
                p["decoder_bx_nl"], p["decoder_Wc"], p["decoder_Wcx"])          # [R, H]
    # deep-output readout (reading A7)
    pre = (s2 @ p["ff_logit_lstm_W"] + p["ff_logit_lstm_b"]
           + e @ p["ff_logit_prev_W"] + p["ff_logit_prev_b"]
           + ctx_r @ p["ff_logit_ctx_W"] + p["ff_logit_ctx_b"])
    if m.dims.readout == "tanh":
        t = np.tanh(pre)
    else:  # maxout: t_k = max(pre_{2k}, pre_{2k+1})
        t = np.maximum(pre[:, 0::2], pre[:, 1::2])
    # whole-vocabulary logits and normaliser ("computations over the whole target vocabulary")
    z = t @ p["ff_logit_W"] + p["ff_logit_b"]                                   # [R, V]
    logZ = logsumexp(z, axis=1)
    argmax = np.argmax(z, axis=1)  # first index of the max = lowest id on ties (reading A21)
    return dict(s1=s1, alpha=alpha, c=ctx_r, s2=s2, t=t, z=z, logZ=logZ, argmax=argmax)


def word_logprob(m: Model, t: np.ndarray, logZ: float, w: int) -> float:
    """log p(w) = z_w - logZ with z_w = t . W_o[:, w] + b_o[w] (column w of z = t W_o + b_o)."""
    return float(t @ m.p["ff_logit_W"][:, w] + m.p["ff_logit_b"][w] - logZ)


@dataclasses.dataclass
class Node:
    parent: int
    word: int                     # y_prev of this node's step (BOS for the root)
    s_in: np.ndarray              # input state of this node's step
    stepped: bool = False
    s_out: Optional[np.ndarray] = None
    t: Optional[np.ndarray] = None
    logZ: float = 0.0
    argmax: int = -1


class Session:
    """Per-sentence state cache ("Cache state pointers and probabilities at target
    nodes"; PAPER.md:136 states reused "at later time").  Node ids are assigned in first-appearance
    order of the (parent-major, candidate-order) request stream (SURVEY §8(b) Determinism)."""

    def __init__(self, m: Model, src: Sequence[int]):
        self.m = m
        self.c = encode(m, src)
        self.nodes: List[Node] = [Node(parent=-1, word=BOS, s_in=self.c.s0)]
        self.children: Dict[Tuple[int, int], int] = {}
        self.n_steps = 0
        self.rows_per_step: List[int] = []

    root = 0

    def inject_state(self, s: np.ndarray, y_prev: int) -> int:
        self.nodes.append(Node(parent=-1, word=int(y_prev), s_in=np.asarray(s, np.float64)))
        return len(self.nodes) - 1

    def _step_nodes(self, ids: List[int], chunk: int = 256) -> None:
        for k in range(0, len(ids), chunk):  # rows are independent (batch independence)
            part = ids[k:k + chunk]
            out = step(self.m, self.c, np.stack([self.nodes[i].s_in for i in part]),
                       [self.nodes[i].word for i in part])
            for r, i in enumerate(part):
                n = self.nodes[i]
                n.stepped, n.s_out, n.t = True, out["s2"][r], out["t"][r]
                n.logZ, n.argmax = float(out["logZ"][r]), int(out["argmax"][r])

    def score_batch(self, parents: Sequence[int], cand_offsets: Sequence[int],
                    cand_words: Sequence[int]) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(parents, candidate CSR) -> (log-probs [N_cand], child ids [N_cand], argmax [n_parents])."""
        parents = [int(x) for x in parents]
        off = [int(x) for x in cand_offsets]
        words = [int(x) for x in cand_words]
        if len(off) != len(parents) + 1 or off[0] != 0 or off[-1] != len(words):
            raise ValueError("bad candidate offsets")
        for p in parents:
            if not 0 <= p < len(self.nodes):
                raise KeyError(f"unknown state {p}")
        for w in words:
            if not 0 <= w < self.m.V:
                raise IndexError(f"word {w} out of range")
        children = np.empty(len(words), np.int64)
        for k, p in enumerate(parents):                      # intern (p, w) in request order
            for i in range(off[k], off[k + 1]):
                key = (p, words[i])
                if key not in self.children:
                    self.nodes.append(Node(parent=p, word=words[i], s_in=None))
                    self.children[key] = len(self.nodes) - 1
                children[i] = self.children[key]
        rows: List[int] = []
        for k, p in enumerate(parents):                      # unique, unstepped, >= 1 candidate
            if off[k + 1] > off[k] and not self.nodes[p].stepped and p not in rows:
                rows.append(p)
        if rows:
            self._step_nodes(rows)
            self.n_steps += 1
            self.rows_per_step.append(len(rows))
        for k, p in enumerate(parents):
            for i in range(off[k], off[k + 1]):
                ch = self.nodes[children[i]]
                if ch.s_in is None:
                    ch.s_in = self.nodes[p].s_out            # child = (s2, w)
        logp = np.array([word_logprob(self.m, self.nodes[p].t, self.nodes[p].logZ, words[i])
                         for k, p in enumerate(parents) for i in range(off[k], off[k + 1])])
        argmax = np.array([self.nodes[p].argmax if self.nodes[p].stepped else -1 for p in parents],
                          np.int64)
        return logp, children, argmax

    def logprobs_full(self, node: int) -> np.ndarray:
        n = self.nodes[node]
        out = step(self.m, self.c, n.s_in[None, :], [n.word])
        return log_softmax(out["z"][0])

    def beam_step(self, parents: Sequence[int], k: int) -> Tuple[np.ndarray, np.ndarray]:
        """Pure-NMT beam step: for each parent, the k words of
        largest log p(w | parent) over the whole vocabulary -> (words [n, k], logp [n, k])."""
        rows = [self.logprobs_full(int(p)) for p in parents]
        words = np.array([topk_words(r, k) for r in rows], np.int64).reshape(len(rows), k)
        return words, np.array([r[w] for r, w in zip(rows, words)]).reshape(len(rows), k)

    def intermediates(self, node: int) -> Dict[str, np.ndarray]:
        n = self.nodes[node]
        out = step(self.m, self.c, n.s_in[None, :], [n.word])
        return {k: v[0] for k, v in out.items()}


def topk_words(logp: np.ndarray, k: int) -> np.ndarray:
    """The k indices of largest value, by value descending then index ascending (a stable sort of
    -logp): the definition of a beam step's expansion set."""
    return np.argsort(-np.asarray(logp, np.float64), kind="stable")[:k]


def score_sequence(m: Model, c: Context, words: Sequence[int], s: Optional[np.ndarray] = None,
                   y_prev: int = BOS) -> Tuple[float, List[float], np.ndarray]:
    """Brute-force sequential scorer with no cache: chained single-row steps."""
    s = c.s0 if s is None else np.asarray(s, np.float64)
    y = y_prev
    lps: List[float] = []
    for w in words:
        out = step(m, c, s[None, :], [y])
        lps.append(float(log_softmax(out["z"][0])[w]))
        s, y = out["s2"][0], int(w)
    return float(sum(lps)), lps, s


def ensemble_combine(member_logp: Sequence[np.ndarray], weights: Sequence[float], mode: int = 0) -> np.ndarray:
    """Ensemble hook ("multiple models ... as separate features", reading A16).

    mode 0: log-linear sum_m lambda_m log p_m(w);  mode 1: log sum_m pi_m p_m(w)."""
    L = np.stack([np.asarray(x, np.float64) for x in member_logp])
    w = np.asarray(weights, np.float64)[:, None]
    if mode == 0:
        return (w * L).sum(axis=0)
    return np.log((w * np.exp(L)).sum(axis=0))


def average_params(members: Sequence[Dict[str, np.ndarray]]) -> Dict[str, np.ndarray]:
    """Checkpoint averaging, NMT-k-Avg ("the element-wise average of all model weights
    in the NMT ensembles and saved the resulting model"): every array is mean_i W_i, in float64."""
    names = list(members[0].keys())
    for m in members[1:]:
        if list(m.keys()) != names or any(m[k].shape != members[0][k].shape for k in names):
            raise ValueError("average_params: members differ in names or shapes")
    return {k: np.mean(np.stack([np.asarray(m[k], np.float64) for m in members]), axis=0) for k in names}


# ---------------------------------------------------------------------------------------------
# ScoreBatch forest driver (Alg. 1) expressed on top of Session.score_batch:
# one call per tree depth.  Used to pin the Fig. 1 structure (tests/golden/fig1_forest.txt).
# ---------------------------------------------------------------------------------------------

def forest_levels(pairs: Sequence[Tuple[int, Tuple[int, ...]]]) -> List[List[Tuple[Tuple[int, Tuple[int, ...]], int]]]:
    """Edges of the per-hypothesis prefix-tree forest grouped by depth: level i holds
    ((h, prefix_{<i}), w_i) for every distinct edge at depth i."""
    levels: List[List] = []
    seen = set()
    depth = max(len(t) for _, t in pairs)
    for i in range(depth):
        lvl = []
        for h, t in sorted(pairs):
            if len(t) > i:
                e = ((h, tuple(t[:i])), t[i])
                if e not in seen:
                    seen.add(e)
                    lvl.append(e)
        levels.append(lvl)
    return levels


def score_forest(sess: Session, hyp_nodes: Sequence[int], pairs: Sequence[Tuple[int, Tuple[int, ...]]]
                 ) -> Dict[Tuple[int, Tuple[int, ...]], float]:
    """Score every (h, t) pair with one score_batch call per forest depth; returns summed log-probs."""
    node_of: Dict[Tuple[int, Tuple[int, ...]], int] = {(h, ()): hyp_nodes[h] for h, _ in pairs}
    acc: Dict[Tuple[int, Tuple[int, ...]], float] = {(h, ()): 0.0 for h, _ in pairs}
    for lvl in forest_levels(pairs):
        parents: List[int] = []
        offsets = [0]
        words: List[int] = []
        keys: List[Tuple[int, Tuple[int, ...]]] = []
        by_parent: Dict[int, List[Tuple[Tuple[int, Tuple[int, ...]], int]]] = {}
        order: List[int] = []
        for (src, w) in lvl:
            pn = node_of[src]
            if pn not in by_parent:
                by_parent[pn] = []
                order.append(pn)
            by_parent[pn].append((src, w))
        for pn in order:
            parents.append(pn)
            for src, w in by_parent[pn]:
                words.append(w)
                keys.append((src[0], src[1] + (w,)))
                acc[keys[-1]] = acc[src]
            offsets.append(len(words))
        logp, children, _ = sess.score_batch(parents, offsets, words)
        for k, lp, ch in zip(keys, logp, children):
            acc[k] += float(lp)
            node_of[k] = int(ch)
    return {(h, tuple(t)): acc[(h, tuple(t))] for h, t in pairs}
