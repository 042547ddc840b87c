"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the method (no GRU, attention, readout or
softmax).  It only draws random numbers with numpy PCG64 and writes/reads the
params container, so that the float64 oracle (``oracle/``) and the CUDA path
(``paper_1605_04809_b200``) can be fed identical inputs while sharing no code.

Recipes follow SURVEY.md §8(d) "Synthetic model generator" and DESIGN.md §3:

* linear maps  ~ N(0, 1/fan_in); recurrent U, Ux, U_nl, Ux_nl: orthogonal blocks
  (DL4MT ``ortho_weight``); embeddings ~ N(0, 1); biases ~ N(0, 0.1^2);
  U_att ~ N(0, (2/sqrt(2H))^2); W_o ~ N(0, sigma^2) with sigma chosen so that the
  logits t.W_o have a NOMINAL std ``logit_std``; b_o[w] = -ln(w+1) (Zipf prior).
* token ids: 1 + zipf(1.1), resampled while >= V, so ids lie in [2, V);
  0 = EOS, 1 = UNK (DL4MT/Nematus convention).

Parameter names/shapes are the Nematus npz names; row-vector
convention x.W with W in R^{in x out}.  PAPER.md:32 fixes emb 500 / hidden 1024.
"""
from __future__ import annotations

import dataclasses
import struct
import zlib
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

EOS = 0
UNK = 1


@dataclasses.dataclass(frozen=True)
class Dims:
    dim_emb: int
    dim_hid: int
    vocab_src: int
    vocab_tgt: int
    readout: str = "tanh"  # "tanh" (DL4MT/Nematus) or "maxout" (Bahdanau 2014 / north_star)

    @property
    def ctx_dim(self) -> int:
        return 2 * self.dim_hid


# Configurations of BASELINE.json:configs.
TINY = Dims(8, 16, 50, 50, "tanh")            # C1
EN_RU = Dims(500, 1024, 50000, 100000, "tanh")  # C2 / C4 / C5
RU_EN = Dims(500, 1024, 100000, 50000, "tanh")  # C3


def param_shapes(d: Dims) -> List[Tuple[str, Tuple[int, int]]]:
    """Ordered (name, (rows, cols)) list; vectors are 1 x n.  Order = payload order."""
    E, H, C = d.dim_emb, d.dim_hid, d.ctx_dim
    ro = E if d.readout == "tanh" else 2 * E
    out: List[Tuple[str, Tuple[int, int]]] = [
        ("Wemb", (d.vocab_src, E)),
        ("Wemb_dec", (d.vocab_tgt, E)),
    ]
    for pre in ("encoder", "encoder_r"):
        out += [(f"{pre}_W", (E, 2 * H)), (f"{pre}_b", (1, 2 * H)), (f"{pre}_U", (H, 2 * H)),
                (f"{pre}_Wx", (E, H)), (f"{pre}_bx", (1, H)), (f"{pre}_Ux", (H, H))]
    out += [("ff_state_W", (C, H)), ("ff_state_b", (1, H))]
    out += [("decoder_W", (E, 2 * H)), ("decoder_b", (1, 2 * H)), ("decoder_U", (H, 2 * H)),
            ("decoder_Wx", (E, H)), ("decoder_bx", (1, H)), ("decoder_Ux", (H, H)),
            ("decoder_U_nl", (H, 2 * H)), ("decoder_b_nl", (1, 2 * H)),
            ("decoder_Ux_nl", (H, H)), ("decoder_bx_nl", (1, H)),
            ("decoder_Wc", (C, 2 * H)), ("decoder_Wcx", (C, H)),
            ("decoder_W_comb_att", (H, C)), ("decoder_Wc_att", (C, C)), ("decoder_b_att", (1, C)),
            ("decoder_U_att", (C, 1)), ("decoder_c_tt", (1, 1))]
    out += [("ff_logit_lstm_W", (H, ro)), ("ff_logit_lstm_b", (1, ro)),
            ("ff_logit_prev_W", (E, ro)), ("ff_logit_prev_b", (1, ro)),
            ("ff_logit_ctx_W", (C, ro)), ("ff_logit_ctx_b", (1, ro)),
            ("ff_logit_W", (E, d.vocab_tgt)), ("ff_logit_b", (1, d.vocab_tgt))]
    return out


def _rng(seed: int, name: str) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, zlib.crc32(name.encode())])))


def _ortho(rng: np.random.Generator, n: int) -> np.ndarray:
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return (q * np.sign(np.diag(r))).astype(np.float32)


# nominal E[t^2] of the readout output, used only to scale W_o
_T_SECOND_MOMENT = {"tanh": 0.6, "maxout": 3.0}


def make_model(d: Dims, seed: int, logit_std: float = 1.0) -> Dict[str, np.ndarray]:
    """Seeded random-weight DL4MT/Nematus cGRU model as float32 arrays (Nematus names)."""
    H = d.dim_hid
    p: Dict[str, np.ndarray] = {}
    for name, (rows, cols) in param_shapes(d):
        g = _rng(seed, name)
        if name in ("Wemb", "Wemb_dec"):
            a = g.standard_normal((rows, cols), dtype=np.float32)
        elif name.endswith("_U") or name.endswith("_U_nl"):
            a = np.concatenate([_ortho(g, H), _ortho(g, H)], axis=1)
        elif name.endswith("_Ux") or name.endswith("_Ux_nl"):
            a = _ortho(g, H)
        elif name == "decoder_U_att":
            a = (g.standard_normal((rows, cols)) * (2.0 / np.sqrt(rows))).astype(np.float32)
        elif name == "ff_logit_W":
            sigma = logit_std / np.sqrt(d.dim_emb * _T_SECOND_MOMENT[d.readout])
            a = (g.standard_normal((rows, cols), dtype=np.float32) * np.float32(sigma))
        elif name == "ff_logit_b":
            a = (-np.log(np.arange(1, cols + 1, dtype=np.float64))).astype(np.float32)[None, :]
        elif rows == 1:  # biases (incl. c_tt)
            a = (g.standard_normal((rows, cols)) * 0.1).astype(np.float32)
        else:  # linear maps ~ N(0, 1/fan_in)
            a = (g.standard_normal((rows, cols), dtype=np.float32) * np.float32(1.0 / np.sqrt(rows)))
        p[name] = np.ascontiguousarray(a, dtype=np.float32)
    return p


def zero_model(d: Dims) -> Dict[str, np.ndarray]:
    return {n: np.zeros(s, np.float32) for n, s in param_shapes(d)}


def zipf_ids(rng: np.random.Generator, n: int, vocab: int, a: float = 1.1) -> np.ndarray:
    """n token ids = 1 + zipf(a), resampled while >= vocab: ids in [2, vocab)."""
    out = np.empty(n, np.int32)
    filled = 0
    while filled < n:
        z = 1 + rng.zipf(a, size=2 * (n - filled) + 8)
        z = z[z < vocab]
        k = min(len(z), n - filled)
        out[filled:filled + k] = z[:k]
        filled += k
    return out


def make_source(vocab_src: int, n_words: int, seed: int) -> np.ndarray:
    """Synthetic BPE source of n_words Zipf ids followed by EOS (caller appends EOS, A11)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.concatenate([zipf_ids(rng, n_words, vocab_src), np.array([EOS], np.int32)]).astype(np.int32)


def make_states(n: int, dim_hid: int, vocab_tgt: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """Injected synthetic parent states s ~ tanh(N(0,1)) (float32) and previous words y ~ Zipf."""
    rng = np.random.Generator(np.random.PCG64(seed))
    s = np.tanh(rng.standard_normal((n, dim_hid))).astype(np.float32)
    y = zipf_ids(rng, n, vocab_tgt)
    return s, y


def make_candidates(n_parents: int, per_parent: int, vocab_tgt: int, seed: int,
                    distinct: bool = True) -> Tuple[np.ndarray, np.ndarray]:
    """CSR candidate lists: offsets [n_parents+1], words [n_parents*per_parent] (Zipf ids)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    words = np.empty((n_parents, per_parent), np.int32)
    for i in range(n_parents):
        if distinct:
            row: List[int] = []
            while len(row) < per_parent:
                for w in zipf_ids(rng, per_parent, vocab_tgt):
                    if int(w) not in row and len(row) < per_parent:
                        row.append(int(w))
            words[i] = row
        else:
            words[i] = zipf_ids(rng, per_parent, vocab_tgt)
    offsets = np.arange(0, n_parents * per_parent + 1, per_parent, dtype=np.int32)
    return offsets, words.reshape(-1)


# ---------------------------------------------------------------------------------------------
# C3 stack-decoding request stream: phrase expansions (h, t) of a stack,
# realised as a sequence of per-depth (parent, candidate) requests over a prefix forest.
# ---------------------------------------------------------------------------------------------
_PHRASE_LEN_P = np.array([.35, .30, .20, .10, .05])
_BRANCH_BY_DEPTH = [6, 3, 2, 2, 1]


def make_stack_expansions(n_expansions: int, n_hyps: int, vocab_tgt: int, seed: int
                          ) -> List[Tuple[int, Tuple[int, ...]]]:
    """Distinct (hypothesis index, target phrase) pairs, hypothesis drawn as zipf(1.3) mod n_hyps.

    Each phrase word at depth k is drawn from a per-(hyp, prefix) candidate set of size
    _BRANCH_BY_DEPTH[k] (PAPER.md:187 - branching shrinks with depth), Zipf(1.1) ids.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    cand_sets: Dict[Tuple[int, Tuple[int, ...]], np.ndarray] = {}
    seen = set()
    out: List[Tuple[int, Tuple[int, ...]]] = []
    guard = 0
    while len(out) < n_expansions and guard < 50 * n_expansions:
        guard += 1
        h = int((rng.zipf(1.3) - 1) % n_hyps)
        L = int(rng.choice(5, p=_PHRASE_LEN_P)) + 1
        prefix: Tuple[int, ...] = ()
        for k in range(L):
            key = (h, prefix)
            if key not in cand_sets:
                cand_sets[key] = zipf_ids(rng, _BRANCH_BY_DEPTH[k], vocab_tgt)
            cs = cand_sets[key]
            prefix = prefix + (int(cs[rng.integers(len(cs))]),)
        if (h, prefix) not in seen:
            seen.add((h, prefix))
            out.append((h, prefix))
    return out


# ---------------------------------------------------------------------------------------------
# Params container (concrete form of SPEC.md:239):
#   "NMTPARAMS 1\n" "dims E H Vs Vt readout=<r> eos=0 unk=1\n" "arrays n\n" "<name> <rows> <cols>\n"...
#   then zero padding to a 64-byte boundary, then the float32 LE payload in header order.
# ---------------------------------------------------------------------------------------------

def params_bytes(d: Dims, params: Dict[str, np.ndarray]) -> bytes:
    names = [n for n, _ in param_shapes(d)]
    hdr = [f"NMTPARAMS 1", f"dims {d.dim_emb} {d.dim_hid} {d.vocab_src} {d.vocab_tgt} "
           f"readout={d.readout} eos={EOS} unk={UNK}", f"arrays {len(names)}"]
    for n in names:
        a = params[n]
        hdr.append(f"{n} {a.shape[0]} {a.shape[1]}")
    head = ("\n".join(hdr) + "\n").encode()
    head += b"\0" * ((-len(head)) % 64)
    body = b"".join(np.ascontiguousarray(params[n], dtype="<f4").tobytes() for n in names)
    return head + body


def write_params(path: str, d: Dims, params: Dict[str, np.ndarray]) -> None:
    with open(path, "wb") as f:
        f.write(params_bytes(d, params))


def read_params(path_or_bytes) -> Tuple[Dims, Dict[str, np.ndarray]]:
    """Parse the container (used by tests to round-trip; no model arithmetic)."""
    if isinstance(path_or_bytes, (bytes, bytearray)):
        buf = bytes(path_or_bytes)
    else:
        with open(path_or_bytes, "rb") as f:
            buf = f.read()
    lines: List[str] = []
    pos = 0
    while True:
        nl = buf.index(b"\n", pos)
        lines.append(buf[pos:nl].decode())
        pos = nl + 1
        if len(lines) >= 3 and len(lines) == 3 + int(lines[2].split()[1]):
            break
    assert lines[0] == "NMTPARAMS 1"
    f = lines[1].split()
    kv = dict(x.split("=") for x in f[5:])
    d = Dims(int(f[1]), int(f[2]), int(f[3]), int(f[4]), kv["readout"])
    pos += (-pos) % 64
    out: Dict[str, np.ndarray] = {}
    for ln in lines[3:]:
        n, r, c = ln.split()
        r, c = int(r), int(c)
        out[n] = np.frombuffer(buf, "<f4", r * c, pos).reshape(r, c).copy()
        pos += 4 * r * c
    return d, out
