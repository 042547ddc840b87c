"""ScoreBatch (Alg. 1; §5.1) as a thin host driver over nmt_score_batch.

Given a set L of (hypothesis, target phrase) pairs, the paper builds a forest of per-hypothesis
prefix trees and runs ONE forward step per tree depth, so the
number of GPU queries is the maximum phrase length, not the number of words (PAPER.md:109-111,
:181).  Here each depth is one nmt_score_batch call whose parents are the (deduplicated) source
nodes of the depth's edges and whose candidates are the edge labels; the library interns
(parent, word) -> child state and steps each distinct unstepped parent once (parent-indexed rows,
DESIGN.md §2 A13).  All arithmetic happens in libnmt.so; this module only groups ids.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Sequence, Tuple

import numpy as np

Pair = Tuple[int, Tuple[int, ...]]


@dataclasses.dataclass
class ForestStats:
    steps: int                      # nmt_score_batch calls (= max phrase length)
    edges_per_depth: List[int]      # collapsed edges = word-scores per depth
    rows_per_depth: List[int]       # decoder rows actually stepped per depth
    naive_words: int                # total words of all phrases (the naive query count)


def forest_levels(pairs: Sequence[Pair]) -> List[List[Tuple[Pair, int]]]:
    """Distinct forest edges grouped by depth: level i holds ((h, prefix_<i), w_i), in
    (hypothesis, prefix) order so that the paper's E_1/H_0 row order results."""
    levels: List[List[Tuple[Pair, int]]] = []
    seen = set()
    depth = max((len(t) for _, t in pairs), default=0)
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


def score_batch(ctx, hyp_states: Sequence[int], pairs: Sequence[Pair]
                ) -> Tuple[Dict[Pair, Tuple[float, int]], ForestStats]:
    """Score every (h, t) in `pairs` from hypothesis states hyp_states[h] (node handles of ctx).

    Returns {(h, t): (sum of log-probs of t's words, state handle after t)} and the forest stats.
    """
    if any(len(t) == 0 for _, t in pairs):
        raise ValueError("empty expansion")
    node_of: Dict[Pair, int] = {}
    acc: Dict[Pair, float] = {}
    for h, _ in pairs:
        node_of[(h, ())] = int(hyp_states[h])
        acc[(h, ())] = 0.0
    levels = forest_levels(pairs)
    edges, rows = [], []
    for lvl in levels:
        by_parent: Dict[int, List[Tuple[Pair, int]]] = {}
        order: List[int] = []
        for src, w in lvl:
            pn = node_of[src]
            if pn not in by_parent:
                by_parent[pn] = []
                order.append(pn)
            by_parent[pn].append((src, w))
        parents, offsets, words, keys, srcs = [], [0], [], [], []
        for pn in order:
            parents.append(pn)
            for src, w in by_parent[pn]:
                words.append(w)
                srcs.append(src)
                keys.append((src[0], src[1] + (w,)))
            offsets.append(len(words))
        _, stepped0 = ctx.stats()
        logp, child, _ = ctx.score_batch(np.asarray(parents, np.int64), np.asarray(offsets, np.int32),
                                         np.asarray(words, np.int32), with_argmax=False)
        _, stepped1 = ctx.stats()
        for k, src, lp, ch in zip(keys, srcs, logp, child):
            acc[k] = acc[src] + float(lp)
            node_of[k] = int(ch)
        edges.append(len(words))
        rows.append(stepped1 - stepped0)
    out = {(h, tuple(t)): (acc[(h, tuple(t))], node_of[(h, tuple(t))]) for h, t in pairs}
    stats = ForestStats(steps=len(levels), edges_per_depth=edges, rows_per_depth=rows,
                        naive_words=sum(len(t) for _, t in pairs))
    return out, stats
