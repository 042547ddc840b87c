"""Checkpoint averaging, NMT-k-Avg ("the element-wise average of all model weights in
the NMT ensembles"): nmt_params_average on the GPU against the float64 oracle's average_params, and
the averaged model's scores against the oracle run on the averaged weights."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu


def _ulp_diff(a: np.ndarray, b: np.ndarray) -> int:
    """max distance in fp32 ulps (equal values, including -0 == +0, are 0 apart)"""
    a = a.astype(np.float32)
    b = b.astype(np.float32)
    ia = a.view(np.int32).astype(np.int64)
    ib = b.view(np.int32).astype(np.int64)
    return int(np.max(np.where(a == b, 0, np.abs(ia - ib))))


@pytest.mark.parametrize("k", [2, 3, 4])
def test_average_matches_oracle_within_one_ulp(k):
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(8, 16, 50, 50, "maxout")
    members = [synth.make_model(d, 100 + i) for i in range(k)]
    blob = nmt.params_average([synth.params_bytes(d, m) for m in members])
    dd, avg = synth.read_params(blob)
    assert dd == d
    ref = O.average_params(members)  # float64 mean; the library returns fp32(fp64 sum / k)
    for name in ref:
        assert _ulp_diff(avg[name], ref[name].astype(np.float32)) <= 1, name


def test_average_of_identical_members_is_the_member():
    from paper_1605_04809_b200 import nmt
    d = synth.TINY
    blob = synth.params_bytes(d, synth.make_model(d, 11))
    assert nmt.params_average([blob, blob, blob, blob]) == blob  # 4x / 4 is exact


@pytest.mark.parametrize("prec", ["fp32class", "bf16"])
def test_averaged_model_scores_match_oracle(prec):
    from paper_1605_04809_b200 import nmt
    d = synth.Dims(8, 16, 50, 50, "tanh")
    members = [synth.make_model(d, 200 + i) for i in range(4)]
    blob = nmt.params_average([synth.params_bytes(d, m) for m in members])
    _, avg = synth.read_params(blob)
    M = nmt.Model(blob, precision=prec)
    src = synth.make_source(d.vocab_src, 6, seed=5)
    ctx = M.encode(src)
    words = np.array([2, 7, 11, 0], np.int32)
    lp, _, _ = ctx.score_batch([ctx.root], [0, 4], words)
    om = O.Model(d, avg)
    c = O.encode(om, src)
    st = O.step(om, c, c.s0[None, :], [O.BOS])
    ref = st["z"][0, words] - st["logZ"][0]
    tol = 1e-3 if prec == "fp32class" else 2e-2
    assert np.max(np.abs(np.asarray(lp) - ref)) < tol
