"""tools/npz_to_params.py: a Nematus-shaped .npz (1-D biases, (2H,1) U_att,
(1,) c_tt, extra non-parameter arrays) converts to exactly the container synth writes for the same
arrays; the DL4MT test-time dropout fold scales only ff_logit_W (reading A17) and leaves the
oracle's log-probs equal to scaling the readout t by the retain probability."""
import io
import os
import sys

import numpy as np
import pytest

import oracle as O
import synth

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import npz_to_params  # noqa: E402


def _nematus_npz(d, p):
    arrs = {}
    for name, (r, c) in synth.param_shapes(d):
        a = p[name]
        arrs[name] = a.reshape(-1) if r == 1 and name != "decoder_c_tt" else a
    arrs["decoder_c_tt"] = p["decoder_c_tt"].reshape(1)
    arrs["history_errs"] = np.zeros(3)
    buf = io.BytesIO()
    np.savez(buf, **arrs)
    buf.seek(0)
    with np.load(buf) as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("readout", ["tanh", "maxout"])
def test_npz_converts_to_the_same_container(readout):
    d = synth.Dims(8, 16, 50, 60, readout)
    p = synth.make_model(d, 3)
    blob = npz_to_params.convert(_nematus_npz(d, p))
    assert blob == synth.params_bytes(d, p)


def test_missing_and_misshaped_arrays_are_named():
    d = synth.Dims(8, 16, 50, 60, "tanh")
    arrs = _nematus_npz(d, synth.make_model(d, 3))
    bad = dict(arrs)
    del bad["decoder_Wcx"]
    with pytest.raises(KeyError, match="decoder_Wcx"):
        npz_to_params.convert(bad)
    bad = dict(arrs)
    bad["decoder_b_att"] = np.zeros(5, np.float32)
    with pytest.raises(ValueError, match="decoder_b_att"):
        npz_to_params.convert(bad)


def test_readout_dropout_fold():
    d = synth.Dims(8, 16, 50, 60, "tanh")
    p = synth.make_model(d, 3)
    d2, q = synth.read_params(npz_to_params.convert(_nematus_npz(d, p), readout_retain=0.5))
    for n in p:
        if n == "ff_logit_W":
            assert np.array_equal(q[n], (p[n].astype(np.float64) * 0.5).astype(np.float32))
        else:
            assert np.array_equal(q[n], p[n]), n
    # log p with the folded W_o == log p with t scaled by 0.5 (non-inverted dropout at test time)
    src = synth.make_source(d.vocab_src, 4, seed=1)
    c = O.encode(O.Model(d, p), src)
    out = O.step(O.Model(d, p), c, c.s0[None, :], [-1])
    z_scaled = 0.5 * out["t"][0] @ p["ff_logit_W"].astype(np.float64) + p["ff_logit_b"][0]
    c2 = O.encode(O.Model(d2, q), src)
    out2 = O.step(O.Model(d2, q), c2, c2.s0[None, :], [-1])
    assert np.allclose(O.log_softmax(out2["z"][0]), O.log_softmax(z_scaled), atol=1e-6)
