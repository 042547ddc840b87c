"""CPU checks of nmt_random_params (the library's seeded synthetic-model generator, SURVEY §8(d);
host only, no GPU): container format, determinism, and the distributions the recipe fixes -
orthogonal recurrent blocks (Q^T Q = I), b_o = -ln(w + 1) exactly, and the stated standard
deviations (within sampling error).  The generator is input-only: it holds no model arithmetic."""
import numpy as np
import pytest

import oracle as O
import synth


def nmt():
    from paper_1605_04809_b200 import nmt as m
    return m


@pytest.fixture(scope="module")
def small():
    b = nmt().random_params(64, 128, 3000, 4000, "maxout", seed=11, logit_std=2.0)
    return b, synth.read_params(b)


def test_container_round_trips_through_synth(small):
    b, (d, p) = small
    assert d == synth.Dims(64, 128, 3000, 4000, "maxout")
    assert [n for n, _ in synth.param_shapes(d)] == list(p.keys())
    for n, shp in synth.param_shapes(d):
        assert p[n].shape == shp, n
    # re-serialising the parsed arrays with synth gives the same bytes
    assert synth.params_bytes(d, p) == b


def test_deterministic_and_seed_dependent(small):
    b, _ = small
    assert nmt().random_params(64, 128, 3000, 4000, "maxout", seed=11, logit_std=2.0) == b
    assert nmt().random_params(64, 128, 3000, 4000, "maxout", seed=12, logit_std=2.0) != b


def test_recurrent_blocks_are_orthogonal(small):
    _, (d, p) = small
    H = d.dim_hid
    for n in ("encoder_U", "encoder_r_U", "decoder_U", "decoder_U_nl"):
        for blk in (p[n][:, :H], p[n][:, H:]):
            q = blk.astype(np.float64)
            assert np.abs(q.T @ q - np.eye(H)).max() < 1e-5, n
    for n in ("encoder_Ux", "encoder_r_Ux", "decoder_Ux", "decoder_Ux_nl"):
        q = p[n].astype(np.float64)
        assert np.abs(q.T @ q - np.eye(H)).max() < 1e-5, n
    # the two blocks of U are independent draws
    assert np.abs(p["decoder_U"][:, :H] - p["decoder_U"][:, H:]).max() > 0.1


def test_distributions(small):
    _, (d, p) = small
    E, H = d.dim_emb, d.dim_hid

    def sd_ok(a, sd, rel=0.05):
        a = a.astype(np.float64).ravel()
        assert abs(a.mean()) < 5 * sd / np.sqrt(a.size)
        assert abs(a.std() / sd - 1) < rel, (a.std(), sd)

    sd_ok(p["Wemb"], 1.0)
    sd_ok(p["Wemb_dec"], 1.0)
    sd_ok(p["encoder_W"], 1 / np.sqrt(E))
    sd_ok(p["decoder_Wc_att"], 1 / np.sqrt(2 * H))
    sd_ok(p["ff_state_W"], 1 / np.sqrt(2 * H))
    sd_ok(p["decoder_U_att"], 2 / np.sqrt(2 * H), rel=0.15)
    sd_ok(np.concatenate([p[n].ravel() for n in ("encoder_b", "decoder_b", "decoder_b_nl", "ff_logit_lstm_b")]),
          0.1, rel=0.1)
    sd_ok(p["ff_logit_W"], 2.0 / np.sqrt(E * 3.0))  # maxout: nominal E[t^2] = 3
    w = np.arange(d.vocab_tgt)
    assert np.array_equal(p["ff_logit_b"][0], (-np.log(w + 1.0)).astype(np.float32))


def test_oracle_runs_on_generated_model(small):
    _, (d, p) = small
    om = O.Model(d, p)
    src = synth.make_source(d.vocab_src, 6, seed=2)
    sess = O.Session(om, src)
    full = sess.logprobs_full(0)
    assert abs(np.exp(full).sum() - 1) < 1e-9


def test_bad_dims_rejected():
    N = nmt()
    with pytest.raises(N.NmtError) as e:
        N.random_params(0, 16, 50, 50)
    assert e.value.name == "NMT_ERR_INVALID_ARG"
    with pytest.raises(N.NmtError):
        N.random_params(8, 16, 50, 50, logit_std=-1.0)
