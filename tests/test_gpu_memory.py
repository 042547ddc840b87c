"""The §8(b) memory boundary (include/nmt.h nmt_opts): the library's device memory comes through the
caller's allocator hook (PyTorch's caching allocator through the binding) or a private pool, and the
state arenas obey the arena_bytes budget (NMT_ERR_CAPACITY before any output is written).  The paper's
own limit was GPU memory."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def nmt():
    from paper_1605_04809_b200 import nmt as m
    return m


def test_torch_allocator_holds_the_library_memory():
    import torch
    d = synth.Dims(500, 1024, 50000, 100000, "maxout")
    blob = synth.params_bytes(d, synth.make_model(d, 2016))
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    n0, b0 = nmt().device_allocations()
    lo0 = nmt().live_objects()
    M = nmt().Model(blob, precision="bf16", allocator="torch")
    after_load = torch.cuda.memory_allocated()
    mem = M.memory()
    assert after_load - base >= 2 << 30, (base, after_load)  # weights + precomputed tables (> 2 GB)
    assert mem["live"] <= after_load - base + (64 << 20)
    src = synth.make_source(d.vocab_src, 49, seed=1)
    R = 4096
    s, y = synth.make_states(R, d.dim_hid, d.vocab_tgt, seed=2)
    off, words = synth.make_candidates(R, 3, d.vocab_tgt, seed=3)
    c = M.encode(src)
    lp, _, _ = c.score_batch(c.inject_states(s, y), off, words)
    assert np.all(np.isfinite(lp))
    after_step = torch.cuda.memory_allocated()
    assert after_step > after_load  # the step workspace and the grown arena came from torch
    assert M.memory()["arena"] > 0
    c.close()
    assert nmt().live_objects() == (lo0[0] + 1, lo0[1] + 1)  # the released context is pooled
    M.close()
    torch.cuda.synchronize()
    assert nmt().live_objects() == lo0, (lo0, nmt().live_objects())
    assert nmt().device_allocations() == (n0, b0), (n0, b0, nmt().device_allocations())  # all freed
    assert torch.cuda.memory_allocated() - base < 16 << 20, torch.cuda.memory_allocated() - base


def test_private_pool_leaves_torch_alone():
    import torch
    d = synth.TINY
    blob = synth.params_bytes(d, synth.make_model(d, 7))
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    M = nmt().Model(blob, precision="fp32class", allocator=None)
    c = M.encode(synth.make_source(d.vocab_src, 4, seed=1))
    lp, _, _ = c.score_batch([0], [0, 3], [5, 9, 2])
    assert np.all(np.isfinite(lp))
    assert torch.cuda.memory_allocated() == base
    assert M.memory()["live"] > 0 and M.memory()["peak"] >= M.memory()["live"]


def test_arena_budget_capacity_error_and_pool_trim():
    N = nmt()
    d = synth.TINY
    blob = synth.params_bytes(d, synth.make_model(d, 7))
    probe = N.Model(blob, precision="fp32class")
    c0 = probe.encode(synth.make_source(d.vocab_src, 4, seed=1))
    one_ctx = probe.memory()["arena"]  # bytes of one fresh context (fixed part + initial arena)
    c0.close()
    probe.close()
    M = N.Model(blob, precision="fp32class", arena_bytes=int(one_ctx * 1.5))
    src = synth.make_source(d.vocab_src, 4, seed=1)
    c = M.encode(src)
    ref, _, _ = c.score_batch([0], [0, 3], [5, 9, 2])
    s, y = synth.make_states(2000, d.dim_hid, d.vocab_tgt, seed=4)  # needs > 1024 state slots: growth
    with pytest.raises(N.NmtError) as e:
        c.inject_states(s, y)
    assert e.value.name == "NMT_ERR_CAPACITY" and "arena" in str(e.value)
    assert c.stats() == (1 + 3, 1)  # nothing was added
    with pytest.raises(N.NmtError) as e:
        M.encode(src)  # a second live context does not fit either
    assert e.value.name == "NMT_ERR_CAPACITY"
    lp, _, _ = c.score_batch([0], [0, 3], [5, 9, 2])  # the context still works
    assert np.array_equal(lp, ref)
    c.close()
    c2 = M.encode(src)  # reuses the released arena
    assert np.array_equal(c2.score_batch([0], [0, 3], [5, 9, 2])[0], ref)
    assert M.memory()["arena"] <= int(one_ctx * 1.5)
    c2.close()
    big = N.Model(blob, precision="fp32class", arena_bytes=int(one_ctx * 3.5))
    cs = [big.encode(src) for _ in range(2)]
    for x in cs:
        x.close()  # two pooled arenas
    c3 = big.encode(src)  # reuses one; growth below frees the other pooled arena to stay in budget
    ids = c3.inject_states(s[:1500], y[:1500])
    assert len(ids) == 1500 and big.memory()["arena"] <= int(one_ctx * 3.5)


def test_max_src_len_checked_against_attention_shared_memory():
    N = nmt()
    d = synth.Dims(8, 1024, 50, 50, "tanh")
    blob = synth.params_bytes(d, synth.make_model(d, 7))
    with pytest.raises(N.NmtError) as e:
        N.Model(blob, precision="bf16", max_src_len=4000)
    assert e.value.name == "NMT_ERR_INVALID_ARG" and "shared memory" in str(e.value)
