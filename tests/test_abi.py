"""CPU checks of the C-ABI boundary: libnmt.so builds for sm_100a, loads without a GPU, exports every
symbol include/nmt.h declares, and the binding's symbol table matches the header."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nmt.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"NMT_API\s+[\w\s\*]*?\b(nmt_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1605_04809_b200 import build
    return build.build()


def test_header_declares_the_north_star_calls():
    syms = header_symbols()
    for s in ("nmt_load", "nmt_encode", "nmt_score_batch", "nmt_ensemble_combine", "nmt_last_error"):
        assert s in syms


def test_library_loads_and_exports_every_header_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for s in header_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (nmt_\w+)", out))
    assert set(header_symbols()) <= exported
    # nothing but the C ABI is exported
    assert all(s.startswith("nmt_") for s in exported)


def test_binding_matches_header():
    from paper_1605_04809_b200 import nmt
    assert sorted(nmt.EXPORTS) == header_symbols()


def test_sass_is_sm100a_tcgen05(libpath):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", libpath], capture_output=True,
                                       text=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass                      # TMA tile loads
    assert "LDTM" in sass                         # tcgen05.ld


def test_no_gpu_calls_fail_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1605_04809_b200 import nmt
    import synth
    with pytest.raises(nmt.NmtError) as e:
        nmt.Model(synth.params_bytes(synth.TINY, synth.make_model(synth.TINY, 7)))
    assert e.value.name == "NMT_ERR_CUDA"


def test_params_errors_are_named():
    """Header validation happens before any device work, so it is testable without a GPU."""
    import numpy as np
    from paper_1605_04809_b200 import nmt
    import synth
    d = synth.TINY
    p = synth.make_model(d, 7)
    q = dict(p)
    del q["decoder_W_comb_att"]
    names = [n for n, _ in synth.param_shapes(d) if n != "decoder_W_comb_att"]
    hdr = "NMTPARAMS 1\ndims 8 16 50 50 readout=tanh eos=0 unk=1\narrays %d\n" % len(names)
    hdr += "".join(f"{n} {q[n].shape[0]} {q[n].shape[1]}\n" for n in names)
    blob = hdr.encode()
    blob += b"\0" * ((-len(blob)) % 64) + b"".join(q[n].astype("<f4").tobytes() for n in names)
    with pytest.raises(nmt.NmtError) as e:
        nmt.Model(blob)
    assert e.value.name == "NMT_ERR_MISSING_PARAM" and "decoder_W_comb_att" in str(e.value)
    q = dict(p)
    q["decoder_Ux"] = np.zeros((16, 15), np.float32)
    blob = synth.params_bytes(d, q)
    with pytest.raises(nmt.NmtError) as e:
        nmt.Model(blob)
    assert e.value.name == "NMT_ERR_SHAPE" and "decoder_Ux" in str(e.value)
    blob = synth.params_bytes(d, p)
    with pytest.raises(nmt.NmtError) as e:
        nmt.Model(blob[:-4])
    assert e.value.name == "NMT_ERR_FORMAT"
    with pytest.raises(nmt.NmtError) as e:
        nmt.Model("/nonexistent/params.bin")
    assert e.value.name == "NMT_ERR_IO"


def test_params_average_validates_before_device_work():
    """nmt_params_average: headers must match; errors are named, no GPU needed."""
    from paper_1605_04809_b200 import nmt
    import synth
    d = synth.TINY
    a = synth.params_bytes(d, synth.make_model(d, 3))
    other = synth.Dims(8, 16, 50, 50, "maxout")
    b = synth.params_bytes(other, synth.make_model(other, 4))
    with pytest.raises(nmt.NmtError) as e:
        nmt.params_average([a, b])
    assert e.value.name == "NMT_ERR_SHAPE" and "member 1" in str(e.value) and "readout" in str(e.value)
    with pytest.raises(nmt.NmtError) as e:
        nmt.params_average([a, a[:-4]])
    assert e.value.name == "NMT_ERR_FORMAT"
    with pytest.raises(nmt.NmtError) as e:
        nmt.params_average([])
    assert e.value.name == "NMT_ERR_INVALID_ARG"


def test_no_unresolved_library_internal_symbols(libpath):
    """every internal C++ symbol of the library is defined in it (an undefined nmt:: symbol would only
    fail at dlopen time on the GPU box)"""
    out = subprocess.run(["nm", "-D", "--undefined-only", libpath], capture_output=True, text=True).stdout
    bad = [ln for ln in out.splitlines() if "nmt" in ln or "ens_" in ln]
    assert not bad, bad
