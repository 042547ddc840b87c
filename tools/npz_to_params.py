"""Nematus / DL4MT .npz checkpoint -> params container (include/nmt.h).

Arrays keep their Nematus names (the container's names are the Nematus ones); 1-D
biases become 1 x n rows, c_tt a 1 x 1 array; the readout type follows from ff_logit_lstm_W's width
(E -> tanh, 2E -> maxout).  Extra arrays (optimizer state, "zipped_params", "history_errs", ...)
are ignored.

Test-time dropout (reading A17): DL4MT's dropout_layer is NOT inverted - at test time it multiplies
the readout t by the retain probability (0.5 in DL4MT session 3) before the output layer.  Pass
--readout-retain p to fold it into ff_logit_W (t.(pW) = (p t).W; b_o is added after the product and
stays).  Other dropout placements (Nematus embedding/hidden dropout) are not folded.

usage: python tools/npz_to_params.py model.npz out.params [--readout-retain 0.5]
"""
import argparse
import os
import sys
from typing import Dict, Optional

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402  (the container writer; no model arithmetic)


def convert(arrays: Dict[str, np.ndarray], readout_retain: Optional[float] = None) -> bytes:
    E = arrays["Wemb"].shape[1]
    H = arrays["encoder_Ux"].shape[0]
    ro = "maxout" if arrays["ff_logit_lstm_W"].shape[1] == 2 * E else "tanh"
    d = synth.Dims(E, H, arrays["Wemb"].shape[0], arrays["Wemb_dec"].shape[0], ro)
    out: Dict[str, np.ndarray] = {}
    for name, (r, c) in synth.param_shapes(d):
        if name not in arrays:
            raise KeyError(f"missing parameter {name}")
        a = np.asarray(arrays[name], dtype=np.float32)
        if a.size != r * c:
            raise ValueError(f"{name}: expected {r}x{c}, got {a.shape}")
        out[name] = a.reshape(r, c)
    if readout_retain is not None:
        out["ff_logit_W"] = (out["ff_logit_W"].astype(np.float64) * readout_retain).astype(np.float32)
    return synth.params_bytes(d, out)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("npz")
    ap.add_argument("out")
    ap.add_argument("--readout-retain", type=float, default=None)
    a = ap.parse_args()
    with np.load(a.npz) as z:
        blob = convert({k: z[k] for k in z.files}, a.readout_retain)
    with open(a.out, "wb") as f:
        f.write(blob)


if __name__ == "__main__":
    main()
