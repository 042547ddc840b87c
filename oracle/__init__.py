"""Float64 CPU oracle (TEST INFRASTRUCTURE: importable only from tests/, smoke() and bench.py's
cpu_baseline / --impl reference legs).  See oracle/nmt_oracle.py for citations and pins."""
from .nmt_oracle import (BOS, Context, Model, Session, average_params, encode, ensemble_combine,  # noqa: F401
                         forest_levels,
                         gru, gru_nl, log_softmax, logsumexp, score_forest, score_sequence, sigmoid, step, topk_words,
                         word_logprob)
