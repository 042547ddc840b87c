"""The oracle's pins bite: each plausible mistake in tools/mutate_oracle.py (query or GRU2 state from
s instead of s1, transposed pctx, unweighted mode-0 combine, maxout pairing, u on the new state, ...)
makes tests/test_oracle.py fail (VERDICT r01 "What's weak" #2)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_oracle_mutation_is_killed():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "mutate_oracle.py")], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "SURVIVED" not in r.stdout
