"""Shared helpers for the tests (golden fixture parsing)."""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden_lines(name):
    """Non-comment, non-empty lines of tests/golden/<name>."""
    out = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            s = line.strip()
            if s and not s.startswith("#"):
                out.append(s)
    return out


def golden_kv(name):
    """key -> list of numeric tokens (stops at the first non-numeric token)."""
    d = {}
    for s in golden_lines(name):
        toks = s.split()
        vals = []
        for t in toks[1:]:
            try:
                vals.append(float(t))
            except ValueError:
                break
        d[toks[0]] = vals
    return d
