"""Readers for tests/golden/*.txt fixtures (each file states its citation)."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(line.split())
    return rows


def read_tables(name):
    """{theta(float): [(oh, ow), ...]} from rows 'theta k oh ow'."""
    out = {}
    for th, k, oh, ow in read_rows(name):
        out.setdefault(float(th), {})[int(k)] = (int(oh), int(ow))
    return {th: [d[k] for k in sorted(d)] for th, d in out.items()}
