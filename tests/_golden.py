"""Reader for tests/golden/*.txt fixtures (values written by hand from the
paper's equations; each file states its derivation and citation)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    out = {}
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, _, rest = line.partition(" ")
            if key == "edges":
                pairs = [p.split() for p in rest.split(";")]
                out[key] = [(int(a), int(b)) for a, b in pairs]
            elif key == "n":
                out[key] = int(rest)
            else:
                vals = [float(v) for v in rest.split()]
                out[key] = vals[0] if len(vals) == 1 else np.array(vals)
    return out


def csr_from_edges(n, edges, w=None):
    """CSR by source from an (s, t) list, preserving input order within a row."""
    src = np.array([e[0] for e in edges], dtype=np.int64)
    dst = np.array([e[1] for e in edges], dtype=np.int32)
    order = np.argsort(src, kind="stable")
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=row_ptr[1:])
    ww = None if w is None else np.asarray(w, dtype=np.float64)[order]
    return row_ptr, dst[order], ww
