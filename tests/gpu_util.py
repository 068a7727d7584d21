"""Helpers shared by the GPU parity tests (test infrastructure)."""
import numpy as np


def rel(a, b):
    """Relative ℓ2 difference (real or complex)."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def record(case: str, **vals):
    """Append the achieved parity numbers of a case to $CNPINT_PARITY_LOG (JSON lines), if set —
    the source of profiles/r02_parity.json (scripts/parity_table.py)."""
    import json
    import os
    path = os.environ.get("CNPINT_PARITY_LOG")
    if not path:
        return
    with open(path, "a") as f:
        f.write(json.dumps({"case": case, **{k: (float(v) if isinstance(v, (int, float, np.floating)) else v)
                                             for k, v in vals.items()}}) + "\n")
