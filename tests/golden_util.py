"""Loading helpers for the committed golden vectors (tests/golden/*.npz)."""
import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_case(name):
    z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
    d = {k: z[k] for k in z.files}
    d["params"] = json.loads(str(d["params"]))
    return d


def oracle_plan(case):
    from oracle.bst_oracle import OraclePlan
    p = case["params"]
    n_ang, n_t = case["sino"].shape
    f = p["filter"]
    roll = f.get("rolloff", 1.0) if f.get("kind", "ramp") == "ramp_apodized" else 1.0
    return OraclePlan(n_t=n_t, n_theta=p["n_theta"], rolloff=roll, **p["plan"])


def _wide(a):
    a = np.asarray(a)
    return a.astype(np.complex128 if np.iscomplexobj(a) else np.float64)


def rel_l2(a, b):
    return float(np.linalg.norm(_wide(a) - b) / np.linalg.norm(b))


def max_rel(a, b):
    return float(np.max(np.abs(_wide(a) - b)) / np.max(np.abs(b)))
