"""Shared test helpers: fixture loading and the reference's error metric."""
import json
import os

import numpy as np

from pyoracle import Plan

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def scaled_max_err(a, b) -> float:
    """oracle_helpers.hpp:43-53: max|a-b| / max(1, max|a|, max|b|)."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    if a.size == 0:
        return 0.0
    scale = max(1.0, float(np.abs(a).max()), float(np.abs(b).max()))
    return float(np.abs(a - b).max()) / scale


def load_plans():
    with open(os.path.join(GOLDEN, "plans.json")) as f:
        return json.load(f)


def small_cases():
    z = np.load(os.path.join(GOLDEN, "small_cases.npz"))
    cases = []
    for n in range(int(z["count"][0])):
        pre = f"c{n}_"
        rows, emb, d, pooling, is64 = (int(x) for x in z[pre + "plan"])
        plan = Plan(rows, emb, list(z[pre + "rf"]), list(z[pre + "cf"]), list(z[pre + "rk"]))
        cases.append(dict(
            plan=plan, pooling=pooling, dtype=np.float64 if is64 else np.float32,
            cores=[z[pre + f"core{k}"] for k in range(d)],
            grads=[z[pre + f"grad{k}"] for k in range(d)],
            after=[z[pre + f"after{k}"] for k in range(d)],
            idx=z[pre + "idx"], off=z[pre + "off"],
            w=z[pre + "w"] if (pre + "w") in z else None,
            grad_out=z[pre + "grad_out"], fwd=z[pre + "fwd"]))
    return cases


def cfg1():
    z = np.load(os.path.join(GOLDEN, "cfg1.npz"))
    plan = Plan(1000000, 16, [100, 100, 100], [2, 2, 4], [1, 16, 16, 1])
    return plan, {k: z[k] for k in z.files}


def cache_case():
    z = np.load(os.path.join(GOLDEN, "cache_case.npz"))
    return {k: z[k] for k in z.files}


CFG2 = Plan(10131227, 16, [200, 220, 250], [2, 2, 4], [1, 32, 32, 1])
CFG3 = Plan(40000000, 64, [200, 200, 1000], [4, 4, 4], [1, 64, 64, 1])
