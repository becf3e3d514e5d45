"""The north-star parity statistic (BASELINE.json north_star; SURVEY.md §7 hard
part 2): per input, ||got - ref||inf / ||ref||inf against the CPU fp32
logits, and top-1 agreement -- raw, and restricted to the inputs whose fp32
top-1 margin exceeds twice that input's measured error (where a 16-bit path
can be expected to decide the same class).  Used by the GPU parity tests and
the bench's ``parity`` block; it only compares arrays (no oracle code here).
"""

from __future__ import annotations

import numpy as np

TOL = 2e-2              # max relative error, north star
TOP1_MIN = 0.999        # identical top-1 on >= 99.9 % of inputs, north star


def stats(got: np.ndarray, ref: np.ndarray) -> dict:
    """got, ref: (n, classes).  Returns the statistic as plain floats/ints."""
    got = np.asarray(got, np.float64).reshape(len(got), -1)
    ref = np.asarray(ref, np.float64).reshape(len(ref), -1)
    scale = np.abs(ref).max(axis=1)
    err = np.abs(got - ref).max(axis=1) / np.maximum(scale, 1e-30)
    top_ref, top_got = ref.argmax(1), got.argmax(1)
    srt = np.sort(ref, axis=1)
    margin = (srt[:, -1] - srt[:, -2]) / np.maximum(scale, 1e-30)
    decided = margin > 2 * err
    agree = top_ref == top_got
    n = len(ref)
    return {
        "n": int(n),
        "max_rel_err": float(err.max()) if n else 0.0,
        "p99_rel_err": float(np.quantile(err, 0.99)) if n else 0.0,
        "mean_rel_err": float(err.mean()) if n else 0.0,
        "top1_raw": float(agree.mean()) if n else 1.0,
        "top1_mismatches": int((~agree).sum()),
        "top1_margin_filtered": float(agree[decided].mean()) if decided.any() else 1.0,
        "margin_filtered_n": int(decided.sum()),
        "mismatch_margins": [float(m) for m in margin[~agree][:8]],
    }


def passes(s: dict) -> bool:
    return s["max_rel_err"] <= TOL and s["top1_raw"] >= TOP1_MIN and s["top1_margin_filtered"] == 1.0
