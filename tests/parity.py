"""Parity helpers: compare CUDA-path records with oracle results.

Tolerances (BASELINE.json north_star): relative Frobenius
error <= 1e-4 on each H block and on b (denominator max(||b||, ||sum |terms|||)
because b -> 0 near the optimum), relative error <= 1e-5 on the error e;
integer results (inliers, invisible, degenerate counts) bit-exact.
"""
import numpy as np

H_TOL = 1e-4
B_TOL = 1e-4
E_TOL = 1e-5


def rel_fro(a, b, den=None):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    d = np.linalg.norm(b) if den is None else den
    if d == 0:
        return float(np.linalg.norm(a - b))
    return float(np.linalg.norm(a - b) / d)


def compare_factor(rec, ref, levels, what=""):
    """rec: one LINEAR_FACTOR_DTYPE record; ref: oracle.linearize dict."""
    errs = {}
    assert rec["inliers"][:levels].tolist() == ref["inliers"].tolist(), \
        f"{what} inliers {rec['inliers'][:levels]} vs {ref['inliers']}"
    assert int(rec["num_invisible"]) == ref["num_invisible"], what
    assert int(rec["num_degenerate"]) == ref["num_degenerate"], what
    for name, sl in (("H_ii", (slice(0, 6), slice(0, 6))), ("H_ij", (slice(0, 6), slice(6, 12))),
                     ("H_jj", (slice(6, 12), slice(6, 12)))):
        refb = ref["H"][sl]
        e = rel_fro(rec[name].reshape(6, 6), refb)
        errs[name] = e
        assert e <= H_TOL, f"{what} {name} rel err {e:.3g}"
    b = np.concatenate([rec["b_i"], rec["b_j"]])
    den = max(np.linalg.norm(ref["b"]), np.linalg.norm(ref["b_abs"]), 1e-300)
    errs["b"] = rel_fro(b, ref["b"], den)
    assert errs["b"] <= B_TOL, f"{what} b rel err {errs['b']:.3g}"
    e_ref = ref["e"]
    errs["e"] = abs(float(rec["error"]) - e_ref) / max(abs(e_ref), 1e-300)
    if e_ref == 0.0:
        assert float(rec["error"]) == 0.0, what
        errs["e"] = 0.0
    assert errs["e"] <= E_TOL, f"{what} e rel err {errs['e']:.3g}"
    return errs


class Margins:
    """Worst relative errors (H blocks, b, e) and integer mismatches over the
    factors compared in one parity test.  When GVOX_MARGINS_OUT names a file,
    `save` appends one JSON line per test (tools/parity_margins.py turns them
    into profiles/*_parity_margins.md); otherwise it only prints."""

    def __init__(self, config):
        self.config = config
        self.worst = {"H_ii": 0.0, "H_ij": 0.0, "H_jj": 0.0, "b": 0.0, "e": 0.0}
        self.factors = 0
        self.int_compared = {}
        self.int_mismatch = {}

    def add_factor(self, errs):
        self.factors += 1
        for k, v in errs.items():
            self.worst[k] = max(self.worst.get(k, 0.0), float(v))

    def add_ints(self, what, compared, mismatches=0):
        self.int_compared[what] = self.int_compared.get(what, 0) + int(compared)
        self.int_mismatch[what] = self.int_mismatch.get(what, 0) + int(mismatches)

    def save(self, test):
        import json
        import os
        rec = {"test": test, "config": self.config, "factors": self.factors, "worst": self.worst,
               "int_compared": self.int_compared, "int_mismatch": self.int_mismatch,
               "tolerances": {"H": H_TOL, "b": B_TOL, "e": E_TOL}}
        print("parity margins:", json.dumps(rec))
        path = os.environ.get("GVOX_MARGINS_OUT")
        if path:
            with open(path, "a") as fh:
                fh.write(json.dumps(rec) + "\n")
