"""Turn the parity tests' margin records (GVOX_MARGINS_OUT JSON lines written by
tests/parity.py::Margins) into a markdown table: per config, the worst
relative errors of H (per block), b and e against the fp64 oracle, next to
the tolerances of BASELINE.json's north star, and every integer result
compared (voxel-key correspondences, inliers, overlap counts, screening
decisions) with its mismatch count.

    python tools/parity_margins.py gpurun_out/margins.jsonl > profiles/r02_parity_margins.md
"""
import json
import sys


def main(path):
    recs = [json.loads(x) for x in open(path) if x.strip()]
    print("| config (test) | factors | max rel H_ii | H_ij | H_jj | b | e | integers compared: mismatches |")
    print("|---|---|---|---|---|---|---|---|")
    for r in recs:
        w = r["worst"]
        ints = ", ".join(f"{k} {r['int_compared'][k]:,}: {r['int_mismatch'][k]}"
                         for k in sorted(r["int_compared"]))
        print(f"| {r['config']} (`{r['test']}`) | {r['factors']} | {w['H_ii']:.2e} | {w['H_ij']:.2e} | "
              f"{w['H_jj']:.2e} | {w['b']:.2e} | {w['e']:.2e} | {ints} |")
    t = recs[0]["tolerances"] if recs else {"H": 1e-4, "b": 1e-4, "e": 1e-5}
    print(f"\nTolerances (north star): H {t['H']:g}, b {t['b']:g} (relative Frobenius; b's "
          f"denominator max(|b|, |sum |terms||), Q13), e {t['e']:g}; integers bit-exact.")


if __name__ == "__main__":
    main(sys.argv[1])
