"""Fit fz_recommend_t's cost model to a `bench.py --study f4` run.

    python tools/f4_fit.py profiles/r02x_f4_study.jsonl

Per (case, t) features from the host count tables (the quantities fz_recommend_t computes): R = |Z(n)|,
P = leading prefixes (a_1..a_L, phi <= n), Q = innermost runs (a_1..a_{L-1}), O = outer prefixes
(a_1..a_{L-2}), E = memo rows sum_{x<=n} |Z(x; tail)|, L = d - t.  Whole-step model (non-negative least
squares on relative error; seconds) -- the form fz_recommend_t evaluates:
  MATERIALIZE: c0 + c1 (4 d R) + c2 P + c3 (4 t E)
  HASH:        c0 + c1 R + c2 P + c3 (4 t E)
  COUNT:       c0 + c1 P + c2 Q + c3 O      (fz_recommend_t splits c1 by walk kind: staged pair walk or not)
(Splitting memo and walk time into separate fits, or adding a per-tail-level term, fitted worse: the small-n
rows are latency-bound.)  Prints the constants and, per case, the model's pick against the measured best t."""
import json
import sys

import numpy as np
from scipy.optimize import nnls


def cum(g, n):
    c = np.zeros(n + 1)
    c[0] = 1
    for gi in g:
        for x in range(gi, n + 1):
            c[x] += c[x - gi]
    return c


def feats(g, n, t, mode):
    d, L = len(g), len(g) - t
    R = cum(g, n)[n]
    P = cum(g[:L], n).sum()
    Q = cum(g[:L - 1], n).sum() if L >= 1 else 0.0
    O = cum(g[:L - 2], n).sum() if L >= 2 else 0.0
    E = cum(g[L:], n).sum()
    if mode == "materialize":
        return [1.0, 4.0 * d * R, P, 4.0 * t * E]
    if mode == "hash":
        return [1.0, R, P, 4.0 * t * E]
    return [1.0, P, Q, O]


def main(path):
    recs = [json.loads(x) for x in open(path) if x.strip()]
    cs = {}
    for mode in ("materialize", "hash", "count"):
        X = [[v / (us * 1e-6) for v in feats(tuple(r["gens"]), r["n"], int(t), mode)]
             for r in recs if r["mode"] == mode for t, us in r["step_us"].items()]
        if not X:
            continue
        cs[mode], _ = nnls(np.array(X), np.ones(len(X)))
        print(f"{mode}: " + ", ".join(f"{v:.4g}" for v in cs[mode]))
    worst = 1.0
    for r in recs:
        mode = r["mode"]
        pred = {int(t): float(np.dot(cs[mode], feats(tuple(r["gens"]), r["n"], int(t), mode))) for t in r["step_us"]}
        meas = {int(t): v for t, v in r["step_us"].items()}
        pick, best = min(pred, key=pred.get), min(meas, key=meas.get)
        ratio = meas[pick] / meas[best]
        worst = max(worst, ratio)
        print(f"{r['case']:>22} {mode:>11}: pick t={pick} ({meas[pick]:.1f} us), best t={best} "
              f"({meas[best]:.1f} us), ratio {ratio:.3f}")
    print(f"worst pick / best = {worst:.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
