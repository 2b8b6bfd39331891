#!/usr/bin/env python
"""Calibrate the synthetic draft noise (delta) so that the mean acceptance rate
alpha = E[sum_v min(p, q)] (PAPER §4.1 P133: "alpha = E(beta)") hits each config's
target.  alpha and the draft confidence are MEASURED WITH THE ORACLE only
(oracle.row_softmax, oracle.confidence); the script prints the constants that go
into paper_2506_01979_b200/synth.py CONFIGS.

    python scripts/calibrate_alpha.py [--rows 256] [--configs c1,c2,...]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2506_01979_b200 import synth  # noqa: E402


def measure(cfg, rows, seed=99):
    G = 7
    B = max(1, rows // (G + 1))
    c = synth.config(cfg.name, B=B, K=1, G=G, layout="fixed", rounds=1, delta=cfg.delta, rho_same=cfg.rho_same)
    inp = synth.to_numpy_inputs(synth.generate(c, device="cpu", seed=seed))
    al, t1 = [], []
    for b in range(B):
        for i in range(G + 1):
            P, _ = oracle.row_softmax(inp["PL"], b, 0, i, V=inp["V"])
            Q, _ = oracle.row_softmax(inp["QL"], b, 0, i, V=inp["V"])
            al.append(np.minimum(P, Q).sum())
            t1.append(Q.max())
    conf = oracle.confidence(inp["QL"], V=inp["V"])
    return float(np.mean(al)), float(np.mean(t1)), float(np.mean(conf["gamma_next"]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=256)
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    a = ap.parse_args()
    for name in a.configs.split(","):
        cfg = synth.config(name)
        lo, hi = 0.0, 4.0
        for _ in range(14):
            mid = 0.5 * (lo + hi)
            al, _, _ = measure(synth.config(name, delta=mid), a.rows)
            if al > cfg.alpha:
                lo = mid
            else:
                hi = mid
        d = round(0.5 * (lo + hi), 3)
        al, t1, gam = measure(synth.config(name, delta=d), a.rows * 2, seed=7)
        print(f"{name}: target alpha {cfg.alpha}  rho_same {cfg.rho_same}  delta {d}  "
              f"-> alpha {al:.4f}, mean draft top-1 {t1:.3f}, mean max(1,stop) over G=7 {gam:.2f}")


if __name__ == "__main__":
    main()
