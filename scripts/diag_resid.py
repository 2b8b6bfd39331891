"""Diagnostic: worst resid_mass errors (GPU vs oracle) on a full-size configuration.
usage: python scripts/diag_resid.py c5 [nseq]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2506_01979_b200 import synth  # noqa: E402
from parity_util import gpu_run, oracle_for  # noqa: E402

name = sys.argv[1]
nseq = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cfg = synth.config(name)
inp = synth.generate(cfg, device="cuda")
g, d, _ = gpu_run(inp)
idx = np.arange(min(nseq, inp["PL"].shape[0]))
it = torch.as_tensor(idx, device="cuda")
sub = synth.to_numpy_inputs({k: (v.index_select(0, it) if torch.is_tensor(v) else v) for k, v in inp.items()})
o = oracle_for(sub, sub["gamma"])
Rg = g["resid_mass"][idx].astype(np.float64)
Ro = o["resid_mass"]
same = g["y_kind"][idx] == o["y_kind"]
err = np.abs(Rg - Ro)
band = err / (1e-5 * np.abs(Ro) + 1e-7)
band[~same] = 0
order = np.argsort(-band)[:15]
print("kind counts", np.bincount(o["y_kind"], minlength=3))
for b in order:
    print(f"b={b} kind={o['y_kind'][b]} sel={o['sel_k'][b]} n={o['n_acc'][b].tolist()} Ro={Ro[b]:.9g} Rg={Rg[b]:.9g} "
          f"err={err[b]:.3g} rel={err[b] / max(Ro[b], 1e-30):.3g} band={band[b]:.3f}")
