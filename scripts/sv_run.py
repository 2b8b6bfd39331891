"""Run the small-batch step a few times without a graph (profiling target):
    python scripts/sv_run.py c2|c1one [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_01979_b200 import api, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg = synth.config(name) if name != "c1one" else synth.config("c1", rounds=1)
inp = synth.generate(cfg, device="cuda")
d = api.dims_for(inp["PL"], V=inp["V"])
buf = api.StepBuffers.alloc(d, "cuda")
for _ in range(reps):
    api.verify_step(d, inp, buf, adaptive=(cfg.layout == "adaptive"))
torch.cuda.synchronize()
print("ok", name)
