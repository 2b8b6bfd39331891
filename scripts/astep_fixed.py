"""k_astep on a fixed workload (C2 shape, gamma = 8 for every sequence: plan items, no
confidence phase) for A/B builds whose results differ (SB_LIB_PATH):
    SB_ASTEP=1 python scripts/astep_fixed.py [B]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_01979_b200 import api, synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = synth.config("c2", B=B, layout="fixed")
inp = synth.generate(cfg, device="cuda")
d = api.dims_for(inp["PL"], V=inp["V"])
buf = api.StepBuffers.alloc(d, "cuda")
g = api.StepGraph(d, inp, buf, adaptive=False)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for r in range(25):
    flush.fill_(r & 255)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    if r >= 5:
        ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
print(f"B={B} fixed gamma=8: median {ts[len(ts)//2]:.1f} us, min {ts[0]:.1f} us")
