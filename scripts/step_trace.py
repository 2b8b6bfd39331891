"""Global-timer timeline of one whole step (confidence -> verify -> select) from an
SB_TRACE build of the library (diagnostics only).

    python -m paper_2506_01979_b200.build --out build/lib_trace.so -- -DSB_TRACE
    SB_LIB_PATH=$PWD/build/lib_trace.so python scripts/step_trace.py c2
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_01979_b200 import _lib, api, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = (synth.config("c1", rounds=1) if name == "c1one" else
       synth.config("c2", layout="fixed") if name == "c2fixed" else synth.config(name))
adaptive = cfg.layout == "adaptive"
inp = synth.generate(cfg, device="cuda")
d = api.dims_for(inp["PL"], V=inp["V"])
buf = api.StepBuffers.alloc(d, "cuda")
g = api.StepGraph(d, inp, buf, adaptive=adaptive)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
L = _lib.lib()
tabs = {}
for t in ("sb_trace_conf", "sb_trace_rows", "sb_trace_select"):
    fn = getattr(L, t + "_read")
    fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    a = np.zeros((160, 8, 64), np.uint64)
    fn(a.ctypes.data, a.nbytes)
    tabs[t] = a
t0 = min(int(a[:, 0, 0][a[:, 0, 0] > 0].min()) for a in tabs.values() if (a[:, 0, 0] > 0).any())


def us(x):
    return (x.astype(np.int64) - t0) / 1000.0


for t, a in tabs.items():
    act = a[:, 0, 0] > 0
    if not act.any():
        print(t, "not launched")
        continue
    launch, post = us(a[act, 0, 0]), us(a[act, 0, 1])
    print(f"{t}: {int(act.sum())} CTAs; CTA start {launch.min():.1f}..{launch.max():.1f} us, "
          f"past griddepcontrol.wait {post.min():.1f}..{post.max():.1f} us")
    for role, lab in ((1, "producer"), (2, "epilogue"), (3, "consumer")):
        ends = a[act, role, 63]
        ends = ends[ends > 0]
        if ends.size:
            e = us(ends)
            print(f"   {lab} done: median {np.median(e):.1f} max {e.max():.1f} us")
    if t == "sb_trace_rows":
        # per CTA: consumer unit (start, publish) pairs, producer first-copy times
        for cta in (0, 1, 70, 147):
            cs = [(round(us(np.array([a[cta, 3, 2 + k]]))[0], 1), round(us(np.array([a[cta, 3, 32 + k]]))[0], 1))
                  for k in range(30) if a[cta, 3, 2 + k] > 0]
            ps = [round(us(np.array([a[cta, 1, 2 + k]]))[0], 1) for k in range(30) if a[cta, 1, 2 + k] > 0]
            es = [round(us(np.array([a[cta, 2, 2 + k]]))[0], 1) for k in range(30) if a[cta, 2, 2 + k] > 0]
            print(f"   CTA {cta}: producer unit issue {ps[:8]}\n            consumer (start, publish) {cs[:8]}"
                  f"\n            epilogue done {es[:8]}")
    if t == "sb_trace_select":
        e = a[act, 2, 2:40]
        e = e[e > 0]
        if e.size:
            print(f"   sequence epilogues: first {us(e).min():.1f} median {np.median(us(e)):.1f} last {us(e).max():.1f} us")
        e62 = us(a[act, 2, 62][a[act, 2, 62] > 0])
        print(f"   CTA exit: max {e62.max():.1f} us")
