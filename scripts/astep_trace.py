"""Timeline of the single-launch adaptive step (k_astep) from an SB_TRACE build:
per CTA, items in grab order with type (C confidence, V verify, S sample), grab time,
consumer done and epilogue done (us from the first CTA start).
    SB_LIB_PATH=$PWD/build/lib_trace.so python scripts/astep_trace.py c2"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_01979_b200 import _lib, api, synth  # noqa: E402

cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c2")
inp = synth.generate(cfg, device="cuda")
d = api.dims_for(inp["PL"], V=inp["V"])
buf = api.StepBuffers.alloc(d, "cuda")
g = api.StepGraph(d, inp, buf, adaptive=True)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
fn = _lib.lib().sb_trace_astep_read
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
a = np.zeros((160, 8, 64), np.uint64)
fn(a.ctypes.data, a.nbytes)
act = a[:, 0, 0] > 0
t0 = int(a[act, 0, 0].min())
us = lambda x: (int(x) - t0) / 1000.0  # noqa: E731
print(f"{int(act.sum())} CTAs; pdl passed {min(us(x) for x in a[act,0,1]):.1f}..{max(us(x) for x in a[act,0,1]):.1f} us")
ends = [us(a[c, 2, 2 + k]) for c in np.where(act)[0] for k in range(60) if a[c, 2, 2 + k] > 0]
print(f"last epilogue item done: {max(ends):.1f} us")
for c in (0, 1, 50, 100, 147):
    row = []
    for k in range(60):
        t = a[c, 0, 2 + k]
        if t == 0:
            break
        typ = "XCVS"[int(t)] if int(t) < 4 else "?"
        row.append(f"{typ}@{us(a[c,1,2+k]):.1f}/{us(a[c,3,2+k]) if a[c,3,2+k] else float('nan'):.1f}/{us(a[c,2,2+k]) if a[c,2,2+k] else float('nan'):.1f}")
    print(f"CTA {c}: " + "  ".join(row))
# when did each phase end overall
for typ, code in (("conf", 1), ("verify", 2), ("sample", 3)):
    ts = [us(a[c, 3, 2 + k]) for c in np.where(act)[0] for k in range(60) if a[c, 0, 2 + k] == code and a[c, 3, 2 + k] > 0]
    gs = [us(a[c, 1, 2 + k]) for c in np.where(act)[0] for k in range(60) if a[c, 0, 2 + k] == code]
    if ts:
        print(f"{typ}: {len(ts)} items, grabbed {min(gs):.1f}..{max(gs):.1f} us, consumers done {min(ts):.1f}..{max(ts):.1f} us")

# consumer split per item type: wait for the first chunk / stream+compute / warp reduction / publish
for typ, code in (("conf", 1), ("verify", 2)):
    w, c_, r_, pub = [], [], [], []
    for cta in np.where(act)[0]:
        prev = None
        for k in range(60):
            if a[cta, 0, 2 + k] == 0:
                break
            t_first, t_comp, t_red, t_done = (a[cta, 4, 2 + k], a[cta, 5, 2 + k], a[cta, 6, 2 + k], a[cta, 3, 2 + k])
            if a[cta, 0, 2 + k] == code and t_first and t_comp and t_red and t_done and prev:
                w.append((int(t_first) - int(prev)) / 1e3)
                c_.append((int(t_comp) - int(t_first)) / 1e3)
                r_.append((int(t_red) - int(t_comp)) / 1e3)
                pub.append((int(t_done) - int(t_red)) / 1e3)
            prev = t_done if t_done else prev
    if w:
        print(f"{typ} items: wait-for-data median {np.median(w):.2f} us, stream+math {np.median(c_):.2f}, "
              f"warp reductions {np.median(r_):.2f}, publish (pempty wait) {np.median(pub):.2f}")

# producer side: grab -> last chunk issued, last chunk issued -> consumers done
for typ, code in (("conf", 1), ("verify", 2), ("sample", 3)):
    gi, ic = [], []
    for cta in np.where(act)[0]:
        for k in range(60):
            if a[cta, 0, 2 + k] != code:
                continue
            g_, i_, c_ = int(a[cta, 1, 2 + k]), int(a[cta, 7, 2 + k]), int(a[cta, 3, 2 + k])
            if g_ and i_ and c_:
                gi.append((i_ - g_) / 1e3)
                ic.append((c_ - i_) / 1e3)
    if gi:
        print(f"{typ}: grab -> last chunk issued median {np.median(gi):.2f} us (p90 {np.percentile(gi, 90):.2f}); "
              f"last issued -> consumers done median {np.median(ic):.2f} us (p90 {np.percentile(ic, 90):.2f})")
