"""Timeline of the split-vocabulary step k_sv from an SB_TRACE build: per barrier the
spread of CTA arrival / departure times, per streaming phase the warps' finish times
(us from the first CTA start).
    SB_LIB_PATH=$PWD/build/lib_trace.so python scripts/sv_trace.py c2|c1one"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_01979_b200 import _lib, api, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = synth.config(name) if name != "c1one" else synth.config("c1", rounds=1)
adaptive = cfg.layout == "adaptive"
inp = synth.generate(cfg, device="cuda")
d = api.dims_for(inp["PL"], V=inp["V"])
buf = api.StepBuffers.alloc(d, "cuda")
g = api.StepGraph(d, inp, buf, adaptive=adaptive)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
fn = _lib.lib().sb_trace_sv_read
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
a = np.zeros((160, 8, 64), np.uint64)
fn(a.ctypes.data, a.nbytes)
act = a[:, 0, 0] > 0
t0 = int(a[act, 0, 0].min())
us = lambda x: (x.astype(np.int64) - t0) / 1000.0  # noqa: E731
print(f"{int(act.sum())} CTAs; start {us(a[act,0,0]).max():.1f} max; pdl passed {us(a[act,0,1]).min():.1f}..{us(a[act,0,1]).max():.1f} us")
for ph, role in (("C", 1), ("V", 2)):
    v = a[act, role, :16]
    v = v[v > 0]
    if v.size:
        t = us(v)
        print(f"stream {ph}: warps done {t.min():.1f} .. median {np.median(t):.1f} .. {t.max():.1f} us")
for n in range(1, 8):
    arr, dep = a[act, 0, 2 * n], a[act, 0, 2 * n + 1]
    if (arr > 0).all():
        print(f"barrier {n}: arrive {us(arr).min():.1f}..{us(arr).max():.1f}  depart {us(dep).min():.1f}..{us(dep).max():.1f} us")
print(f"exit: {us(a[act,0,40]).min():.1f}..{us(a[act,0,40]).max():.1f} us")

# per warp (first task): combine V: start, folds done, epilogue done, decision done; locate: start, sampled, committed, offsets
for role, nm in ((3, "combine V"), (4, "locate")):
    rows = []
    for c in np.where(act)[0]:
        for w in range(16):
            ev = a[c, role, 4 * w:4 * w + 4]
            if ev[0] > 0:
                rows.append([us(np.array([x]))[0] if x > 0 else np.nan for x in ev])
    if rows:
        r = np.array(rows)
        d1, d2, d3 = r[:, 1] - r[:, 0], r[:, 2] - r[:, 1], r[:, 3] - r[:, 2]
        print(f"{nm}: {len(r)} warps; start {np.nanmin(r[:,0]):.1f}..{np.nanmax(r[:,0]):.1f}; step1 med {np.nanmedian(d1):.2f} max {np.nanmax(d1):.2f}; "
              f"step2 med {np.nanmedian(d2):.2f} max {np.nanmax(d2):.2f}; step3 med {np.nanmedian(d3):.2f} max {np.nanmax(d3):.2f} us")

pr = a[0, 5]
if pr[0] > 0:
    print(f"probe: 16 dependent L2 loads {(int(pr[1]) - int(pr[0])) / 16:.0f} ns each; 16 dependent HBM loads {(int(pr[2]) - int(pr[1])) / 16:.0f} ns each; "
          f"clock64 {int(pr[3])} cycles over {(int(pr[2]) - int(pr[0]))} ns = {int(pr[3]) / max(1, int(pr[2]) - int(pr[0])):.2f} GHz")
