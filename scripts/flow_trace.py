"""Timeline of the fused small-batch kernel (k_flow) from its SB_FLOW_TRACE build.

    python -m paper_2506_01979_b200.build --out paper_2506_01979_b200/libspecbranch_trace.so -- -DSB_FLOW_TRACE
    SB_LIB_PATH=paper_2506_01979_b200/libspecbranch_trace.so python scripts/flow_trace.py c2 [adaptive]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_01979_b200 import _lib, api, synth  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
adaptive = len(sys.argv) > 2 and sys.argv[2] == "adaptive"
c = synth.config(cfgname) if cfgname != "c1one" else synth.config("c1", rounds=1)
inp = synth.generate(c, device="cuda")
d = api.dims_for(inp["PL"], V=inp["V"])
buf = api.StepBuffers.alloc(d, "cuda")
for _ in range(3):
    api.verify_step(d, inp, buf, adaptive=adaptive)
torch.cuda.synchronize()
L = _lib.lib()
tr = np.zeros((1024, 2, 64), np.uint64)
L.sb_flow_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
L.sb_flow_trace_read(tr.ctypes.data, tr.nbytes)
api.verify_step(d, inp, buf, adaptive=adaptive)
torch.cuda.synchronize()
tr[:] = 0
L.sb_flow_trace_read(tr.ctypes.data, tr.nbytes)  # cleared? (symbol persists: read after a fresh run)
api.verify_step(d, inp, buf, adaptive=adaptive)
torch.cuda.synchronize()
L.sb_flow_trace_read(tr.ctypes.data, tr.nbytes)
act = tr[:, 0, 0] > 0
t0 = tr[act, :, 0].min()
rel = lambda x: (x.astype(np.int64) - int(t0)) / 1000.0  # us  # noqa: E731
ncta = int(act.sum())
print(f"{cfgname} adaptive={adaptive}: {ncta} CTAs traced")
starts = rel(tr[act, 0, 0])
print(f"start: min {starts.min():.1f} max {starts.max():.1f} us")
if adaptive:
    print(f"C items done (stream w0): median {np.median(rel(tr[act,0,1])):.1f} max {rel(tr[act,0,1]).max():.1f}")
    print(f"conf barrier passed: median {np.median(rel(tr[act,0,2])):.1f} max {rel(tr[act,0,2]).max():.1f}")
r_end = rel(tr[act, 0, 40])
f_end = rel(tr[act, 1, 40])
print(f"R streaming done (w0): median {np.median(r_end):.1f} max {r_end.max():.1f}")
print(f"R finalize done (w6): median {np.median(f_end):.1f} max {f_end.max():.1f}")
has_s = tr[act, 0, 41] > 0
if has_s.any():
    w0 = rel(tr[act, 0, 41][has_s]); w1 = rel(tr[act, 0, 42][has_s]); w2 = rel(tr[act, 0, 43][has_s])
    print(f"S item wait start: median {np.median(w0):.1f}; ready seen: median {np.median(w1):.1f} max {w1.max():.1f}; "
          f"sums done: median {np.median(w2):.1f} max {w2.max():.1f}")
end = rel(tr[act, 0, 63])
endf = rel(tr[act, 1, 63])
print(f"end (w0): median {np.median(end):.1f} max {end.max():.1f}; end (w6): max {endf.max():.1f}")
# per item handoff times of CTA 0
items = [(k - 4, rel(tr[0, 0, k]), rel(tr[0, 1, k])) for k in range(4, 36) if tr[0, 0, k] > 0 or tr[0, 1, k] > 0]
print("CTA0 items (li, stream handoff us, finalize us):", [(i, round(a, 1), round(b, 1)) for i, a, b in items[:12]])
