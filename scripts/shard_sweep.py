"""Per-rank work of the vocabulary-sharded C5 step on one GPU (time the
shard row kernel at V/2, V/4, V/8 before a multi-GPU run): for G = 1, 2, 4, 8 the local
verify pass (sb_shard_verify_local: k_plan + k_rows_tma in partial mode) and the local
select pass (sb_shard_select_local) of rank 0's column slice, each replayed from a CUDA
graph; GB/s over the slice's bytes.  The exchanges are not timed (one GPU).
    python scripts/shard_sweep.py [c5]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_01979_b200 import api, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = synth.config(name)
inp = synth.generate(cfg, device="cuda")
V = inp["V"]
es = inp["PL"].element_size()
peak = 6550.4
for G in (1, 2, 4, 8):
    v0, n = api.shard_bounds(V, G)[0]
    d, pv = api.shard_view(inp["PL"], V, v0, n)
    _, qv = api.shard_view(inp["QL"], V, v0, n)
    ws = api.make_workspace(d, "cuda")
    part = torch.empty(api.sb_shard_partial_bytes(d), dtype=torch.uint8, device="cuda")
    buf = api.StepBuffers.alloc(d, "cuda")

    def local(s_):
        api.sb_shard_verify_local(d, pv, qv, inp["tok"], inp["u"], inp["gamma"], inp["branch_pos"], part, ws, s_)

    g = api.CallGraph(local)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    # rows read in partial mode: every tested row pair plus the bonus rows (Lr = gamma + 1)
    B, K, Gm = cfg.B, cfg.K, cfg.G
    pairs = B * ((Gm + 1) + (K - 1) * Gm)  # s_b = 0, gamma_b = G: Lr = G+1 rows in slot 0, G in slots 1..K-1
    nbytes = pairs * 2 * n * es
    print(f"G={G}: slice {n} columns ({n * es} B rows), local verify {ms * 1e3:.1f} us, "
          f"{nbytes / (ms * 1e-3) / 1e9:.0f} GB/s = {nbytes / (ms * 1e-3) / 1e9 / peak:.3f} of peak")
