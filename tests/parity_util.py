"""Parity harness: run the CUDA path (through the C ABI) and the fp64 oracle on the same
bytes and compare element by element.  Test infrastructure (imports oracle/).

Bars (BASELINE.json north_star; SURVEY §8.4 "Pass criteria"):
  * discrete outputs bit-exact, except sequences the oracle flags as near ties
    (|u - P/Q| < 1e-6, sample |t - F| < 1e-6, R < 1e-4, |stat - eps| < 1e-6,
    Eq. 7 argument within 1e-6 of an integer);
  * continuous outputs |gpu - ref| <= 1e-5 |ref| + 1e-7 (lse: 1e-5 max(1, |ref|)).
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_2506_01979_b200 import api, synth

REL, ABS = 1e-5, 1e-7


def gpu_run(inp: dict, rule=0, adaptive=False, eps=0.2, k_max=6, fused=True):
    d = api.dims_for(inp["PL"], V=inp["V"])
    buf = api.StepBuffers.alloc(d, inp["PL"].device)
    gamma = api.verify_step(d, inp, buf, rule=rule, adaptive=adaptive, eps=eps, k_max=k_max, fused=fused)
    torch.cuda.synchronize()
    out = {k: getattr(buf, k).cpu().numpy() for k in buf.__dataclass_fields__
           if k not in ("workspace", "conf_workspace")}
    out["acc_mask"] = out["acc_mask"].view(np.uint32)
    out["keep_mask"] = out["keep_mask"].view(np.uint32)
    out["gamma_used"] = gamma.cpu().numpy().astype(np.int32)
    return out, d, buf


def _close(g, r, rel=REL, ab=ABS):
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    nan_ok = np.array_equal(np.isnan(g), np.isnan(r))
    m = ~np.isnan(r)
    err = np.abs(g[m] - r[m])
    ok = bool(np.all(err <= rel * np.abs(r[m]) + ab)) if m.any() else True
    relerr = float(np.max(err / np.maximum(np.abs(r[m]), 1e-30))) if m.any() else 0.0
    return nan_ok and ok, relerr


def _band(g, r):
    """max |gpu - ref| / (1e-5 |ref| + 1e-7): <= 1 means inside the pass band."""
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    m = ~np.isnan(r) & ~np.isnan(g)
    if not m.any():
        return 0.0
    return float(np.max(np.abs(g[m] - r[m]) / (REL * np.abs(r[m]) + ABS)))


def sample_candidates(inp_np: dict, o: dict, b: int, band: float = 1e-6):
    """The tokens an inverse-CDF draw may return for oracle sequence b when t = us R lies
    within `band` (probability mass) of a CDF breakpoint: every id with mass whose
    interval [F(j-1), F(j)) comes within the band of t (SURVEY §8.0 "Inverse CDF"), from
    the oracle's own fp64 softmax of the sampled row."""
    g = int(o["_gamma"][b]) if "_gamma" in o else int(inp_np["gamma"][b])
    G = inp_np["PL"].shape[2] - 1
    g = min(max(g, 0), G)
    s = min(max(int(inp_np["branch_pos"][b]), 0), g)
    L = g if s < g else g + 1
    ks, kind = int(o["sel_k"][b]), int(o["y_kind"][b])
    if ks < 0:
        row, slot = min(int(o["n_acc"][b, 0]), s), 0
    else:
        n = int(o["n_acc"][b, ks])
        row, slot = (n, 0 if n <= s else ks) if n < L else (g, ks)
    V = inp_np["V"]
    P, _ = oracle.row_softmax(inp_np["PL"][b:b + 1], 0, slot, row, V=V)
    if kind == 1:
        Q, _ = oracle.row_softmax(inp_np["QL"][b:b + 1], 0, slot, row, V=V)
        r = np.maximum(0.0, P - Q)
        if r.sum() == 0.0:
            r = P
    else:
        r = P
    F = np.cumsum(r)
    t = float(inp_np["us"][b]) * F[-1]
    ok = (r > 0) & (F - r - band <= t) & (t < F + band)
    cand = set(np.nonzero(ok)[0].tolist())
    if t >= F[-1] - band:
        cand.add(int(np.nonzero(r > 0)[0][-1]))
    return cand


def compare(g: dict, o: dict, sel=None, strict=True, inp_np=None):
    """Compare gpu outputs g with oracle outputs o on sequences `sel` (indices into g).
    With inp_np (the oracle's inputs), a near-tie sample is not skipped: the GPU's token
    must be one of the ids adjacent to the CDF breakpoint (sample_candidates)."""
    B = o["status"].shape[0]
    sel = np.arange(B) if sel is None else np.asarray(sel)
    gs = {k: (v[sel] if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] >= len(sel) and k not in ("offsets", "packed_tok") else v)
          for k, v in g.items()}
    rep = {"n": B, "fail": []}
    ties = o["ties"]
    t_dec = (ties & (oracle.TIE_ACC_DEC)) != 0
    t_mask = (ties & oracle.TIE_ACC_MASK) != 0
    t_samp = (ties & (oracle.TIE_SAMPLE | oracle.TIE_ILLCOND)) != 0
    rep["ties"] = {"acc_mask": int(t_mask.sum()), "decision": int(t_dec.sum()), "sample": int(t_samp.sum())}

    def fail(name, idx):
        idx = np.atleast_1d(idx)
        if idx.size:
            rep["fail"].append((name, idx[:8].tolist()))

    # continuous
    for k in ("lse_p", "lse_q"):
        r = o[k]
        gg = gs[k].astype(np.float64)
        nan_ok = np.array_equal(np.isnan(gg), np.isnan(r))
        m = ~np.isnan(r)
        err = np.abs(gg[m] - r[m]) / np.maximum(1.0, np.abs(r[m]))
        rep[f"max_err_{k}"] = float(err.max()) if err.size else 0.0
        if not nan_ok or (err.size and err.max() > REL):
            fail(k, np.where(np.any((np.isnan(gg) != np.isnan(r)).reshape(len(sel), -1), axis=1))[0])
            if err.size and err.max() > REL:
                rep["fail"].append((k + "_tol", float(err.max())))
    for k in ("top1_q", "entropy_q", "p_tok", "q_tok"):
        ok, relerr = _close(gs[k], o[k])
        rep[f"max_rel_{k}"] = relerr
        rep[f"max_band_{k}"] = _band(gs[k], o[k])
        if not ok:
            bad = ~np.isclose(gs[k].astype(np.float64), o[k], rtol=REL, atol=ABS, equal_nan=True)
            fail(k, np.where(bad.reshape(len(sel), -1).any(axis=1))[0])
    # discrete
    ok_id = gs["top1_id_q"] == o["top1_id_q"]
    fail("top1_id_q", np.where(~ok_id.reshape(len(sel), -1).all(axis=1))[0])
    fail("status", np.where(gs["status"] != o["status"])[0])
    am = (gs["acc_mask"] != o["acc_mask"]).any(axis=1) & ~t_mask
    fail("acc_mask", np.where(am)[0])
    nd = (gs["n_acc"] != o["n_acc"]).any(axis=1) & ~t_dec
    fail("n_acc", np.where(nd)[0])
    for k in ("sel_k", "commit_len", "y_kind", "path_rolled", "branch_discarded"):
        fail(k, np.where((gs[k] != o[k]) & ~t_dec)[0])
    fail("keep_mask", np.where((gs["keep_mask"] != o["keep_mask"]).any(axis=1) & ~t_dec)[0])
    fail("y_tok", np.where((gs["y_tok"] != o["y_tok"]) & ~t_dec & ~t_samp)[0])
    ot = (gs["out_tok"] != o["out_tok"]).any(axis=1) & ~t_dec & ~t_samp
    fail("out_tok", np.where(ot)[0])
    rep["tie_samples_checked"] = 0
    rep["tie_samples_differ"] = 0
    if inp_np is not None:
        # flagged samples: the GPU token must be a valid draw at the breakpoint, and the
        # rest of the commit must agree
        for b in np.where(t_samp & ~t_dec & (o["y_kind"] != 0))[0]:
            rep["tie_samples_checked"] += 1
            if gs["y_tok"][b] == o["y_tok"][b]:
                continue
            rep["tie_samples_differ"] += 1
            if int(gs["y_tok"][b]) not in sample_candidates(inp_np, o, b):
                fail("y_tok_tie_invalid", [b])
            n = int(o["commit_len"][b]) - 1
            if not np.array_equal(gs["out_tok"][b, :n], o["out_tok"][b, :n]) or gs["out_tok"][b, n] != gs["y_tok"][b]:
                fail("out_tok_tie", [b])
        m = o["margin_sample"][t_samp]
        rep["tie_margin_hist"] = np.histogram(np.log10(np.maximum(m, 1e-12)), bins=[-12, -9, -8, -7, -6])[0].tolist()
        # flagged accept decisions (|u - P/Q| < 1e-6 somewhere on a path): the GPU's
        # acceptance bits may differ from the oracle's only at rows whose own test is that
        # close, and its n_k must be the first rejection of its own bits
        rep["tie_decisions_checked"] = 0
        G = inp_np["PL"].shape[2] - 1
        K = inp_np["PL"].shape[1]
        for b in np.where(t_dec)[0]:
            rep["tie_decisions_checked"] += 1
            g_b = int(o["_gamma"][b]) if "_gamma" in o else int(inp_np["gamma"][b])
            g_b = min(max(g_b, 0), G)
            s_b = min(max(int(inp_np["branch_pos"][b]), 0), g_b)
            L = g_b if s_b < g_b else g_b + 1
            for k in range(K):
                gm, om = int(gs["acc_mask"][b, k]), int(o["acc_mask"][b, k])
                rej = [r for r in range(L) if not (gm >> r) & 1]
                if int(gs["n_acc"][b, k]) != (rej[0] if rej else L):
                    fail("n_acc_tie_inconsistent", [b])
                for r in range(L):
                    if ((gm ^ om) >> r) & 1:
                        ts = 0 if r < s_b else k
                        uu = float(inp_np["u"][b, ts, r])
                        pt, qt = float(gs["p_tok"][b, ts, r]), float(gs["q_tok"][b, ts, r])
                        if not (qt > 0 and abs(uu - pt / qt) < 2e-6):
                            fail("acc_tie_invalid", [b])
    same = (gs["y_kind"] == o["y_kind"]) & ~t_dec & ~t_samp
    ok, relerr = _close(gs["resid_mass"][same], o["resid_mass"][same])
    rep["max_rel_resid_mass"] = relerr
    rep["max_band_resid_mass"] = _band(gs["resid_mass"][same], o["resid_mass"][same])
    if not ok:
        rep["fail"].append(("resid_mass", relerr))
    rep["exact_seq"] = int((~t_dec & ~t_samp).sum())
    rep["y_compared"] = int(((gs["y_kind"] != 0) & ~t_dec & ~t_samp).sum())
    if strict:
        assert not rep["fail"], rep
    return rep


def internal_consistency(g: dict, G: int):
    """offsets = exclusive scan of commit_len; packed stream = concatenated commits."""
    cl = g["commit_len"]
    assert g["offsets"][0] == 0 and np.array_equal(np.diff(g["offsets"]), cl)
    for b in range(len(cl)):
        seg = g["packed_tok"][g["offsets"][b]: g["offsets"][b + 1]]
        assert np.array_equal(seg, g["out_tok"][b, : cl[b]])
        assert (g["out_tok"][b, cl[b]:] == -1).all()


def oracle_for(inp_np: dict, gamma, rule=0, nthreads=0):
    return oracle.verify(inp_np["PL"], inp_np["QL"], inp_np["tok"], inp_np["u"], inp_np["us"],
                         gamma, inp_np["branch_pos"], rule=rule, nthreads=nthreads, V=inp_np["V"])


def subset(inp_np: dict, idx):
    out = {k: (v[idx] if isinstance(v, np.ndarray) else v) for k, v in inp_np.items()}
    return out
