"""Exact laws through the GPU path (SURVEY §8.3 pins table: "Run the same enumeration
batch through the GPU (fp32 -> 1e-6)").

K = 1, s_b = 0 is vanilla speculative sampling (§3 P94): the first committed token is
distributed exactly as the target p.  The enumeration batch of the oracle pin
(tests/test_oracle_pins.py::enum_first_token_cases — every drafted x ~ q, the accept /
reject interval of u and every residual inverse-CDF interval of us, at interval
midpoints, with its probability weight) is run through sb_verify_branches +
sb_select_branch on the device; the weighted law of the GPU's committed tokens must equal
p within 1e-6 (fp32 arithmetic: a midpoint can only land in the wrong interval when the
interval is narrower than the fp32 error, and then its weight is below it).
The heterogeneous first-rejection law P(n = k) = prod_{i<k} beta_i (1 - beta_k) (Eq. 2
generalised to per-row rates) is checked the same way."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2506_01979_b200.build import build

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    build()


def gpu_round(PL, QL, tok, u, us, gamma, bpos):
    """One verify + select round on the device (fp32 logits, fp32 uniforms)."""
    from paper_2506_01979_b200 import api

    dev = "cuda"
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), device=dev).to(dt)  # noqa: E731
    inp = {"PL": t(PL, torch.float32), "QL": t(QL, torch.float32), "tok": t(tok, torch.int32),
           "u": t(u, torch.float32), "us": t(us, torch.float32), "gamma": t(gamma, torch.int32),
           "branch_pos": t(bpos, torch.int32), "V": PL.shape[-1]}
    d = api.dims_for(inp["PL"], V=inp["V"])
    buf = api.StepBuffers.alloc(d, dev)
    api.verify_step(d, inp, buf, fused=False)
    torch.cuda.synchronize()
    return {k: getattr(buf, k).cpu().numpy() for k in ("out_tok", "n_acc", "status", "commit_len")}


@pytest.mark.parametrize("V", [2, 4, 8])
def test_gpu_losslessness_enumeration(V):
    from test_oracle_pins import enum_first_token_cases, first_token_law

    rng = np.random.default_rng(2506 + V)
    batches = []
    for t in range(200):
        P0 = rng.dirichlet(np.ones(V))
        Q0 = rng.dirichlet(np.ones(V))
        if t % 10 == 0:
            Q0[rng.integers(V)] = 0.0  # masked draft tokens
            Q0 /= Q0.sum()
        batches.append(enum_first_token_cases(P0, Q0, V))
    PL = np.concatenate([b[0] for b in batches])
    QL = np.concatenate([b[1] for b in batches])
    tok = np.concatenate([b[2] for b in batches])
    u = np.concatenate([b[3] for b in batches]).astype(np.float32)
    us = np.concatenate([b[4] for b in batches]).astype(np.float32)
    n = len(us)
    g = gpu_round(PL, QL, tok, u, us, np.ones(n), np.zeros(n))
    assert (g["status"] == 0).all() and (g["commit_len"] >= 1).all()
    worst, off = 0.0, 0
    for (_, _, _, _, _, w, Pe) in batches:
        m = len(w)
        law = first_token_law(g["out_tok"][off:off + m, 0], w, V)
        worst = max(worst, float(np.abs(law - Pe).max()))
        off += m
    print(f"V={V}: {n} enumerated rounds, max |law - p| = {worst:.3g}")
    assert worst < 1e-6, worst


def test_gpu_heterogeneous_first_rejection_law():
    """P(n_0 = k) over the enumeration of (x_i, accept/reject interval of u_i), V = 3,
    gamma = 3, per-row (p_i, q_i): equals prod_{i<k} beta_i (1 - beta_k) within 1e-6."""
    from test_oracle_pins import logits_from_probs, softmax64

    rng = np.random.default_rng(3)
    V, G = 3, 3
    for trial in range(4):
        P = rng.dirichlet(np.ones(V), size=G + 1)
        Q = rng.dirichlet(np.ones(V), size=G + 1)
        lp, lq = logits_from_probs(P), logits_from_probs(Q)
        Pe = np.array([softmax64(r) for r in lp])
        Qe = np.array([softmax64(r) for r in lq])
        beta = np.minimum(Pe, Qe).sum(axis=1)
        cases = []
        for xs in np.ndindex(*(V,) * G):
            for pat in np.ndindex(*(2,) * G):
                w, us_ = 1.0, []
                for i in range(G):
                    a = min(1.0, Pe[i, xs[i]] / Qe[i, xs[i]])
                    w *= Qe[i, xs[i]] * (a if pat[i] == 0 else 1 - a)
                    us_.append(a / 2 if pat[i] == 0 else (1 + a) / 2)
                if w > 0:
                    cases.append((xs, us_, w))
        n = len(cases)
        PL = np.broadcast_to(lp[None, None], (n, 1, G + 1, V)).copy()
        QL = np.broadcast_to(lq[None, None], (n, 1, G + 1, V)).copy()
        tok = np.zeros((n, 1, G + 1), np.int32)
        u = np.zeros((n, 1, G + 1), np.float32)
        for b, (xs, us_, _) in enumerate(cases):
            tok[b, 0, :G] = xs
            u[b, 0, :G] = us_
        g = gpu_round(PL, QL, tok, u, np.full(n, 0.5, np.float32), np.full(n, G), np.zeros(n))
        law = np.zeros(G + 1)
        np.add.at(law, g["n_acc"][:, 0], [c[2] for c in cases])
        ref = np.array([np.prod(beta[:k]) * (1 - beta[k]) for k in range(G)] + [np.prod(beta[:G])])
        assert np.abs(law - ref).max() < 1e-6, (trial, law, ref)
