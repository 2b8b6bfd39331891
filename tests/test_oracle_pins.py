"""Pins that hold the fp64 oracle to what the paper and the mathematics fix.

None of these re-types the oracle's formula and compares it with itself: each checks
a closed form (Lemma 1, Eq. 2, softmax of a uniform / one-hot / two-point row), an
exact law obtained by enumeration (losslessness of speculative sampling, P94; the
heterogeneous first-rejection law), a Monte-Carlo law (truncated geometric, Eq. 2
P135, S162/S680), an invariant (p = q accepts everything, shift invariance,
compaction identities) or a worked example printed in SPEC.md / the paper
(tests/golden/spec_examples.json, each with its citation).
"""
import json
import math
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------- helpers
def logits_from_probs(rows):
    """fp32 logits ln p (-inf where p = 0) for a list of probability rows."""
    a = np.asarray(rows, dtype=np.float64)
    with np.errstate(divide="ignore"):
        return np.log(a).astype(np.float32)


def softmax64(l):
    l = l.astype(np.float64)
    m = l.max()
    e = np.exp(l - m)
    return e / e.sum()


def one_round(P_rows, Q_rows, tok, u, us=0.5, K=1, s=0, gamma=None, rule=0, orc=None, f64=False):
    """Single-sequence round from per-(slot,row) probability rows.
    P_rows/Q_rows: [K][G+1][V] probabilities; tok, u: [K][G+1]."""
    PL = logits_from_probs(P_rows)[None]
    QL = logits_from_probs(Q_rows)[None]
    G = PL.shape[2] - 1
    gamma = G if gamma is None else gamma
    return orc.verify(PL, QL, np.asarray(tok, np.int32)[None], np.asarray(u)[None],
                      np.asarray([us]), gamma=[gamma], branch_pos=[s], rule=rule, f64_uniforms=f64)


# ---------------------------------------------------------------- softmax stats
def test_uniform_row_closed_form(orc):
    V = 7
    QL = np.full((1, 1, 2, V), 1.5, np.float32)
    P, lse = orc.row_softmax(QL, 0, 0, 0)
    assert np.allclose(P, 1.0 / V, rtol=0, atol=1e-15)
    assert abs(lse - (1.5 + math.log(V))) < 1e-14
    c = orc.confidence(QL, mode=orc.CONF_TOP1)
    assert abs(c["top1_prob"][0, 0, 0] - 1.0 / V) < 1e-15
    assert c["top1_id"][0, 0, 0] == 0  # ties -> smallest id (S393, S443)
    assert abs(c["entropy"][0, 0, 0] - math.log(V)) < 1e-14  # H(uniform) = ln V


def test_one_hot_row(orc):
    QL = np.full((1, 1, 2, 4), -np.inf, np.float32)
    QL[0, 0, 0, 1] = 2.0
    P, lse = orc.row_softmax(QL, 0, 0, 0)
    assert P.tolist() == [0.0, 1.0, 0.0, 0.0] and lse == 2.0
    c = orc.confidence(QL)
    assert c["top1_prob"][0, 0, 0] == 1.0 and c["top1_id"][0, 0, 0] == 1 and c["entropy"][0, 0, 0] == 0.0


def test_two_point_closed_form(orc):
    QL = np.zeros((1, 1, 2, 2), np.float32)
    QL[0, 0, 0] = [0.0, 1.0]
    P, lse = orc.row_softmax(QL, 0, 0, 0)
    e = math.e
    assert abs(P[1] - e / (1 + e)) < 1e-15 and abs(lse - math.log(1 + e)) < 1e-15
    h = -(P[0] * math.log(1 / (1 + e)) + P[1] * math.log(e / (1 + e)))
    assert abs(orc.confidence(QL)["entropy"][0, 0, 0] - h) < 1e-15


def test_shift_invariance(orc):
    rng = np.random.default_rng(1)
    V = 50
    base = (rng.integers(-64, 64, size=(1, 1, 3, V)) / 8.0).astype(np.float32)  # exact dyadics
    shifted = (base + np.float32(16.0)).astype(np.float32)
    assert np.all(shifted - base == 16.0)
    a, b = orc.confidence(base), orc.confidence(shifted)
    for k in ("top1_prob", "entropy"):
        assert np.allclose(a[k], b[k], rtol=1e-13, atol=1e-15)
    assert np.array_equal(a["top1_id"], b["top1_id"])
    for i in range(2):
        Pa, la = orc.row_softmax(base, 0, 0, i)
        Pb, lb = orc.row_softmax(shifted, 0, 0, i)
        assert np.allclose(Pa, Pb, rtol=1e-13, atol=1e-16) and abs(lb - la - 16.0) < 1e-12


def test_bf16_widening_is_exact(orc):
    # 0x3FC0 = 1.5, 0xC000 = -2.0, 0x7F80 = +inf, 0xFF80 = -inf
    L = np.array([0x3FC0, 0xC000, 0xFF80, 0x3F80], np.uint16).reshape(1, 1, 1, 4)
    L = np.concatenate([L, L], axis=2)
    P, lse = orc.row_softmax(L, 0, 0, 0)
    ref = softmax64(np.array([1.5, -2.0, -np.inf, 1.0]))
    assert np.allclose(P, ref, atol=1e-16)


def test_softmax_is_plain_at_any_magnitude(orc):
    """oracle_row_softmax is the plain definition for every finite row, whatever its
    magnitude (the library's input domain is a separate validation step, DESIGN reading
    34): a row at -2^98 with one entry 2^91 above the rest is a point mass; a row whose
    entries are all equal is uniform; finfo(bf16).min masks contribute exactly 0."""
    V = 6
    L = np.full((1, 1, 2, V), -(2.0 ** 98), np.float32)
    P, lse = orc.row_softmax(L, 0, 0, 0)
    assert np.allclose(P, 1.0 / V, atol=1e-15) and lse == -(2.0 ** 98) + math.log(V)
    L[0, 0, 0, 3] = -(2.0 ** 98) + 2.0 ** 91
    P, _ = orc.row_softmax(L, 0, 0, 0)
    assert P.tolist() == [0, 0, 0, 1.0, 0, 0]
    assert orc.row_domain(L, 0, 0, 0) == orc.ST_RANGE
    bmin = np.float32(-3.3895313892515355e38)  # finfo(bfloat16).min, exact in fp32
    L2 = np.full((1, 1, 2, V), bmin, np.float32)
    a = float(np.float32(math.log(3.0)))  # exactly the stored fp32 value
    L2[0, 0, 0, :2] = [0.0, a]
    P, lse = orc.row_softmax(L2, 0, 0, 0)
    ea = math.exp(a)
    assert np.allclose(P, [1 / (1 + ea), ea / (1 + ea), 0, 0, 0, 0], atol=1e-15)
    assert abs(lse - math.log1p(ea)) < 1e-15
    assert orc.row_domain(L2, 0, 0, 0) == 0


def test_row_domain_classes(orc):
    """The validation step's classes, in its stated order (oracle.h)."""
    V = 4

    def dom(vals):
        L = np.zeros((1, 1, 1, V), np.float32)
        L[0, 0, 0] = vals
        return orc.row_domain(L, 0, 0, 0)

    assert dom([0.0, 1.0, -np.inf, 2.0 ** 24 - 2]) == 0
    assert dom([0.0, 1.0, 2.0 ** 24, 3.0]) == orc.ST_RANGE
    assert dom([-(2.0 ** 24), -(2.0 ** 25), -np.inf, -np.inf]) == orc.ST_RANGE
    assert dom([-np.inf] * 4) == orc.ST_NONFINITE
    assert dom([0.0, np.inf, 1.0, 2.0]) == orc.ST_NONFINITE
    assert dom([0.0, np.nan, 1.0, 2.0]) == orc.ST_NONFINITE
    assert dom([np.nan, -(2.0 ** 30), 1e30, 2.0]) == orc.ST_RANGE  # range checked before NaN
    assert dom([np.nan] * 4) == orc.ST_NONFINITE


# ---------------------------------------------------------------- accept test (P94, S123-149)
@pytest.mark.parametrize("case", GOLD["accept_prob"])
def test_accept_prob_examples(orc, case):
    p, q = case["p"], case["q"]
    P = [[[p, 1 - p], [0.5, 0.5]]]
    Q = [[[q, 1 - q], [0.5, 0.5]]]
    beta = case["beta"]
    for du, acc in ((-1e-3, 1), (1e-3, 0)):
        u = min(max(beta + du, 0.0), 0.999)
        if beta >= 1.0 and du > 0:
            continue  # beta = 1 accepts every u in [0,1)
        o = one_round(P, Q, [[0, 0]], [[u, 0.0]], K=1, s=0, gamma=1, orc=orc)
        ratio = o["p_tok"][0, 0, 0] / o["q_tok"][0, 0, 0]
        assert abs(min(1.0, ratio) - beta) < 1e-6
        assert (o["acc_mask"][0, 0] & 1) == acc


def test_verify_sequence_hand_trace(orc):
    case = GOLD["verify_sequence"][0]
    # row 0: p = q (ratio 1.0); row 1: p = (.2,.8), q = (.5,.5) at x = 0 -> ratio 0.4
    P = [[[0.5, 0.5], [0.2, 0.8], [0.5, 0.5]]]
    Q = [[[0.5, 0.5], [0.5, 0.5], [0.5, 0.5]]]
    o = one_round(P, Q, [[0, 0, 0]], [case["r"] + [0.0]], K=1, s=0, gamma=2, orc=orc)
    assert o["n_acc"][0, 0] == case["n"]
    # rejection at 0-based row 1 -> residual norm(max(0, p - q)) = (0, 1) -> y = 1 (P94, P554)
    assert o["y_kind"][0] == 1 and o["y_tok"][0] == 1
    assert o["commit_len"][0] == 2 and o["out_tok"][0, :2].tolist() == [0, 1]


@pytest.mark.parametrize("case", GOLD["residual"])
def test_residual_examples(orc, case):
    p, q, res = case["p"], case["q"], case["residual"]
    x = int(np.argmax(q))  # a token q proposes
    assert p[x] < q[x]
    u = 0.999  # > p/q: rejected
    for us in (0.01, 0.5, 0.99):
        o = one_round([[p, p]], [[q, q]], [[x, 0]], [[u, 0.0]], us=us, gamma=1, orc=orc)
        assert o["n_acc"][0, 0] == 0 and o["y_kind"][0] == 1
        assert o["y_tok"][0] == int(np.argmax(res))  # the residual is a point mass


def test_p_equals_q_accepts_everything(orc):
    """Identical p and q accept every drafted token (north_star; S131, S148)."""
    from paper_2506_01979_b200 import synth

    cfg = synth.config("c2", V=64, B=24, K=3, G=6, layout="mixed")
    inp = synth.to_numpy_inputs(synth.generate(cfg, seed=7))
    o = orc.verify(inp["PL"], inp["PL"], inp["tok"], inp["u"], inp["us"], inp["gamma"], inp["branch_pos"])
    for b in range(cfg.B):
        g, s = inp["gamma"][b], inp["branch_pos"][b]
        L = g if s < g else g + 1
        assert (o["n_acc"][b] == L).all()
        assert (o["acc_mask"][b] == (1 << L) - 1).all()
        assert o["path_rolled"][b] == 0


def test_point_mass_mismatch_rejects(orc):
    P = [[[1.0, 0.0], [0.5, 0.5]]]
    Q = [[[0.0, 1.0], [0.5, 0.5]]]
    o = one_round(P, Q, [[1, 0]], [[0.3, 0.0]], gamma=1, orc=orc)  # x=1: p/q = 0 (S79)
    assert o["n_acc"][0, 0] == 0 and o["y_tok"][0] == 0  # residual is all on token 0
    o = one_round(P, Q, [[1, 0]], [[0.0, 0.0]], gamma=1, orc=orc)  # u = 0 accepts (reading #2)
    assert o["n_acc"][0, 0] == 1


def test_q_zero_accepts(orc):
    P = [[[0.5, 0.5], [0.5, 0.5]]]
    Q = [[[1.0, 0.0], [0.5, 0.5]]]
    o = one_round(P, Q, [[1, 0]], [[0.999, 0.0]], gamma=1, orc=orc)  # q[x]=0 -> accept (S127)
    assert o["n_acc"][0, 0] == 1


# ---------------------------------------------------------------- exact laws by enumeration
def enum_first_token_cases(P0, Q0, V):
    """Batch of one-row rounds (K = 1, s_b = 0, gamma_b = 1) covering every (x,
    u-interval, us-interval) at interval midpoints, with the probability weight of each:
    x ~ Q, then u < a = min(1, P/Q) (accept) or u in (a, 1) followed by the residual's
    inverse-CDF intervals of us.  Returns (PL, QL, tok, u, us, w, Pe)."""
    toks, us_l, uu, w = [], [], [], []
    lp = logits_from_probs([P0, P0])
    lq = logits_from_probs([Q0, Q0])
    Pe, Qe = softmax64(lp[0]), softmax64(lq[0])
    r = np.maximum(0.0, Pe - Qe)
    R = r.sum()
    F = np.cumsum(r)
    for x in range(V):
        if Qe[x] == 0:
            continue
        rho = Pe[x] / Qe[x]
        a = min(1.0, rho)
        toks.append(x); uu.append(a / 2); us_l.append(0.5); w.append(Qe[x] * a)
        if a < 1.0:
            for j in range(V):
                if r[j] <= 0:
                    continue
                lo = (F[j] - r[j]) / R
                toks.append(x); uu.append((1 + a) / 2); us_l.append(lo + r[j] / R / 2)
                w.append(Qe[x] * (1 - a) * r[j] / R)
    n = len(toks)
    PL = np.broadcast_to(lp, (n, 1, 2, V)).copy()
    QL = np.broadcast_to(lq, (n, 1, 2, V)).copy()
    tok = np.zeros((n, 1, 2), np.int32)
    tok[:, 0, 0] = toks
    u = np.zeros((n, 1, 2))
    u[:, 0, 0] = uu
    return PL, QL, tok, u, np.asarray(us_l), np.asarray(w), Pe


def first_token_law(out_tok0, w, V):
    law = np.zeros(V)
    np.add.at(law, out_tok0, w)
    return law


def _enumerate_first_token_law(orc, P0, Q0, V):
    PL, QL, tok, u, us, w, Pe = enum_first_token_cases(P0, Q0, V)
    n = len(w)
    o = orc.verify(PL, QL, tok, u, us, gamma=np.ones(n), branch_pos=np.zeros(n), f64_uniforms=True)
    return first_token_law(o["out_tok"][:, 0], w, V), Pe


def test_losslessness_enumeration(orc):
    """K=1, s_b=0 is vanilla speculative sampling (P94): the first committed token is
    distributed exactly as p, for 600 random (p,q) pairs, V in {2,4,8} (S150-161)."""
    rng = np.random.default_rng(2506)
    worst = 0.0
    for t in range(600):
        V = (2, 4, 8)[t % 3]
        P0 = rng.dirichlet(np.ones(V))
        Q0 = rng.dirichlet(np.ones(V))
        if t % 10 == 0:
            Q0[rng.integers(V)] = 0.0  # some q zeros (masked draft tokens)
            Q0 /= Q0.sum()
        law, Pe = _enumerate_first_token_law(orc, P0, Q0, V)
        worst = max(worst, np.abs(law - Pe).max())
    assert worst < 1e-12, worst


def test_heterogeneous_first_rejection_law(orc):
    """P(n=k) = prod_{i<k} beta_i (1 - beta_k), beta_i = sum_v min(p_i, q_i) (P94; Eq. 2
    generalised to per-row rates), by exact enumeration over x_i ~ q_i and u_i."""
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
        u = np.zeros((n, 1, G + 1))
        for b, (xs, us_, _) in enumerate(cases):
            tok[b, 0, :G] = xs
            u[b, 0, :G] = us_
        o = orc.verify(PL, QL, tok, u, np.full(n, 0.5), gamma=np.full(n, G), branch_pos=np.zeros(n),
                       f64_uniforms=True)
        law = np.zeros(G + 1)
        for b, (_, _, w) in enumerate(cases):
            law[o["n_acc"][b, 0]] += w
        ref = [np.prod(beta[:k]) * (1 - beta[k]) for k in range(G)] + [np.prod(beta[:G])]
        assert np.abs(law - np.asarray(ref)).max() < 1e-12


def _iid_rows(alpha, V):
    """(P, Q) with sum_v min(P,Q) = alpha exactly: P = alpha Q + (1-alpha) delta_{V-1}, Q(V-1)=0."""
    Q = np.r_[np.full(V - 1, 1.0 / (V - 1)), 0.0]
    P = alpha * Q
    P[V - 1] = 1 - alpha
    return P, Q


@pytest.mark.parametrize("case", GOLD["lemma1"])
def test_lemma1_mean_by_enumeration(orc, case):
    """E[n] for i.i.d. rows equals Lemma 1, alpha(1-alpha^gamma)/(1-alpha) (P566-582), and
    the law is Eq. 2's truncated geometric (P135), by exact enumeration of the oracle."""
    a, G = case["alpha"], case["gamma"]
    V = 2
    P, Q = _iid_rows(a, V)  # Q = (1, 0): x = 0 always; accept w.p. alpha
    lp, lq = logits_from_probs([P] * (G + 1)), logits_from_probs([Q] * (G + 1))
    alpha_real = min(softmax64(lp[0])[0] / softmax64(lq[0])[0], 1.0)
    # enumerate first-rejection position k in [0, G]: rows < k accept-mid, row k reject-mid
    n = G + 1
    u = np.zeros((n, 1, G + 1))
    w = np.zeros(n)
    for k in range(n):
        u[k, 0, :k] = alpha_real / 2
        if k < G:
            u[k, 0, k] = (1 + alpha_real) / 2
        w[k] = alpha_real**k * ((1 - alpha_real) if k < G else 1.0)
    o = orc.verify(np.broadcast_to(lp[None, None], (n, 1, G + 1, V)).copy(),
                   np.broadcast_to(lq[None, None], (n, 1, G + 1, V)).copy(),
                   np.zeros((n, 1, G + 1), np.int32), u, np.full(n, 0.5),
                   gamma=np.full(n, G), branch_pos=np.zeros(n), f64_uniforms=True)
    assert o["n_acc"][:, 0].tolist() == list(range(n))
    EX = float((w * o["n_acc"][:, 0]).sum())
    closed = alpha_real * (1 - alpha_real**G) / (1 - alpha_real)
    assert abs(EX - closed) < 1e-12
    assert abs(closed - case["EX"]) < case.get("tol", 1e-12) + 1e-6  # the paper-level value
    if "pmf" in case:
        assert np.allclose(w, case["pmf"], atol=1e-6)


@pytest.mark.parametrize("alpha", [0.3, 0.5, 0.7, 0.9])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_truncated_geometric_monte_carlo(orc, alpha, G):
    """x_i ~ q, u_i ~ U(0,1) i.i.d.: n ~ TruncGeo(alpha, gamma), Eq. 2 (P135); TV < 0.01
    at 10^5 rounds (S162, S680)."""
    V, n = 6, 100_000
    P, Q = _iid_rows(alpha, V)
    lp, lq = logits_from_probs([P] * (G + 1)), logits_from_probs([Q] * (G + 1))
    rng = np.random.default_rng(int(alpha * 100) + G)
    tok = np.zeros((n, 1, G + 1), np.int32)
    tok[:, 0, :G] = rng.integers(0, V - 1, size=(n, G))  # x ~ Q (uniform on V-1 tokens)
    u = rng.random((n, 1, G + 1)).astype(np.float32)
    o = orc.verify(np.broadcast_to(lp[None, None], (n, 1, G + 1, V)).copy(),
                   np.broadcast_to(lq[None, None], (n, 1, G + 1, V)).copy(),
                   tok, u, rng.random(n).astype(np.float32), gamma=np.full(n, G), branch_pos=np.zeros(n))
    hist = np.bincount(o["n_acc"][:, 0], minlength=G + 1) / n
    pmf = np.array([(1 - alpha) * alpha**k for k in range(G)] + [alpha**G])
    assert 0.5 * np.abs(hist - pmf).sum() < 0.01
    assert abs(o["n_acc"][:, 0].mean() - alpha * (1 - alpha**G) / (1 - alpha)) < 0.03


# ---------------------------------------------------------------- branch-point verification
def _branch_round(orc, p_branch, q_branch, rule=0, u_branch=None, toks=(1, 2), V=4):
    """K = len(toks) branches at row s_b = gamma_b = 0 (Alg.-1 form, P538; L_b = 1)."""
    K = len(toks)
    P = np.full(V, (1 - sum(p_branch)) / (V - K))
    Q = np.full(V, (1 - sum(q_branch)) / (V - K))
    for t, pp, qq in zip(toks, p_branch, q_branch):
        P[t], Q[t] = pp, qq
    Prow = [[P] for _ in range(K)]
    Qrow = [[Q] for _ in range(K)]
    tok = [[t] for t in toks]
    u = [[0.5 if u_branch is None else u_branch[k]] for k in range(K)]
    return one_round(Prow, Qrow, tok, u, K=K, s=0, gamma=0, rule=rule, orc=orc)


def test_branch_select_eq9_trace(orc):
    case = GOLD["branch_point"][0]
    o = _branch_round(orc, case["p_branch"], case["p_branch"])  # p = q at both: both accepted
    assert o["n_acc"][0].tolist() == [1, 1]
    assert o["sel_k"][0] == case["selected"]
    assert o["y_kind"][0] == 0 and o["commit_len"][0] == 1 and o["out_tok"][0, 0] == 2
    # Algorithm-1 variant: argmax r_b (P540)
    o = _branch_round(orc, [0.1, 0.4], [0.1, 0.4], rule=1, u_branch=[0.9, 0.2])
    assert o["sel_k"][0] == 0


def test_branch_single_p_eq_q(orc):
    o = _branch_round(orc, [0.3], [0.3], toks=(2,))
    assert o["sel_k"][0] == GOLD["branch_point"][1]["selected"] and o["n_acc"][0, 0] == 1


def test_branch_none_accepted_is_rollback(orc):
    # p(x_b) = 0.01 << q(x_b) = 0.4 for both, u = 0.5 -> both rejected (P655)
    o = _branch_round(orc, [0.01, 0.01], [0.4, 0.4])
    assert o["sel_k"][0] == GOLD["branch_point"][2]["selected"]
    assert o["y_kind"][0] == 1 and o["commit_len"][0] == 1
    assert o["y_tok"][0] not in (1, 2)  # residual has no mass on the over-drafted tokens


def test_branch_eq9_ties_smaller_token_then_k(orc):
    # equal target logits at the two branch tokens -> smaller token id wins (S443)
    o = _branch_round(orc, [0.3, 0.3], [0.3, 0.3], toks=(3, 1))
    assert o["sel_k"][0] == 1
    o = _branch_round(orc, [0.3, 0.3], [0.3, 0.3], toks=(2, 2))  # same token -> smaller k
    assert o["sel_k"][0] == 0


def test_branch_alg1_ties_smaller_k(orc):
    """Alg. 1 argmax r_b (P540) with equal uniforms: the smaller branch index wins
    (DESIGN reading 36), whatever the tokens' ids."""
    o = _branch_round(orc, [0.3, 0.3], [0.3, 0.3], rule=1, u_branch=[0.25, 0.25], toks=(3, 1))
    assert o["n_acc"][0].tolist() == [1, 1] and o["sel_k"][0] == 0


def test_k1_branch_coupling_equals_single_token_test(orc):
    """K=1 at the branch row (s=gamma) makes the same accept decision as the plain test
    with the same uniform (S438)."""
    rng = np.random.default_rng(5)
    for _ in range(50):
        V = 5
        P, Q = rng.dirichlet(np.ones(V)), rng.dirichlet(np.ones(V))
        x = int(rng.integers(V))
        u = float(rng.random())
        a = one_round([[P]], [[Q]], [[x]], [[u]], K=1, s=0, gamma=0, orc=orc)  # branch form
        b = one_round([[P, P]], [[Q, Q]], [[x, 0]], [[u, 0.0]], K=1, s=0, gamma=1, orc=orc)  # SD form
        assert a["n_acc"][0, 0] == b["n_acc"][0, 0]


# ---------------------------------------------------------------- compaction invariants
def test_compaction_invariants(orc):
    from paper_2506_01979_b200 import synth

    cfg = synth.config("c2", V=40, B=64, K=3, G=6, layout="mixed", delta=2.0, rho_same=0.5)
    inp = synth.to_numpy_inputs(synth.generate(cfg, seed=11))
    for rule in (0, 1):
        o = orc.verify(inp["PL"], inp["QL"], inp["tok"], inp["u"], inp["us"], inp["gamma"],
                       inp["branch_pos"], rule=rule)
        K = cfg.K
        assert o["offsets"][0] == 0 and (np.diff(o["offsets"]) == o["commit_len"]).all()
        kinds = set()
        for b in range(cfg.B):
            g, s = int(inp["gamma"][b]), int(inp["branch_pos"][b])
            L = g if s < g else g + 1
            ks = o["sel_k"][b]
            n = o["n_acc"][b, ks] if ks >= 0 else min(o["n_acc"][b, 0], s)
            y = o["y_kind"][b] != 0
            kinds.add(int(o["y_kind"][b]))
            assert o["commit_len"][b] == n + y
            kp = max(ks, 0)
            path = [inp["tok"][b, 0 if i < s else kp, i] for i in range(n)]
            assert o["out_tok"][b, :n].tolist() == path
            assert (o["out_tok"][b, n + y:] == -1).all()
            assert o["path_rolled"][b] == L - n
            assert n + o["path_rolled"][b] + o["branch_discarded"][b] == s + K * (L - s)
            assert o["packed_tok"][o["offsets"][b]: o["offsets"][b + 1]].tolist() == o["out_tok"][b, : n + y].tolist()
            # A = {k : n_k > s}; empty <=> sel_k = -1 (Eq. 9, P655)
            assert (ks == -1) == (not (o["n_acc"][b] > s).any())
            if ks >= 0:
                assert o["n_acc"][b, ks] > s
        assert kinds == {0, 1, 2}


# ---------------------------------------------------------------- confidence (Eq. 6, Eq. 7, §4.2)
def _conf_rows(confs, V=10):
    rows = []
    for c in confs:
        r = np.full(V, (1 - c) / (V - 1))
        r[0] = c
        rows.append(r)
    rows.append(np.full(V, 1.0 / V))
    return logits_from_probs(rows)[None, None]


@pytest.mark.parametrize("case", GOLD["confidence_stop"])
def test_confidence_stop_examples(orc, case):
    QL = _conf_rows(case["conf"])
    o = orc.confidence(QL, mode=orc.CONF_TOP1, eps=case["eps"], k_max=6)
    assert o["stop"][0, 0] == case["stop"]
    assert o["gamma_next"][0, 0] == max(1, case["stop"])
    if case["stop"] < len(case["conf"]):
        c = case["conf"][case["stop"]]
        assert o["k_next"][0, 0] == max(1, math.floor(6 * (1 - c) + 1e-9))
    else:
        assert o["k_next"][0, 0] == -1


def test_entropy_stop_uniform4(orc):
    case = GOLD["entropy_stop"][0]
    QL = np.zeros((1, 1, 2, case["uniform_over"]), np.float32)
    o = orc.confidence(QL, mode=orc.CONF_ENTROPY, eps=case["eps"], lam=case["lambda"])
    assert abs(o["stat"][0, 0, 0] - (1 - math.sqrt(math.log(4)))) < 1e-14
    assert o["stop"][0, 0] == 0
    QL = np.full((1, 1, 2, 4), -np.inf, np.float32)
    QL[..., 0] = 0.0  # point mass: H = 0, statistic 1 -> no stop (S320)
    assert orc.confidence(QL, mode=orc.CONF_ENTROPY, eps=0.2)["stop"][0, 0] == 1


@pytest.mark.parametrize("case", GOLD["adaptive_k"])
def test_adaptive_k_examples(orc, case):
    assert orc.adaptive_k(case["q"], case["k_max"]) == case["k"]


def test_token_mode_uses_drafted_token(orc):
    QL = _conf_rows([0.9, 0.9, 0.9])
    tok = np.zeros((1, 1, 4), np.int32)
    tok[0, 0, 1] = 5  # q(x_1) = 0.1/9 <= 0.2 -> stop at 1 in TOKEN mode (Eq. 6 P198, Alg. 1 P517)
    o = orc.confidence(QL, tok=tok, mode=orc.CONF_TOKEN, eps=0.2)
    assert o["stop"][0, 0] == 1
    assert abs(o["tok_prob"][0, 0, 1] - 0.1 / 9) < 1e-7
    assert o["k_next"][0, 0] == max(1, math.floor(6 * (1 - 0.1 / 9)))


# ---------------------------------------------------------------- degenerate cases and status
def test_gamma0_branch_row_only(orc):
    """gamma_b = 0, s_b = 0: the branch point is the first token (H-RAD s_t = 0, P669)."""
    o = _branch_round(orc, [0.2, 0.2], [0.2, 0.2])
    assert o["commit_len"][0] == 1 and o["y_kind"][0] == 0


def test_status_flags(orc):
    P = [[[0.5, 0.5], [0.5, 0.5]]]
    o = one_round(P, P, [[7, 0]], [[0.1, 0.0]], gamma=1, orc=orc)  # token out of range
    assert o["status"][0] & orc.ST_BAD_TOKEN and o["n_acc"][0, 0] == 0
    PL = logits_from_probs(P)[None]
    PL[0, 0, 0, 1] = np.nan
    o = orc.verify(PL, PL, np.zeros((1, 1, 2), np.int32), np.zeros((1, 1, 2)), np.array([0.5]),
                   gamma=[1], branch_pos=[0])
    assert o["status"][0] & orc.ST_NONFINITE
    # input domain (DESIGN reading 34): a finite row whose maximum has |m| >= 2^24 is
    # not evaluated (ST_RANGE, NaN outputs); masks below an in-range maximum are exact
    M = np.full_like(PL, -(2.0 ** 98))
    o = orc.verify(M, M, np.zeros((1, 1, 2), np.int32), np.zeros((1, 1, 2)), np.array([0.5]),
                   gamma=[1], branch_pos=[0])
    assert o["status"][0] == orc.ST_RANGE and np.isnan(o["lse_p"][0, 0, 0])
    M[..., 1] = -3.0
    o = orc.verify(M, M, np.ones((1, 1, 2), np.int32), np.zeros((1, 1, 2)), np.array([0.5]),
                   gamma=[1], branch_pos=[0])
    assert o["status"][0] == 0 and o["n_acc"][0, 0] == 1 and o["lse_p"][0, 0, 0] == -3.0
    A = np.full_like(PL, -np.inf)
    o = orc.verify(A, A, np.zeros((1, 1, 2), np.int32), np.zeros((1, 1, 2)), np.array([0.5]),
                   gamma=[1], branch_pos=[0])
    assert o["status"][0] == orc.ST_NONFINITE
    o = orc.verify(PL * 0, PL * 0, np.zeros((1, 1, 2), np.int32), np.zeros((1, 1, 2)), np.array([0.5]),
                   gamma=[5], branch_pos=[9])
    assert o["status"][0] & orc.ST_GAMMA_CLAMPED and o["status"][0] & orc.ST_BRANCH_CLAMPED


# ---------------------------------------------------------------- branch spawn (f1, Eq. 7)
@pytest.mark.parametrize("case", GOLD["spawn_branches"])
def test_spawn_examples(orc, case):
    q = case["q"]
    QL = logits_from_probs([q, q])[None, None]
    o = orc.spawn(QL, k_max=case["k_max"])
    k = case["k"]
    assert o["k"][0] == k
    assert o["btok"][0, :k].tolist() == case["tokens"]
    assert (o["btok"][0, k:] == -1).all()
    assert np.allclose(o["bprob"][0, :k], np.asarray(q)[case["tokens"]], rtol=1e-6)


def test_spawn_topk_is_max_mass_subset_bruteforce(orc):
    """The spawned set has the largest q-mass of all k-subsets (S437) and respects Eq. 7."""
    import itertools

    rng = np.random.default_rng(77)
    for t in range(200):
        V = int(rng.integers(2, 9))
        q = rng.dirichlet(np.ones(V) * 0.7)
        if t % 5 == 0:  # ties
            q = np.round(q * 8) / 8 + 1e-3
            q /= q.sum()
        k_max = int(rng.integers(1, 9))
        QL = logits_from_probs([q, q])[None, None]
        o = orc.spawn(QL, k_max=k_max)
        Q = softmax64(QL[0, 0, 0])
        c = Q.max()
        k_ref = min(V, max(1, math.floor(k_max * (1 - c) + 0.0)))
        if not (o["ties"][0] & orc.TIE_EQ7):
            assert o["k"][0] == k_ref
        k = o["k"][0]
        chosen = o["btok"][0, :k]
        assert len(set(chosen.tolist())) == k
        best = max(sum(Q[list(sub)]) for sub in itertools.combinations(range(V), k))
        assert abs(Q[chosen].sum() - best) < 1e-12
        # order: descending q, ties -> smaller id
        pairs = [(-Q[x], x) for x in chosen]
        assert pairs == sorted(pairs)


def test_kv_rollback_rows_are_keep_mask(orc):
    """f2 pin: the gathered rows are exactly the verify oracle's keep_mask positions
    (P241 keep the selected branch's KV, discard the rest) — two independent statements
    of the committed draft positions — and nothing at or past n_b is kept."""
    import oracle
    from paper_2506_01979_b200 import synth

    c = synth.config("c2", V=512, B=32, K=3, G=6, layout="mixed")
    inp_np = synth.to_numpy_inputs(synth.generate(c, device="cpu", seed=41))
    inp_np["gamma"][:3] = [9, 4, 3]  # clamped layouts: gamma > G, s > gamma, s < 0
    inp_np["branch_pos"][:3] = [1, 6, -2]
    o = oracle.verify(inp_np["PL"], inp_np["QL"], inp_np["tok"], inp_np["u"], inp_np["us"], inp_np["gamma"],
                      inp_np["branch_pos"])
    kv = np.arange(c.B * c.K * (c.G + 1) * 4, dtype=np.int64).reshape(c.B, c.K, c.G + 1, 4)
    out = oracle.kv_rollback(kv, inp_np["branch_pos"], inp_np["gamma"], o["sel_k"], o["commit_len"], o["y_kind"])
    for b in range(c.B):
        n = int(o["commit_len"][b]) - int(o["y_kind"][b] != 0)
        kept = [(k, i) for k in range(c.K) for i in range(c.G + 1) if (int(o["keep_mask"][b, k]) >> i) & 1]
        assert sorted(i for _, i in kept) == list(range(n)), b  # one kept row per committed position
        for k, i in kept:
            assert np.array_equal(out[b, i], kv[b, k, i])
        assert not out[b, n:].any()


def _branch_as_tree(inp_np, b):
    """Map sequence b of a branch-layout round (SURVEY §8.0 slot maps) to a token tree:
    shared prefix tokens i < s as a chain, then K chains for i in [s, L).  Context row
    after token i of branch k is the physical row ls(k, i+1) = (i+1 <= s ? 0 : k)."""
    PL, QL, tok, u = inp_np["PL"][b], inp_np["QL"][b], inp_np["tok"][b], inp_np["u"][b]
    K, R1, V = PL.shape
    g, s = int(inp_np["gamma"][b]), int(inp_np["branch_pos"][b])
    L = g if s < g else g + 1
    rows_p, rows_q = [PL[0, 0]], [QL[0, 0]]
    par, tk, uu, where = [], [], [], {}
    for i in range(s):
        par.append(i - 1)
        tk.append(tok[0, i]); uu.append(u[0, i])
        rows_p.append(PL[0, i + 1]); rows_q.append(QL[0, i + 1])
        where[(0, i)] = len(par) - 1
    for k in range(K):
        prev = s - 1
        for i in range(s, L):
            par.append(prev)
            tk.append(tok[k, i]); uu.append(u[k, i])
            ls = 0 if i + 1 <= s else k
            rows_p.append(PL[ls, i + 1]); rows_q.append(QL[ls, i + 1])
            prev = len(par) - 1
            where[(k, i)] = prev
    return (np.stack(rows_p), np.stack(rows_q), np.array(par, np.int32), np.array(tk, np.int32),
            np.array(uu, np.float32), L, s, where)


@pytest.mark.parametrize("K,dtype", [(1, "f32"), (3, "bf16"), (4, "f32")])
def test_tree_verify_reduces_to_branch_contract(orc, K, dtype):
    """f3 pin: a prefix-plus-K-chains tree is exactly SpecBranch's branch layout, so the
    tree walk (Eq. 9 at every node) must reproduce oracle.verify's commit, selected
    path and sampled y; K = 1 is the chain of plain speculative decoding (Alg. 1, P94).
    Cases with s = gamma (no bonus row inside the tensor) are skipped by construction."""
    import oracle
    from paper_2506_01979_b200 import synth

    c = synth.config("c2", V=400, B=40, K=K, G=6, layout="mixed", dtype=dtype)
    inp_np = synth.to_numpy_inputs(synth.generate(c, device="cpu", seed=71))
    o = oracle.verify(inp_np["PL"], inp_np["QL"], inp_np["tok"], inp_np["u"], inp_np["us"], inp_np["gamma"],
                      inp_np["branch_pos"])
    checked = 0
    for b in range(c.B):
        if int(inp_np["branch_pos"][b]) >= int(inp_np["gamma"][b]):
            continue
        PLt, QLt, par, tk, uu, L, s, where = _branch_as_tree(inp_np, b)
        t = oracle.tree_verify(PLt[None], QLt[None], par[None], tk[None], uu[None], inp_np["us"][b:b + 1])
        assert t["commit_len"][0] == o["commit_len"][b], b
        assert np.array_equal(t["out_tok"][0, : t["commit_len"][0]], o["out_tok"][b, : o["commit_len"][b]]), b
        assert t["y_kind"][0] == o["y_kind"][b] and t["y_tok"][0] == o["y_tok"][b], b
        for (k, i), j in where.items():
            assert ((int(t["acc_mask"][0]) >> j) & 1) == ((int(o["acc_mask"][b, k]) >> i) & 1), (b, k, i)
            assert ((int(t["keep_mask"][0]) >> j) & 1) == ((int(o["keep_mask"][b, k]) >> i) & 1), (b, k, i)
        checked += 1
    assert checked >= 10


@pytest.mark.parametrize("shape,kw", [("dense", dict(branching=(3, 2, 2))), ("random", dict(N=40, depth=7)),
                                      ("chain", dict(N=12))])
def test_tree_walk_is_valid(orc, shape, kw):
    """f3 pin: the committed path is a root path of accepted nodes; at every step the
    chosen child has the largest raw target logit among its accepted siblings (ties to
    the smaller token); the walk stops at a node none of whose children is accepted,
    and y is residual there iff that node has children (a leaf gives the bonus)."""
    import oracle
    from paper_2506_01979_b200 import synth

    c = synth.config("c2", V=257, dtype="f32")
    t = synth.tree_to_numpy(synth.generate_tree(c, shape, B=48, seed=5, **kw))
    o = oracle.tree_verify(t["PL"], t["QL"], t["parent"], t["tok"], t["u"], t["us"])
    N = t["N"]
    for b in range(48):
        par, tk, acc = t["parent"][b], t["tok"][b], int(o["acc_mask"][b])
        kids = lambda p: [j for j in range(N) if par[j] == p]  # noqa: E731
        c_node, path = -1, []
        while True:
            a = [j for j in kids(c_node) if (acc >> j) & 1]
            if not a:
                break
            key = lambda j: (-float(t["PL"][b, c_node + 1, tk[j]]), int(tk[j]), j)  # noqa: E731
            c_node = min(a, key=key)
            path.append(c_node)
        assert o["stop_node"][b] == c_node
        n = len(path)
        assert np.array_equal(o["out_tok"][b, :n], tk[path])
        assert int(o["keep_mask"][b]) == sum(1 << j for j in path)
        assert o["y_kind"][b] == (1 if kids(c_node) else 2)
        assert o["commit_len"][b] == n + 1 and 0 <= o["y_tok"][b] < c.V


def test_tree_accept_test_closed_form(orc):
    """f3 pin: a two-node tree with hand-set rows.  Root context p = (1/2, 1/4, 1/4),
    q = (1/4, 1/4, 1/2) (logits ln of these): child token 2 has p/q = 1/2 so u = 0.4
    accepts and u = 0.6 rejects (P94); token 0 has p/q = 2 and always accepts."""
    import oracle

    lp = np.log(np.array([0.5, 0.25, 0.25], np.float32))
    lq = np.log(np.array([0.25, 0.25, 0.5], np.float32))
    PL = np.stack([lp, lp, lp])[None].astype(np.float32)
    QL = np.stack([lq, lq, lq])[None].astype(np.float32)
    for u2, acc2 in [(0.4, 1), (0.6, 0)]:
        t = oracle.tree_verify(PL, QL, np.array([[-1, -1]], np.int32), np.array([[2, 0]], np.int32),
                               np.array([[u2, 0.99]], np.float32), np.array([0.5], np.float32))
        assert int(t["acc_mask"][0]) == (acc2 * 1 | 2)
        # both accepted -> Eq. 9 picks the larger target logit: token 0 (p = 1/2)
        assert t["stop_node"][0] == 1 and t["out_tok"][0, 0] == 0 and t["y_kind"][0] == 2


# ---------------------------------------------------------------- H-RAD MLP (f4, Eq. 4-5, P745)
def _bf16_bits(x):
    import torch

    return torch.tensor(np.asarray(x, np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def _bf16_vals(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def test_hrad_matches_library_matmul(orc):
    """Plain-loop oracle vs numpy's float64 matmul on the same widened bytes (a library
    routine, an independent implementation of the three affine layers)."""
    from paper_2506_01979_b200 import synth

    n = synth.hrad_to_numpy(synth.hrad_inputs(37, 320, G=6, seed=3))
    o = orc.hrad(n["z"], n["w1"], n["b1"], n["w2"], n["b2"], n["w3"], n["b3"], n["stop"], n["G"])
    z, w1 = _bf16_vals(n["z"]), _bf16_vals(n["w1"])
    h1 = np.maximum(z @ w1.T + n["b1"].astype(np.float64), 0.0)
    h2 = np.maximum(h1 @ n["w2"].astype(np.float64).T + n["b2"], 0.0)
    lg = h2 @ n["w3"].astype(np.float64).T + n["b3"]
    assert np.allclose(o["h1"], h1, rtol=1e-12, atol=1e-12)
    assert np.allclose(o["logits"], lg, rtol=1e-12, atol=1e-12)
    assert np.array_equal(o["s_t"], np.argmax(lg, axis=1))


def test_hrad_closed_form_identity_network(orc):
    """W1 = I, W2 = [I 0], W3 = [I 0] -> logits = relu(relu(z[:3]) ) + b3, so the class is
    the argmax of the first three (bf16-exact) features; ReLU clips negatives."""
    Dz = 256
    rng = np.random.default_rng(5)
    zv = rng.choice([-2.0, -0.5, 0.25, 0.75, 1.5, 3.0], size=(9, Dz))
    z = _bf16_bits(zv)
    w1 = _bf16_bits(np.eye(256, Dz))
    w2 = np.eye(64, 256, dtype=np.float32)
    w3 = np.eye(3, 64, dtype=np.float32)
    zero = lambda n: np.zeros(n, np.float32)  # noqa: E731
    o = orc.hrad(z, w1, zero(256), w2, zero(64), w3, zero(3))
    expect = np.maximum(zv[:, :3], 0.0)
    assert np.array_equal(o["logits"], expect)
    first_max = np.array([int(np.flatnonzero(r == r.max())[0]) for r in expect])
    assert np.array_equal(o["s_t"], first_max)  # ties -> smaller class (incl. all-zero rows)


def test_hrad_ties_and_branch_layout(orc):
    """Ties go to the smaller class; H_t maps s_t = 0/1/2 to (gamma, s) = (0,0) /
    (stop, stop) / (G, G) (P194-201, P669; DESIGN reading 35)."""
    Dz, G = 64, 8
    z = _bf16_bits(np.zeros((6, Dz)))
    w1 = _bf16_bits(np.zeros((256, Dz)))
    zero = lambda n: np.zeros(n, np.float32)  # noqa: E731
    w2, w3 = np.zeros((64, 256), np.float32), np.zeros((3, 64), np.float32)
    stop = np.array([0, 3, 8, 11, -2, 5], np.int32)
    for b3, cls in (([1, 1, 0], 0), ([0, 2, 2], 1), ([0, 1, 2], 2), ([5, 5, 5], 0)):
        o = orc.hrad(z, w1, zero(256), w2, zero(64), w3, np.array(b3, np.float32), stop, G)
        assert (o["s_t"] == cls).all()
        exp = {0: np.zeros(6), 1: np.clip(stop, 0, G), 2: np.full(6, G)}[cls]
        assert np.array_equal(o["gamma"], exp) and np.array_equal(o["branch_pos"], exp)
