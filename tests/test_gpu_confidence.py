"""GPU parity of sb_draft_confidence against the fp64 oracle, in
all three statistic modes: TOP1 max_x q(x) (§4.2 P170, App. E.6 P954), TOKEN q(x_i) of
the drafted token (Eq. 6 P198, Alg. 1 'Mask' P517) and ENTROPY 1 - sqrt(lambda H)
(§4.2 P170; SPEC S313-321), with the tok_prob output, K > 1 (b,k) groups, several eps,
lambda and k_max values, bf16 / fp32, ragged V and the register-staged fallback.

Bars: per-row continuous outputs within 1e-5 |ref| + 1e-7; top1_id, stop,
k_next and gamma_next bit-exact except groups the oracle flags as near ties
(|stat - eps| < 1e-6 before the stop, or k_max (1 - c) within 1e-6 of an integer)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REL, ABS = 1e-5, 1e-7


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2506_01979_b200.build import build

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    build()


def _band(g, r):
    g = np.asarray(g, np.float64)
    r = np.asarray(r, np.float64)
    assert np.array_equal(np.isnan(g), np.isnan(r)), "NaN pattern differs"
    m = ~np.isnan(r)
    return float(np.max(np.abs(g[m] - r[m]) / (REL * np.abs(r[m]) + ABS))) if m.any() else 0.0


def run_conf(QL, tok, mode, eps, lam, k_max, V):
    from paper_2506_01979_b200 import api

    d = api.dims_for(QL, V=V)
    B, K, G = d.B, d.K, d.G
    dev = QL.device
    e = lambda *s, dt=torch.float32: torch.full(s, -7, dtype=dt, device=dev)  # noqa: E731
    out = dict(top1_prob=e(B, K, G), top1_id=e(B, K, G, dt=torch.int32), entropy=e(B, K, G),
               tok_prob=e(B, K, G), stat=e(B, K, G), stop=e(B, K, dt=torch.int32),
               k_next=e(B, K, dt=torch.int32), gamma_next=e(B, K, dt=torch.int32))
    ws = api.make_workspace(d, dev)
    api.sb_draft_confidence(d, QL, tok, mode, eps, lam, k_max, out["top1_prob"], out["top1_id"], out["entropy"],
                            out["tok_prob"] if tok is not None else None, out["stat"], out["stop"], out["k_next"],
                            out["gamma_next"], ws)
    torch.cuda.synchronize()
    o = {k: v.cpu().numpy() for k, v in out.items()}
    if tok is None:
        o["tok_prob"] = None
    return o


def check(g, o, mode, with_tok):
    import oracle

    rep = {}
    for k in ("top1_prob", "entropy", "stat") + (("tok_prob",) if with_tok else ()):
        rep[k] = _band(g[k], o[k])
        assert rep[k] <= 1.0, (k, rep[k])
    assert np.array_equal(g["top1_id"], o["top1_id"])
    tie_c = (o["ties"] & oracle.TIE_CONF) != 0
    tie_7 = (o["ties"] & oracle.TIE_EQ7) != 0
    ok = ~tie_c
    assert np.array_equal(g["stop"][ok], o["stop"][ok]), "stop"
    assert np.array_equal(g["gamma_next"][ok], o["gamma_next"][ok]), "gamma_next"
    ok7 = ~tie_c & ~tie_7
    assert np.array_equal(g["k_next"][ok7], o["k_next"][ok7]), "k_next"
    # near ties are checked for validity, not skipped: a stop may only move to a row whose
    # statistic is within 1e-6 of eps (all earlier rows above eps - 1e-6), and Eq. 7's
    # floor may only move by one when k_max (1 - c) is within 1e-6 of an integer
    G = o["stat"].shape[-1]
    for b, k in zip(*np.nonzero(tie_c | tie_7)):
        st = o["stat"][b, k]
        gs = int(g["stop"][b, k])
        valid = {i for i in range(G) if st[i] <= eps_of(o) + 1e-6 and np.all(~(st[:i] <= eps_of(o) - 1e-6))}
        if np.all(~(st <= eps_of(o) - 1e-6)):
            valid.add(G)
        assert gs in valid, (b, k, gs, valid)
        if gs == int(o["stop"][b, k]):
            kn, ko = int(g["k_next"][b, k]), int(o["k_next"][b, k])
            assert kn == ko or (tie_7[b, k] and abs(kn - ko) == 1 and kn >= 1), (b, k, kn, ko)
    rep["ties"] = int((tie_c | tie_7).sum())
    rep["groups"] = int(o["stop"].size)
    rep["stops"] = np.bincount(o["stop"].ravel()).tolist()
    return rep


def eps_of(o):
    return o["_eps"]


CASES = [
    # name, synth config overrides, mode, eps, lambda, k_max
    ("top1_bf16_K1", dict(name="c2", B=48, K=1), "TOP1", 0.2, 1.0, 6),
    ("top1_bf16_K4_eps05", dict(name="c2", B=24, K=4), "TOP1", 0.5, 1.0, 16),
    ("token_bf16_K3", dict(name="c2", V=9000, B=32, K=3, G=12), "TOKEN", 0.2, 1.0, 6),
    ("token_bf16_eps005_kmax1", dict(name="c3", B=8, K=2, G=16), "TOKEN", 0.05, 1.0, 1),
    ("token_f32_ragged", dict(name="c1", V=3001, B=40, K=2, G=6, rounds=1), "TOKEN", 0.3, 1.0, 8),
    ("entropy_bf16_K2", dict(name="c2", B=40, K=2), "ENTROPY", 0.2, 1.0, 6),
    ("entropy_bf16_lam03", dict(name="c4", B=8, K=3, G=8), "ENTROPY", 0.1, 0.3, 6),
    ("entropy_f32", dict(name="c1", B=32, K=2, rounds=1), "ENTROPY", 0.4, 1.0, 6),
    ("entropy_bf16_ragged_V5003", dict(name="c2", V=5003, B=32, K=3, G=7), "ENTROPY", 0.2, 2.0, 6),
    ("top1_tiny_V8", dict(name="c2", V=8, B=64, K=2, G=4, delta=2.0, rho_same=0.5), "TOP1", 0.3, 1.0, 6),
]


@pytest.mark.parametrize("tma", ["tma", "fallback"])
@pytest.mark.parametrize("name,kw,mode,eps,lam,k_max", CASES, ids=[c[0] for c in CASES])
def test_confidence_modes(name, kw, mode, eps, lam, k_max, tma, monkeypatch):
    import oracle
    from paper_2506_01979_b200 import api, synth

    if tma == "fallback":
        monkeypatch.setenv("SB_DISABLE_TMA", "1")
    kw = dict(kw)
    c = synth.config(kw.pop("name"), layout="fixed", **kw)
    inp = synth.generate(c, device="cuda", seed=77)
    m = {"TOP1": api.SB_CONF_TOP1, "TOKEN": api.SB_CONF_TOKEN, "ENTROPY": api.SB_CONF_ENTROPY}[mode]
    # TOKEN needs the drafted tokens; pass them in the other modes too so tok_prob is checked
    g = run_conf(inp["QL"], inp["tok"], m, eps, lam, k_max, inp["V"])
    n = synth.to_numpy_inputs(inp)
    o = oracle.confidence(n["QL"], n["tok"], mode=m, eps=eps, lam=lam, k_max=k_max, V=n["V"])
    o["_eps"] = eps
    rep = check(g, o, mode, with_tok=True)
    print(name, tma, rep)


def test_confidence_without_tokens_leaves_tok_prob_out():
    """TOP1 / ENTROPY without tok: tok_prob may be NULL, stat and stop as with tokens."""
    import oracle
    from paper_2506_01979_b200 import api, synth

    c = synth.config("c2", B=16, K=2, layout="fixed")
    inp = synth.generate(c, device="cuda", seed=78)
    g = run_conf(inp["QL"], None, api.SB_CONF_ENTROPY, 0.2, 1.0, 6, inp["V"])
    n = synth.to_numpy_inputs(inp)
    o = oracle.confidence(n["QL"], None, mode=api.SB_CONF_ENTROPY, eps=0.2, k_max=6, V=n["V"])
    o["_eps"] = 0.2
    check(g, o, "ENTROPY", with_tok=False)


def test_confidence_special_rows():
    """Non-finite / out-of-domain / one-hot / uniform rows: NaN statistics (no stop on
    them), exact closed forms on the others (H of a uniform row = ln V, one-hot: 0)."""
    import oracle
    from paper_2506_01979_b200 import api, synth

    c = synth.config("c2", V=4000, B=8, K=2, G=5, layout="fixed")
    inp = synth.generate(c, device="cuda", seed=79)
    QL = inp["QL"]
    QL[0, 0, 1] = 0.5  # uniform row
    QL[1, 1, 0] = float("-inf")
    QL[1, 1, 0, 17] = 3.0  # one-hot
    QL[2, 0, 2, 5] = float("nan")
    QL[3, 1, 3] = float("-inf")  # no distribution
    QL[4, 0, 0] = torch.finfo(torch.bfloat16).min  # outside the input domain
    QL[5, 0, 4, ::3] = torch.finfo(torch.bfloat16).min  # masks under an in-range maximum
    for mode in (api.SB_CONF_TOP1, api.SB_CONF_TOKEN, api.SB_CONF_ENTROPY):
        g = run_conf(QL, inp["tok"], mode, 0.2, 1.0, 6, inp["V"])
        n = synth.to_numpy_inputs(inp)
        o = oracle.confidence(n["QL"], n["tok"], mode=mode, eps=0.2, k_max=6, V=n["V"])
        o["_eps"] = 0.2
        check(g, o, mode, with_tok=True)
        assert abs(g["entropy"][0, 0, 1] - np.log(4000)) < 1e-5 * np.log(4000)
        assert abs(g["entropy"][1, 1, 0]) <= 1e-7 and abs(g["top1_prob"][1, 1, 0] - 1.0) <= 2e-7
        assert g["top1_id"][1, 1, 0] == 17
        assert np.isnan(g["stat"][2, 0, 2]) and np.isnan(g["stat"][3, 1, 3]) and np.isnan(g["stat"][4, 0, 0])
