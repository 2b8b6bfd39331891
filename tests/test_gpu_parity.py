"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by
element on the same seeded bytes.  Small cases span several tiles plus ragged tails;
the BASELINE configurations run at full size in bench.py's launch configuration and
are checked on sampled sequences (SURVEY §8.4 "Parity coverage")."""
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


def _check_chunk(inp, g, idx, adaptive, rule, nthreads):
    """Oracle on sequences idx of the GPU run g (same bytes), compared element by element."""
    import oracle
    from paper_2506_01979_b200 import synth

    from parity_util import compare, oracle_for

    it = torch.as_tensor(idx, device=inp["PL"].device)
    sub = synth.to_numpy_inputs({k: (v.index_select(0, it) if torch.is_tensor(v) else v) for k, v in inp.items()})
    if adaptive:
        c = oracle.confidence(np.ascontiguousarray(sub["QL"][:, :1]), mode=oracle.CONF_TOP1, eps=0.2,
                              k_max=6, V=sub["V"], nthreads=nthreads)
        tie = (c["ties"][:, 0] & oracle.TIE_CONF) != 0
        assert np.array_equal(c["stop"][:, 0][~tie], g["c_stop"][idx, 0][~tie])
        assert np.array_equal(c["k_next"][:, 0][~tie], g["c_knext"][idx, 0][~tie]) or (c["ties"][:, 0] & oracle.TIE_EQ7).any()
        G = sub["PL"].shape[2] - 1
        for key, gk in (("top1_prob", "c_top1"), ("entropy", "c_ent"), ("stat", "c_stat")):
            ref = c[key][:, 0, :G]
            got = g[gk][idx, 0, :G].astype(np.float64)
            assert np.allclose(got, ref, rtol=1e-5, atol=1e-7, equal_nan=True), key
        assert np.array_equal(c["top1_id"][:, 0, :G], g["c_id"][idx, 0, :G])
        gamma = c["gamma_next"][:, 0]
        keep = gamma == g["gamma_used"][idx]
    else:
        gamma = sub["gamma"]
        keep = np.ones(len(idx), bool)
    o = oracle_for(sub, gamma, rule=rule, nthreads=nthreads)
    o["_gamma"] = np.asarray(gamma)
    keep_idx = np.where(keep)[0]
    osub = {k: (v[keep_idx] if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == len(idx) else v)
            for k, v in o.items()}
    isub = {k: (v[keep_idx] if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == len(idx) else v)
            for k, v in sub.items()}
    return compare(g, osub, sel=idx[keep_idx], inp_np=isub)


def _merge(reps):
    out = {"n": 0, "ties": {"acc_mask": 0, "decision": 0, "sample": 0}, "exact_seq": 0, "y_compared": 0,
           "tie_samples_checked": 0, "tie_samples_differ": 0, "tie_decisions_checked": 0,
           "tie_margin_hist": [0, 0, 0, 0]}
    for r in reps:
        for k in ("n", "exact_seq", "y_compared", "tie_samples_checked", "tie_samples_differ",
                  "tie_decisions_checked"):
            out[k] += r.get(k, 0)
        for k in out["ties"]:
            out["ties"][k] += r["ties"][k]
        out["tie_margin_hist"] = [a + b for a, b in zip(out["tie_margin_hist"], r.get("tie_margin_hist", [0] * 4))]
        for k, v in r.items():
            if k.startswith("max_"):
                out[k] = max(out.get(k, 0.0), v)
    return out


def _run(cfg, row_pad=0, rule=0, seed=None, adaptive=False, sample=None, nthreads=0, fused=True, chunk=None):
    from paper_2506_01979_b200 import synth

    from parity_util import gpu_run, internal_consistency

    inp = synth.generate(cfg, device="cuda", seed=seed, row_pad=row_pad)
    g, d, _ = gpu_run(inp, rule=rule, adaptive=adaptive, fused=fused)
    internal_consistency(g, cfg.G)
    B = inp["PL"].shape[0]
    idx = np.arange(B) if sample is None else np.unique(np.r_[0, B - 1, np.random.default_rng(1).choice(B, sample - 2, replace=False)])
    step = len(idx) if chunk is None else chunk
    reps = [_check_chunk(inp, g, idx[j:j + step], adaptive, rule, nthreads) for j in range(0, len(idx), step)]
    return _merge(reps), g


def cfg(name, **kw):
    from paper_2506_01979_b200 import synth

    return synth.config(name, **kw)


SMALL = [
    ("bf16_V32000_mixed", dict(name="c2", B=48, layout="mixed"), 0, 0),
    ("bf16_ragged_V5003", dict(name="c2", V=5003, B=40, K=3, G=7, layout="mixed"), 0, 0),
    ("bf16_strided_V5000", dict(name="c2", V=5000, B=32, layout="mixed"), 24, 0),
    ("f32_mixed_V32000", dict(name="c1", B=48, rounds=1, layout="mixed"), 0, 0),
    ("f32_ragged_alg1", dict(name="c1", V=3001, B=40, K=4, G=6, rounds=1, layout="mixed"), 0, 1),
    ("bf16_alg1_K8", dict(name="c5", V=9000, B=24, K=8, G=16, layout="mixed"), 0, 1),
    ("tiny_V8", dict(name="c2", V=8, B=64, K=2, G=4, layout="mixed", delta=2.0, rho_same=0.5), 0, 0),
    ("tiny_V2_f32", dict(name="c1", V=2, B=64, K=1, G=3, rounds=1, layout="mixed", delta=2.0), 0, 0),
    ("K1_vanilla_sd", dict(name="c4", V=20000, B=64, K=1, G=5, layout="mixed"), 0, 0),
    ("bf16_large_V_few_seq", dict(name="c3", B=6, layout="mixed"), 0, 0),
    ("gamma_max_31", dict(name="c2", V=4096, B=16, K=2, G=31, layout="mixed"), 0, 0),
    ("B1_single_round_f32", dict(name="c1", B=1, rounds=1, layout="fixed"), 0, 0),
]


@pytest.mark.parametrize("fused", ["single_launch", "astep", "verify_select", "two_calls"])
@pytest.mark.parametrize("name,kw,pad,rule", SMALL, ids=[c[0] for c in SMALL])
def test_small_parity(name, kw, pad, rule, fused, monkeypatch):
    """single_launch: the persistent TMA-ring k_step_tma (SB_FUSED_STEP=1); astep: the
    persistent work-queue kernel k_astep with plan items (opt-in for sb_verify_select,
    SB_ASTEP=1); verify_select: the two streaming kernels behind sb_verify_select (the
    default); two_calls: sb_verify_branches then sb_select_branch."""
    kw = dict(kw)
    c = cfg(kw.pop("name"), **kw)
    monkeypatch.setenv("SB_ASTEP", "1" if fused == "astep" else "0")
    if fused == "single_launch":
        monkeypatch.setenv("SB_FUSED_STEP", "1")  # the persistent k_step_tma kernel
    rep, g = _run(c, row_pad=pad, rule=rule, fused=(fused != "two_calls"))
    assert rep["exact_seq"] >= 0.9 * rep["n"], rep
    kinds = set(np.unique(g["y_kind"]).tolist())
    if c.B >= 32 and c.G >= 4:
        assert {1, 2} <= kinds or 0 in kinds, kinds


@pytest.mark.parametrize("name,kw,pad,rule", SMALL, ids=[c[0] for c in SMALL])
def test_rows_warp_kernel_parity(name, kw, pad, rule, monkeypatch):
    """k_rows_warp (one warp per row pair, per-warp cp.async ring) on every small shape
    (SB_ROWS_VARIANT=9 forces it; unaligned rows keep the register-staged kernel)."""
    monkeypatch.setenv("SB_ROWS_VARIANT", "9")
    kw = dict(kw)
    rep, _ = _run(cfg(kw.pop("name"), **kw), row_pad=pad, rule=rule, fused=False)
    assert rep["exact_seq"] >= 0.9 * rep["n"], rep


def test_rows_warp_kernel_default_route():
    """Many short rows take k_rows_warp by default (>= 16384 row slots of <= 64 KB): 512
    sequences x K = 4 x 9 rows of 16 KB, checked on a sample of 96 sequences."""
    rep, _ = _run(cfg("c2", V=8192, B=512, K=4, G=8, layout="mixed"), sample=96, fused=False)
    assert rep["exact_seq"] >= 0.9 * rep["n"], rep


@pytest.mark.parametrize("name,kw", [("bf16", dict(name="c2", B=40, layout="mixed")),
                                     ("f32", dict(name="c1", B=40, rounds=1, layout="mixed"))])
def test_register_staged_fallback_parity(monkeypatch, name, kw):
    """The non-TMA kernels (used for unaligned rows) on aligned inputs too."""
    monkeypatch.setenv("SB_DISABLE_TMA", "1")
    kw = dict(kw)
    rep, _ = _run(cfg(kw.pop("name"), **kw), adaptive=(name == "bf16"))
    assert rep["exact_seq"] >= 0.9 * rep["n"], rep


ADAPTIVE = [
    ("c2_B64", dict(name="c2", B=64), 0, 60),
    ("bf16_ragged_mixed", dict(name="c2", V=5000, B=40, K=3, G=12, layout="mixed"), 0, 36),
    ("bf16_K8_G16_alg1", dict(name="c5", V=9000, B=24, K=8, G=16, layout="mixed"), 1, 20),
    ("f32_mixed", dict(name="c1", V=4000, B=40, K=3, G=8, rounds=1, layout="mixed"), 0, 36),
    ("f32_unaligned_V3001", dict(name="c1", V=3001, B=24, K=2, G=6, rounds=1, layout="mixed"), 0, 20),
    ("bf16_B300_more_than_sms", dict(name="c2", V=2048, B=300, K=4, G=8), 0, 280),
    ("tiny_V8", dict(name="c2", V=8, B=64, K=2, G=4, layout="mixed", delta=2.0, rho_same=0.5), 0, 50),
    ("gamma_max_31", dict(name="c2", V=4096, B=16, K=2, G=31, layout="mixed"), 0, 14),
]


@pytest.mark.parametrize("path", ["astep", "three_calls"])
@pytest.mark.parametrize("name,kw,rule,nmin", ADAPTIVE, ids=[a[0] for a in ADAPTIVE])
def test_adaptive_confidence_parity(name, kw, rule, nmin, path, monkeypatch):
    """The adaptive-gamma step through sb_step_adaptive: the single persistent launch
    k_astep (default; confidence -> verify -> select items in one grid) and the three
    streaming kernels (SB_ASTEP=0: confidence -> verify reusing its rows -> select), on shapes with several items per CTA, more sequences than SMs,
    ragged / unaligned rows (the latter always take the three kernels), K = 8,
    gamma_max = 31 and Alg. 1."""
    monkeypatch.setenv("SB_ASTEP", "0" if path == "three_calls" else "1")
    kw = dict(kw)
    rep, g = _run(cfg(kw.pop("name"), **kw), adaptive=True, rule=rule)
    assert rep["n"] >= nmin, rep
    assert rep["exact_seq"] >= 0.85 * rep["n"], rep


def test_deterministic_run_to_run():
    from paper_2506_01979_b200 import synth

    from parity_util import gpu_run

    inp = synth.generate(cfg("c2", B=32, layout="mixed"), device="cuda", seed=5)
    a, _, _ = gpu_run(inp, adaptive=False)
    b, _, _ = gpu_run(inp, adaptive=False)
    n = a["offsets"][-1]
    a["packed_tok"], b["packed_tok"] = a["packed_tok"][:n], b["packed_tok"][:n]  # tail unwritten
    for k in a:
        if k.startswith("c_"):
            continue  # draft-confidence buffers are not written without adaptive gamma
        assert np.array_equal(a[k], b[k], equal_nan=True), k


@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_sequence_shards_bit_identical(nranks):
    """sequence-sharded output at every G is bit-identical to G = 1.  Each
    rank's contiguous slice [g B / G, (g+1) B / G) (bench.py rank_slice) generated on its
    own (the counter-keyed generator gives the same bytes) and run alone must reproduce the
    full batch's per-sequence outputs exactly."""
    from paper_2506_01979_b200 import synth

    from parity_util import gpu_run

    c = cfg("c2", V=8000, B=48, layout="mixed")
    full, _, _ = gpu_run(synth.generate(c, device="cuda"))
    per = ("lse_p", "lse_q", "p_tok", "q_tok", "acc_mask", "n_acc", "top1_q", "top1_id_q", "entropy_q", "status",
           "sel_k", "commit_len", "out_tok", "y_tok", "y_kind", "path_rolled", "branch_discarded", "keep_mask",
           "resid_mass")
    for g in range(nranks):
        b0, b1 = g * c.B // nranks, (g + 1) * c.B // nranks
        part, _, _ = gpu_run(synth.generate(c, device="cuda", b0=b0, b1=b1))
        for k in per:
            assert np.array_equal(part[k], full[k][b0:b1], equal_nan=True), (nranks, g, k)


def test_workspace_reuse_across_calls():
    """One workspace, three rounds of different inputs: the self-resetting counters
    leave it re-usable (include/specbranch.h workspace contract)."""
    import torch

    from paper_2506_01979_b200 import api, synth

    from parity_util import compare, oracle_for

    c = cfg("c2", V=8000, B=40, layout="mixed")
    inp0 = synth.generate(c, device="cuda", seed=21)
    d = api.dims_for(inp0["PL"], V=inp0["V"])
    buf = api.StepBuffers.alloc(d, "cuda")
    for seed in (21, 22, 23):
        inp = synth.generate(c, device="cuda", seed=seed)
        api.verify_step(d, inp, buf)
        torch.cuda.synchronize()
        g = {k: getattr(buf, k).cpu().numpy() for k in buf.__dataclass_fields__ if not k.endswith("workspace")}
        g["acc_mask"] = g["acc_mask"].view(np.uint32)
        g["keep_mask"] = g["keep_mask"].view(np.uint32)
        inp_np = synth.to_numpy_inputs(inp)
        compare(g, oracle_for(inp_np, inp_np["gamma"]))


def test_identical_p_q_accepts_all_on_gpu():
    from paper_2506_01979_b200 import synth

    from parity_util import gpu_run

    inp = synth.generate(cfg("c2", V=6000, B=40, layout="mixed"), device="cuda", seed=3)
    inp["QL"] = inp["PL"].clone()
    g, _, _ = gpu_run(inp)
    gam, s = inp["gamma"].cpu().numpy(), inp["branch_pos"].cpu().numpy()
    L = np.where(s < gam, gam, gam + 1)
    assert (g["n_acc"] == L[:, None]).all()
    assert (g["path_rolled"] == 0).all()


@pytest.mark.parametrize("path", ["astep", "three_calls"])
def test_adaptive_special_values(path, monkeypatch):
    """The adaptive step (k_astep and the three kernels) on rows that break the usual
    assumptions: NaN / +inf / all -inf / one-hot / finfo(bf16).min-masked draft rows in
    slot 0 (the confidence pass and its reused q states), NaN target rows, out-of-range
    tokens, a clamped branch row; statistics, stop / k / gamma and every verify / select
    output against the oracle (_check_chunk's adaptive path)."""
    from paper_2506_01979_b200 import synth

    monkeypatch.setenv("SB_ASTEP", "1" if path == "astep" else "0")
    c = cfg("c2", V=4096, B=24, K=3, G=6, layout="adaptive")
    inp = synth.generate(c, device="cuda", seed=13)
    bmin = torch.finfo(torch.bfloat16).min
    inp["QL"][0, 0, 0, 100] = float("nan")      # confidence row 0 of b=0 poisoned
    inp["QL"][1, 0, 2, 7] = float("inf")
    inp["QL"][2, 0, 1, :] = float("-inf")        # an all -inf draft row
    inp["QL"][3, 0, 0, :] = float("-inf")
    inp["QL"][3, 0, 0, 11] = 5.0                 # one-hot: top-1 = 1, H = 0 exactly
    inp["QL"][4, 0, 3, 1::2] = bmin              # half the row masked with finfo.min
    inp["PL"][5, 0, 0, 3] = float("nan")         # target row NaN at the first row
    inp["PL"][6, 1, 2, :] = float("-inf")
    inp["tok"][7, 0, 0] = 99999                  # out-of-range token
    inp["branch_pos"][8] = 40                    # clamped branch row
    rep, g = _run_inp(inp, c, adaptive=True)
    assert rep["n"] >= 16, rep


def _run_inp(inp, c, adaptive=False, rule=0):
    """_run on given inputs (all sequences, one chunk)."""
    from parity_util import gpu_run, internal_consistency

    g, d, _ = gpu_run(inp, rule=rule, adaptive=adaptive)
    internal_consistency(g, c.G)
    idx = np.arange(inp["PL"].shape[0])
    return _check_chunk(inp, g, idx, adaptive, rule, 0), g


def test_special_values_and_status():
    """NaN / +inf / all -inf rows, out-of-range tokens and clamped layouts are reported
    per sequence in status and match the oracle's handling."""
    from paper_2506_01979_b200 import synth

    from parity_util import compare, gpu_run, oracle_for

    c = cfg("c2", V=3000, B=16, K=2, G=4, layout="fixed")
    inp = synth.generate(c, device="cuda", seed=9)
    inp["PL"][0, 0, 1, 17] = float("nan")
    inp["QL"][1, 0, 0, 5] = float("inf")
    inp["PL"][2, 1, 2, :] = float("-inf")
    inp["QL"][3, 0, 0, :] = float("-inf")
    inp["QL"][3, 0, 0, 7] = 1.0  # one-hot draft row
    inp["tok"][3, :, 0] = 7
    inp["tok"][4, 0, 2] = 999999
    inp["tok"][5, 1, 3] = -4
    inp["gamma"][6] = 40
    inp["branch_pos"][7] = 3
    inp["gamma"][7] = 2
    inp["QL"][8, 0, 2, :100] = float("-inf")  # masked draft logits
    inp["QL"][9, 0, 1, :] = -(2.0 ** 98)  # finite, max outside the input domain (reading 34)
    inp["PL"][10, 0, 0, ::2] = float("-inf")  # half-masked target and draft rows
    inp["QL"][10, 0, 0, 1::3] = float("-inf")
    inp["QL"][11, 0, 1, 3:] = -(2.0 ** 97)  # masked tail at exactly -2^97 (in domain)
    bmin = torch.finfo(torch.bfloat16).min
    inp["QL"][12, 1, 2, :] = float("-inf")  # an all -inf draft row (bf16 clamp tie-break)
    inp["QL"][13, 1, 2, :] = bmin  # a draft row fully masked with finfo(bf16).min: RANGE
    inp["PL"][14, 0, 3, 5::2] = bmin  # finfo.min masks under an in-range maximum: exact
    inp["QL"][14, 0, 3, 7::3] = bmin
    inp["PL"][15, 0, 2, :] = 3.0e7  # a target row whose maximum is >= 2^24: RANGE
    g, _, _ = gpu_run(inp)
    inp_np = synth.to_numpy_inputs(inp)
    o = oracle_for(inp_np, inp_np["gamma"])
    compare(g, o)
    st = g["status"]
    assert st[0] & 8 and st[4] & 4 and st[6] & 1 and st[7] & 2
    assert st[9] & 64 and not st[10] & 72 and not st[11] & 72
    assert st[12] == 8 and st[13] == 64 and st[14] == 0 and st[15] == 64


@pytest.mark.slow
@pytest.mark.parametrize("name,adaptive,chunk", [("c1", False, 256), ("c2", True, 64), ("c3", True, 64),
                                                 ("c4", False, 256), ("c5", False, 64)])
def test_baseline_config_full_size(name, adaptive, chunk):
    """Full BASELINE sizes in bench.py's launch configuration; the oracle checks EVERY
    sequence (in chunks that bound host memory), SURVEY §8.4 "Parity coverage".  Near-tie
    samples are not skipped: the GPU's token must be a valid draw at the breakpoint."""
    c = cfg(name)
    rep, g = _run(c, adaptive=adaptive, nthreads=0, chunk=chunk)
    assert rep["n"] == c.B * c.rounds or adaptive, rep
    assert rep["ties"]["decision"] <= 0.1 * rep["n"], rep
    print(name, rep)


@pytest.mark.parametrize("name,kw", [("bf16_mixed_V32000", dict(name="c2", B=48, layout="mixed")),
                                     ("f32_mixed_ragged", dict(name="c1", V=3001, B=40, K=3, G=6, rounds=1,
                                                                layout="mixed")),
                                     ("bf16_K8_G16", dict(name="c5", V=9000, B=24, K=8, G=16, layout="mixed"))])
def test_verify_reuse_of_confidence_states(name, kw):
    """sb_verify_branches_reuse: slot-0 draft rows i < G are not re-read; their q state
    comes from the preceding sb_draft_confidence.  Same bars against the oracle on mixed
    layouts (branch rows s_b > 0, Algorithm-1 form, gamma = 0), with the step's select."""
    import oracle
    from paper_2506_01979_b200 import api, synth

    from parity_util import compare, oracle_for

    c = cfg(kw.pop("name"), **kw)
    inp = synth.generate(c, device="cuda", seed=31)
    d = api.dims_for(inp["PL"], V=inp["V"])
    buf = api.StepBuffers.alloc(d, inp["PL"].device)
    api.sb_draft_confidence(api.conf_dims(d), inp["QL"], None, api.SB_CONF_TOP1, 0.2, 1.0, 6, buf.c_top1, buf.c_id,
                            buf.c_ent, None, buf.c_stat, buf.c_stop, buf.c_knext, buf.c_gamma, buf.conf_workspace)
    api.sb_verify_branches_reuse(d, inp["PL"], inp["QL"], inp["tok"], inp["u"], inp["gamma"], inp["branch_pos"],
                                 buf.lse_p, buf.lse_q, buf.p_tok, buf.q_tok, buf.acc_mask, buf.n_acc, buf.top1_q,
                                 buf.top1_id_q, buf.entropy_q, buf.status, buf.conf_workspace, buf.workspace)
    api.sb_select_branch(d, inp["PL"], inp["QL"], inp["tok"], inp["u"], inp["us"], inp["gamma"], inp["branch_pos"],
                         buf.n_acc, 0, buf.sel_k, buf.commit_len, buf.out_tok, buf.y_tok, buf.y_kind, buf.offsets,
                         buf.packed_tok, buf.path_rolled, buf.branch_discarded, buf.keep_mask, buf.resid_mass,
                         buf.status, buf.workspace)
    torch.cuda.synchronize()
    g = {k: getattr(buf, k).cpu().numpy() for k in buf.__dataclass_fields__ if k not in ("workspace", "conf_workspace")}
    g["acc_mask"] = g["acc_mask"].view(np.uint32)
    g["keep_mask"] = g["keep_mask"].view(np.uint32)
    inp_np = synth.to_numpy_inputs(inp)
    o = oracle_for(inp_np, inp_np["gamma"])
    rep = compare(g, o)
    assert rep["exact_seq"] >= 0.9 * rep["n"], rep
