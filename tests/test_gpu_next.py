"""§8(f) NEXT rows on the GPU against the oracle: f1 branch spawn (Eq. 7), f2 KV rollback."""
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


SPAWN = [("bf16_V128256", dict(name="c3", B=40, layout="mixed"), 6, 0),
         ("bf16_V32000_k16", dict(name="c2", B=64, layout="mixed"), 16, 0),
         ("f32_V3001_ragged", dict(name="c1", V=3001, B=48, rounds=1, layout="mixed"), 8, 0),
         ("bf16_token_mode", dict(name="c2", V=5000, B=48, layout="mixed"), 6, 1),
         ("tiny_V5", dict(name="c2", V=5, B=64, K=2, G=3, layout="mixed"), 8, 0),
         # B > 5 x SMs: the 64-thread-CTA geometry
         ("bf16_V5000_B1000", dict(name="c2", V=5000, B=1000, layout="mixed"), 16, 0),
         ("f32_V3001_B800_ragged", dict(name="c1", V=3001, B=800, rounds=1, layout="mixed"), 8, 0)]


@pytest.mark.parametrize("name,kw,k_max,mode", SPAWN, ids=[c[0] for c in SPAWN])
def test_spawn_matches_oracle(name, kw, k_max, mode):
    import oracle
    from paper_2506_01979_b200 import api, synth

    kw = dict(kw)
    c = synth.config(kw.pop("name"), **kw)
    inp = synth.generate(c, device="cuda", seed=17)
    d = api.dims_for(inp["QL"], V=inp["V"])
    B = d.B
    k = torch.empty(B, dtype=torch.int32, device="cuda")
    bt = torch.empty((B, k_max), dtype=torch.int32, device="cuda")
    bp = torch.empty((B, k_max), dtype=torch.float32, device="cuda")
    cf = torch.empty(B, dtype=torch.float32, device="cuda")
    api.sb_spawn_branches(d, inp["QL"], inp["branch_pos"], inp["tok"], mode, k_max, k, bt, bp, cf)
    torch.cuda.synchronize()
    inp_np = synth.to_numpy_inputs(inp)
    o = oracle.spawn(inp_np["QL"], inp_np["branch_pos"], inp_np["tok"], mode=mode, k_max=k_max, V=inp_np["V"])
    tie = (o["ties"] & oracle.TIE_EQ7) != 0
    kg, btg = k.cpu().numpy(), bt.cpu().numpy()
    assert np.array_equal(kg[~tie], o["k"][~tie])
    for b in np.where(~tie)[0]:
        n = o["k"][b]
        assert np.array_equal(btg[b], o["btok"][b]), b
        assert np.allclose(bp.cpu().numpy()[b, :n], o["bprob"][b, :n], rtol=1e-5, atol=1e-7)
    assert np.allclose(cf.cpu().numpy(), o["conf"], rtol=1e-5, atol=1e-7, equal_nan=True)


@pytest.mark.parametrize("inplace", [False, True])
def test_kv_rollback_matches_oracle(inplace):
    """The kept rows are exactly the committed draft positions of the oracle's decision
    (the decisions fed to both sides come from the oracle, never from the GPU path)."""
    import oracle
    from paper_2506_01979_b200 import api, synth

    c = synth.config("c2", V=2048, B=48, K=4, G=8, layout="mixed")
    inp = synth.generate(c, device="cpu", seed=23)
    inp["gamma"][:3] = torch.tensor([11, 5, 4], dtype=torch.int32)  # clamped layouts
    inp["branch_pos"][:3] = torch.tensor([2, 7, -1], dtype=torch.int32)
    inp_np = synth.to_numpy_inputs(inp)
    o = oracle.verify(inp_np["PL"], inp_np["QL"], inp_np["tok"], inp_np["u"], inp_np["us"], inp_np["gamma"],
                      inp_np["branch_pos"])
    g = torch.Generator().manual_seed(5)
    kv = torch.randint(-30000, 30000, (c.B, c.K, c.G + 1, 2, 8, 64), generator=g, dtype=torch.int16)
    ref = oracle.kv_rollback(kv.numpy(), inp_np["branch_pos"], inp_np["gamma"], o["sel_k"], o["commit_len"],
                             o["y_kind"])
    # the kept set is the oracle's keep_mask, an independent statement of the same decision
    for b in range(c.B):
        for k in range(c.K):
            for i in range(c.G + 1):
                if (int(o["keep_mask"][b, k]) >> i) & 1:
                    assert np.array_equal(ref[b, i], kv.numpy()[b, k, i])
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")  # noqa: E731
    kvd = kv.cuda()
    args = (dev(o["keep_mask"].view(np.int32)),)
    n = o["commit_len"] - (o["y_kind"] != 0)
    if inplace:
        api.sb_kv_rollback(kvd, *args)
        torch.cuda.synchronize()
        got = kvd.cpu().numpy()[:, 0]
    else:
        out = torch.zeros((c.B, c.G + 1) + kv.shape[3:], dtype=kv.dtype, device="cuda")
        api.sb_kv_rollback(kvd, *args, out_kv=out)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
    for b in range(c.B):
        assert np.array_equal(got[b, : n[b]], ref[b, : n[b]]), b


TREES = [("dense_2222_bf16_V32000", "c2", dict(), "dense", dict(branching=(2, 2, 2, 2)), 64),
         ("dense_32_f32_V3001", "c1", dict(V=3001), "dense", dict(branching=(3, 2, 2)), 48),
         ("random63_bf16_V128256", "c3", dict(), "random", dict(N=63, depth=8), 24),
         ("chain8_bf16_V151936", "c4", dict(), "chain", dict(N=8), 32),
         ("random_tiny_V7", "c2", dict(V=7), "random", dict(N=30, depth=5), 96)]


@pytest.mark.parametrize("name,cfg,over,shape,kw,B", TREES, ids=[t[0] for t in TREES])
def test_tree_verify_matches_oracle(name, cfg, over, shape, kw, B):
    """f3 tree verify through the C-ABI against oracle.tree_verify: acceptance masks
    exact except at near-ties the oracle flags; the walk, commit and sample bit-exact
    on every sequence the oracle does not flag."""
    import oracle
    from paper_2506_01979_b200 import api, synth

    c = synth.config(cfg, **over)
    inp = synth.generate_tree(c, shape, B=B, seed=13, **kw)
    t = synth.tree_to_numpy(inp)
    o = oracle.tree_verify(t["PL"], t["QL"], t["parent"], t["tok"], t["u"], t["us"])
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    d = api.tree_dims(dev["PL"])
    buf = api.TreeBuffers(d)
    api.sb_tree_verify(d, dev["PL"], dev["QL"], dev["parent"], dev["tok"], dev["u"], dev["us"], buf)
    torch.cuda.synchronize()
    g = {k: getattr(buf, k).cpu().numpy() for k in ("acc_mask", "keep_mask", "stop_node", "commit_len", "out_tok",
                                                     "y_tok", "y_kind", "status", "resid_mass")}
    assert np.array_equal(g["status"], o["status"])
    # decisions: every sequence without an acceptance near-tie (|u - P/Q| < 1e-6)
    dec = (o["ties"] & oracle.TIE_ACC_DEC) == 0
    assert dec.mean() > 0.9
    assert np.array_equal(g["acc_mask"].view(np.uint64)[dec], o["acc_mask"][dec])
    assert np.array_equal(g["keep_mask"].view(np.uint64)[dec], o["keep_mask"][dec])
    for k in ("stop_node", "commit_len", "y_kind"):
        assert np.array_equal(g[k][dec], o[k][dec]), k
    n = o["commit_len"] - (o["y_kind"] != 0)
    for b in np.where(dec)[0]:
        assert np.array_equal(g["out_tok"][b, : n[b]], o["out_tok"][b, : n[b]]), b
    # the sample: bit-exact unless the oracle's CDF puts t within 1e-6 of a breakpoint
    # (bulk tokens of a V = 152k row carry ~3e-6 each) or the residual is ill-conditioned
    smp = dec & ((o["ties"] & (oracle.TIE_SAMPLE | oracle.TIE_ILLCOND)) == 0)
    assert smp.sum() >= len(smp) // 2
    assert np.array_equal(g["y_tok"][smp], o["y_tok"][smp])
    assert np.array_equal(g["out_tok"][smp], o["out_tok"][smp])
    assert ((g["y_tok"] >= 0) & (g["y_tok"] < c.V))[o["y_kind"] != 0].all()
    assert np.allclose(g["resid_mass"][dec], o["resid_mass"][dec], rtol=1e-5, atol=1e-7)


def test_tree_bad_parent_and_nonfinite():
    """Status bits: a parent pointer that is not earlier in topological order rejects
    that node (SB_ST_BAD_PARENT); a NaN context row rejects its children (NONFINITE)."""
    import oracle
    from paper_2506_01979_b200 import api, synth

    c = synth.config("c2", V=1000, dtype="f32")
    inp = synth.generate_tree(c, "dense", B=8, seed=3, branching=(2, 2))
    inp["parent"][1, 3] = 5  # not < 3
    inp["PL"][2, 1, 17] = float("nan")  # context after node 0
    t = synth.tree_to_numpy(inp)
    o = oracle.tree_verify(t["PL"], t["QL"], t["parent"], t["tok"], t["u"], t["us"])
    assert o["status"][1] & oracle.ST_BAD_PARENT and o["status"][2] & oracle.ST_NONFINITE
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    d = api.tree_dims(dev["PL"])
    buf = api.TreeBuffers(d)
    api.sb_tree_verify(d, dev["PL"], dev["QL"], dev["parent"], dev["tok"], dev["u"], dev["us"], buf)
    torch.cuda.synchronize()
    assert np.array_equal(buf.status.cpu().numpy(), o["status"])
    ok = o["ties"] == 0
    assert np.array_equal(buf.commit_len.cpu().numpy()[ok], o["commit_len"][ok])
    assert np.array_equal(buf.out_tok.cpu().numpy()[ok], o["out_tok"][ok])


# ---------------------------------------------------------------- f4: H-RAD MLP (tcgen05)
HRAD = [("B1_Dz64", 1, 64), ("B100_Dz320", 100, 320), ("B129_Dz256", 129, 256), ("B128_Dz5120", 128, 5120),
        ("B300_Dz2048", 300, 2048), ("B256_Dz20480", 256, 20480), ("B2048_Dz20480", 2048, 20480)]


@pytest.mark.parametrize("name,B,Dz", HRAD, ids=[h[0] for h in HRAD])
def test_hrad_matches_oracle(name, B, Dz):
    """Layer 1 on the tensor cores (fp32 accumulation of exact bf16 products), layers 2-3
    in fp32, vs the fp64 oracle.  Tolerance: a fp32 sum of Dz O(1)-bounded partials is
    off by ~sqrt(Dz/16) * 2^-24 relative; 1e-4 absolute on O(1) logits leaves > 10x
    margin.  s_t is exact except where the oracle's top-2 gap is below 1e-3 (flagged)."""
    import oracle
    from paper_2506_01979_b200 import api, synth

    G = 8
    inp = synth.hrad_inputs(B, Dz, G=G, seed=B + Dz, device="cuda")
    s_t, lg, gm, bp = api.sb_hrad_predict(inp["z"], inp["w1"], inp["b1"], inp["w2"], inp["b2"], inp["w3"],
                                          inp["b3"], G, stop=inp["stop"])
    torch.cuda.synchronize()
    n = synth.hrad_to_numpy(inp)
    o = oracle.hrad(n["z"], n["w1"], n["b1"], n["w2"], n["b2"], n["w3"], n["b3"], n["stop"], G)
    lg = lg.cpu().numpy()
    assert np.allclose(lg, o["logits"], rtol=1e-4, atol=1e-4), np.abs(lg - o["logits"]).max()
    tie = o["margin"] < 1e-3
    assert tie.mean() < 0.05
    assert np.array_equal(s_t.cpu().numpy()[~tie], o["s_t"][~tie])
    assert np.array_equal(gm.cpu().numpy()[~tie], o["gamma"][~tie])
    assert np.array_equal(bp.cpu().numpy()[~tie], o["branch_pos"][~tie])
    # run-to-run deterministic (fixed-order cluster reduction, no atomics)
    s2, lg2, _, _ = api.sb_hrad_predict(inp["z"], inp["w1"], inp["b1"], inp["w2"], inp["b2"], inp["w3"],
                                        inp["b3"], G, stop=inp["stop"])
    assert np.array_equal(lg2.cpu().numpy(), lg) and torch.equal(s2, s_t)


def test_hrad_rejects_unsupported_shapes():
    from paper_2506_01979_b200 import api, synth

    inp = synth.hrad_inputs(4, 200, G=4, seed=1, device="cuda")  # Dz not a multiple of 64
    with pytest.raises(RuntimeError):
        api.sb_hrad_predict(inp["z"], inp["w1"], inp["b1"], inp["w2"], inp["b2"], inp["w3"], inp["b3"], 4)
