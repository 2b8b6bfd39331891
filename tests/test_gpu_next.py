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
         ("tiny_V5", dict(name="c2", V=5, B=64, K=2, G=3, layout="mixed"), 8, 0)]


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
    inp_np = synth.to_numpy_inputs(inp)
    o = oracle.verify(inp_np["PL"], inp_np["QL"], inp_np["tok"], inp_np["u"], inp_np["us"], inp_np["gamma"],
                      inp_np["branch_pos"])
    g = torch.Generator().manual_seed(5)
    kv = torch.randint(-30000, 30000, (c.B, c.K, c.G + 1, 2, 8, 64), generator=g, dtype=torch.int16)
    ref = oracle.kv_rollback(kv.numpy(), inp_np["branch_pos"], o["sel_k"], o["commit_len"], o["y_kind"])
    # the kept set is the oracle's keep_mask, an independent statement of the same decision
    for b in range(c.B):
        for k in range(c.K):
            for i in range(c.G + 1):
                if (int(o["keep_mask"][b, k]) >> i) & 1:
                    assert np.array_equal(ref[b, i], kv.numpy()[b, k, i])
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")  # noqa: E731
    kvd = kv.cuda()
    args = (dev(inp_np["branch_pos"]), dev(o["sel_k"]), dev(o["commit_len"]), dev(o["y_kind"]))
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
