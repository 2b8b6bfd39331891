"""a7: vocabulary-sharded verify-and-branch.  On one GPU the G
shards run through the split-phase C ABI with in-process exchanges (loopback); every
rank's outputs must equal the unsharded oracle on the full vocabulary and each other.
The NCCL communicator path (sb_comm_*) runs with a single rank."""
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


def _np(buf):
    out = {k: getattr(buf, k).cpu().numpy() for k in buf.__dataclass_fields__ if not k.endswith("workspace")}
    out["acc_mask"] = out["acc_mask"].view(np.uint32)
    out["keep_mask"] = out["keep_mask"].view(np.uint32)
    return out


CASES = [
    ("bf16_K8_G16", dict(name="c5", V=12288, B=24, layout="mixed"), (1, 2, 4, 8), 0),
    ("bf16_V32000_alg1", dict(name="c2", V=32000, B=24, layout="mixed"), (2, 8), 1),
    ("f32_V4096", dict(name="c1", V=4096, B=32, rounds=1, K=3, G=6, layout="mixed"), (2, 4), 0),
    ("bf16_uneven_V5000", dict(name="c4", V=5000, B=16, K=2, G=5, layout="mixed"), (3,), 0),
    # ragged last slices (row lengths not 16-byte multiples): register-staged partial pass
    ("f32_ragged_V3001", dict(name="c1", V=3001, B=24, rounds=1, K=3, G=6, layout="mixed"), (2, 3, 8), 0),
    ("bf16_ragged_V5003", dict(name="c2", V=5003, B=24, K=3, G=7, layout="mixed"), (2, 4), 1),
]


@pytest.mark.parametrize("warp_kernel", [False, True], ids=["tma_rows", "warp_rows"])
@pytest.mark.parametrize("name,kw,granks,rule", CASES, ids=[c[0] for c in CASES])
def test_sharded_loopback_matches_oracle(name, kw, granks, rule, warp_kernel, monkeypatch):
    """warp_rows: the partial pass through k_rows_warp (one warp per row pair; forced with
    SB_ROWS_VARIANT=9, the default for many rows of <= 64 KB such as C5's shards at G >= 4)."""
    if warp_kernel:
        monkeypatch.setenv("SB_ROWS_VARIANT", "9")
    from paper_2506_01979_b200 import api, synth

    from parity_util import compare, internal_consistency, oracle_for

    kw = dict(kw)
    c = synth.config(kw.pop("name"), **kw)
    inp = synth.generate(c, device="cuda", seed=31)
    inp_np = synth.to_numpy_inputs(inp)
    o = oracle_for(inp_np, inp_np["gamma"], rule=rule)
    for G in granks:
        bufs = api.sharded_step_loopback(inp, G, rule=rule)
        torch.cuda.synchronize()
        outs = [_np(b) for b in bufs]
        for g in outs[1:]:  # decisions replicated on every rank
            for k in ("n_acc", "acc_mask", "sel_k", "out_tok", "y_tok", "commit_len", "status", "lse_p", "p_tok"):
                assert np.array_equal(g[k], outs[0][k], equal_nan=True), (G, k)
        internal_consistency(outs[0], c.G)
        rep = compare(outs[0], o)
        assert rep["exact_seq"] >= 0.85 * rep["n"], (G, rep)


def test_nccl_comm_single_rank():
    """The library-owned NCCL path (sb_comm_create + comm argument) with one rank."""
    from paper_2506_01979_b200 import api, synth

    from parity_util import compare, oracle_for

    c = synth.config("c5", V=8192, B=16, layout="mixed")
    inp = synth.generate(c, device="cuda", seed=41)
    d, pv = api.shard_view(inp["PL"], inp["V"], 0, inp["V"])
    _, qv = api.shard_view(inp["QL"], inp["V"], 0, inp["V"])
    comm = api.Comm(1, 0, d)
    try:
        buf = api.StepBuffers.alloc(d, "cuda")
        api.verify_step(d, inp, buf, comm=comm, views=(pv, qv))
        torch.cuda.synchronize()
        inp_np = synth.to_numpy_inputs(inp)
        compare(_np(buf), oracle_for(inp_np, inp_np["gamma"]))
        comm.check()  # no asynchronous NCCL error recorded
    finally:
        comm.close()


def test_nccl_comm_abort():
    """sb_comm_abort releases a communicator (the failure path's teardown)."""
    from paper_2506_01979_b200 import api

    d = api.L.sb_dims(4, 2, 4, 1024, 0, 1024, 1024, 0, api.L.SB_BF16, 0)
    comm = api.Comm(1, 0, d)
    comm.check()
    comm.abort()
    assert not comm.handle


def test_sharded_dims_without_comm_rejected():
    from paper_2506_01979_b200 import _lib, api, synth

    c = synth.config("c2", V=1024, B=4, layout="mixed")
    inp = synth.generate(c, device="cuda", seed=1)
    d, pv = api.shard_view(inp["PL"], 1024, 0, 512)
    _, qv = api.shard_view(inp["QL"], 1024, 0, 512)
    buf = api.StepBuffers.alloc(d, "cuda")
    with pytest.raises(RuntimeError, match="invalid argument"):
        api.verify_step(d, inp, buf, views=(pv, qv))
