"""Vocabulary-sharded verify-and-branch with REAL ranks: two
processes, one vocabulary slice each, exchanging through torch.distributed (gloo, CPU
tensors) between the split-phase C-ABI calls — the rank-order plumbing of the three
exchanges (all-gather of the row partials, all-gather of the masses, all-reduce MAX of
the sampled token) that sb_comm runs with NCCL on a multi-GPU box.  Both processes share
the one GPU of this box.  Every rank's outputs must be identical and equal the unsharded
fp64 oracle (same bars as tests/parity_util.compare)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = {"bf16_c5_shape": dict(name="c5", V=20000, B=12, K=4, G=8, layout="mixed"),
         "f32_ragged": dict(name="c1", V=3001, B=16, K=3, G=6, rounds=1, layout="mixed")}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, case):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2506_01979_b200 import api, synth

    kw = dict(CASES[case])
    c = synth.config(kw.pop("name"), **kw)
    host = synth.generate(c, device="cpu", seed=61)  # the same bytes on every rank
    inp = {k: (v.cuda() if torch.is_tensor(v) else v) for k, v in host.items()}
    V = inp["V"]
    v0, n = api.shard_bounds(V, world)[rank]
    d, pv = api.shard_view(inp["PL"], V, v0, n)
    _, qv = api.shard_view(inp["QL"], V, v0, n)
    buf = api.StepBuffers.alloc(d, "cuda")
    part = torch.empty(api.sb_shard_partial_bytes(d), dtype=torch.uint8, device="cuda")
    api.sb_shard_verify_local(d, pv, qv, inp["tok"], inp["u"], inp["gamma"], inp["branch_pos"], part, buf.workspace)
    torch.cuda.synchronize()
    parts = [torch.empty_like(part.cpu()) for _ in range(world)]
    dist.all_gather(parts, part.cpu())  # exchange 1, rank order
    gathered = torch.cat(parts).cuda()
    api.sb_shard_verify_combine(d, gathered, world, inp["tok"], inp["u"], buf)
    mass = torch.empty((d.B, 2), dtype=torch.float64, device="cuda")
    api.sb_shard_select_local(d, pv, qv, inp["tok"], inp["u"], buf.n_acc, 0, mass, buf.workspace)
    torch.cuda.synchronize()
    ms = [torch.empty_like(mass.cpu()) for _ in range(world)]
    dist.all_gather(ms, mass.cpu())  # exchange 2
    gmass = torch.cat(ms).cuda()
    yc = torch.empty(d.B, dtype=torch.int32, device="cuda")
    api.sb_shard_select_sample(d, gmass, world, rank, pv, qv, inp["us"], yc, buf.workspace)
    torch.cuda.synchronize()
    y = yc.cpu()
    dist.all_reduce(y, op=dist.ReduceOp.MAX)  # exchange 3
    api.sb_shard_select_commit(d, y.cuda(), inp["tok"], buf)
    torch.cuda.synchronize()
    out = {k: getattr(buf, k).cpu().numpy() for k in buf.__dataclass_fields__ if not k.startswith("c_")
           and not k.endswith("workspace")}
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", list(CASES))
def test_vocab_shards_two_processes(tmp_path, case):
    import torch.multiprocessing as mp

    from paper_2506_01979_b200 import synth
    from paper_2506_01979_b200.build import build

    from parity_util import compare, oracle_for

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    build()
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), case), nprocs=world, join=True)
    outs = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    for k in outs[0]:
        if k == "packed_tok":
            continue
        assert np.array_equal(outs[0][k], outs[1][k], equal_nan=True), k  # decisions replicated
    kw = dict(CASES[case])
    c = synth.config(kw.pop("name"), **kw)
    inp_np = synth.to_numpy_inputs(synth.generate(c, device="cpu", seed=61))
    g = outs[0]
    g["acc_mask"] = g["acc_mask"].view(np.uint32)
    g["keep_mask"] = g["keep_mask"].view(np.uint32)
    rep = compare(g, oracle_for(inp_np, inp_np["gamma"]), inp_np=inp_np)
    assert rep["exact_seq"] >= 0.8 * rep["n"], rep
