"""world_size-2 gloo tests (CPU) of the multi-rank host logic: sequence sharding of the
inputs, the max/sum-over-ranks reduction bench.py reports, and the fact that sharding
sequences across ranks does not change any sequence's result (checked on the oracle:
sequences are independent units)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, scaling):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import oracle
    from paper_2506_01979_b200 import synth

    cfg = synth.config("c2", V=256, B=6, K=3, G=5, layout="mixed")
    b0, b1 = bench.rank_slice(cfg, rank, world, scaling)
    inp = synth.to_numpy_inputs(synth.generate(cfg, device="cpu", b0=b0, b1=b1))
    o = oracle.verify(inp["PL"], inp["QL"], inp["tok"], inp["u"], inp["us"], inp["gamma"], inp["branch_pos"],
                      nthreads=1, V=inp["V"])
    # gather every rank's shard and result on rank 0
    parts = [None] * world
    dist.all_gather_object(parts, {"PL": inp["PL"], "tok": inp["tok"], "out_tok": o["out_tok"],
                                   "n_acc": o["n_acc"], "commit_len": o["commit_len"]})
    ms, toks, comm, nbytes = bench.reduce_over_ranks(1.0 + rank, 10 * (rank + 1), 3, 100, "cpu", world)
    if rank == 0:
        np.savez(os.path.join(out_dir, "res.npz"),
                 PL=np.concatenate([p["PL"] for p in parts]), tok=np.concatenate([p["tok"] for p in parts]),
                 out_tok=np.concatenate([p["out_tok"] for p in parts]),
                 n_acc=np.concatenate([p["n_acc"] for p in parts]),
                 commit_len=np.concatenate([p["commit_len"] for p in parts]),
                 red=np.array([ms, toks, comm, nbytes]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_sequence_sharding_world2_gloo(tmp_path, scaling):
    """strong (bench default): the 6 sequences split 3 + 3 over the ranks;
    weak: every rank 6 sequences with global keys rank*6 ...  Either way the shards are
    the same bytes and results as the unsharded batch."""
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), scaling), nprocs=world, join=True)
    r = np.load(tmp_path / "res.npz")
    sys.path.insert(0, ROOT)
    import oracle
    from paper_2506_01979_b200 import synth

    cfg = synth.config("c2", V=256, B=6, K=3, G=5, layout="mixed")
    n = cfg.B if scaling == "strong" else world * cfg.B
    full = synth.to_numpy_inputs(synth.generate(cfg, device="cpu", b0=0, b1=n))
    # shard bytes == the same sequences of the unsharded batch (counter-keyed generator)
    assert np.array_equal(r["PL"], full["PL"]) and np.array_equal(r["tok"], full["tok"])
    o = oracle.verify(full["PL"], full["QL"], full["tok"], full["u"], full["us"], full["gamma"],
                      full["branch_pos"], nthreads=1, V=full["V"])
    for k in ("out_tok", "n_acc", "commit_len"):
        assert np.array_equal(r[k], o[k]), k
    # time = max over ranks, tokens / committed / bytes = sums
    assert r["red"].tolist() == [2.0, 30.0, 6.0, 200.0]
