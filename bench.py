#!/usr/bin/env python
"""Benchmark of the SpecBranch verify-and-branch step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One step = one pass of the whole hot path over one batch of synthetic input
([draft confidence ->] sb_verify_branches -> sb_select_branch, through the C ABI).
Default workload: BASELINE config C4 (Qwen V=151936, 2048 sequences, K=4, gamma=8,
bf16) — the configuration the metric's "1/2/4/8 GPUs" is quoted on.  Sequences shard
across ranks with no data-path collective: by default the 2048 sequences are split over
the N ranks (strong scaling; --scaling weak gives every rank 2048).
`python bench.py --gpus N` without torchrun re-launches itself as N ranks.  Rank 0 prints
one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "verified draft tokens/sec and logit HBM GB/s (% of B200 peak) at 1/2/4/8 GPUs"


def peaks():
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        if self.index < 0:
            return self
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in self.rows for j in range(4) if len(r) > 3 + j and r[3 + j] == "Active"})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(pw) if pw else None}


def verified_tokens(gamma, bpos, K):
    """sum_b [s_b + K (L_b - s_b)]."""
    t = 0
    for g, s in zip(gamma, bpos):
        L = g if s < g else g + 1
        t += s + K * (L - s)
    return t


def bytes_model(gamma, bpos, y_kind, K, V, es, G, conf_rows=0, bonus_rows=False):
    """Algorithmic bytes of one step: a1 row pairs, a4 sampled
    rows (2 for a residual, 1 for a bonus; a bonus row needs 2 passes), a6 draft rows,
    plus 12 B per path token (token + uniform + output)."""
    units = sum(L + (K - 1) * (L - 1 - s) for g, s in zip(gamma, bpos)
                for L in [(g if s < g else g + 1) if not bonus_rows else g + 1])
    a1 = units * 2 * V * es
    # sharded mode reads bonus rows in a1; its sample pass streams the row once per kind
    a4 = sum(2 if k == 1 else (1 if k == 2 else 0) for k in y_kind) * V * es
    a6 = conf_rows * V * es
    small = verified_tokens(gamma, bpos, K) * 12
    return a1, a4, a6, small, units


def launches_per_step(cfg, d, adaptive, vocab, es):
    """The library's kernel launches in one step: the adaptive step of a small problem is
    one k_astep launch (sb_step_adaptive's rule: B K (G+1) <= 4096, 16-byte rows, not
    SB_ASTEP=0); otherwise confidence (adaptive) + k_plan + k_rows_tma + k_select_tma,
    plus the three shard kernels of the vocabulary-sharded path."""
    if adaptive and not vocab and os.environ.get("SB_ASTEP") != "0" and (d.V * es) % 16 == 0 \
            and d.B * d.K * (d.G + 1) <= 4096:
        return 1
    return (1 if adaptive else 0) + (6 if vocab else 3)


def rank_slice(cfg, rank, world, scaling="strong"):
    """Sequences [b0, b1) a rank owns (global sequence keys; no data-path collective).
    strong (default): the configuration's batch split contiguously, rank g
    owns [g B / N, (g + 1) B / N) (C4 at 8 GPUs: 256 each); weak: every rank a full
    per-GPU batch with keys rank * B .. (rank + 1) * B - 1."""
    Bl = cfg.B * cfg.rounds
    if scaling == "weak":
        return rank * Bl, (rank + 1) * Bl
    return rank * Bl // world, (rank + 1) * Bl // world


def reduce_over_ranks(ms_step, toks, committed, nbytes, device, world):
    """Step time = MAX over ranks; tokens / bytes = SUM over ranks (torch.distributed)."""
    if world <= 1:
        return ms_step, toks, committed, nbytes
    import torch

    t = torch.tensor([ms_step, float(toks), float(committed), float(nbytes)], device=device, dtype=torch.float64)
    mx = t[:1].clone()
    sm = t[1:].clone()
    torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
    torch.distributed.all_reduce(sm, op=torch.distributed.ReduceOp.SUM)
    return float(mx[0]), float(sm[0]), float(sm[1]), float(sm[2])


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2506_01979_b200 import api, synth
    from paper_2506_01979_b200.build import build

    build()
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = synth.config(args.config, **({"delta": args.delta} if args.delta is not None else {}))
    Btot = cfg.B * cfg.rounds
    b0, b1 = rank_slice(cfg, rank, world, args.scaling)
    vocab = args.mode == "vocab"
    if vocab:  # every rank sees all sequences and owns a vocabulary slice (a7)
        b0, b1 = 0, Btot
    Bl = b1 - b0  # this rank's sequences
    t0 = time.time()
    inp = synth.generate(cfg, device=dev, b0=b0, b1=b1)
    gen_s = time.time() - t0
    comm, views = None, None
    if vocab:
        v0, vn = api.shard_bounds(inp["V"], world)[rank]
        d, pv = api.shard_view(inp["PL"], inp["V"], v0, vn)
        _, qv = api.shard_view(inp["QL"], inp["V"], v0, vn)
        views = (pv, qv)
        uid = [None]
        if rank == 0:
            import ctypes

            from paper_2506_01979_b200 import _lib
            b = ctypes.create_string_buffer(int(_lib.lib().sb_comm_unique_id_bytes()))
            _lib.check(_lib.lib().sb_comm_unique_id(b), "sb_comm_unique_id")
            uid = [b.raw]
        if world > 1:
            torch.distributed.broadcast_object_list(uid, src=0)
        comm = api.Comm(world, rank, d, unique_id=uid[0])
    else:
        d = api.dims_for(inp["PL"], V=inp["V"])
    buf = api.StepBuffers.alloc(d, dev)
    adaptive = cfg.layout == "adaptive"
    stream = torch.cuda.current_stream()
    es = 2 if cfg.dtype == "bf16" else 4

    def step():
        return api.verify_step(d, inp, buf, adaptive=adaptive, stream=stream, comm=comm, views=views)

    # Inputs of a small configuration (C2: 147 MB of logits) are rotated over several
    # independently drawn sets so that no timed step can find its bytes in the 126 MB L2
    # (>= 3 x L2 of logits across the sets); every set is its own graph, replayed in turn.
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    in_bytes = inp["PL"].numel() * inp["PL"].element_size() * 2
    nsets = 1 if (vocab or in_bytes >= 3 * l2) else min(8, -(-3 * l2 // in_bytes))
    sets = [inp] + [synth.generate(cfg, device=dev, b0=b0, b1=b1, seed=7919 * r + 1) for r in range(1, nsets)]
    stats = []
    for x in sets:  # warm-up per set, then its verified tokens / bytes / commits
        for _ in range(max(args.warmup, 3)):
            api.verify_step(d, x, buf, adaptive=adaptive, stream=stream, comm=comm, views=views if x is inp else None)
        torch.cuda.synchronize()
        gamma = (buf.c_gamma.view(-1) if adaptive else x["gamma"]).cpu().tolist()
        bpos = x["branch_pos"].cpu().tolist()
        ykind = buf.y_kind.cpu().tolist()
        bm = bytes_model(gamma, bpos, ykind, cfg.K, d.V, es, cfg.G, conf_rows=(Bl * cfg.G if adaptive else 0),
                         bonus_rows=vocab)
        stats.append((bm, verified_tokens(gamma, bpos, cfg.K), int(buf.commit_len.sum())))
    # set 0 is the one the per-call breakdown and the roofline kernel are timed on
    (a1, a4, a6, small, units), _, _ = stats[0]
    api.verify_step(d, inp, buf, adaptive=adaptive, stream=stream, comm=comm, views=views)
    torch.cuda.synchronize()
    # the per-call timings replay set 0 alone: small sets get an L2 flush (a write of 2 x L2,
    # outside the events) before every timed replay
    flush_buf = torch.empty(2 * l2 // 4 if nsets > 1 else 0, dtype=torch.float32, device=dev)

    def flush_l2():
        if flush_buf.numel():
            flush_buf.zero_()

    seq = [stats[k % nsets] for k in range(args.steps)]  # the timed steps' sets, in order
    toks = sum(t for _, t, _ in seq) / args.steps
    committed = sum(c for _, _, c in seq) / args.steps
    step_bytes = sum(sum(bm[:4]) for bm, _, _ in seq) / args.steps

    # ---- timed region: exactly K whole steps, replayed from a CUDA graph of the C-ABI
    # launches (no per-step host/ctypes overhead), bracketed by barrier + synchronize
    kt_first = {}
    gam0 = buf.c_gamma.view(-1) if adaptive else inp["gamma"]
    PLv0, QLv0 = views if views is not None else (inp["PL"], inp["QL"])
    ver_fn = (lambda s_: api.sb_verify_branches(
        d, PLv0, QLv0, inp["tok"], inp["u"], gam0, inp["branch_pos"], buf.lse_p, buf.lse_q, buf.p_tok, buf.q_tok,
        buf.acc_mask, buf.n_acc, buf.top1_q, buf.top1_id_q, buf.entropy_q, buf.status, buf.workspace, s_, comm))
    if not args.no_graph:  # the roofline kernel, timed right before the step region
        vg = api.CallGraph(ver_fn)
        ve = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        torch.cuda.synchronize()
        for e0, e1 in ve:
            flush_l2()
            e0.record(torch.cuda.current_stream())
            vg.replay()
            e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        kt_first["verify"] = sum(e0.elapsed_time(e1) for e0, e1 in ve) / args.steps
    graphs = [api.CallGraph(lambda s_, x=x: api.verify_step(d, x, buf, adaptive=adaptive, stream=s_, comm=comm,
                                                          views=views if x is inp else None))
              for x in sets] if not args.no_graph else None
    clk = Clocks(local_rank if not args.no_clocks else -1).__enter__()
    time.sleep(0.3)  # let nvidia-smi start sampling before the timed region
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    run_stream = torch.cuda.current_stream()  # CUDAGraph.replay() launches on the current stream
    start.record(run_stream)
    for k in range(args.steps):
        if graphs is not None:
            graphs[k % nsets].replay()
        else:
            api.verify_step(d, sets[k % nsets], buf, adaptive=adaptive, stream=stream, comm=comm,
                            views=views if k % nsets == 0 else None)
    end.record(run_stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = start.elapsed_time(end)
    if nsets > 1:  # set 0's state again for the per-call timings and the parity record
        step()
        torch.cuda.synchronize()

    # ---- kernel timing region (roofline): each C-ABI call captured alone in a CUDA
    # graph and replayed K times, CUDA events around every replay on the launching stream
    gam = buf.c_gamma.view(-1) if adaptive else inp["gamma"]
    PLv, QLv = views if views is not None else (inp["PL"], inp["QL"])
    calls = {
        "conf": (lambda s: api.sb_draft_confidence(
            api.conf_dims(d), inp["QL"], None, api.SB_CONF_TOP1, 0.2, 1.0, 6, buf.c_top1, buf.c_id,
            buf.c_ent, None, buf.c_stat, buf.c_stop, buf.c_knext, buf.c_gamma, buf.conf_workspace, s))
        if adaptive else None,
        "verify": lambda s: api.sb_verify_branches(
            d, PLv, QLv, inp["tok"], inp["u"], gam, inp["branch_pos"], buf.lse_p, buf.lse_q,
            buf.p_tok, buf.q_tok, buf.acc_mask, buf.n_acc, buf.top1_q, buf.top1_id_q, buf.entropy_q,
            buf.status, buf.workspace, s, comm),
        "verify_reuse": (lambda s: api.sb_verify_branches_reuse(
            d, PLv, QLv, inp["tok"], inp["u"], gam, inp["branch_pos"], buf.lse_p, buf.lse_q,
            buf.p_tok, buf.q_tok, buf.acc_mask, buf.n_acc, buf.top1_q, buf.top1_id_q, buf.entropy_q,
            buf.status, buf.conf_workspace, buf.workspace, s))
        if adaptive and comm is None else None,
        "fused": (lambda s: api.sb_verify_select(
            d, PLv, QLv, inp["tok"], inp["u"], inp["us"], gam, inp["branch_pos"], 0, buf, s))
        if comm is None else None,
        "select": lambda s: api.sb_select_branch(
            d, PLv, QLv, inp["tok"], inp["u"], inp["us"], gam, inp["branch_pos"], buf.n_acc, 0,
            buf.sel_k, buf.commit_len, buf.out_tok, buf.y_tok, buf.y_kind, buf.offsets, buf.packed_tok,
            buf.path_rolled, buf.branch_discarded, buf.keep_mask, buf.resid_mass, buf.status, buf.workspace, s,
            comm),
    }
    kt = {}
    for name, fn in calls.items():
        if fn is None or name in kt_first:
            kt[name] = 0.0
            continue
        cg = api.CallGraph(fn) if not args.no_graph else None
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream()
        for e0, e1 in evs:
            flush_l2()
            e0.record(cur)
            cg.replay() if cg is not None else fn(cur)
            e1.record(cur)
        torch.cuda.synchronize()
        kt[name] = sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps
    clk.__exit__()
    kt.update(kt_first)
    t_conf, t_ver, t_sel, t_fused = kt["conf"], kt["verify"], kt["select"], kt["fused"]
    ms_step = ms / args.steps
    ms_step_all, toks_all, comm_all, bytes_all = reduce_over_ranks(
        ms_step, toks, committed, step_bytes, dev, world)
    if vocab:  # every rank verifies the same tokens: count them once
        toks_all, comm_all = float(toks), float(committed)

    # ---- C1 also has a latency number: one round of batch 1 as its own
    # dependent step, replayed from a CUDA graph (rotating over 8 distinct rounds)
    round_lat = None
    if cfg.name == "c1" and not vocab and world == 1:
        c1 = synth.config("c1", rounds=1)
        one = [synth.generate(c1, device=dev, seed=1000 + r) for r in range(8)]
        d1 = api.dims_for(one[0]["PL"], V=one[0]["V"])
        b1s = [api.StepBuffers.alloc(d1, dev) for _ in one]
        gs = [api.CallGraph(lambda s_, x=x, bb=bb: api.verify_step(d1, x, bb, stream=s_)) for x, bb in zip(one, b1s)]
        for g_ in gs:
            g_.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nrep = 200
        e0.record(torch.cuda.current_stream())
        for k in range(nrep):
            gs[k % len(gs)].replay()
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        round_lat = round(1e3 * e0.elapsed_time(e1) / nrep, 2)

    # ---- e2e through the public API with host buffers (pinned), H2D + D2H inside
    e2e = None
    if not args.no_e2e and not vocab:
        e2e = run_e2e(args, inp, d, buf, adaptive, stream, dev, world)
    if comm is not None:
        comm.close()
    if rank != 0:
        return None
    peak, peak_src = peaks()
    # dominant kernel (93% of the C4 step in the ncu launch list): sb_verify_branches
    rf_kernel = "sb_verify_branches (k_plan + k_rows_tma" + (" + NCCL all-gather + k_shard_combine)" if vocab else ")")
    rf_bytes, rf_ms = a1 + small, t_ver
    ver_gbs = rf_bytes / (rf_ms * 1e-3) / 1e9
    step_gbs = bytes_all / (ms_step_all * 1e-3) / 1e9
    value = toks_all / (ms_step_all * 1e-3)
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "verified draft tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": round(ms_step_all, 4), "higher_is_better": True,
        "scaling": "strong" if vocab else args.scaling,
        "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic (seeded, DESIGN.md §Input recipe)",
        "config": {"workload": f"{cfg.name.upper()}: {cfg.note}", "V": cfg.V, "K": cfg.K, "G": cfg.G,
                   "per_rank_batch": Bl, "global_batch": Btot if (vocab or args.scaling == "strong") else Btot * world,
                   "layout": cfg.layout,
                   "parallelism": (f"vocabulary-sharded x{world} (NCCL all-gather / all-reduce, sb_comm)"
                                   if vocab else f"sequence-sharded x{world} (no data-path collective)"),
                   "l2": ("inputs larger than L2 (%.1f GB of logits per rank vs %.0f MB)" % (in_bytes / 1e9, l2 / 1e6)
                          if nsets == 1 else "%d rotating input sets (%d x %.0f MB of logits vs %.0f MB L2)"
                          % (nsets, nsets, in_bytes / 1e6, l2 / 1e6))},
        "logit_GBps": round(step_gbs, 1), "logit_frac_of_peak": round(step_gbs / world / peak, 4),
        "committed_tokens_per_s": round(comm_all / (ms_step_all * 1e-3), 1),
        "breakdown_ms": {"draft_confidence": round(t_conf, 4), "verify": round(t_ver, 4),
                         "verify_reusing_confidence_rows": round(kt["verify_reuse"], 4),
                         "select": round(t_sel, 4), "verify_select": round(t_fused, 4),
                         "source": "each call replayed alone from its own CUDA graph, CUDA events"},
        "timing": "CUDA graph replay of the whole step" if not args.no_graph else "eager C-ABI calls",
        "roofline": {"bound": "hbm", "kernel": rf_kernel,
                     "achieved": round(ver_gbs, 1), "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(ver_gbs / peak, 4), "traffic": traffic_from_profiles(cfg.name),
                     "algorithmic_bytes_per_launch": rf_bytes, "row_pairs_per_launch": units},
        "gpu_launches": args.steps * launches_per_step(cfg, d, adaptive, vocab, es),
        "clocks": clk.summary(),
        "generation_s": round(gen_s, 1),
    }
    if e2e is not None:
        line["e2e"] = e2e
    if round_lat is not None:
        line["per_round_latency_us"] = round_lat
        line["per_round_note"] = ("one C1 round (batch 1, K=2, gamma=8, fp32) as a dependent step: "
                                  "conf-free verify + select from a CUDA graph; latency-bound (4 MB of rows)")
    if not args.no_cpu_baseline and world == 1 and not vocab:
        line["cpu_baseline"] = cpu_baseline(cfg, inp, adaptive, buf, budget_s=args.cpu_budget)
    return line


def tensor_peak():
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(pk["bf16_tflops"]), "measured (MEASURED_PEAKS.json bf16_tflops, burst)"
    except Exception:
        return 1590.0, "fallback (B200_PROFILING.md 1.59 PFLOP/s)"


def run_hrad(args, rank, world, local_rank):
    """--config hrad: the f4 row, H-RAD MLP inference (sb_hrad_predict) on synthetic
    LLaMA-3.1-8B-shaped features (Dz = 4 layers x 4096 + 4096 embedding = 20480, P400)
    for a batch of sequences per rank.  Three input sets rotate so no launch finds its
    z / W1 in L2 (3 x 94 MB > 126 MB)."""
    import numpy as np
    import torch

    from paper_2506_01979_b200 import _lib, api, synth
    from paper_2506_01979_b200.build import build

    build()
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    B, Dz, G = args.hrad_batch, synth.HRAD_DZ["llama31_8b"], 16
    sets = [synth.hrad_inputs(B, Dz, G=G, seed=1000 * rank + j, device=dev) for j in range(3)]
    nws = int(_lib.lib().sb_hrad_workspace_bytes(B, Dz))
    outs = [(torch.empty(B, dtype=torch.int32, device=dev), torch.empty((B, 3), device=dev),
             torch.empty(B, dtype=torch.int32, device=dev), torch.empty(B, dtype=torch.int32, device=dev),
             torch.empty(nws, dtype=torch.uint8, device=dev)) for _ in range(3)]

    def call(j, s_):
        x, o = sets[j], outs[j]
        api.sb_hrad_predict(x["z"], x["w1"], x["b1"], x["w2"], x["b2"], x["w3"], x["b3"], G, stop=x["stop"],
                            s_t=o[0], logits=o[1], gamma=o[2], branch_pos=o[3], workspace=o[4], stream=s_)

    graphs = [api.CallGraph(lambda s_, j=j: call(j, s_)) for j in range(3)]
    for k in range(max(args.warmup, 3)):
        graphs[k % 3].replay()
    torch.cuda.synchronize()
    clk = Clocks(local_rank if not args.no_clocks else -1).__enter__()
    time.sleep(0.3)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    cur = torch.cuda.current_stream()
    for k, (e0, e1) in enumerate(evs):
        e0.record(cur)
        graphs[k % 3].replay()
        e1.record(cur)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk.__exit__()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps
    ms_all, rows_all, _, _ = reduce_over_ranks(ms, B, 0, 0, dev, world)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        n = synth.hrad_to_numpy({k: (v[:64] if k in ("z", "stop") else v) for k, v in sets[0].items()})
        nthreads = os.cpu_count() or 1
        t0 = time.time()
        oracle.hrad(n["z"], n["w1"], n["b1"], n["w2"], n["b2"], n["w3"], n["b3"], n["stop"], G, nthreads=nthreads)
        dt = time.time() - t0
        cpu = {"value": round(64 / dt, 1), "unit": "H-RAD predictions/s", "cores": nthreads, "kind": "oracle",
               "sample": f"64 of {B} sequences, {dt:.2f} s, fp64 plain loops, OpenMP over sequences"}
    if rank != 0:
        return None
    peak, peak_src = peaks()
    tpk, tpk_src = tensor_peak()
    nbytes = B * Dz * 2 + 256 * Dz * 2 + B * 4 * 4 + 256 * 4 + 64 * 256 * 4
    flops = 2.0 * B * Dz * 256 + 2.0 * B * 256 * 64 + 2.0 * B * 64 * 3
    gbs = nbytes / (ms * 1e-3) / 1e9
    tfs = flops / (ms * 1e-3) / 1e12
    return {
        "metric": "H-RAD length predictions/s (SURVEY §8.6 f4)", "value": round(rows_all / (ms_all * 1e-3), 1),
        "unit": "predictions/s", "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": round(ms_all, 5), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (seeded features and random-init weights; no trained H-RAD exists)",
        "config": {"workload": f"H-RAD MLP {Dz}-256-64-3, batch {B} per GPU (LLaMA-3.1-8B features, L_f = 4)",
                   "l2": "3 rotating input sets (3 x %.0f MB > 126 MB L2)" % (nbytes / 1e6)},
        "roofline": {"bound": "hbm", "kernel": "k_hrad (tcgen05 layer 1, split-K) + k_hrad_tail (PDL)",
                     "achieved": round(gbs, 1), "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(gbs / peak, 4), "traffic": None, "algorithmic_bytes_per_launch": nbytes},
        "tensor": {"achieved_tflops": round(tfs, 1), "peak": tpk, "peak_source": tpk_src,
                   "frac": round(tfs / tpk, 4), "flops_per_launch": flops},
        "gpu_launches": 2 * args.steps, "clocks": clk.summary(),
        **({"cpu_baseline": cpu} if cpu else {}),
    }


def run_next(args, rank, world, local_rank):
    """--config spawn | kv | tree: the SURVEY §8.6 NEXT rows f1-f3, each timed alone
    (CUDA graph of the C-ABI call, CUDA events per replay) against the HBM roofline."""
    import torch

    from paper_2506_01979_b200 import api, synth
    from paper_2506_01979_b200.build import build

    build()
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    t0 = time.time()
    if args.config == "spawn":  # f1: Eq. 7 TopK spawn on the branch row, C4 shape
        c = synth.config("c4")
        B, V, k_max = c.B, c.V, 6
        QL = synth.draft_rows(c, B, seed=1, device=dev).view(B, 1, 1, V)  # the branch rows (s_b = 0)
        d = api.dims_for(QL, V=V)
        bpos = torch.zeros(B, dtype=torch.int32, device=dev)
        k = torch.empty(B, dtype=torch.int32, device=dev)
        bt = torch.empty((B, k_max), dtype=torch.int32, device=dev)
        bp = torch.empty((B, k_max), dtype=torch.float32, device=dev)
        cf = torch.empty(B, dtype=torch.float32, device=dev)
        fn = lambda s_: api.sb_spawn_branches(d, QL, bpos, None, api.SB_CONF_TOP1, k_max, k, bt, bp, cf, s_)  # noqa
        nbytes, units, unit = B * V * 2, B, "branch spawns/s"
        work = f"f1 Eq. 7 branch spawn (k_max = {k_max}), batch {B}, V = {V} bf16 (C4 shape)"
        kern = "k_spawn"
    elif args.config == "kv":  # f2: KV rollback of a C4-shaped round, 8 KB of draft KV per position
        c = synth.config("c4")
        B, K, G, row = c.B, c.K, c.G, 8192
        g = torch.Generator(device="cpu").manual_seed(11)
        kv = torch.empty((B, K, G + 1, row // 2), dtype=torch.bfloat16, device=dev)
        kv.view(torch.int16).random_(-30000, 30000)
        out = torch.empty((B, G + 1, row // 2), dtype=torch.bfloat16, device=dev)
        sel = torch.randint(-1, K, (B,), generator=g, dtype=torch.int32).to(dev)
        cl = torch.randint(1, G + 2, (B,), generator=g, dtype=torch.int32).to(dev)
        yk = torch.ones(B, dtype=torch.int32, device=dev)
        bpos = torch.zeros(B, dtype=torch.int32, device=dev)
        # keep mask of the round (as sb_select_branch writes it): slot 0 below s_b = 0 is
        # empty, the selected slot (0 on rollback) keeps positions i < n_b
        n_b = (cl - yk.ne(0).to(torch.int32)).clamp(min=0)
        bits = ((1 << n_b.to(torch.int64)) - 1).to(torch.int32)
        keep = torch.zeros((B, K), dtype=torch.int32, device=dev)
        keep[torch.arange(B, device=dev), sel.clamp(min=0).long()] = bits
        fn = lambda s_: api.sb_kv_rollback(kv, keep, out_kv=out, stream=s_)  # noqa: E731
        moved = int((cl - 1).clamp(min=0).sum())
        nbytes, units, unit = 2 * moved * row, moved, "KV positions kept/s"
        work = f"f2 KV rollback, batch {B}, K = {K}, gamma = {G}, {row} B per position (out of place)"
        kern = "k_kv_rollback"
    else:  # f3: dense SpecInfer-style trees (branching 2,2,2,2: 30 nodes), Vicuna vocab
        c = synth.config("c2")
        B = 256
        inp = synth.generate_tree(c, "dense", B=B, seed=13, branching=(2, 2, 2, 2), device=dev)
        d = api.tree_dims(inp["PL"])
        buf = api.TreeBuffers(d, dev)
        fn = lambda s_: api.sb_tree_verify(d, inp["PL"], inp["QL"], inp["parent"], inp["tok"], inp["u"],  # noqa
                                           inp["us"], buf, s_)
        par = inp["parent"][0].tolist()
        inner = len(set(par))  # contexts with children: their p and q rows are read
        nbytes, units, unit = B * inner * 2 * c.V * 2, B * inp["N"], "tree nodes verified/s"
        work = f"f3 token-tree verify, {B} dense trees of {inp['N']} nodes (2,2,2,2), V = {c.V} bf16"
        kern = "k_tree_* (context-row stats + walk + sample)"
    gen_s = time.time() - t0
    g = api.CallGraph(fn)
    for _ in range(max(args.warmup, 3)):
        g.replay()
    torch.cuda.synchronize()
    clk = Clocks(local_rank if not args.no_clocks else -1).__enter__()
    time.sleep(0.3)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    cur = torch.cuda.current_stream()
    for e0, e1 in evs:
        e0.record(cur)
        g.replay()
        e1.record(cur)
    torch.cuda.synchronize()
    clk.__exit__()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps
    if rank != 0:
        return None
    peak, peak_src = peaks()
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {
        "metric": f"SURVEY §8.6 {args.config}: {unit}", "value": round(units / (ms * 1e-3), 1), "unit": unit,
        "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded, DESIGN.md §Input recipe)",
        "config": {"workload": work, "l2": "inputs %.0f MB per call vs 126 MB L2" % (nbytes / 1e6)},
        "roofline": {"bound": "hbm", "kernel": kern, "achieved": round(gbs, 1), "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": round(gbs / peak, 4), "traffic": None,
                     "algorithmic_bytes_per_launch": nbytes},
        "gpu_launches": args.steps * (2 if args.config == "tree" else 1), "clocks": clk.summary(),
        "generation_s": round(gen_s, 1),
    }


def traffic_from_profiles(name):
    p = os.path.join(ROOT, "profiles", f"traffic_{name}.json")
    try:
        return json.load(open(p))["dram_bytes_per_launch"]
    except Exception:
        return None


def run_e2e(args, inp, d, buf, adaptive, stream, dev, world):
    import torch

    from paper_2506_01979_b200 import api

    keys = ("PL", "QL", "tok", "u", "us", "gamma", "branch_pos")
    need = sum(inp[k].numel() * inp[k].element_size() for k in keys)
    # every rank pins its own inputs: skip (all ranks alike) rather than exhaust host memory
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = float("inf")
    host, ok = None, need * world <= 0.6 * avail
    if ok:
        try:
            host = {k: torch.empty(inp[k].shape, dtype=inp[k].dtype, pin_memory=True) for k in keys}
        except Exception:
            host, ok = None, False
    if world > 1:
        f = torch.tensor([1 if ok else 0], device=dev)
        torch.distributed.all_reduce(f, op=torch.distributed.ReduceOp.MIN)
        ok = bool(f.item())
    if not ok:
        del host
        return {"unavailable": "pinned host copies of %d ranks x %.1f GB of inputs exceed 60 %% of the %.0f GB "
                               "of available host memory" % (world, need / 1e9, avail / 1e9)}
    for k in keys:
        host[k].copy_(inp[k])
    dv = {k: inp[k] for k in keys}
    dv["V"] = inp["V"]
    h2d = sum(host[k].numel() * host[k].element_size() for k in keys)
    outs = ("commit_len", "out_tok", "y_tok", "sel_k", "offsets")
    hout = {k: torch.empty(getattr(buf, k).shape, dtype=torch.int32, pin_memory=True) for k in outs}
    d2h = sum(v.numel() * 4 for v in hout.values())
    steps = max(1, min(args.steps, args.e2e_steps))
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(steps):
        for k in keys:
            dv[k].copy_(host[k], non_blocking=True)
        api.verify_step(d, dv, buf, adaptive=adaptive, stream=stream)
        for k in outs:
            hout[k].copy_(getattr(buf, k), non_blocking=True)
    e.record(stream)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    gamma = (buf.c_gamma.view(-1) if adaptive else inp["gamma"]).cpu().tolist()
    toks = verified_tokens(gamma, inp["branch_pos"].cpu().tolist(), d.K)
    if world > 1:  # time = max over ranks, tokens = sum over ranks
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t[0])
        n = torch.tensor([float(toks)], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(n, op=torch.distributed.ReduceOp.SUM)
        toks = float(n[0])
    return {"value": round(toks / (ms * 1e-3), 1), "unit": "verified draft tokens/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 3),
            "steps": steps, "path": "pinned host -> H2D -> verify_step (C ABI) -> D2H of the commit"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(cfg, inp, adaptive, buf, budget_s=15.0):
    """The fp64 oracle as it stands, on this host's cores, over a bounded sample."""
    import numpy as np
    import torch

    import oracle
    from paper_2506_01979_b200 import synth

    nthreads = os.cpu_count() or 1
    B = inp["PL"].shape[0]
    gamma_all = (buf.c_gamma.view(-1) if adaptive else inp["gamma"]).cpu().numpy()

    last = {}

    def run(idx, nth=nthreads):
        it = torch.as_tensor(idx, device=inp["PL"].device)
        sub = synth.to_numpy_inputs({k: (v.index_select(0, it) if torch.is_tensor(v) else v) for k, v in inp.items()})
        t0 = time.time()
        if adaptive:
            c = oracle.confidence(np.ascontiguousarray(sub["QL"][:, :1]), V=sub["V"], nthreads=nth)
            g = c["gamma_next"][:, 0]
        else:
            g = sub["gamma"]
        o = oracle.verify(sub["PL"], sub["QL"], sub["tok"], sub["u"], sub["us"], g, sub["branch_pos"],
                          nthreads=nth, V=sub["V"])
        dt_ = time.time() - t0
        last.update(idx=np.asarray(idx), o=o, gamma=np.asarray(g))
        return dt_, verified_tokens(g.tolist(), sub["branch_pos"].tolist(), cfg.K)

    n = min(B, nthreads)
    dt, tk = run(np.arange(n))
    if dt < budget_s and n < B:
        n2 = int(min(B, max(n, n * budget_s / max(dt, 1e-3))))
        n2 = max(n, (n2 // nthreads) * nthreads)
        if n2 > n:
            dt, tk = run(np.arange(n2))
            n = n2
    parity = parity_stats(last["o"], buf, last["idx"], last["gamma"], gamma_all)
    # the same oracle on one core, over a few sequences (SURVEY §8.4 "a 1-thread run")
    n1 = min(B, 4)
    dt1, tk1 = run(np.arange(n1), nth=1)
    return {"value": round(tk / dt, 1), "unit": "verified draft tokens/s", "cores": nthreads,
            "kind": "oracle", "sample": f"{n} of {B} sequences of {cfg.name.upper()} (first {n}), {dt:.1f} s, "
                                        f"OpenMP over sequences, fp64 plain loops",
            "cpu_model": cpu_model(),
            "single_core_value": round(tk1 / dt1, 1),
            "single_core_sample": f"{n1} sequences on 1 thread, {dt1:.1f} s",
            "parity": parity}


def parity_stats(o, buf, idx, gamma_o, gamma_gpu):
    """The bench's own outputs against the oracle on the cpu_baseline sample (SURVEY §5
    run record): discrete mismatches outside the oracle's near-tie flags, flagged
    sequences, and the largest continuous error in units of the pass band
    |gpu - ref| <= 1e-5 |ref| + 1e-7 (lse: relative to max(1, |lse|))."""
    import numpy as np

    import oracle

    g = {k: getattr(buf, k)[idx].cpu().numpy() for k in ("n_acc", "sel_k", "commit_len", "y_tok", "y_kind",
                                                          "out_tok", "lse_p", "lse_q", "p_tok", "q_tok",
                                                          "top1_q", "entropy_q", "resid_mass")}
    same_gamma = np.asarray(gamma_o) == np.asarray(gamma_gpu)[idx]
    ties = o["ties"]
    dec = (ties & oracle.TIE_ACC_DEC) != 0
    samp = (ties & (oracle.TIE_SAMPLE | oracle.TIE_ILLCOND)) != 0
    ok = same_gamma & ~dec
    mism = np.zeros(len(idx), bool)
    for k in ("n_acc", "out_tok"):
        mism |= (g[k] != o[k]).reshape(len(idx), -1).any(axis=1)
    for k in ("sel_k", "commit_len", "y_kind"):
        mism |= g[k] != o[k]
    mism |= (g["y_tok"] != o["y_tok"]) & ~samp
    band = 0.0
    for k in ("lse_p", "lse_q"):
        r, x = o[k][ok], g[k][ok].astype(np.float64)
        m = ~np.isnan(r) & ~np.isnan(x)
        if m.any():
            band = max(band, float(np.max(np.abs(x[m] - r[m]) / (1e-5 * np.maximum(1.0, np.abs(r[m]))))))
    for k in ("p_tok", "q_tok", "top1_q", "entropy_q", "resid_mass"):
        r, x = o[k][ok], g[k][ok].astype(np.float64)
        m = ~np.isnan(r) & ~np.isnan(x)
        if k == "resid_mass":
            m &= (g["y_kind"][ok] == o["y_kind"][ok]) & ~samp[ok]
        if m.any():
            band = max(band, float(np.max(np.abs(x[m] - r[m]) / (1e-5 * np.abs(r[m]) + 1e-7))))
    return {"sequences": int(ok.sum()), "discrete_mismatch": int((mism & ok).sum()),
            "flagged_ties": int((dec | samp).sum()), "max_continuous_band": round(band, 4),
            "note": "GPU outputs of the timed step vs the oracle on the cpu_baseline sample; band <= 1 passes"}


def run_reference(args, rank, world):
    """--impl reference: the oracle (the only reference this tier has), on host cores."""
    if rank != 0:
        return None
    import numpy as np
    import torch

    import oracle
    from paper_2506_01979_b200 import synth

    cfg = synth.config(args.config)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    nthreads = os.cpu_count() or 1
    per_step = max(nthreads, int(args.ref_seqs))
    adaptive = cfg.layout == "adaptive"
    total_steps = args.warmup + args.steps
    inp = synth.generate(cfg, device=dev, b0=0, b1=per_step * min(total_steps, 2))
    sub_all = synth.to_numpy_inputs(inp)
    times, toks = [], 0
    for k in range(total_steps):
        lo = (k % 2) * per_step
        sub = {kk: (v[lo:lo + per_step] if isinstance(v, np.ndarray) else v) for kk, v in sub_all.items()}
        t0 = time.time()
        if adaptive:
            c = oracle.confidence(np.ascontiguousarray(sub["QL"][:, :1]), V=sub["V"], nthreads=nthreads)
            g = c["gamma_next"][:, 0]
        else:
            g = sub["gamma"]
        oracle.verify(sub["PL"], sub["QL"], sub["tok"], sub["u"], sub["us"], g, sub["branch_pos"],
                      nthreads=nthreads, V=sub["V"])
        dt = time.time() - t0
        if k >= args.warmup:
            times.append(dt)
            toks += verified_tokens(g.tolist(), sub["branch_pos"].tolist(), cfg.K)
    tot = sum(times)
    value = toks / tot
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "verified draft tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot / len(times), 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, DESIGN.md §Input recipe)",
        "config": {"workload": f"{cfg.name.upper()}: {cfg.note}", "V": cfg.V, "K": cfg.K, "G": cfg.G,
                   "per_rank_batch": cfg.B * cfg.rounds, "layout": cfg.layout,
                   "step_sample": f"{per_step} sequences per step"},
        "cpu_baseline": {"value": round(value, 1), "unit": "verified draft tokens/s", "cores": nthreads,
                         "kind": "oracle", "sample": f"{per_step} sequences of {cfg.name.upper()} per step"},
        "e2e": {"value": round(value, 1), "unit": "verified draft tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def emit(line, args):
    """Print the bench line; with --record also append it to a JSONL run record."""
    print(json.dumps(line), flush=True)
    if args.record:
        import socket

        rec = dict(line, recorded_at=time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), host=socket.gethostname(),
                   argv=sys.argv[1:])
        os.makedirs(os.path.dirname(os.path.abspath(args.record)), exist_ok=True)
        with open(args.record, "a") as fh:
            fh.write(json.dumps(rec) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5", "hrad", "spawn", "kv", "tree"])
    ap.add_argument("--hrad-batch", type=int, default=2048)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="issue the C-ABI calls eagerly each step")
    ap.add_argument("--delta", type=float, default=None, help="override the generator's draft noise")
    ap.add_argument("--no-clocks", action="store_true", help="do not run the nvidia-smi sampler")
    ap.add_argument("--mode", default=None, choices=["seq", "vocab"],
                    help="seq: sequences sharded across ranks; vocab: vocabulary sharded (a7). "
                         "Default: vocab for c5, seq otherwise")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-seqs", type=int, default=32)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="sequence-sharded configs: strong = the config's batch split over the ranks "
                         "(SURVEY §8.5, default); weak = a full batch per rank")
    ap.add_argument("--record", default=os.environ.get("SB_RUN_RECORD"),
                    help="append the JSON line (plus time and host) to this JSONL run record (SURVEY §5)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test-only multi-rank runs on one GPU (LOCAL_RANK modulo the device count)")
    args = ap.parse_args()
    if args.mode is None:
        args.mode = "vocab" if args.config == "c5" else "seq"
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl != "reference":
        # launched as `python bench.py --gpus N`: become N ranks (one process per GPU)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl != "reference" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dist_backend == "gloo" and args.impl != "reference":
        import torch

        local_rank %= max(1, torch.cuda.device_count())
    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if line is not None:
            emit(line, args)
        return
    if world > 1:
        import torch

        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:  # test-only: several ranks sharing one GPU (gloo collectives on CPU tensors)
            torch.distributed.init_process_group("gloo")
    runner = {"hrad": run_hrad, "spawn": run_next, "kv": run_next, "tree": run_next}.get(args.config, run_ours)
    line = runner(args, rank, world, local_rank)
    if line is not None:
        emit(line, args)
    if world > 1:
        import torch

        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
