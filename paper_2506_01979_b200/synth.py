"""Seeded synthetic inputs for the verify-and-branch step (DESIGN.md §"Input recipe").

This module is the ONLY thing shared between the CUDA path and the oracle: it draws
the logits, draft tokens and uniforms both sides consume.  It holds none of the
method's arithmetic (no softmax, no acceptance test, no residual, no statistic): the
logits are built from closed-form parameters and the draft tokens are drawn by
Gumbel-max / TopK over the draft logits, which is how a draft model would have
produced them (P94 "proposes gamma candidate tokens"; Eq. 7 P218 TopK branch tokens).

Shapes follow SURVEY.md §8.0: PL, QL [B][K][G+1][V] (bf16 or fp32), tok int32
[B][K][G+1], u fp32 [B][K][G+1] in [0,1), us fp32 [B] in [0,1), gamma / branch_pos
int32 [B].  Each sequence b is drawn from its own counter-keyed generator
(seed, b), so any contiguous slice of sequences (one rank's shard) is bit-identical
to the same slice of the full batch generated on the same device type.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import torch

SEED_BASE = 2506_01979


@dataclass(frozen=True)
class Config:
    name: str
    V: int
    dtype: str          # "bf16" | "f32"
    B: int
    K: int
    G: int
    layout: str         # "fixed" (gamma=G, s=0) | "adaptive" (s=0, gamma from a6) | "mixed"
    alpha: float        # target mean acceptance sum_v min(p,q) (P133: alpha = E[beta])
    pi_low: float       # probability a row is a low-confidence row (c ~ U[.02,.2])
    delta: float        # draft logit noise scale (calibrated, scripts/calibrate_alpha.py)
    rho_same: float     # probability the draft peak sits on the target peak
    rounds: int = 1     # C1: independent rounds folded into the batch axis
    note: str = ""
    extra: dict = field(default_factory=dict)


# delta from scripts/calibrate_alpha.py (alpha measured with the oracle only, 512 rows):
# c1/c2 alpha 0.617, c3/c5 0.904, c4 0.802 (profiles/r1_calibration.txt).
CONFIGS = {
    "c1": Config("c1", 32000, "f32", 1, 2, 8, "fixed", 0.6, 0.15, 1.34, 0.85, rounds=256,
                 note="Vicuna 68M&13B vocab, batch 1, K=2, gamma=8, fp32, 256 verify rounds"),
    "c2": Config("c2", 32000, "bf16", 64, 4, 8, "adaptive", 0.6, 0.15, 1.34, 0.85,
                 note="V=32000, batch 64, K=4, gamma<=8 adaptive via draft confidence"),
    "c3": Config("c3", 128256, "bf16", 256, 4, 16, "adaptive", 0.9, 0.08, 0.318, 0.97,
                 note="Llama-3 V=128256, batch 256, K=4, gamma<=16 adaptive"),
    "c4": Config("c4", 151936, "bf16", 2048, 4, 8, "fixed", 0.8, 0.08, 0.622, 0.93,
                 note="Qwen V=151936, batch 2048, K=4, gamma=8, sequence-sharded"),
    "c5": Config("c5", 128256, "bf16", 512, 8, 16, "fixed", 0.9, 0.08, 0.318, 0.97,
                 note="Llama-3 V=128256, batch 512, K=8, gamma=16, vocab-sharded"),
}


def config(name: str, **over) -> Config:
    return replace(CONFIGS[name], **over)


def _gen(seed: int, b: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1_000_003 + b * 7_919 + 12_345) % (2**63 - 1))
    return g


def _peak_height(c: torch.Tensor, V: int) -> torch.Tensor:
    """Logit height h that puts mass ~c on one token above V-1 bulk logits 2z, z~N(0,1):
    E[exp(2z)] = e^2, so c = e^h / (e^h + (V-1) e^2).  Closed form, no data touched."""
    return torch.log(c / (1.0 - c)) + math.log(V - 1) + 2.0


def _rows(cfg: Config, g: torch.Generator, shape: tuple, device):
    """Target / draft logit rows of the recipe (DESIGN.md §"Input recipe"), shape + (V,)."""
    V = cfg.V
    f32 = torch.float32
    z = torch.randn(shape + (V,), generator=g, device=device, dtype=f32)
    lp = 2.0 * z
    vstar = torch.randint(0, V, shape, generator=g, device=device)
    low = torch.rand(shape, generator=g, device=device) < cfg.pi_low
    c_low = 0.02 + 0.18 * torch.rand(shape, generator=g, device=device)
    c_high = 0.30 + 0.69 * torch.rand(shape, generator=g, device=device)
    h = _peak_height(torch.where(low, c_low, c_high), V)
    lp.scatter_(-1, vstar.unsqueeze(-1), h.unsqueeze(-1))
    # draft logits: target plus noise; with prob 1 - rho_same the draft peak moves
    z2 = torch.randn(shape + (V,), generator=g, device=device, dtype=f32)
    lq = lp + cfg.delta * z2
    move = torch.rand(shape, generator=g, device=device) >= cfg.rho_same
    vmove = torch.randint(0, V, shape, generator=g, device=device)
    bulk_at_star = 2.0 * z.gather(-1, vstar.unsqueeze(-1)).squeeze(-1)
    noise_star = z2.gather(-1, vstar.unsqueeze(-1)).squeeze(-1)
    noise_move = z2.gather(-1, vmove.unsqueeze(-1)).squeeze(-1)
    # the draft bulk mass grows by E[exp(delta z')] = exp(delta^2/2); lifting the draft
    # peak by delta^2/2 keeps the draft's own top-1 confidence distributed like c
    hq = h + 0.5 * cfg.delta * cfg.delta
    new_star = torch.where(move, bulk_at_star + cfg.delta * noise_star, hq + cfg.delta * noise_star)
    lq.scatter_(-1, vstar.unsqueeze(-1), new_star.unsqueeze(-1))
    cur_move = lq.gather(-1, vmove.unsqueeze(-1)).squeeze(-1)
    lq.scatter_(-1, vmove.unsqueeze(-1), torch.where(move, hq + cfg.delta * noise_move, cur_move).unsqueeze(-1))
    return lp, lq


def draft_rows(cfg: Config, B: int, seed: int = 0, device="cpu", chunk: int = 128):
    """B draft rows of the recipe (the branch rows Eq. 7 spawns from), [B][V] in the
    config's dtype; row b from its own counter-keyed generator."""
    ldt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    out = torch.empty((B, cfg.V), dtype=ldt, device=device)
    for b0 in range(0, B, chunk):
        n = min(chunk, B - b0)
        _, lq = _rows(cfg, _gen(SEED_BASE + 31 * seed, b0, device), (n,), device)
        out[b0:b0 + n] = lq.to(ldt)
    return out


def _one_sequence(cfg: Config, seed: int, b: int, device, gamma_b: int, s_b: int):
    K, G, V = cfg.K, cfg.G, cfg.V
    R1 = G + 1
    g = _gen(seed, b, device)
    f32 = torch.float32
    lp, lq = _rows(cfg, g, (K, R1), device)
    ldt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    PL = lp.to(ldt)
    QL = lq.to(ldt)
    del lp, lq
    # draft tokens: Gumbel-max samples from each draft row (x_i ~ q_i, Alg. 1 P505/P516)
    gum = torch.rand((K, R1, V), generator=g, device=device, dtype=f32).clamp_(min=1e-12)
    gum = -torch.log(-torch.log(gum))
    tok = torch.argmax(QL.float() + gum, dim=2).to(torch.int32)
    del gum
    # branch tokens at row s_b: TopK of the shared draft row (Eq. 7, P218)
    kk = min(K, V)
    top = torch.topk(QL[0, s_b].float(), kk).indices.to(torch.int32)
    tok[:kk, s_b] = top
    u = torch.rand((K, R1), generator=g, device=device, dtype=f32)
    us = torch.rand((1,), generator=g, device=device, dtype=f32)
    return PL, QL, tok, u, us


def layout_for(cfg: Config, b: int, seed: int):
    """(gamma_b, s_b) for the fixed and mixed layouts; adaptive uses gamma from a6, s=0."""
    if cfg.layout == "fixed":
        return cfg.extra.get("gamma", cfg.G), cfg.extra.get("s", 0)
    if cfg.layout == "adaptive":
        return cfg.G, 0
    if cfg.layout == "mixed":
        g = torch.Generator().manual_seed(seed * 31 + b)
        gam = int(torch.randint(0, cfg.G + 1, (1,), generator=g))
        s = int(torch.randint(0, gam + 1, (1,), generator=g))
        return gam, s
    raise ValueError(cfg.layout)


def generate(cfg: Config, device="cpu", seed: int | None = None, b0: int = 0, b1: int | None = None,
             row_pad: int = 0):
    """Draw sequences [b0, b1) of config cfg on `device`.

    Returns dict(PL, QL, tok, u, us, gamma, branch_pos).  For cfg.rounds > 1 the rounds
    are folded into the batch axis (B_total = B * rounds).  row_pad > 0 leaves a gap of
    row_pad elements after every row (row_stride = V + row_pad) to exercise strides.
    """
    seed = SEED_BASE + 1000 * int(cfg.name[1:] if cfg.name[1:].isdigit() else 0) if seed is None else seed
    Btot = cfg.B * cfg.rounds
    b1 = Btot if b1 is None else b1
    n = b1 - b0
    K, R1, V = cfg.K, cfg.G + 1, cfg.V
    ldt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    stride = V + row_pad
    PL = torch.empty((n, K, R1, stride), dtype=ldt, device=device)
    QL = torch.empty((n, K, R1, stride), dtype=ldt, device=device)
    if row_pad:
        PL[..., V:] = float("nan")
        QL[..., V:] = float("nan")
    tok = torch.empty((n, K, R1), dtype=torch.int32, device=device)
    u = torch.empty((n, K, R1), dtype=torch.float32, device=device)
    us = torch.empty((n,), dtype=torch.float32, device=device)
    gamma = torch.empty((n,), dtype=torch.int32)
    bpos = torch.empty((n,), dtype=torch.int32)
    for j, b in enumerate(range(b0, b1)):
        gb, sb = layout_for(cfg, b, seed)
        p, q, t, uu, uss = _one_sequence(cfg, seed, b, device, gb, sb)
        PL[j, :, :, :V] = p
        QL[j, :, :, :V] = q
        tok[j] = t
        u[j] = uu
        us[j] = uss[0]
        gamma[j] = gb
        bpos[j] = sb
    return dict(PL=PL, QL=QL, tok=tok, u=u, us=us, gamma=gamma.to(device), branch_pos=bpos.to(device),
                V=V, row_stride=stride)


def to_numpy_inputs(inp: dict):
    """Host copies with the exact bytes: bf16 logits as raw uint16, everything else as is."""
    out = {}
    for k in ("PL", "QL"):
        t = inp[k].detach().cpu().contiguous()
        out[k] = t.view(torch.int16).numpy().view("uint16") if t.dtype == torch.bfloat16 else t.numpy()
    for k in ("tok", "u", "us", "gamma", "branch_pos"):
        out[k] = inp[k].detach().cpu().contiguous().numpy()
    out["V"] = inp["V"]
    return out


# ---------------------------------------------------------------- token trees (f3)
def tree_parents(shape: str, N: int | None = None, branching=(2, 2, 2, 2), depth: int = 6, b: int = 0,
                 seed: int = 0) -> list[int]:
    """Parent pointers in topological (BFS) order, -1 = the committed context.

    dense:  every node of level l has branching[l] children (SpecInfer-style dense tree,
            Appendix F P1057: (k^gamma - 1)/(k - 1) nodes for a k-ary tree);
    chain:  N nodes in one path (plain speculative decoding, Alg. 1);
    random: N nodes, each attached to a uniformly drawn earlier node (or the root) of
            depth < `depth` (a sparse tree of mixed widths)."""
    if shape == "dense":
        par, level = [], [-1]
        for k in branching:
            nxt = []
            for p in level:
                for _ in range(k):
                    par.append(p)
                    nxt.append(len(par) - 1)
            level = nxt
        return par
    if shape == "chain":
        return list(range(-1, N - 1))
    if shape == "random":
        g = torch.Generator().manual_seed(seed * 7_919 + b * 104_729 + 3)
        par, dep = [], []
        for j in range(N):
            while True:
                p = int(torch.randint(-1, j, (1,), generator=g)) if j > 0 else -1
                d = 0 if p < 0 else dep[p] + 1
                if d < depth:
                    break
            par.append(p)
            dep.append(d)
        # BFS renumbering keeps parent < child and groups siblings
        order = sorted(range(N), key=lambda j: (dep[j], j))
        new = {old: i for i, old in enumerate(order)}
        return [(-1 if par[o] < 0 else new[par[o]]) for o in order]
    raise ValueError(shape)


def generate_tree(cfg: Config, shape: str = "dense", B: int | None = None, N: int | None = None,
                  branching=(2, 2, 2, 2), depth: int = 6, device="cpu", seed: int = 7):
    """Seeded token-tree inputs: rows [B][N+1][V] (row 0 = committed context, row j+1 =
    context after node j), parent / tok int32 [B][N], u f32 [B][N], us f32 [B].
    Children of one context are the TopK of its draft row (distinct tokens, the SpecInfer
    expansion); a lone child is a Gumbel-max sample of the draft row (x ~ q)."""
    B = cfg.B if B is None else B
    ldt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    pars = [tree_parents(shape, N, branching, depth, b, seed) for b in range(B)]
    N = len(pars[0])
    assert all(len(p) == N for p in pars) and 1 <= N <= 63
    V = cfg.V
    PL = torch.empty((B, N + 1, V), dtype=ldt, device=device)
    QL = torch.empty((B, N + 1, V), dtype=ldt, device=device)
    tok = torch.empty((B, N), dtype=torch.int32)
    u = torch.empty((B, N), dtype=torch.float32)
    us = torch.empty((B,), dtype=torch.float32)
    for b in range(B):
        g = _gen(seed + 77, b, device)
        lp, lq = _rows(cfg, g, (N + 1,), device)
        PL[b] = lp.to(ldt)
        QL[b] = lq.to(ldt)
        q = QL[b].float()
        kids: dict[int, list[int]] = {}
        for j, p in enumerate(pars[b]):
            kids.setdefault(p, []).append(j)
        for p, js in kids.items():
            row = q[p + 1]
            if len(js) == 1:
                gum = torch.rand((V,), generator=g, device=device).clamp_(min=1e-12)
                t = [int(torch.argmax(row - torch.log(-torch.log(gum))))]
            else:
                t = torch.topk(row, min(len(js), V)).indices.tolist()
            for j, x in zip(js, t + [t[-1]] * (len(js) - len(t))):
                tok[b, j] = x
        u[b] = torch.rand((N,), generator=g, device=device).cpu()
        us[b] = float(torch.rand((1,), generator=g, device=device))
    parent = torch.tensor(pars, dtype=torch.int32)
    return dict(PL=PL, QL=QL, parent=parent.to(device), tok=tok.to(device), u=u.to(device), us=us.to(device),
                V=V, N=N)


def tree_to_numpy(inp: dict):
    out = {}
    for k in ("PL", "QL"):
        t = inp[k].detach().cpu().contiguous()
        out[k] = t.view(torch.int16).numpy().view("uint16") if t.dtype == torch.bfloat16 else t.numpy()
    for k in ("parent", "tok", "u", "us"):
        out[k] = inp[k].detach().cpu().contiguous().numpy()
    out["V"], out["N"] = inp["V"], inp["N"]
    return out


# ---------------------------------------------------------------- H-RAD (f4)
# Feature width of z_t = Concat(h^1..h^{L_f}, e_t) (Eq. 4, P190): L_f = 4 target layers
# (P400, Table 5) of the target hidden size plus the token embedding.  LLaMA-3.1-8B
# (hidden 4096) -> 5 * 4096 = 20480; Vicuna-13B (hidden 5120) -> 25600.
HRAD_DZ = {"llama31_8b": 5 * 4096, "vicuna_13b": 5 * 5120}


def hrad_inputs(B: int, Dz: int, G: int = 8, seed: int = 0, device="cpu"):
    """Synthetic H-RAD inputs (random-init weights: no trained checkpoint exists here).

    z ~ N(0, 1) rounded to bf16 (hidden-state-like scale); W1 ~ N(0, 2/Dz) bf16 (He
    init for the ReLU layer), b1 ~ N(0, 0.1); W2 ~ N(0, 2/256), b2 ~ N(0, 0.1);
    W3 ~ N(0, 1/64), b3 = 0; stop ~ U{0..G} stands in for a6's confidence stop.
    Holds none of the MLP's arithmetic."""
    g = torch.Generator(device="cpu").manual_seed(SEED_BASE + 7919 * seed + 17)
    z = torch.randn(B, Dz, generator=g).to(torch.bfloat16)
    w1 = (torch.randn(256, Dz, generator=g) * math.sqrt(2.0 / Dz)).to(torch.bfloat16)
    b1 = torch.randn(256, generator=g) * 0.1
    w2 = torch.randn(64, 256, generator=g) * math.sqrt(2.0 / 256)
    b2 = torch.randn(64, generator=g) * 0.1
    w3 = torch.randn(3, 64, generator=g) * math.sqrt(1.0 / 64)
    b3 = torch.zeros(3)
    stop = torch.randint(0, G + 1, (B,), generator=g, dtype=torch.int32)
    out = {"z": z, "w1": w1, "b1": b1, "w2": w2, "b2": b2, "w3": w3, "b3": b3, "stop": stop, "G": G}
    return {k: (v.to(device) if torch.is_tensor(v) else v) for k, v in out.items()}


def hrad_to_numpy(inp: dict):
    """The exact bytes both sides consume: bf16 as raw uint16, the rest float32 / int32."""
    u16 = lambda t: t.detach().cpu().contiguous().view(torch.int16).numpy().view("uint16")  # noqa: E731
    f = lambda t: t.detach().cpu().float().numpy()  # noqa: E731
    return {"z": u16(inp["z"]), "w1": u16(inp["w1"]), "b1": f(inp["b1"]), "w2": f(inp["w2"]),
            "b2": f(inp["b2"]), "w3": f(inp["w3"]), "b3": f(inp["b3"]),
            "stop": inp["stop"].cpu().numpy().astype("int32"), "G": inp["G"]}
