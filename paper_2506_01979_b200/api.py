"""Python binding of the C ABI (include/specbranch.h) — same names, torch tensors in.

Argument marshalling only: tensors are checked for device / dtype / contiguity and
passed as raw device pointers; every step of the verify-and-branch path runs in
libspecbranch.so.  PyTorch provides device memory and streams, nothing else.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib as L
from ._lib import (SB_BF16, SB_CONF_ENTROPY, SB_CONF_TOKEN, SB_CONF_TOP1, SB_F32,  # noqa: F401
                   SB_SELECT_ALG1, SB_SELECT_EQ9)


def dims_for(logits: torch.Tensor, V: int | None = None, K: int | None = None,
             seq_stride: int = 0) -> L.sb_dims:
    """sb_dims of a [B][K][G+1][row_stride] logits tensor (row_stride >= V)."""
    if logits.dim() != 4:
        raise ValueError("logits must be [B][K][G+1][row_stride]")
    B, K0, R1, rs = logits.shape
    if logits.stride(3) != 1 or logits.stride(2) != rs or logits.stride(1) != R1 * rs:
        raise ValueError("logits rows must be contiguous with row_stride = shape[3]")
    dt = {torch.bfloat16: SB_BF16, torch.float32: SB_F32}.get(logits.dtype)
    if dt is None:
        raise TypeError("logits must be bfloat16 or float32")
    V = rs if V is None else V
    K = K0 if K is None else K
    ss = seq_stride or (logits.stride(0) if logits.stride(0) != K * R1 * rs else 0)
    return L.sb_dims(B, K, R1 - 1, V, 0, V, rs, ss, dt, 0)


def _ptr(t: torch.Tensor | None, dtype=None, what=""):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{what}: expected a CUDA tensor")
    if dtype is not None and t.dtype not in (dtype if isinstance(dtype, tuple) else (dtype,)):
        raise TypeError(f"{what}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous() and what not in ("p_logits", "q_logits"):
        raise ValueError(f"{what}: expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def sb_workspace_bytes(d: L.sb_dims) -> int:
    return int(L.lib().sb_workspace_bytes(ctypes.byref(d)))


def make_workspace(d: L.sb_dims, device) -> torch.Tensor:
    """Zero-filled device workspace (the ABI requires zero before first use)."""
    n = sb_workspace_bytes(d)
    if n == 0:
        raise ValueError("invalid sb_dims")
    return torch.zeros(n, dtype=torch.uint8, device=device)


I32, F32 = torch.int32, torch.float32
LOG = (torch.bfloat16, torch.float32)


def sb_verify_branches(d, p_logits, q_logits, tok, u, gamma, branch_pos, lse_p, lse_q, p_tok,
                       q_tok, acc_mask, n_acc, top1_q, top1_id_q, entropy_q, status, workspace,
                       stream=None, comm=None):
    rc = L.lib().sb_verify_branches(
        ctypes.byref(d), _ptr(p_logits, LOG, "p_logits"), _ptr(q_logits, LOG, "q_logits"),
        _ptr(tok, I32, "tok"), _ptr(u, F32, "u"), _ptr(gamma, I32, "gamma"),
        _ptr(branch_pos, I32, "branch_pos"), _ptr(lse_p, F32, "lse_p"), _ptr(lse_q, F32, "lse_q"),
        _ptr(p_tok, F32, "p_tok"), _ptr(q_tok, F32, "q_tok"), _ptr(acc_mask, I32, "acc_mask"),
        _ptr(n_acc, I32, "n_acc"), _ptr(top1_q, F32, "top1_q"), _ptr(top1_id_q, I32, "top1_id_q"),
        _ptr(entropy_q, F32, "entropy_q"), _ptr(status, I32, "status"), comm.handle if comm else None,
        _ptr(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream))
    L.check(rc, "sb_verify_branches")


def sb_verify_branches_reuse(d, p_logits, q_logits, tok, u, gamma, branch_pos, lse_p, lse_q, p_tok,
                             q_tok, acc_mask, n_acc, top1_q, top1_id_q, entropy_q, status, conf_workspace,
                             workspace, stream=None):
    """sb_verify_branches reusing the slot-0 draft-row states of a preceding
    sb_draft_confidence(conf_dims(d), ...) whose workspace is conf_workspace."""
    rc = L.lib().sb_verify_branches_reuse(
        ctypes.byref(d), _ptr(p_logits, LOG, "p_logits"), _ptr(q_logits, LOG, "q_logits"),
        _ptr(tok, I32, "tok"), _ptr(u, F32, "u"), _ptr(gamma, I32, "gamma"),
        _ptr(branch_pos, I32, "branch_pos"), _ptr(lse_p, F32, "lse_p"), _ptr(lse_q, F32, "lse_q"),
        _ptr(p_tok, F32, "p_tok"), _ptr(q_tok, F32, "q_tok"), _ptr(acc_mask, I32, "acc_mask"),
        _ptr(n_acc, I32, "n_acc"), _ptr(top1_q, F32, "top1_q"), _ptr(top1_id_q, I32, "top1_id_q"),
        _ptr(entropy_q, F32, "entropy_q"), _ptr(status, I32, "status"),
        _ptr(conf_workspace, torch.uint8, "conf_workspace"),
        _ptr(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream))
    L.check(rc, "sb_verify_branches_reuse")


def sb_select_branch(d, p_logits, q_logits, tok, u, us, gamma, branch_pos, n_acc, rule, sel_k,
                     commit_len, out_tok, y_tok, y_kind, offsets, packed_tok, path_rolled,
                     branch_discarded, keep_mask, resid_mass, status, workspace, stream=None, comm=None):
    rc = L.lib().sb_select_branch(
        ctypes.byref(d), _ptr(p_logits, LOG, "p_logits"), _ptr(q_logits, LOG, "q_logits"),
        _ptr(tok, I32, "tok"), _ptr(u, F32, "u"), _ptr(us, F32, "us"), _ptr(gamma, I32, "gamma"),
        _ptr(branch_pos, I32, "branch_pos"), _ptr(n_acc, I32, "n_acc"), int(rule),
        _ptr(sel_k, I32, "sel_k"), _ptr(commit_len, I32, "commit_len"), _ptr(out_tok, I32, "out_tok"),
        _ptr(y_tok, I32, "y_tok"), _ptr(y_kind, I32, "y_kind"), _ptr(offsets, I32, "offsets"),
        _ptr(packed_tok, I32, "packed_tok"), _ptr(path_rolled, I32, "path_rolled"),
        _ptr(branch_discarded, I32, "branch_discarded"), _ptr(keep_mask, I32, "keep_mask"),
        _ptr(resid_mass, F32, "resid_mass"), _ptr(status, I32, "status"), comm.handle if comm else None,
        _ptr(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream))
    L.check(rc, "sb_select_branch")


def sb_verify_select(d, p_logits, q_logits, tok, u, us, gamma, branch_pos, rule, buf: "StepBuffers",
                     stream=None):
    """The fused verify + select call (outputs into a StepBuffers)."""
    rc = L.lib().sb_verify_select(
        ctypes.byref(d), _ptr(p_logits, LOG, "p_logits"), _ptr(q_logits, LOG, "q_logits"), _ptr(tok, I32, "tok"),
        _ptr(u, F32, "u"), _ptr(us, F32, "us"), _ptr(gamma, I32, "gamma"), _ptr(branch_pos, I32, "branch_pos"),
        int(rule), _ptr(buf.lse_p, F32, "lse_p"), _ptr(buf.lse_q, F32, "lse_q"), _ptr(buf.p_tok, F32, "p_tok"),
        _ptr(buf.q_tok, F32, "q_tok"), _ptr(buf.acc_mask, I32, "acc_mask"), _ptr(buf.n_acc, I32, "n_acc"),
        _ptr(buf.top1_q, F32, "top1_q"), _ptr(buf.top1_id_q, I32, "top1_id_q"),
        _ptr(buf.entropy_q, F32, "entropy_q"), _ptr(buf.status, I32, "status"), _ptr(buf.sel_k, I32, "sel_k"),
        _ptr(buf.commit_len, I32, "commit_len"), _ptr(buf.out_tok, I32, "out_tok"), _ptr(buf.y_tok, I32, "y_tok"),
        _ptr(buf.y_kind, I32, "y_kind"), _ptr(buf.offsets, I32, "offsets"), _ptr(buf.packed_tok, I32, "packed_tok"),
        _ptr(buf.path_rolled, I32, "path_rolled"), _ptr(buf.branch_discarded, I32, "branch_discarded"),
        _ptr(buf.keep_mask, I32, "keep_mask"), _ptr(buf.resid_mass, F32, "resid_mass"),
        _ptr(buf.workspace, torch.uint8, "workspace"), buf.workspace.numel(), _stream(stream))
    L.check(rc, "sb_verify_select")


def sb_step_adaptive(d, p_logits, q_logits, tok, u, us, branch_pos, rule, eps, k_max, buf: "StepBuffers",
                     stream=None):
    """The adaptive-gamma step ([confidence -> gamma] -> verify -> select) in one C-ABI call;
    confidence outputs into buf.c_* (slot-0 view, K = 1), the rest as sb_verify_select."""
    rc = L.lib().sb_step_adaptive(
        ctypes.byref(d), _ptr(p_logits, LOG, "p_logits"), _ptr(q_logits, LOG, "q_logits"), _ptr(tok, I32, "tok"),
        _ptr(u, F32, "u"), _ptr(us, F32, "us"), _ptr(branch_pos, I32, "branch_pos"), int(rule), float(eps),
        int(k_max), _ptr(buf.c_top1, F32, "c_top1"), _ptr(buf.c_id, I32, "c_id"), _ptr(buf.c_ent, F32, "c_ent"),
        _ptr(buf.c_stat, F32, "c_stat"), _ptr(buf.c_stop, I32, "c_stop"), _ptr(buf.c_knext, I32, "c_knext"),
        _ptr(buf.c_gamma, I32, "c_gamma"), _ptr(buf.lse_p, F32, "lse_p"), _ptr(buf.lse_q, F32, "lse_q"),
        _ptr(buf.p_tok, F32, "p_tok"), _ptr(buf.q_tok, F32, "q_tok"), _ptr(buf.acc_mask, I32, "acc_mask"),
        _ptr(buf.n_acc, I32, "n_acc"), _ptr(buf.top1_q, F32, "top1_q"), _ptr(buf.top1_id_q, I32, "top1_id_q"),
        _ptr(buf.entropy_q, F32, "entropy_q"), _ptr(buf.status, I32, "status"), _ptr(buf.sel_k, I32, "sel_k"),
        _ptr(buf.commit_len, I32, "commit_len"), _ptr(buf.out_tok, I32, "out_tok"), _ptr(buf.y_tok, I32, "y_tok"),
        _ptr(buf.y_kind, I32, "y_kind"), _ptr(buf.offsets, I32, "offsets"), _ptr(buf.packed_tok, I32, "packed_tok"),
        _ptr(buf.path_rolled, I32, "path_rolled"), _ptr(buf.branch_discarded, I32, "branch_discarded"),
        _ptr(buf.keep_mask, I32, "keep_mask"), _ptr(buf.resid_mass, F32, "resid_mass"),
        _ptr(buf.conf_workspace, torch.uint8, "conf_workspace"), buf.conf_workspace.numel(),
        _ptr(buf.workspace, torch.uint8, "workspace"), buf.workspace.numel(), _stream(stream))
    L.check(rc, "sb_step_adaptive")


def sb_draft_confidence(d, q_logits, tok, mode, eps, lam, k_max, top1_prob, top1_id, entropy,
                        tok_prob, stat, stop, k_next, gamma_next, workspace, stream=None):
    rc = L.lib().sb_draft_confidence(
        ctypes.byref(d), _ptr(q_logits, LOG, "q_logits"), _ptr(tok, I32, "tok"), int(mode),
        float(eps), float(lam), int(k_max), _ptr(top1_prob, F32, "top1_prob"),
        _ptr(top1_id, I32, "top1_id"), _ptr(entropy, F32, "entropy"), _ptr(tok_prob, F32, "tok_prob"),
        _ptr(stat, F32, "stat"), _ptr(stop, I32, "stop"), _ptr(k_next, I32, "k_next"),
        _ptr(gamma_next, I32, "gamma_next"), None, _ptr(workspace, torch.uint8, "workspace"),
        workspace.numel(), _stream(stream))
    L.check(rc, "sb_draft_confidence")


def sb_spawn_branches(d, q_logits, branch_pos, tok, mode, k_max, k_out, branch_tok, branch_prob=None,
                      conf=None, stream=None):
    L.check(L.lib().sb_spawn_branches(
        ctypes.byref(d), _ptr(q_logits, LOG, "q_logits"), _ptr(branch_pos, I32, "branch_pos"), _ptr(tok, I32, "tok"),
        int(mode), int(k_max), _ptr(k_out, I32, "k_out"), _ptr(branch_tok, I32, "branch_tok"),
        _ptr(branch_prob, F32, "branch_prob"), _ptr(conf, F32, "conf"), _stream(stream)), "sb_spawn_branches")


def sb_kv_rollback(kv: torch.Tensor, keep_mask, out_kv=None, stream=None):
    """kv: [B][K][G+1][...] device tensor (any dtype); the trailing dims of a position
    must be contiguous, positions may be strided (e.g. a slice of a larger cache).
    keep_mask: int32 [B][K] from sb_select_branch.  out_kv: [B][G+1][...] or None."""
    if kv.dim() < 4:
        raise ValueError("kv must be [B][K][G+1][...]")
    B, K, R1 = kv.shape[:3]
    _ptr(kv[0, 0, 0], None, "kv position")  # device + contiguous trailing dims
    if not kv.is_cuda or kv.stride(1) != R1 * kv.stride(2) or kv.stride(0) != K * kv.stride(1):
        raise ValueError("kv: expected [B][K][G+1] positions at a uniform stride on the device")
    row = kv[0, 0, 0].numel() * kv.element_size()
    stride = kv.stride(2) * kv.element_size()
    if out_kv is not None:
        if tuple(out_kv.shape) != (B, R1) + tuple(kv.shape[3:]) or out_kv.dtype != kv.dtype:
            raise ValueError("out_kv must be [B][G+1][...] of kv's dtype")
        _ptr(out_kv[0, 0], None, "out_kv position")
        if out_kv.stride(1) * out_kv.element_size() != stride or out_kv.stride(0) != R1 * out_kv.stride(1):
            raise ValueError("out_kv: positions must use kv's position stride")
    L.check(L.lib().sb_kv_rollback(
        B, K, R1 - 1, ctypes.c_void_p(kv.data_ptr()), row, stride, _ptr(keep_mask, I32, "keep_mask"),
        None if out_kv is None else ctypes.c_void_p(out_kv.data_ptr()), _stream(stream)), "sb_kv_rollback")


class TreeBuffers:
    """Outputs + workspace of sb_tree_verify for B sequences of N nodes."""

    def __init__(self, d: L.sb_dims, device="cuda"):
        B, N = d.B, d.G
        i32 = dict(dtype=I32, device=device)
        self.acc_mask = torch.zeros(B, dtype=torch.int64, device=device)
        self.keep_mask = torch.zeros(B, dtype=torch.int64, device=device)
        self.stop_node = torch.empty(B, **i32)
        self.commit_len = torch.empty(B, **i32)
        self.out_tok = torch.empty((B, N + 1), **i32)
        self.y_tok = torch.empty(B, **i32)
        self.y_kind = torch.empty(B, **i32)
        self.resid_mass = torch.empty(B, dtype=F32, device=device)
        self.status = torch.empty(B, **i32)
        n = int(L.lib().sb_tree_workspace_bytes(ctypes.byref(d)))
        if n == 0:
            raise ValueError("invalid tree dims")
        self.workspace = torch.empty(n, dtype=torch.uint8, device=device)


def tree_dims(logits: torch.Tensor, V: int | None = None) -> L.sb_dims:
    """sb_dims of [B][N+1][row_stride] context rows (K = 1, G = N)."""
    if logits.dim() != 3:
        raise ValueError("tree logits must be [B][N+1][row_stride]")
    return dims_for(logits.unsqueeze(1), V=V)


def sb_tree_verify(d, p_logits, q_logits, parent, tok, u, us, buf: TreeBuffers, stream=None):
    """Token-tree verify (include/specbranch.h sb_tree_verify)."""
    L.check(L.lib().sb_tree_verify(
        ctypes.byref(d), _ptr(p_logits, LOG, "p_logits"), _ptr(q_logits, LOG, "q_logits"),
        _ptr(parent, I32, "parent"), _ptr(tok, I32, "tok"), _ptr(u, F32, "u"), _ptr(us, F32, "us"),
        _ptr(buf.acc_mask, torch.int64, "acc_mask"), _ptr(buf.keep_mask, torch.int64, "keep_mask"),
        _ptr(buf.stop_node, I32, "stop_node"), _ptr(buf.commit_len, I32, "commit_len"),
        _ptr(buf.out_tok, I32, "out_tok"), _ptr(buf.y_tok, I32, "y_tok"), _ptr(buf.y_kind, I32, "y_kind"),
        _ptr(buf.resid_mass, F32, "resid_mass"), _ptr(buf.status, I32, "status"),
        _ptr(buf.workspace, torch.uint8, "workspace"), buf.workspace.numel(), _stream(stream)), "sb_tree_verify")


# ------------------------------------------------------------------ convenience layer
@dataclass
class StepBuffers:
    """Every output of one verify-and-branch round, preallocated on the device."""
    lse_p: torch.Tensor
    lse_q: torch.Tensor
    p_tok: torch.Tensor
    q_tok: torch.Tensor
    acc_mask: torch.Tensor
    n_acc: torch.Tensor
    top1_q: torch.Tensor
    top1_id_q: torch.Tensor
    entropy_q: torch.Tensor
    status: torch.Tensor
    sel_k: torch.Tensor
    commit_len: torch.Tensor
    out_tok: torch.Tensor
    y_tok: torch.Tensor
    y_kind: torch.Tensor
    offsets: torch.Tensor
    packed_tok: torch.Tensor
    path_rolled: torch.Tensor
    branch_discarded: torch.Tensor
    keep_mask: torch.Tensor
    resid_mass: torch.Tensor
    # draft confidence (slot-0 rows) for the adaptive-gamma configurations
    c_top1: torch.Tensor
    c_id: torch.Tensor
    c_ent: torch.Tensor
    c_stat: torch.Tensor
    c_stop: torch.Tensor
    c_knext: torch.Tensor
    c_gamma: torch.Tensor
    workspace: torch.Tensor
    conf_workspace: torch.Tensor

    @staticmethod
    def alloc(d: L.sb_dims, device) -> "StepBuffers":
        B, K, G = d.B, d.K, d.G
        R1 = G + 1
        e = lambda *s, dt=F32: torch.empty(s, dtype=dt, device=device)  # noqa: E731
        dc = L.sb_dims(B, 1, G, d.V, 0, d.V, d.row_stride,
                       d.seq_stride or K * R1 * d.row_stride, d.dtype, 0)
        return StepBuffers(
            lse_p=e(B, K, R1), lse_q=e(B, K, R1), p_tok=e(B, K, R1), q_tok=e(B, K, R1),
            acc_mask=e(B, K, dt=I32), n_acc=e(B, K, dt=I32), top1_q=e(B, K, R1),
            top1_id_q=e(B, K, R1, dt=I32), entropy_q=e(B, K, R1), status=e(B, dt=I32),
            sel_k=e(B, dt=I32), commit_len=e(B, dt=I32), out_tok=e(B, G + 2, dt=I32),
            y_tok=e(B, dt=I32), y_kind=e(B, dt=I32), offsets=e(B + 1, dt=I32),
            packed_tok=e(B * (G + 2), dt=I32), path_rolled=e(B, dt=I32),
            branch_discarded=e(B, dt=I32), keep_mask=e(B, K, dt=I32), resid_mass=e(B),
            c_top1=e(B, 1, max(G, 1)), c_id=e(B, 1, max(G, 1), dt=I32), c_ent=e(B, 1, max(G, 1)),
            c_stat=e(B, 1, max(G, 1)), c_stop=e(B, 1, dt=I32), c_knext=e(B, 1, dt=I32),
            c_gamma=e(B, 1, dt=I32),
            workspace=make_workspace(d, device), conf_workspace=make_workspace(dc, device))


def conf_dims(d: L.sb_dims) -> L.sb_dims:
    """Slot-0 view of a [B][K][G+1] draft tensor (the drafted path before branching).
    Unsharded dims only (verify_step rejects adaptive gamma on vocabulary shards)."""
    if d.v_total and d.v_total != d.V:
        raise ValueError("conf_dims: vocabulary-shard dims (the confidence pass is unsharded)")
    return L.sb_dims(d.B, 1, d.G, d.V, 0, d.V, d.row_stride,
                     d.seq_stride or d.K * (d.G + 1) * d.row_stride, d.dtype, 0)


def verify_step(d: L.sb_dims, inp: dict, buf: StepBuffers, rule: int = SB_SELECT_EQ9,
                adaptive: bool = False, eps: float = 0.2, k_max: int = 6, stream=None, comm=None,
                views=None, fused: bool = True):
    """One whole hot-path step: [draft confidence -> adaptive gamma] -> verify -> select.

    inp: PL, QL, tok, u, us, gamma, branch_pos device tensors (synth.generate layout).
    With adaptive=True gamma_b = max(1, stop_b) of the slot-0 draft rows (Eq. 6, TOP1)
    replaces inp["gamma"]: with fused=True through sb_step_adaptive
    (one call; one launch for small batches), with fused=False as sb_draft_confidence ->
    sb_verify_branches_reuse (the confidence pass's slot-0 draft-row states) ->
    sb_select_branch.  Otherwise fused=True runs verify + select through sb_verify_select,
    fused=False issues the two calls.
    """
    gamma = inp["gamma"]
    if adaptive and (comm is not None or (d.v_total and d.v_total != d.V)):
        # sb_draft_confidence scores whole draft rows; a vocabulary shard would score its
        # slice only and every rank would take a different gamma
        raise ValueError("adaptive gamma is not supported on vocabulary shards (sb_draft_confidence is unsharded)")
    PL, QL = views if views is not None else (inp["PL"], inp["QL"])
    if adaptive and fused and comm is None:  # the whole adaptive step in one call
        sb_step_adaptive(d, PL, QL, inp["tok"], inp["u"], inp["us"], inp["branch_pos"], rule, eps, k_max, buf,
                         stream)
        return buf.c_gamma.view(-1)
    if adaptive:
        sb_draft_confidence(conf_dims(d), inp["QL"], None, SB_CONF_TOP1, eps, 1.0, k_max,
                            buf.c_top1, buf.c_id, buf.c_ent, None, buf.c_stat, buf.c_stop,
                            buf.c_knext, buf.c_gamma, buf.conf_workspace, stream)
        gamma = buf.c_gamma.view(-1)
    if adaptive and comm is None:  # the confidence pass already streamed slot 0's draft rows
        sb_verify_branches_reuse(d, PL, QL, inp["tok"], inp["u"], gamma, inp["branch_pos"],
                                 buf.lse_p, buf.lse_q, buf.p_tok, buf.q_tok, buf.acc_mask, buf.n_acc,
                                 buf.top1_q, buf.top1_id_q, buf.entropy_q, buf.status, buf.conf_workspace,
                                 buf.workspace, stream)
    elif fused and comm is None:
        sb_verify_select(d, PL, QL, inp["tok"], inp["u"], inp["us"], gamma, inp["branch_pos"], rule, buf, stream)
        return gamma
    else:
        sb_verify_branches(d, PL, QL, inp["tok"], inp["u"], gamma, inp["branch_pos"],
                           buf.lse_p, buf.lse_q, buf.p_tok, buf.q_tok, buf.acc_mask, buf.n_acc,
                           buf.top1_q, buf.top1_id_q, buf.entropy_q, buf.status, buf.workspace, stream, comm)
    sb_select_branch(d, PL, QL, inp["tok"], inp["u"], inp["us"], gamma,
                     inp["branch_pos"], buf.n_acc, rule, buf.sel_k, buf.commit_len, buf.out_tok,
                     buf.y_tok, buf.y_kind, buf.offsets, buf.packed_tok, buf.path_rolled,
                     buf.branch_discarded, buf.keep_mask, buf.resid_mass, buf.status,
                     buf.workspace, stream, comm)
    return gamma


class CallGraph:
    """CUDA graph of a sequence of C-ABI calls (captured once after one warm-up run,
    replayed on the current stream).  Removes per-call host/ctypes overhead; the
    captured tensors are re-read at every replay (update inputs in place)."""

    def __init__(self, fn):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn(side)  # warm-up: one-time function attributes are set outside capture
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=side):
            self.result = fn(side)

    def replay(self):
        self.graph.replay()


class StepGraph(CallGraph):
    """The whole step ([confidence ->] verify -> select) as one CUDA graph."""

    def __init__(self, d: L.sb_dims, inp: dict, buf: StepBuffers, rule: int = SB_SELECT_EQ9,
                 adaptive: bool = False, eps: float = 0.2, k_max: int = 6):
        super().__init__(lambda s: verify_step(d, inp, buf, rule, adaptive, eps, k_max, s))
        self.gamma = self.result


# ------------------------------------------------------------------ vocabulary shards (a7)
def shard_bounds(V_total: int, nranks: int, align: int = 8):
    """Contiguous slices in rank order; every slice starts on a 16-byte boundary."""
    per = -(-V_total // nranks)
    per = -(-per // align) * align
    out, v0 = [], 0
    for _ in range(nranks):
        n = max(0, min(per, V_total - v0))
        out.append((v0, n))
        v0 += n
    return out


def shard_view(logits: torch.Tensor, V_total: int, v0: int, n: int):
    """(sb_dims, view) of columns [v0, v0+n) of a full [B][K][G+1][row_stride] tensor;
    the view shares memory (row_stride of the full tensor, pointer offset v0)."""
    d = dims_for(logits, V=V_total)
    dd = L.sb_dims(d.B, d.K, d.G, n, v0, V_total, d.row_stride, d.seq_stride, d.dtype, 0)
    return dd, logits[..., v0:v0 + n]


def sb_shard_partial_bytes(d) -> int:
    return int(L.lib().sb_shard_partial_bytes(ctypes.byref(d)))


def sb_shard_verify_local(d, p_view, q_view, tok, u, gamma, branch_pos, partial, workspace, stream=None):
    L.check(L.lib().sb_shard_verify_local(
        ctypes.byref(d), _ptr(p_view, LOG, "p_logits"), _ptr(q_view, LOG, "q_logits"), _ptr(tok, I32, "tok"),
        _ptr(u, F32, "u"), _ptr(gamma, I32, "gamma"), _ptr(branch_pos, I32, "branch_pos"),
        _ptr(partial, torch.uint8, "partial"), _ptr(workspace, torch.uint8, "workspace"), workspace.numel(),
        _stream(stream)), "sb_shard_verify_local")


def sb_shard_verify_combine(d, gathered, nranks, tok, u, buf: "StepBuffers", stream=None):
    L.check(L.lib().sb_shard_verify_combine(
        ctypes.byref(d), _ptr(gathered, torch.uint8, "gathered"), int(nranks), _ptr(tok, I32, "tok"),
        _ptr(u, F32, "u"), _ptr(buf.lse_p, F32, "lse_p"), _ptr(buf.lse_q, F32, "lse_q"),
        _ptr(buf.p_tok, F32, "p_tok"), _ptr(buf.q_tok, F32, "q_tok"), _ptr(buf.acc_mask, I32, "acc_mask"),
        _ptr(buf.n_acc, I32, "n_acc"), _ptr(buf.top1_q, F32, "top1_q"), _ptr(buf.top1_id_q, I32, "top1_id_q"),
        _ptr(buf.entropy_q, F32, "entropy_q"), _ptr(buf.status, I32, "status"),
        _ptr(buf.workspace, torch.uint8, "workspace"), buf.workspace.numel(), _stream(stream)),
        "sb_shard_verify_combine")


def sb_shard_select_local(d, p_view, q_view, tok, u, n_acc, rule, mass, workspace, stream=None):
    L.check(L.lib().sb_shard_select_local(
        ctypes.byref(d), _ptr(p_view, LOG, "p_logits"), _ptr(q_view, LOG, "q_logits"), _ptr(tok, I32, "tok"),
        _ptr(u, F32, "u"), _ptr(n_acc, I32, "n_acc"), int(rule), _ptr(mass, torch.float64, "mass"),
        _ptr(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream)), "sb_shard_select_local")


def sb_shard_select_sample(d, gathered_mass, nranks, rank, p_view, q_view, us, ycand, workspace, stream=None):
    L.check(L.lib().sb_shard_select_sample(
        ctypes.byref(d), _ptr(gathered_mass, torch.float64, "gathered_mass"), int(nranks), int(rank),
        _ptr(p_view, LOG, "p_logits"), _ptr(q_view, LOG, "q_logits"), _ptr(us, F32, "us"),
        _ptr(ycand, I32, "ycand"), _ptr(workspace, torch.uint8, "workspace"), workspace.numel(),
        _stream(stream)), "sb_shard_select_sample")


def sb_shard_select_commit(d, y, tok, buf: "StepBuffers", stream=None):
    L.check(L.lib().sb_shard_select_commit(
        ctypes.byref(d), _ptr(y, I32, "y"), _ptr(tok, I32, "tok"), _ptr(buf.sel_k, I32, "sel_k"),
        _ptr(buf.commit_len, I32, "commit_len"), _ptr(buf.out_tok, I32, "out_tok"), _ptr(buf.y_tok, I32, "y_tok"),
        _ptr(buf.y_kind, I32, "y_kind"), _ptr(buf.offsets, I32, "offsets"), _ptr(buf.packed_tok, I32, "packed_tok"),
        _ptr(buf.path_rolled, I32, "path_rolled"), _ptr(buf.branch_discarded, I32, "branch_discarded"),
        _ptr(buf.keep_mask, I32, "keep_mask"), _ptr(buf.resid_mass, F32, "resid_mass"),
        _ptr(buf.status, I32, "status"), _ptr(buf.workspace, torch.uint8, "workspace"), buf.workspace.numel(),
        _stream(stream)), "sb_shard_select_commit")


def sharded_step_loopback(inp: dict, nranks: int, rule: int = SB_SELECT_EQ9):
    """G vocabulary shards emulated in one process on one device: the split-phase C-ABI
    calls of every rank with the three exchanges done as device concatenations / max.
    Returns one StepBuffers per rank (all ranks' outputs must be identical)."""
    PL, QL, V = inp["PL"], inp["QL"], inp["V"]
    ranks = []
    for r, (v0, n) in enumerate(shard_bounds(V, nranks)):
        d, pv = shard_view(PL, V, v0, n)
        _, qv = shard_view(QL, V, v0, n)
        buf = StepBuffers.alloc(d, PL.device)
        part = torch.empty(sb_shard_partial_bytes(d), dtype=torch.uint8, device=PL.device)
        ranks.append((d, pv, qv, buf, part))
    for d, pv, qv, buf, part in ranks:
        sb_shard_verify_local(d, pv, qv, inp["tok"], inp["u"], inp["gamma"], inp["branch_pos"], part, buf.workspace)
    gathered = torch.cat([r[4] for r in ranks])  # exchange 1 (all-gather)
    for d, pv, qv, buf, part in ranks:
        sb_shard_verify_combine(d, gathered, nranks, inp["tok"], inp["u"], buf)
    masses = []
    for d, pv, qv, buf, part in ranks:
        m = torch.empty((d.B, 2), dtype=torch.float64, device=PL.device)
        sb_shard_select_local(d, pv, qv, inp["tok"], inp["u"], buf.n_acc, rule, m, buf.workspace)
        masses.append(m)
    gmass = torch.cat(masses)  # exchange 2 (all-gather)
    cands = []
    for r, (d, pv, qv, buf, part) in enumerate(ranks):
        yc = torch.empty(d.B, dtype=torch.int32, device=PL.device)
        sb_shard_select_sample(d, gmass, nranks, r, pv, qv, inp["us"], yc, buf.workspace)
        cands.append(yc)
    y = torch.stack(cands).max(dim=0).values.contiguous()  # exchange 3 (all-reduce max)
    for d, pv, qv, buf, part in ranks:
        sb_shard_select_commit(d, y, inp["tok"], buf)
    return [r[3] for r in ranks]


class Comm:
    """NCCL communicator of the vocabulary-shard ranks (sb_comm_*).  The unique id is
    created on rank 0 and broadcast with torch.distributed (plumbing)."""

    def __init__(self, nranks: int, rank: int, max_dims: L.sb_dims, unique_id: bytes | None = None):
        n = int(L.lib().sb_comm_unique_id_bytes())
        if unique_id is None:
            buf = ctypes.create_string_buffer(n)
            L.check(L.lib().sb_comm_unique_id(buf), "sb_comm_unique_id")
            unique_id = buf.raw
        self.unique_id = unique_id
        self.handle = ctypes.c_void_p()
        L.check(L.lib().sb_comm_create(ctypes.create_string_buffer(unique_id, n), int(nranks), int(rank),
                                       ctypes.byref(max_dims), ctypes.byref(self.handle)), "sb_comm_create")

    def check(self):
        """Raise if NCCL has recorded an asynchronous error on this communicator."""
        L.check(L.lib().sb_comm_check(self.handle), "sb_comm_check")

    def abort(self):
        """Release a failed communicator without waiting for its pending collectives."""
        if self.handle:
            L.check(L.lib().sb_comm_abort(self.handle), "sb_comm_abort")
            self.handle = ctypes.c_void_p()

    def close(self):
        if self.handle:
            L.check(L.lib().sb_comm_destroy(self.handle), "sb_comm_destroy")
            self.handle = ctypes.c_void_p()


def sb_hrad_predict(z: torch.Tensor, w1: torch.Tensor, b1, w2, b2, w3, b3, G: int, stop=None,
                    logits=None, s_t=None, gamma=None, branch_pos=None, workspace=None, stream=None):
    """H-RAD MLP inference (include/specbranch.h sb_hrad_predict).  z [B][Dz] and
    w1 [256][Dz] bf16; b1, w2, b2, w3, b3 fp32; stop int32 [B] or None.  Returns
    (s_t, logits, gamma, branch_pos), allocating any output not given."""
    B, Dz = z.shape
    dev = z.device
    s_t = torch.empty(B, dtype=I32, device=dev) if s_t is None else s_t
    logits = torch.empty((B, 3), dtype=F32, device=dev) if logits is None else logits
    gamma = torch.empty(B, dtype=I32, device=dev) if gamma is None else gamma
    branch_pos = torch.empty(B, dtype=I32, device=dev) if branch_pos is None else branch_pos
    BF = torch.bfloat16
    nws = int(L.lib().sb_hrad_workspace_bytes(B, Dz))
    if workspace is None or workspace.numel() < nws:
        workspace = torch.empty(max(nws, 16), dtype=torch.uint8, device=dev)
    L.check(L.lib().sb_hrad_predict(
        B, Dz, int(G), _ptr(z, BF, "z"), _ptr(w1, BF, "w1"), _ptr(b1, F32, "b1"), _ptr(w2, F32, "w2"),
        _ptr(b2, F32, "b2"), _ptr(w3, F32, "w3"), _ptr(b3, F32, "b3"), _ptr(stop, I32, "stop"),
        _ptr(logits, F32, "logits"), _ptr(s_t, I32, "s_t"), _ptr(gamma, I32, "gamma"),
        _ptr(branch_pos, I32, "branch_pos"), _ptr(workspace, torch.uint8, "workspace"), ctypes.c_size_t(nws),
        _stream(stream)), "sb_hrad_predict")
    return s_t, logits, gamma, branch_pos
