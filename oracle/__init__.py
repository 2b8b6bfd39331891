"""ctypes wrapper of the fp64 CPU oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of bench.py.  The product package
(paper_2506_01979_b200) never imports this module.

Inputs are numpy arrays holding the exact bytes the GPU path consumes:
logits as uint16 (raw bf16) or float32, shaped [B][K][G+1][V] (or with a larger row
stride), tokens int32 [B][K][G+1], uniforms float32.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

OR_BF16, OR_F32 = 0, 1
ST_GAMMA_CLAMPED, ST_BRANCH_CLAMPED, ST_BAD_TOKEN, ST_NONFINITE, ST_ZERO_RESID, ST_BAD_PARENT = 1, 2, 4, 8, 16, 32
ST_RANGE = 64  # row outside the input domain (|row max| >= 2^24), oracle.h
TIE_ACC_MASK, TIE_ACC_DEC, TIE_SAMPLE, TIE_ILLCOND, TIE_CONF, TIE_EQ7 = 1, 2, 4, 8, 16, 32
CONF_TOP1, CONF_TOKEN, CONF_ENTROPY = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, OpenMP across sequences only)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wall", "-o", _SO, _SRC, "-lm"]
        )
    return _SO


class _Dims(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int32), ("K", ctypes.c_int32), ("G", ctypes.c_int32), ("V", ctypes.c_int32),
        ("row_stride", ctypes.c_int64), ("seq_stride", ctypes.c_int64),
        ("dtype", ctypes.c_int32), ("pad_", ctypes.c_int32),
    ]


_P = ctypes.c_void_p
_VERIFY_FIELDS = [
    ("lse_p", np.float64, "row"), ("lse_q", np.float64, "row"),
    ("top1_q", np.float64, "row"), ("entropy_q", np.float64, "row"),
    ("top1_id_q", np.int32, "row"),
    ("p_tok", np.float64, "row"), ("q_tok", np.float64, "row"),
    ("acc_mask", np.uint32, "bk"), ("n_acc", np.int32, "bk"),
    ("sel_k", np.int32, "b"), ("commit_len", np.int32, "b"),
    ("out_tok", np.int32, "out"),
    ("y_tok", np.int32, "b"), ("y_kind", np.int32, "b"),
    ("offsets", np.int32, "b1"), ("packed_tok", np.int32, "packed"),
    ("path_rolled", np.int32, "b"), ("branch_discarded", np.int32, "b"),
    ("keep_mask", np.uint32, "bk"), ("resid_mass", np.float64, "b"),
    ("status", np.int32, "b"), ("ties", np.uint32, "b"),
    ("margin_acc", np.float64, "b"), ("margin_sample", np.float64, "b"),
]
_CONF_FIELDS = [
    ("top1_prob", np.float64, "row"), ("top1_id", np.int32, "row"),
    ("entropy", np.float64, "row"), ("tok_prob", np.float64, "row"),
    ("stat", np.float64, "row"), ("stop", np.int32, "bk"), ("k_next", np.int32, "bk"),
    ("gamma_next", np.int32, "bk"), ("ties", np.uint32, "bk"),
]


_SPAWN_FIELDS = [("k", np.int32, "b"), ("btok", np.int32, "bkm"), ("bprob", np.float64, "bkm"),
                 ("conf", np.float64, "b"), ("ties", np.uint32, "b")]


_TREE_FIELDS = [("acc_mask", np.uint64, "b"), ("keep_mask", np.uint64, "b"), ("stop_node", np.int32, "b"),
                ("commit_len", np.int32, "b"), ("out_tok", np.int32, "bn1"), ("y_tok", np.int32, "b"),
                ("y_kind", np.int32, "b"), ("resid_mass", np.float64, "b"), ("status", np.int32, "b"),
                ("ties", np.uint32, "b")]


class _TreeOut(ctypes.Structure):
    _fields_ = [(n, _P) for n, _, _ in _TREE_FIELDS]


class _SpawnOut(ctypes.Structure):
    _fields_ = [(n, _P) for n, _, _ in _SPAWN_FIELDS]


class _VerifyOut(ctypes.Structure):
    _fields_ = [(n, _P) for n, _, _ in _VERIFY_FIELDS]


class _ConfOut(ctypes.Structure):
    _fields_ = [(n, _P) for n, _, _ in _CONF_FIELDS]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_verify.restype = ctypes.c_int
        _lib.oracle_verify_f64u.restype = ctypes.c_int
        _lib.oracle_confidence.restype = ctypes.c_int
        _lib.oracle_row_softmax.restype = ctypes.c_double
        _lib.oracle_row_domain.restype = ctypes.c_uint32
        _lib.oracle_adaptive_k.restype = ctypes.c_int
        _lib.oracle_adaptive_k.argtypes = [ctypes.c_double, ctypes.c_int]
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _dims(L: np.ndarray, B, K, G, V):
    if L.dtype == np.uint16:
        dt = OR_BF16
    elif L.dtype == np.float32:
        dt = OR_F32
    else:
        raise TypeError("logits must be uint16 (raw bf16) or float32")
    assert L.flags.c_contiguous and L.shape[:3] == (B, K, G + 1)
    return _Dims(B, K, G, V, L.shape[3], 0, dt, 0)


def _shape(kind, B, K, G, rowlen):
    return {"row": (B, K, rowlen), "bk": (B, K), "b": (B,), "b1": (B + 1,),
            "out": (B, G + 2), "packed": (B * (G + 2),)}[kind]


def verify(PL, QL, tok, u, us, gamma=None, branch_pos=None, rule=0, nthreads=0, V=None,
           f64_uniforms=False):
    """One verify-and-branch round on the oracle.  Returns a dict of numpy arrays."""
    B, K, R1, stride = PL.shape
    G = R1 - 1
    V = stride if V is None else V
    d = _dims(PL, B, K, G, V)
    d.row_stride = stride
    assert QL.shape == PL.shape and QL.dtype == PL.dtype
    tok = np.ascontiguousarray(tok, dtype=np.int32)
    out = {n: np.empty(_shape(kind, B, K, G, R1), dtype=dt) for n, dt, kind in _VERIFY_FIELDS}
    o = _VerifyOut(*[_ptr(out[n]) for n, _, _ in _VERIFY_FIELDS])
    g = None if gamma is None else np.ascontiguousarray(gamma, dtype=np.int32)
    s = None if branch_pos is None else np.ascontiguousarray(branch_pos, dtype=np.int32)
    if f64_uniforms:
        uu = np.ascontiguousarray(u, dtype=np.float64)
        uss = np.ascontiguousarray(us, dtype=np.float64)
        fn = lib().oracle_verify_f64u
    else:
        uu = np.ascontiguousarray(u, dtype=np.float32)
        uss = np.ascontiguousarray(us, dtype=np.float32)
        fn = lib().oracle_verify
    rc = fn(ctypes.byref(d), _ptr(PL), _ptr(QL), _ptr(tok), _ptr(uu), _ptr(uss), _ptr(g), _ptr(s),
            ctypes.c_int(rule), ctypes.c_int(nthreads), ctypes.byref(o))
    if rc != 0:
        raise ValueError("oracle_verify rejected its arguments")
    out["packed_tok"] = out["packed_tok"][: out["offsets"][-1]]
    return out


def confidence(QL, tok=None, mode=CONF_TOP1, eps=0.2, lam=1.0, k_max=6, nthreads=0, V=None):
    """Draft confidence over rows 0..G-1 of every (b,k) group (SURVEY §8.0 Confidence)."""
    B, K, R1, stride = QL.shape
    G = R1 - 1
    V = stride if V is None else V
    d = _dims(QL, B, K, G, V)
    d.row_stride = stride
    out = {n: np.empty(_shape(kind, B, K, G, G), dtype=dt) for n, dt, kind in _CONF_FIELDS}
    o = _ConfOut(*[_ptr(out[n]) for n, _, _ in _CONF_FIELDS])
    t = None if tok is None else np.ascontiguousarray(tok, dtype=np.int32)
    rc = lib().oracle_confidence(ctypes.byref(d), _ptr(QL), _ptr(t), ctypes.c_int(mode),
                                 ctypes.c_double(eps), ctypes.c_double(lam), ctypes.c_int(k_max),
                                 ctypes.c_int(nthreads), ctypes.byref(o))
    if rc != 0:
        raise ValueError("oracle_confidence rejected its arguments")
    return out


def row_softmax(L, b, slot, i, V=None):
    """fp64 softmax of one physical row: (P[V], lse)."""
    B, K, R1, stride = L.shape
    V = stride if V is None else V
    d = _dims(L, B, K, R1 - 1, V)
    d.row_stride = stride
    P = np.empty(V, dtype=np.float64)
    lse = lib().oracle_row_softmax(ctypes.byref(d), _ptr(L), b, slot, i, _ptr(P))
    return P, lse


def row_domain(L, b, slot, i, V=None):
    """Input-domain validation of one physical row: 0, ST_NONFINITE or ST_RANGE."""
    B, K, R1, stride = L.shape
    V = stride if V is None else V
    d = _dims(L, B, K, R1 - 1, V)
    d.row_stride = stride
    return int(lib().oracle_row_domain(ctypes.byref(d), _ptr(L), b, slot, i))


def adaptive_k(c: float, k_max: int) -> int:
    return lib().oracle_adaptive_k(c, k_max)


def spawn(QL, branch_pos=None, tok=None, mode=CONF_TOP1, k_max=6, nthreads=0, V=None):
    """Eq. 7 branch spawn at each sequence's branch row (slot 0): k_b and TopK tokens."""
    B, K, R1, stride = QL.shape
    V = stride if V is None else V
    d = _dims(QL, B, K, R1 - 1, V)
    d.row_stride = stride
    shapes = {"b": (B,), "bkm": (B, k_max)}
    out = {n: np.empty(shapes[kind], dtype=dt) for n, dt, kind in _SPAWN_FIELDS}
    o = _SpawnOut(*[_ptr(out[n]) for n, _, _ in _SPAWN_FIELDS])
    s = None if branch_pos is None else np.ascontiguousarray(branch_pos, dtype=np.int32)
    t = None if tok is None else np.ascontiguousarray(tok, dtype=np.int32)
    lib().oracle_spawn.restype = ctypes.c_int
    rc = lib().oracle_spawn(ctypes.byref(d), _ptr(QL), _ptr(s), _ptr(t), ctypes.c_int(mode), ctypes.c_int(k_max),
                            ctypes.c_int(nthreads), ctypes.byref(o))
    if rc != 0:
        raise ValueError("oracle_spawn rejected its arguments")
    return out


def tree_verify(PL, QL, parent, tok, u, us, nthreads=0, V=None):
    """Tree-structured verify (oracle.h oracle_tree_verify; R31).
    PL, QL [B][N+1][stride] context rows; parent, tok int32 [B][N]; u f32 [B][N]; us f32 [B]."""
    B, R1, stride = PL.shape
    N = R1 - 1
    V = stride if V is None else V
    d = _dims(PL.reshape(B, 1, R1, stride), B, 1, N, V)
    d.row_stride = stride
    assert QL.shape == PL.shape and QL.dtype == PL.dtype
    shapes = {"b": (B,), "bn1": (B, N + 1)}
    out = {n: np.empty(shapes[kind], dtype=dt) for n, dt, kind in _TREE_FIELDS}
    o = _TreeOut(*[_ptr(out[n]) for n, _, _ in _TREE_FIELDS])
    par = np.ascontiguousarray(parent, dtype=np.int32)
    t = np.ascontiguousarray(tok, dtype=np.int32)
    uu = np.ascontiguousarray(u, dtype=np.float32)
    uss = np.ascontiguousarray(us, dtype=np.float32)
    lib().oracle_tree_verify.restype = ctypes.c_int
    rc = lib().oracle_tree_verify(ctypes.byref(d), _ptr(PL), _ptr(QL), _ptr(par), _ptr(t), _ptr(uu), _ptr(uss),
                                  ctypes.c_int(nthreads), ctypes.byref(o))
    if rc != 0:
        raise ValueError("oracle_tree_verify rejected its arguments")
    return out


def kv_rollback(kv, branch_pos, gamma, sel_k, commit_len, y_kind):
    """Plain gather of the committed draft KV rows: out[b][i] =
    kv[b][ts(k*, i)][i] for i < n_b = commit_len - [y sampled], ts(k, i) = (i < s_b ? 0
    : k), with gamma_b and s_b clamped as the verify contract clamps them (SURVEY §8.0
    Shapes: gamma_b to [0, G], s_b to [0, gamma_b]).  Rows past n_b are zeros."""
    B, K, R1 = kv.shape[:3]
    G = R1 - 1
    out = np.zeros((B, R1) + kv.shape[3:], dtype=kv.dtype)
    for b in range(B):
        n = int(commit_len[b]) - (1 if y_kind[b] != 0 else 0)
        ks = int(sel_k[b])
        g = G if gamma is None else min(max(int(gamma[b]), 0), G)
        s = min(max(int(branch_pos[b]), 0), g)
        for i in range(n):
            slot = 0 if (i < s or ks < 0) else ks
            out[b, i] = kv[b, slot, i]
    return out


def hrad(z, w1, b1, w2, b2, w3, b3, stop=None, G=0, nthreads=0):
    """H-RAD MLP + H_t mapping (oracle.h oracle_hrad; reading 35).
    z [B][Dz], w1 [256][Dz] as uint16 (raw bf16); the rest float32."""
    z = np.ascontiguousarray(z, dtype=np.uint16)
    w1 = np.ascontiguousarray(w1, dtype=np.uint16)
    B, Dz = z.shape
    assert w1.shape == (256, Dz)
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    b1, w2, b2, w3, b3 = f32(b1), f32(w2), f32(b2), f32(w3), f32(b3)
    assert b1.shape == (256,) and w2.shape == (64, 256) and b2.shape == (64,)
    assert w3.shape == (3, 64) and b3.shape == (3,)
    st = None if stop is None else np.ascontiguousarray(stop, dtype=np.int32)
    o = {"h1": np.empty((B, 256)), "logits": np.empty((B, 3)), "s_t": np.empty(B, np.int32),
         "gamma": np.empty(B, np.int32), "branch_pos": np.empty(B, np.int32), "margin": np.empty(B)}
    f = lib().oracle_hrad
    f.restype = ctypes.c_int
    rc = f(ctypes.c_int(B), ctypes.c_int(Dz), _ptr(z), _ptr(w1), _ptr(b1), _ptr(w2), _ptr(b2), _ptr(w3),
           _ptr(b3), _ptr(st), ctypes.c_int(G), ctypes.c_int(nthreads), _ptr(o["h1"]), _ptr(o["logits"]),
           _ptr(o["s_t"]), _ptr(o["gamma"]), _ptr(o["branch_pos"]), _ptr(o["margin"]))
    if rc != 0:
        raise ValueError("oracle_hrad rejected its arguments")
    return o
