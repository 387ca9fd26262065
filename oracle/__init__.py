"""CPU oracle for the SubGCache hot path -- TEST INFRASTRUCTURE, never the product.

Two checkers live here:

* ``liboracle.so`` -- the plain-C restatement in ``sgc_oracle.c`` (every function
  cites the reference file:line it restates), loaded with ctypes;
* ``ref_driver`` -- our driver over the unmodified reference library compiled from
  ``/root/reference/proj/src`` into ``oracle/_ref`` (see ``oracle/Makefile``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference arm may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
LIB_PATH = os.path.join(REF_DIR, "liboracle.so")
DRIVER_PATH = os.path.join(REF_DIR, "ref_driver")
REFERENCE_SRC = "/root/reference/proj"

LINKAGES = {"ward": 0, "single": 1, "average": 2, "complete": 3, "centroid": 4}
VOCAB = 260


def build(ref: bool | None = None) -> None:
    """Compile the restatement (always) and the reference (when its sources exist)."""
    targets = ["restatement"]
    if ref is None:
        ref = os.path.isdir(REFERENCE_SRC)
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build(ref=False)
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        f32p, f64p, u32p, i32p = P(C.c_float), P(C.c_double), P(C.c_uint32), P(C.c_int32)
        L.sgo_splitmix64_once.restype = C.c_uint64
        L.sgo_splitmix64_once.argtypes = [C.c_uint64]
        L.sgo_text_projection.argtypes = [f32p, C.c_uint32, C.c_uint64]
        L.sgo_text_embed.argtypes = [f32p, C.c_uint32, C.c_uint64, C.c_char_p, C.c_size_t, f32p]
        L.sgo_text_hash.restype = C.c_size_t
        L.sgo_text_hash.argtypes = [C.c_char_p, C.c_size_t, C.c_uint64, u32p, P(C.c_int8), C.c_size_t]
        L.sgo_gnn_weights.argtypes = [f32p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64]
        L.sgo_gnn_encode.argtypes = [f32p, C.c_uint32, C.c_uint32, C.c_uint32, f32p, C.c_uint32,
                                     u32p, u32p, f32p, C.c_uint32, f32p]
        L.sgo_pairwise.argtypes = [f32p, C.c_uint32, C.c_uint32, f64p]
        L.sgo_agglomerate.argtypes = [f32p, C.c_uint32, C.c_uint32, C.c_int, C.c_uint32, u32p,
                                      u32p, u32p, f64p, P(C.c_uint64)]
        L.sgo_naive_agglomerate.argtypes = [f32p, C.c_uint32, C.c_uint32, C.c_int, C.c_uint32,
                                            u32p, f64p]
        L.sgo_build_prefix.restype = C.c_long
        L.sgo_build_prefix.argtypes = [P(C.c_char_p), u32p, C.c_uint32, P(C.c_char_p), u32p,
                                       C.c_uint32, C.c_uint32, i32p, u32p, u32p]
        L.sgo_question_tokens.restype = C.c_long
        L.sgo_question_tokens.argtypes = [C.c_char_p, C.c_size_t, C.c_uint32, i32p]
        L.sgo_csv_quote.restype = C.c_size_t
        L.sgo_csv_quote.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p]
        L.sgo_lm_create.restype = C.c_void_p
        L.sgo_lm_create.argtypes = [C.c_uint32] * 5 + [C.c_uint64]
        L.sgo_lm_destroy.argtypes = [C.c_void_p]
        L.sgo_lm_weight.restype = f32p
        L.sgo_lm_weight.argtypes = [C.c_void_p, C.c_int, C.c_uint32, P(C.c_size_t)]
        L.sgo_kv_create.restype = C.c_void_p
        L.sgo_kv_create.argtypes = [C.c_void_p]
        L.sgo_kv_fork.restype = C.c_void_p
        L.sgo_kv_fork.argtypes = [C.c_void_p]
        L.sgo_kv_destroy.argtypes = [C.c_void_p]
        L.sgo_kv_tokens.restype = C.c_uint32
        L.sgo_kv_tokens.argtypes = [C.c_void_p]
        L.sgo_kv_data.restype = f32p
        L.sgo_kv_data.argtypes = [C.c_void_p, C.c_int, C.c_uint32]
        L.sgo_lm_prefill.argtypes = [C.c_void_p, C.c_void_p, i32p, C.c_uint32, f32p, f32p, f32p]
        L.sgo_lm_extend.argtypes = [C.c_void_p, C.c_void_p, i32p, C.c_uint32, f32p, f32p]
        L.sgo_greedy_argmax.restype = C.c_int32
        L.sgo_greedy_argmax.argtypes = [f32p, C.c_uint32, C.c_int32, C.c_float]
        L.sgo_hint_found.argtypes = [i32p, C.c_uint32, C.c_uint32, i32p, C.c_uint32]
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def splitmix64_once(x: int) -> int:
    return lib().sgo_splitmix64_once(x & (2**64 - 1))


# ----------------------------------------------------------------- encoders

def text_projection(dim: int, seed: int = 1) -> np.ndarray:
    out = np.empty(dim * 4096, np.float32)
    lib().sgo_text_projection(_p(out, C.c_float), dim, seed)
    return out


def text_hash(text: bytes, salt: int = 55):
    cap = len(text) + 1
    b = np.zeros(cap, np.uint32)
    s = np.zeros(cap, np.int8)
    n = lib().sgo_text_hash(text, len(text), salt, _p(b, C.c_uint32), _p(s, C.c_int8), cap)
    return b[:n].copy(), s[:n].copy()


def text_embed(proj: np.ndarray, dim: int, text: bytes, salt: int = 55) -> np.ndarray:
    out = np.zeros(dim, np.float32)
    lib().sgo_text_embed(_p(proj, C.c_float), dim, salt, text, len(text), _p(out, C.c_float))
    return out


def gnn_weights(layers: int, heads: int, dim: int, seed: int) -> np.ndarray:
    w = np.empty(layers * heads * dim * dim, np.float32)
    lib().sgo_gnn_weights(_p(w, C.c_float), layers, heads, dim, seed)
    return w


def gnn_encode(w, layers, heads, dim, node_feat, msg_src, msg_dst, msg_gate) -> np.ndarray:
    node_feat = np.ascontiguousarray(node_feat, np.float32)
    msg_src = np.ascontiguousarray(msg_src, np.uint32)
    msg_dst = np.ascontiguousarray(msg_dst, np.uint32)
    msg_gate = np.ascontiguousarray(msg_gate, np.float32).reshape(-1)
    out = np.zeros(dim, np.float32)
    rc = lib().sgo_gnn_encode(_p(w, C.c_float), layers, heads, dim, _p(node_feat, C.c_float),
                              node_feat.shape[0], _p(msg_src, C.c_uint32), _p(msg_dst, C.c_uint32),
                              _p(msg_gate, C.c_float), len(msg_src), _p(out, C.c_float))
    if rc:
        raise ValueError("DomainError: empty subgraph")
    return out


# --------------------------------------------------------------- clustering

def pairwise(emb: np.ndarray) -> np.ndarray:
    emb = np.ascontiguousarray(emb, np.float32)
    m, d = emb.shape
    out = np.empty((m, m), np.float64)
    lib().sgo_pairwise(_p(emb, C.c_float), m, d, _p(out, C.c_double))
    return out


def agglomerate(emb: np.ndarray, linkage: str, c: int):
    emb = np.ascontiguousarray(emb, np.float32)
    m, d = emb.shape
    labels = np.zeros(m, np.uint32)
    nm = max(m - c, 1)
    left = np.zeros(nm, np.uint32)
    right = np.zeros(nm, np.uint32)
    dist = np.zeros(nm, np.float64)
    ops = C.c_uint64(0)
    rc = lib().sgo_agglomerate(_p(emb, C.c_float), m, d, LINKAGES[linkage], c,
                               _p(labels, C.c_uint32), _p(left, C.c_uint32), _p(right, C.c_uint32),
                               _p(dist, C.c_double), C.byref(ops))
    if rc:
        raise ValueError("DomainError: bad cluster count")
    k = m - c
    return labels, left[:k], right[:k], dist[:k], ops.value


def naive_agglomerate(emb: np.ndarray, linkage: str, c: int):
    emb = np.ascontiguousarray(emb, np.float32)
    m, d = emb.shape
    labels = np.zeros(m, np.uint32)
    dist = np.zeros(max(m - c, 1), np.float64)
    lib().sgo_naive_agglomerate(_p(emb, C.c_float), m, d, LINKAGES[linkage], c,
                                _p(labels, C.c_uint32), _p(dist, C.c_double))
    return labels, dist[: m - c]


# ------------------------------------------------- representative / prompt

def csv_quote(field: bytes) -> bytes:
    n = lib().sgo_csv_quote(field, len(field), None)
    buf = C.create_string_buffer(n)
    lib().sgo_csv_quote(field, len(field), buf)
    return buf.raw[:n]


def build_prefix(node_rows, edge_rows, budget_tokens: int):
    """node_rows/edge_rows: lists of bytes (already selected, ascending)."""
    nn, ne = len(node_rows), len(edge_rows)
    NR = (C.c_char_p * max(nn, 1))(*node_rows)
    ER = (C.c_char_p * max(ne, 1))(*edge_rows)
    nl = np.array([len(r) for r in node_rows] or [0], np.uint32)
    el = np.array([len(r) for r in edge_rows] or [0], np.uint32)
    cap = 86 + int(nl.sum()) + int(el.sum()) + nn + ne + 8
    toks = np.zeros(cap, np.int32)
    dn, de = C.c_uint32(0), C.c_uint32(0)
    n = lib().sgo_build_prefix(NR, _p(nl, C.c_uint32), nn, ER, _p(el, C.c_uint32), ne,
                               budget_tokens, _p(toks, C.c_int32), C.byref(dn), C.byref(de))
    if n < 0:
        raise OverflowError("CapacityError: prompt headers alone exceed the prefix budget")
    return toks[:n].copy(), dn.value, de.value


def question_tokens(q: bytes, question_budget: int = 128) -> np.ndarray:
    toks = np.zeros(question_budget + 32, np.int32)
    n = lib().sgo_question_tokens(q, len(q), question_budget, _p(toks, C.c_int32))
    if n < 0:
        raise ValueError("DomainError: question budget smaller than the template")
    return toks[:n].copy()


# -------------------------------------------------------------------- ToyLm

class ToyLm:
    """Restated ToyLm (lm_core.cpp:122-406) with the scalar kernel order."""

    def __init__(self, layers=4, heads=4, model_dim=64, ffn_hidden=256, max_seq_len=1024, seed=3):
        self.cfg = dict(layers=layers, heads=heads, model_dim=model_dim, ffn_hidden=ffn_hidden,
                        max_seq_len=max_seq_len, seed=seed)
        self._h = lib().sgo_lm_create(layers, heads, model_dim, ffn_hidden, max_seq_len, seed)
        if not self._h:
            raise ValueError("DomainError: bad lm config")

    def __del__(self):
        if getattr(self, "_h", None):
            lib().sgo_lm_destroy(self._h)
            self._h = None

    def weight(self, which: str, layer: int = 0) -> np.ndarray:
        idx = ["tok", "head", "wqkv", "wo", "w1", "w2", "rope_cos", "rope_sin"].index(which)
        n = C.c_size_t(0)
        p = lib().sgo_lm_weight(self._h, idx, layer, C.byref(n))
        return np.ctypeslib.as_array(p, shape=(n.value,)).copy()

    def new_cache(self):
        return KV(self, lib().sgo_kv_create(self._h))

    def prefill(self, tokens, soft=None, collect=False):
        kv = self.new_cache()
        t = np.ascontiguousarray(tokens, np.int32)
        lg = np.zeros(VOCAB, np.float32)
        tot = len(t) + (soft is not None)
        allg = np.zeros((max(tot, 1), VOCAB), np.float32) if collect else None
        s = None if soft is None else np.ascontiguousarray(soft, np.float32)
        rc = lib().sgo_lm_prefill(self._h, kv._h, _p(t, C.c_int32), len(t), _p(s, C.c_float),
                                  _p(lg, C.c_float), _p(allg, C.c_float))
        _raise(rc)
        kv.last_logits = lg
        kv.all_logits = allg
        return kv

    def extend(self, kv, tokens):
        t = np.ascontiguousarray(tokens, np.int32)
        if len(t) == 0:
            return kv.last_logits
        lg = np.zeros(VOCAB, np.float32)
        rc = lib().sgo_lm_extend(self._h, kv._h, _p(t, C.c_int32), len(t), _p(lg, C.c_float), None)
        _raise(rc)
        kv.last_logits = lg
        return lg


def _raise(rc):
    if rc == 2:
        raise OverflowError("CapacityError: sequence length exceeds max_seq_len")
    if rc == 1:
        raise ValueError("DomainError")


class KV:
    def __init__(self, lm, h):
        self.lm, self._h = lm, h
        self.last_logits = None

    def __del__(self):
        if getattr(self, "_h", None):
            lib().sgo_kv_destroy(self._h)
            self._h = None

    def fork(self):
        k = KV(self.lm, lib().sgo_kv_fork(self._h))
        k.last_logits = None if self.last_logits is None else self.last_logits.copy()
        return k

    @property
    def tokens(self):
        return lib().sgo_kv_tokens(self._h)

    def data(self, is_v: bool, layer: int) -> np.ndarray:
        n = self.tokens * self.lm.cfg["model_dim"]
        p = lib().sgo_kv_data(self._h, int(is_v), layer)
        return np.ctypeslib.as_array(p, shape=(n,)).copy()


def greedy_argmax(logits, bias_target=-1, bonus=0.0) -> int:
    lg = np.ascontiguousarray(logits, np.float32)
    return lib().sgo_greedy_argmax(_p(lg, C.c_float), len(lg), bias_target, bonus)


def hint_found(ctx, limit, answer) -> bool:
    c = np.ascontiguousarray(ctx, np.int32)
    a = np.ascontiguousarray(answer, np.int32)
    return bool(lib().sgo_hint_found(_p(c, C.c_int32), len(c), limit, _p(a, C.c_int32), len(a)))


# --------------------------------------------------- the compiled reference

def ref_available() -> bool:
    return os.path.exists(DRIVER_PATH)


def run_ref(spec: dict, timeout: float = 600) -> dict:
    """Run oracle/_ref/ref_driver (the unmodified reference library) on a spec."""
    if not ref_available():
        raise FileNotFoundError("oracle/_ref/ref_driver not built (reference sources absent)")
    with tempfile.TemporaryDirectory() as td:
        sp, op = os.path.join(td, "spec.json"), os.path.join(td, "out.json")
        with open(sp, "w") as f:
            json.dump(spec, f)
        subprocess.run([DRIVER_PATH, sp, op], check=True, timeout=timeout)
        with open(op) as f:
            return json.load(f)
