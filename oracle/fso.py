"""ctypes binding of the C oracle (oracle/fso.c).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module.  The product path never does.
"""
import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libfso.so")

Q, K, V, O, GATE, UP, DOWN, ATTN_NORM, MLP_NORM, BQ, BK, BV = range(12)
EMBED, HEAD, FINAL_NORM = 16, 17, 18


class Cfg(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
                ("vocab", C.c_int32), ("qkv_bias", C.c_int32), ("bf16", C.c_int32),
                ("cache_weights", C.c_int32), ("rms_eps", C.c_double),
                ("rope_theta", C.c_double), ("seed", C.c_uint64)]


def build(force=False):
    src = os.path.join(_HERE, "fso.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC",
                               "-shared", "-o", _SO, src, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        P = C.c_void_p
        i32p = C.POINTER(C.c_int32)
        f32p = C.POINTER(C.c_float)
        L.fso_mix64.restype = C.c_uint64
        L.fso_mix64.argtypes = [C.c_uint64]
        L.fso_gen_value.restype = C.c_float
        L.fso_gen_value.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_int32, C.c_int32]
        L.fso_round_bf16.restype = C.c_float
        L.fso_round_bf16.argtypes = [C.c_float]
        L.fso_model_create.restype = P
        L.fso_model_create.argtypes = [C.POINTER(Cfg)]
        L.fso_model_free.argtypes = [P]
        L.fso_model_materialise.argtypes = [P]
        L.fso_tensor_numel.restype = C.c_int64
        L.fso_tensor_numel.argtypes = [P, C.c_int32]
        L.fso_gen_tensor.argtypes = [P, C.c_int32, C.c_int32, f32p]
        L.fso_kv_create.restype = P
        L.fso_kv_create.argtypes = [P, C.c_int32]
        L.fso_kv_free.argtypes = [P]
        L.fso_kv_get.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, f32p]
        L.fso_kv_move.argtypes = [P, C.c_int32, C.c_int32, i32p, i32p, C.c_int32]
        L.fso_kv_synth.argtypes = [P, C.c_int32, C.c_uint64]
        L.fso_forward.argtypes = [P, P, C.c_int32, C.c_int32, C.c_int32, i32p, i32p, i32p,
                                  i32p, i32p, f32p, f32p, f32p]
        L.fso_set_mutant.argtypes = [C.c_int32]
        _lib = L
    return _lib


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(C.POINTER(C.c_int32))


def _f32(a):
    if a is None:
        return None, None
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(C.POINTER(C.c_float))


class Model:
    """Synthetic random-init decoder (weights from the counter generator)."""

    def __init__(self, shape, seed, cache_weights=False):
        self.shape = shape
        self.seed = seed
        c = Cfg(shape.n_layers, shape.d_model, shape.n_heads, shape.n_kv_heads,
                shape.head_dim, shape.ffn, shape.vocab, shape.qkv_bias, shape.bf16,
                int(cache_weights), shape.rms_eps, shape.rope_theta, seed)
        self._cfg = c
        self.h = lib().fso_model_create(C.byref(c))
        if not self.h:
            raise ValueError("fso_model_create: bad shape")
        if cache_weights:
            lib().fso_model_materialise(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.fso_model_free(self.h)
            self.h = None

    def tensor(self, which, layer=0):
        s = self.shape
        rows = {Q: s.n_heads * s.head_dim, K: s.n_kv_heads * s.head_dim,
                V: s.n_kv_heads * s.head_dim, O: s.d_model, GATE: s.ffn, UP: s.ffn,
                DOWN: s.d_model, EMBED: s.vocab, HEAD: s.vocab}.get(which, 1)
        n = lib().fso_tensor_numel(self.h, which)
        out = np.empty(n, np.float32)
        rc = lib().fso_gen_tensor(self.h, layer, which, out.ctypes.data_as(C.POINTER(C.c_float)))
        if rc:
            raise ValueError("fso_gen_tensor failed")
        return out.reshape(rows, n // rows) if rows > 1 else out


class KV:
    def __init__(self, model, max_slots):
        self.model = model
        self.max_slots = max_slots
        self.h = lib().fso_kv_create(model.h, max_slots)
        if not self.h:
            raise MemoryError("fso_kv_create")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.fso_kv_free(self.h)
            self.h = None

    def get(self, layer, which, kvh, slot):
        out = np.empty(self.model.shape.head_dim, np.float32)
        rc = lib().fso_kv_get(self.h, layer, which, kvh, slot, out.ctypes.data_as(C.POINTER(C.c_float)))
        if rc:
            raise IndexError("fso_kv_get")
        return out

    def move(self, layer_begin, layer_end, frm, to):
        if len(frm) == 0:
            return
        a, pa = _i32(frm)
        b, pb = _i32(to)
        if lib().fso_kv_move(self.h, layer_begin, layer_end, pa, pb, len(a)):
            raise IndexError("fso_kv_move")

    def synth(self, n, kv_seed):
        if lib().fso_kv_synth(self.h, n, kv_seed):
            raise IndexError("fso_kv_synth")


def forward(model, kv, layer_begin, layer_end, tokens, pos, slot, vis, h_in=None,
            want_hidden=False, want_logits=True):
    """Decoder forward of len(pos) rows; vis[m] = list of visible KV slots."""
    s = model.shape
    n = len(pos)
    toks, ptok = _i32(tokens if tokens is not None else np.zeros(n, np.int32))
    posa, ppos = _i32(pos)
    slota, pslot = _i32(slot)
    off = np.zeros(n + 1, np.int32)
    for m in range(n):
        off[m + 1] = off[m] + len(vis[m])
    flat = np.concatenate([np.asarray(v, np.int32) for v in vis]) if off[-1] else np.zeros(1, np.int32)
    offa, poff = _i32(off)
    flata, pflat = _i32(flat)
    hin, phin = _f32(h_in)
    hout = np.empty((n, s.d_model), np.float32) if want_hidden else None
    logits = np.empty((n, s.vocab), np.float32) if (want_logits and layer_end == s.n_layers) else None
    rc = lib().fso_forward(model.h, kv.h, layer_begin, layer_end, n, ptok, ppos, pslot,
                           poff, pflat, phin,
                           hout.ctypes.data_as(C.POINTER(C.c_float)) if hout is not None else None,
                           logits.ctypes.data_as(C.POINTER(C.c_float)) if logits is not None else None)
    if rc:
        raise ValueError("fso_forward: bad arguments")
    return hout, logits
