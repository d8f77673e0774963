"""Thin ctypes binding of libflowspec.so (include/flowspec.h).

Argument marshalling only: every step of the path runs in the CUDA kernels
behind the C-ABI.  PyTorch provides the device arena (torch.empty), the CUDA
stream and the process-group bootstrap of the NCCL id.  There is no CPU
fallback: importing this module on a machine without the built library raises.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libflowspec.so")

FS_OK, FS_EINVAL, FS_ENOMEM, FS_ESTATE, FS_ECAPACITY, FS_ECUDA, FS_ENCCL, FS_EPOISONED, FS_ERANGE = \
    0, -1, -2, -3, -4, -5, -6, -7, -8
FS_MAX_LIVE, FS_MAX_SEG, FS_MAX_STAGES = 512, 64, 8
FS_PREFILL, FS_SYNTH_KV = 0, 1
FS_NEW_ROUND, FS_APPEND = 1, 2
FS_ORDER_BFS = 4   # OR into submit flags: breadth-first order (w/o-SBD ablation)
FS_MERGE = 8       # submit kind: merge a tree rooted at the current root (f4 expansion)
FS_SUBMIT_ASYNC = 16   # OR into NEW_ROUND / APPEND: do not wait (errors poison at the next verify)
FS_ACCEPT_GREEDY, FS_ACCEPT_STOCHASTIC = 0, 1
FS_Q_STATE, FS_Q_NODE, FS_Q_TOKEN, FS_Q_PARENT, FS_Q_POS, FS_Q_ANC, FS_Q_CU, FS_Q_RETAIN = range(8)

i32 = C.c_int32


class fs_config(C.Structure):
    _fields_ = [("n_layers", i32), ("d_model", i32), ("n_heads", i32), ("n_kv_heads", i32),
                ("head_dim", i32), ("ffn", i32), ("vocab", i32), ("qkv_bias", i32), ("bf16", i32),
                ("rms_eps", C.c_double), ("rope_theta", C.c_double),
                ("n_stages", i32), ("rank", i32), ("layers_per_stage", C.POINTER(i32)),
                ("max_ctx", i32), ("max_live", i32), ("max_seg", i32), ("device", i32),
                ("arena", C.c_void_p), ("arena_bytes", C.c_size_t), ("stream", C.c_void_p),
                ("nccl_id", C.POINTER(C.c_uint8)), ("local_group", C.c_void_p), ("sampling", i32),
                ("max_prefill", i32)]


class fs_submit_out(C.Structure):
    _fields_ = [("n", i32), ("s_base", i32), ("order", i32 * FS_MAX_LIVE), ("n_segs", i32),
                ("seg_begin", i32 * (FS_MAX_LIVE + 1)), ("seg_id0", i32), ("merged", i32 * FS_MAX_LIVE)]


class fs_step_out(C.Structure):
    _fields_ = [("seg_id", i32), ("s_begin", i32), ("n_rows", i32), ("node", i32 * FS_MAX_SEG),
                ("am", i32 * FS_MAX_SEG), ("margin", C.c_float * FS_MAX_SEG)]


class fs_accept_out(C.Structure):
    _fields_ = [("progress", i32), ("n_acc", i32), ("acc_ids", i32 * FS_MAX_LIVE),
                ("acc_tokens", i32 * FS_MAX_LIVE), ("x_new", i32), ("n_new", i32), ("cont", i32),
                ("n_flagged", i32), ("flagged_ids", i32 * FS_MAX_LIVE)]


class fs_state(C.Structure):
    _fields_ = [("l_glo", i32), ("x_new", i32), ("live", i32), ("n_live", i32), ("next_id", i32),
                ("n_stages", i32), ("rank", i32), ("layer_begin", i32), ("layer_end", i32),
                ("n_cached", i32 * FS_MAX_STAGES), ("layers_per_stage", i32 * FS_MAX_STAGES),
                ("n_queue", i32), ("queue", (i32 * 3) * FS_MAX_LIVE),
                ("inflight", (i32 * 3) * FS_MAX_STAGES), ("launches", C.c_uint64)]


class fs_profile(C.Structure):
    _fields_ = [("gemm_launches", C.c_uint64), ("gemm_ms", C.c_double), ("gemm_bytes", C.c_double),
                ("attn_launches", C.c_uint64), ("attn_ms", C.c_double), ("attn_bytes", C.c_double)]


EXPORTS = ["fs_layers_per_stage", "fs_debug_gemm", "fs_bench_kernel", "fs_set_profiling", "fs_get_profile", "fs_arena_bytes", "fs_nccl_unique_id", "fs_init", "fs_load_random_weights",
           "fs_set_prefix", "fs_submit_segment", "fs_verify_step", "fs_set_logits_buffer",
           "fs_accept", "fs_prune_and_compact", "fs_query", "fs_read_kv", "fs_destroy",
           "fs_last_error", "fs_strerror", "fs_local_group_create", "fs_local_group_destroy", "fs_set_acceptance", "fs_debug_write_kv"]
EXPORTS.sort()

_lib = None


def lib():
    """Load libflowspec.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise ImportError(f"{SO} missing: run `python -m paper_2507_02620_b200.build`")
        L = C.CDLL(SO)
        P = C.c_void_p
        ip = C.POINTER(i32)
        L.fs_arena_bytes.restype = C.c_size_t
        L.fs_arena_bytes.argtypes = [C.POINTER(fs_config)]
        L.fs_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8)]
        L.fs_layers_per_stage.argtypes = [C.POINTER(fs_config), C.POINTER(i32)]
        L.fs_init.argtypes = [C.POINTER(fs_config), C.POINTER(P)]
        L.fs_load_random_weights.argtypes = [P, C.c_uint64]
        L.fs_set_prefix.argtypes = [P, ip, i32, i32, C.c_uint64, ip]
        L.fs_submit_segment.argtypes = [P, i32, ip, ip, C.POINTER(C.c_float), i32, i32, i32,
                                        C.POINTER(fs_submit_out)]
        L.fs_verify_step.argtypes = [P, C.POINTER(fs_step_out)]
        L.fs_set_logits_buffer.argtypes = [P, C.c_void_p, i32]
        L.fs_accept.argtypes = [P, C.POINTER(fs_accept_out)]
        L.fs_prune_and_compact.argtypes = [P, C.POINTER(fs_accept_out)]
        L.fs_query.argtypes = [P, i32, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.fs_read_kv.argtypes = [P, i32, i32, i32, i32, C.POINTER(C.c_float)]
        L.fs_debug_write_kv.argtypes = [P, i32, i32, i32, i32, C.POINTER(C.c_float)]
        L.fs_set_profiling.argtypes = [P, i32]
        L.fs_get_profile.argtypes = [P, C.POINTER(fs_profile)]
        L.fs_bench_kernel.argtypes = [P, i32, i32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.fs_debug_gemm.argtypes = [P, i32, i32, C.POINTER(C.c_float), i32, C.POINTER(C.c_float)]
        L.fs_destroy.argtypes = [P]
        L.fs_local_group_create.argtypes = [i32, C.POINTER(P)]
        L.fs_set_acceptance.argtypes = [P, i32, C.c_float, C.c_uint64, C.c_void_p, i32]
        L.fs_local_group_destroy.argtypes = [P]
        L.fs_last_error.restype = C.c_char_p
        L.fs_last_error.argtypes = [P]
        L.fs_strerror.restype = C.c_char_p
        L.fs_strerror.argtypes = [i32]
        _lib = L
    return _lib


class FlowSpecError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{msg} (code {code})")
        self.code = code


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(C.POINTER(i32))


def make_config(shape, n_stages=1, rank=0, max_ctx=4096, max_live=512, max_seg=16, device=0,
                layers_per_stage=None, sampling=0, max_prefill=0):
    c = fs_config()
    c.sampling = sampling
    c.max_prefill = max_prefill
    for k in ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim", "ffn", "vocab",
              "qkv_bias", "bf16"):
        setattr(c, k, int(getattr(shape, k)))
    c.rms_eps = float(shape.rms_eps)
    c.rope_theta = float(shape.rope_theta)
    c.n_stages, c.rank = n_stages, rank
    c.max_ctx, c.max_live, c.max_seg, c.device = max_ctx, max_live, max_seg, device
    c._lps = None
    if layers_per_stage is not None:
        arr = (i32 * n_stages)(*layers_per_stage)
        c._lps = arr
        c.layers_per_stage = C.cast(arr, C.POINTER(i32))
    return c


class Pipeline:
    """One rank of the pipelined tree verifier (same call names as the C-ABI)."""

    def __init__(self, shape, n_stages=1, rank=0, max_ctx=4096, max_live=512, max_seg=16,
                 device=0, layers_per_stage=None, nccl_id=None, stream=None, local_group=None,
                 sampling=0, max_prefill=0):
        import torch
        self.torch = torch
        self.L = lib()
        self.shape = shape
        self.cfg = make_config(shape, n_stages, rank, max_ctx, max_live, max_seg, device,
                               layers_per_stage, sampling, max_prefill)
        nbytes = self.L.fs_arena_bytes(C.byref(self.cfg))
        if nbytes == 0:
            raise FlowSpecError(FS_EINVAL, "invalid configuration")
        dev = torch.device("cuda", device)
        self.arena = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=dev)
        self.cfg.arena = self.arena.data_ptr()
        self.cfg.arena_bytes = nbytes
        self.cfg.stream = self.stream.cuda_stream
        self._nid = None
        if n_stages > 1 and local_group is not None:
            self.cfg.local_group = local_group
        elif n_stages > 1:
            if nccl_id is None:
                raise ValueError("nccl_id (or local_group) required for n_stages > 1")
            self._nid = (C.c_uint8 * 128)(*bytes(nccl_id))
            self.cfg.nccl_id = C.cast(self._nid, C.POINTER(C.c_uint8))
        h = C.c_void_p()
        self._chk(self.L.fs_init(C.byref(self.cfg), C.byref(h)), "fs_init", ctx=False)
        self.h = h
        self.logits = None

    def _chk(self, rc, what, ctx=True):
        if rc != FS_OK:
            msg = what + ": " + self.L.fs_strerror(rc).decode()
            if ctx and getattr(self, "h", None):
                msg += " — " + self.L.fs_last_error(self.h).decode()
            raise FlowSpecError(rc, msg)

    def close(self):
        if getattr(self, "h", None):
            self.L.fs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- calls
    def fs_load_random_weights(self, seed):
        self._chk(self.L.fs_load_random_weights(self.h, seed), "fs_load_random_weights")

    def fs_set_prefix(self, tokens, mode=FS_PREFILL, kv_seed=0):
        t, pt = _i32(tokens)
        x = i32()
        self._chk(self.L.fs_set_prefix(self.h, pt, len(t), mode, kv_seed, C.byref(x)), "fs_set_prefix")
        return x.value

    def fs_submit_segment(self, flags, parent, token, own, l_max, l_top=0):
        p, pp = _i32(parent)
        t, pt = _i32(token)
        o = np.ascontiguousarray(own, dtype=np.float32)
        out = fs_submit_out()
        self._chk(self.L.fs_submit_segment(self.h, flags, pp, pt, o.ctypes.data_as(C.POINTER(C.c_float)),
                                           len(p), l_top, l_max, C.byref(out)), "fs_submit_segment")
        bounds = [(out.seg_begin[k], out.seg_begin[k + 1]) for k in range(out.n_segs)]
        order = [] if flags & FS_SUBMIT_ASYNC else list(out.order[:out.n])   # async: not read back
        r = dict(order=order, s_base=out.s_base, bounds=bounds, seg_id0=out.seg_id0)
        if (flags & ~(FS_ORDER_BFS | FS_SUBMIT_ASYNC)) == FS_MERGE:
            r["merged"] = list(out.merged[:len(p)])
        return r

    def enable_logits(self, rows_cap=None):
        rows_cap = rows_cap or self.cfg.max_seg
        self.logits = self.torch.zeros((rows_cap, self.shape.vocab), dtype=self.torch.float32,
                                       device=self.arena.device)
        self._chk(self.L.fs_set_logits_buffer(self.h, self.logits.data_ptr(), rows_cap), "logits")

    def fs_set_acceptance(self, mode, temperature=1.0, seed=0, q=None):
        """q: torch float32 CUDA tensor [q_rows, vocab] (row = node id), kept alive here."""
        self._q = q
        ptr = q.data_ptr() if q is not None else None
        rows = q.shape[0] if q is not None else 0
        self._chk(self.L.fs_set_acceptance(self.h, mode, temperature, seed, ptr, rows), "fs_set_acceptance")

    def fs_verify_step(self):
        out = fs_step_out()
        self._chk(self.L.fs_verify_step(self.h, C.byref(out)), "fs_verify_step")
        n = out.n_rows
        r = dict(seg_id=out.seg_id, s_begin=out.s_begin, n_rows=n, node=list(out.node[:n]),
                 am=list(out.am[:n]), margin=list(out.margin[:n]))
        if self.logits is not None and n > 0 and out.seg_id >= 0:
            r["logits"] = self.logits[:n].cpu().numpy().copy()
        return r

    def fs_accept(self):
        out = fs_accept_out()
        self._chk(self.L.fs_accept(self.h, C.byref(out)), "fs_accept")
        return out

    @staticmethod
    def decision_dict(out):
        if not out.progress:
            return dict(progress=0)
        n = out.n_acc
        return dict(progress=1, acc_ids=list(out.acc_ids[:n]), acc_tokens=list(out.acc_tokens[:n]),
                    x_new=out.x_new, n_new_id=out.n_new, cont=out.cont,
                    flagged=list(out.flagged_ids[:out.n_flagged]))

    @staticmethod
    def decision_struct(d):
        o = fs_accept_out()
        o.progress = 1
        o.n_acc = len(d["acc_ids"])
        for k, v in enumerate(d["acc_ids"]):
            o.acc_ids[k] = v
        for k, v in enumerate(d.get("acc_tokens", [])):
            o.acc_tokens[k] = v
        o.x_new = d["x_new"]
        o.n_new = d["n_new_id"]
        o.cont = d["cont"]
        return o

    def fs_prune_and_compact(self, decision):
        if isinstance(decision, dict):
            decision = self.decision_struct(decision)
        self._chk(self.L.fs_prune_and_compact(self.h, C.byref(decision)), "fs_prune_and_compact")

    def state(self):
        s = fs_state()
        self._chk(self.L.fs_query(self.h, FS_Q_STATE, C.byref(s), C.sizeof(s), None), "fs_query")
        P = s.n_stages
        return dict(l_glo=s.l_glo, x_new=s.x_new, live=s.live, n_live=s.n_live, next_id=s.next_id,
                    rank=s.rank,
                    n_cached=list(s.n_cached[:P]), layers_per_stage=list(s.layers_per_stage[:P]),
                    layer_begin=s.layer_begin, layer_end=s.layer_end,
                    queue=[tuple(s.queue[i]) for i in range(s.n_queue)],
                    inflight=[tuple(s.inflight[p]) for p in range(P)], launches=s.launches)

    def query(self, what):
        need = C.c_size_t()
        self._chk(self.L.fs_query(self.h, what, None, 0, C.byref(need)), "fs_query")
        n = need.value // 4
        dt = np.float32 if what == FS_Q_CU else (np.uint32 if what in (FS_Q_ANC, FS_Q_RETAIN) else np.int32)
        buf = np.zeros(max(n, 1), dt)
        self._chk(self.L.fs_query(self.h, what, buf.ctypes.data, buf.nbytes, None), "fs_query")
        return buf[:n]

    def set_profiling(self, on):
        self._chk(self.L.fs_set_profiling(self.h, 1 if on else 0), "fs_set_profiling")

    def get_profile(self):
        p = fs_profile()
        self._chk(self.L.fs_get_profile(self.h, C.byref(p)), "fs_get_profile")
        return {k: getattr(p, k) for k, _ in fs_profile._fields_}

    def bench_kernel(self, kind, iters=20):
        us, by = C.c_double(), C.c_double()
        self._chk(self.L.fs_bench_kernel(self.h, kind, iters, C.byref(us), C.byref(by)), "fs_bench_kernel")
        return us.value, by.value

    def debug_gemm(self, layer, which, X, n_out):
        X = np.ascontiguousarray(X, dtype=np.float32)
        Y = self.torch.zeros((X.shape[0], n_out), dtype=self.torch.float32, device=self.arena.device)
        self._chk(self.L.fs_debug_gemm(self.h, layer, which, X.ctypes.data_as(C.POINTER(C.c_float)),
                                       X.shape[0], C.cast(Y.data_ptr(), C.POINTER(C.c_float))),
                  "fs_debug_gemm")
        return Y.cpu().numpy()

    def debug_write_kv(self, layer, which, kvh, slot, row):
        row = np.ascontiguousarray(row, dtype=np.float32)
        assert row.shape == (self.shape.head_dim,)
        self._chk(self.L.fs_debug_write_kv(self.h, layer, which, kvh, slot,
                                           row.ctypes.data_as(C.POINTER(C.c_float))), "fs_debug_write_kv")

    def read_kv(self, layer, which, kvh, slot):
        out = np.zeros(self.shape.head_dim, np.float32)
        self._chk(self.L.fs_read_kv(self.h, layer, which, kvh, slot,
                                    out.ctypes.data_as(C.POINTER(C.c_float))), "fs_read_kv")
        return out


class LocalPipeline:
    """A P-stage pipeline inside ONE process: one context per stage (each on its
    own CUDA stream, all on `devices[p]`, default one device), joined by an
    fs_local_group so the stage transport is a device copy instead of NCCL
    (include/flowspec.h).  SPMD as under torchrun: every call is made on every
    stage with the same host inputs; the collective calls run one host thread
    per stage.  Results are the last stage's (the one that holds the head)."""

    COLLECTIVE = ("fs_set_prefix", "fs_verify_step")

    def __init__(self, shape, n_stages, max_ctx=4096, max_live=512, max_seg=16, devices=None,
                 layers_per_stage=None, sampling=0, max_prefill=0):
        from concurrent.futures import ThreadPoolExecutor
        self.L = lib()
        self.P = n_stages
        g = C.c_void_p()
        rc = self.L.fs_local_group_create(n_stages, C.byref(g))
        if rc != FS_OK:
            raise FlowSpecError(rc, "fs_local_group_create")
        self.group = g
        devices = devices or [0] * n_stages
        self.stages = [Pipeline(shape, n_stages=n_stages, rank=p, max_ctx=max_ctx, max_live=max_live,
                                max_seg=max_seg, device=devices[p], layers_per_stage=layers_per_stage,
                                local_group=g, sampling=sampling, max_prefill=max_prefill)
                       for p in range(n_stages)]
        self.shape = shape
        self.cfg = self.stages[-1].cfg
        self.pool = ThreadPoolExecutor(max_workers=n_stages)

    @property
    def last(self):
        return self.stages[-1]

    def _all(self, name, *a, **kw):
        if name in self.COLLECTIVE:
            futs = [self.pool.submit(getattr(st, name), *a, **kw) for st in self.stages]
            res = [f.result() for f in futs]
        else:
            res = [getattr(st, name)(*a, **kw) for st in self.stages]
        return res[-1]

    def fs_load_random_weights(self, seed):
        return self._all("fs_load_random_weights", seed)

    def fs_set_prefix(self, tokens, mode=FS_PREFILL, kv_seed=0):
        return self._all("fs_set_prefix", tokens, mode, kv_seed)

    def fs_submit_segment(self, flags, parent, token, own, l_max, l_top=0):
        return self._all("fs_submit_segment", flags, parent, token, own, l_max, l_top)

    def fs_verify_step(self):
        return self._all("fs_verify_step")

    def fs_set_acceptance(self, mode, temperature=1.0, seed=0, q=None):
        return self._all("fs_set_acceptance", mode, temperature, seed, q)

    def fs_accept(self):
        return self._all("fs_accept")

    def fs_prune_and_compact(self, decision):
        return self._all("fs_prune_and_compact", decision)

    def enable_logits(self, rows_cap=None):
        self.last.enable_logits(rows_cap)

    decision_dict = staticmethod(Pipeline.decision_dict)

    def state(self):
        return self.last.state()

    def query(self, what):
        return self.last.query(what)

    def stage_of_layer(self, layer):
        for st in self.stages:
            s = st.state()
            if s["layer_begin"] <= layer < s["layer_end"]:
                return st
        raise ValueError(layer)

    def read_kv(self, layer, which, kvh, slot):
        return self.stage_of_layer(layer).read_kv(layer, which, kvh, slot)

    def close(self):
        for st in getattr(self, "stages", []):
            st.close()
        self.stages = []
        if getattr(self, "group", None):
            self.L.fs_local_group_destroy(self.group)
            self.group = None
        if getattr(self, "pool", None):
            self.pool.shutdown()
            self.pool = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def layers_per_stage(shape, n_stages):
    cfg = make_config(shape, n_stages=n_stages, max_ctx=4096)
    out = (i32 * n_stages)()
    rc = lib().fs_layers_per_stage(C.byref(cfg), out)
    if rc != FS_OK:
        raise FlowSpecError(rc, "fs_layers_per_stage")
    return list(out)


def nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    rc = lib().fs_nccl_unique_id(buf)
    if rc != FS_OK:
        raise FlowSpecError(rc, "fs_nccl_unique_id")
    return bytes(buf)
