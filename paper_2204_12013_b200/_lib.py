"""ctypes binding of include/bamboo.h — argument marshalling only.

Every step of the hot path runs inside libbamboo.so (CUDA kernels + its own
CUDA-IPC transport);
this module converts Python/numpy arguments into the C structs and pointers
the C ABI takes and turns bb_status codes into exceptions. There is no
fallback: if the library cannot be loaded, importing the product fails.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BB_LIB", os.path.join(_HERE, "libbamboo.so"))   # BB_LIB: A/B builds

BB_OK, BB_E_INVAL, BB_E_CUDA, BB_E_NCCL, BB_E_OOM = 0, -1, -2, -3, -4
BB_E_PREEMPTED, BB_E_FATAL, BB_E_STATE, BB_E_UNSUPPORTED = -5, -6, -7, -8
STATUS_NAMES = {0: "BB_OK", -1: "BB_E_INVAL", -2: "BB_E_CUDA", -3: "BB_E_NCCL", -4: "BB_E_OOM",
                -5: "BB_E_PREEMPTED", -6: "BB_E_FATAL", -7: "BB_E_STATE", -8: "BB_E_UNSUPPORTED"}
PREC = {"bf16": 0, "fp32": 1}
STATE = {"params": 0, "grads": 1, "adam_m": 2, "adam_v": 3}

RC = {"none": 0, "eflb": 1, "lflb": 2, "efeb": 3}
EXPORTED = ["bb_default_opts", "bb_session_id", "bb_init", "bb_load_params", "bb_step",
            "bb_stage_inputs", "bb_preempt", "bb_recover", "bb_rejoin", "bb_read_state",
            "bb_write_state", "bb_stage_memory", "bb_stage_params", "bb_schedule_dump", "bb_recovery_dump",
            "bb_kernel_stats", "bb_node_stats", "bb_plan_dump", "bb_last_error", "bb_destroy",
            "bb_xport_pingpong",
            "bb_op_gemm", "bb_op_attention_fwd", "bb_op_attention_bwd", "bb_op_layernorm_fwd",
            "bb_op_layernorm_bwd", "bb_op_cross_entropy", "bb_op_adam"]


class BambooError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")


class BBModel(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in
                ("n_layer", "d_model", "n_head", "d_ff", "vocab", "seq_len", "causal")]


class BBOpts(ctypes.Structure):
    _fields_ = [("micro_batch", ctypes.c_int), ("rc", ctypes.c_int), ("prec", ctypes.c_int),
                ("layers_per_stage", ctypes.POINTER(ctypes.c_int)),
                ("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("world_rank", ctypes.c_int),
                ("world_size", ctypes.c_int), ("device", ctypes.c_int),
                ("node_rank", ctypes.POINTER(ctypes.c_int)), ("session_id", ctypes.c_void_p),
                ("profile", ctypes.c_int), ("frc_retain_bytes", ctypes.c_size_t),
                ("frc_persistent", ctypes.c_int), ("timing", ctypes.c_int),
                ("detect_ms", ctypes.c_int), ("pipelines", ctypes.c_int),
                ("frc_swap_bytes", ctypes.c_size_t)]


class BBStepStats(ctypes.Structure):
    _fields_ = [("loss", ctypes.c_float), ("step_ms", ctypes.c_float),
                ("device_ms", ctypes.c_float), ("gpu_launches", ctypes.c_int),
                ("h2d_bytes", ctypes.c_uint64), ("d2h_bytes", ctypes.c_uint64)]


class BBRecoveryStats(ctypes.Structure):
    _fields_ = [("victim", ctypes.c_int), ("shadow", ctypes.c_int), ("successor", ctypes.c_int),
                ("commit", ctypes.c_int), ("brc_mb", ctypes.c_int), ("frc_done_mb", ctypes.c_int),
                ("resent_mb", ctypes.c_int), ("recover_ms", ctypes.c_float),
                ("loss", ctypes.c_float), ("interrupted_step_ms", ctypes.c_float),
                ("frc_recomputed_mb", ctypes.c_int), ("bytes_resent", ctypes.c_uint64),
                ("frc_swapped_mb", ctypes.c_int)]


class BBNodeStat(ctypes.Structure):
    _fields_ = [("node", ctypes.c_int), ("n_fwd", ctypes.c_int), ("n_bwd", ctypes.c_int),
                ("n_frc", ctypes.c_int), ("step_ms", ctypes.c_float), ("busy_ms", ctypes.c_float),
                ("bubble_ms", ctypes.c_float), ("frc_ms", ctypes.c_float),
                ("frc_hidden_ms", ctypes.c_float)]


class BBKernelStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_int), ("ms", ctypes.c_double),
                ("work", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.bb_init.argtypes = [ctypes.POINTER(BBModel), ctypes.c_int, ctypes.c_int,
                                 ctypes.POINTER(BBOpts), ctypes.POINTER(ctypes.c_void_p)]
        for name in ("bb_load_params", "bb_step", "bb_preempt", "bb_recover", "bb_read_state",
                     "bb_write_state", "bb_stage_memory", "bb_stage_params", "bb_schedule_dump", "bb_recovery_dump",
                     "bb_kernel_stats", "bb_node_stats", "bb_last_error", "bb_session_id"):
            getattr(_lib, name).restype = ctypes.c_int
        _lib.bb_load_params.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
        _lib.bb_step.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.POINTER(BBStepStats)]
        _lib.bb_preempt.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        _lib.bb_stage_inputs.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib.bb_recover.argtypes = [ctypes.c_void_p, ctypes.POINTER(BBRecoveryStats)]
        _lib.bb_rejoin.argtypes = [ctypes.c_void_p]
        _lib.bb_read_state.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_void_p, ctypes.c_size_t]
        _lib.bb_write_state.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_size_t]
        _lib.bb_node_stats.argtypes = [ctypes.c_void_p, ctypes.POINTER(BBNodeStat), ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_int)]
        _lib.bb_stage_memory.argtypes = [ctypes.c_void_p, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_size_t),
                                         ctypes.POINTER(ctypes.c_int)]
        _lib.bb_stage_params.argtypes = [ctypes.c_void_p, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_size_t),
                                         ctypes.POINTER(ctypes.c_size_t)]
        for name in ("bb_schedule_dump", "bb_recovery_dump"):
            getattr(_lib, name).argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t,
                                            ctypes.POINTER(ctypes.c_size_t)]
        _lib.bb_kernel_stats.argtypes = [ctypes.c_void_p, ctypes.POINTER(BBKernelStat),
                                         ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        _lib.bb_last_error.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t]
        _lib.bb_destroy.argtypes = [ctypes.c_void_p]
        _lib.bb_destroy.restype = None
        _lib.bb_default_opts.argtypes = [ctypes.POINTER(BBOpts)]
        _lib.bb_default_opts.restype = None
        _lib.bb_session_id.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
        _lib.bb_xport_pingpong.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_float)]
        _lib.bb_plan_dump.argtypes = [ctypes.POINTER(BBModel), ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(BBOpts), ctypes.c_int, ctypes.c_int,
                                      ctypes.c_char_p, ctypes.c_size_t,
                                      ctypes.POINTER(ctypes.c_size_t)]
        vp, ci = ctypes.c_void_p, ctypes.c_int
        _lib.bb_op_gemm.argtypes = [ci, ci, ci, ci, ci, vp, ci, ci, vp, ci, ci, ci, vp, ci, vp, vp,
                                    vp, vp]
        _lib.bb_op_attention_fwd.argtypes = [ci, ci, ci, ci, ci, ci, vp, vp, vp, vp]
        _lib.bb_op_attention_bwd.argtypes = [ci, ci, ci, ci, ci, ci, vp, vp, vp, vp, vp, vp]
        _lib.bb_op_layernorm_fwd.argtypes = [ci, ci, ci, vp, vp, vp, vp, vp, vp, vp]
        _lib.bb_op_layernorm_bwd.argtypes = [ci, ci, ci, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        _lib.bb_op_cross_entropy.argtypes = [ci, ci, ci, vp, vp, ctypes.c_float, vp, vp]
        _lib.bb_op_adam.argtypes = [ctypes.c_size_t, vp, vp, vp, vp, vp, ci, ctypes.c_float,
                                    ctypes.c_float, ctypes.c_float, ctypes.c_float, vp]
    return _lib


def _model(m):
    get = (lambda k: m[k]) if isinstance(m, dict) else (lambda k: getattr(m, k))
    return BBModel(get("n_layer"), get("d_model"), get("n_head"), get("d_ff"), get("vocab"),
                   get("seq_len"), int(bool(get("causal"))))


def _ints(xs):
    if xs is None:
        return None, None
    arr = (ctypes.c_int * len(xs))(*xs)
    return arr, ctypes.cast(arr, ctypes.POINTER(ctypes.c_int))


def make_opts(micro_batch=1, rc=True, prec="bf16", layers_per_stage=None, lr=1e-4, beta1=0.9,
              beta2=0.999, eps=1e-8, world_rank=0, world_size=1, device=0, node_rank=None,
              session_id=None, profile=False, frc_retain_bytes=0, frc_persistent=False,
              timing=False, detect_ms=0, pipelines=1, frc_swap_bytes=0):
    """rc: True (= "eflb"), False (= "none") or a mode name in RC."""
    o = BBOpts()
    lib().bb_default_opts(ctypes.byref(o))
    keep = []
    o.micro_batch = micro_batch
    o.rc = RC[rc] if isinstance(rc, str) else (1 if rc else 0)
    o.prec = PREC[prec]
    a, p = _ints(layers_per_stage)
    keep.append(a)
    o.layers_per_stage = p
    o.lr, o.beta1, o.beta2, o.eps = lr, beta1, beta2, eps
    o.world_rank, o.world_size, o.device = world_rank, world_size, device
    a, p = _ints(node_rank)
    keep.append(a)
    o.node_rank = p
    if session_id is not None:
        buf = ctypes.create_string_buffer(bytes(session_id), len(session_id))
        keep.append(buf)
        o.session_id = ctypes.cast(buf, ctypes.c_void_p)
    o.profile = int(bool(profile))
    o.frc_retain_bytes = int(frc_retain_bytes)
    o.frc_persistent = int(bool(frc_persistent))
    o.timing = int(bool(timing))
    o.detect_ms = int(detect_ms)
    o.pipelines = int(pipelines)
    o.frc_swap_bytes = int(frc_swap_bytes)
    return o, keep


def session_id():
    """32 random bytes (rank 0); broadcast them to the other ranks."""
    buf = ctypes.create_string_buffer(32)
    st = lib().bb_session_id(buf, 32)
    if st != BB_OK:
        raise BambooError(st, "bb_session_id")
    return buf.raw


def xport_pingpong(rank, world, device, session, nbytes, iters):
    """Mean one-way microseconds per message over the library's transport."""
    us = ctypes.c_float(0)
    buf = ctypes.create_string_buffer(bytes(session), len(session))
    st = lib().bb_xport_pingpong(rank, world, device, buf, nbytes, iters, ctypes.byref(us))
    if st != BB_OK:
        raise BambooError(st, "bb_xport_pingpong")
    return us.value


def _text(fn, *args):
    need = ctypes.c_size_t(0)
    fn(*args, None, 0, ctypes.byref(need))
    buf = ctypes.create_string_buffer(need.value)
    st = fn(*args, buf, need.value, ctypes.byref(need))
    if st != BB_OK:
        raise BambooError(st, "dump")
    return buf.value.decode()


def plan_dump(model, stages, microbatches, victim=-1, at_instr=-1, **opts):
    o, keep = make_opts(**opts)
    m = _model(model)
    return _text(lib().bb_plan_dump, ctypes.byref(m), stages, microbatches, ctypes.byref(o),
                 victim, at_instr)


class Pipeline:
    """One process's share of the pipeline (bb_init ... bb_destroy)."""

    def __init__(self, model, stages, microbatches, **opts):
        self._o, self._keep = make_opts(**opts)
        self._m = _model(model)
        self.stages, self.microbatches = stages, microbatches
        # int32 elements per tokens / targets array: D*M*mb sequences
        self._n_in = (max(1, self._o.pipelines) * microbatches * self._o.micro_batch *
                      self._m.seq_len)
        h = ctypes.c_void_p()
        st = lib().bb_init(ctypes.byref(self._m), stages, microbatches, ctypes.byref(self._o),
                           ctypes.byref(h))
        self._h = h
        if st != BB_OK:
            msg = self.last_error()
            self.close()
            raise BambooError(st, msg)

    def last_error(self):
        if not self._h:
            return ""
        buf = ctypes.create_string_buffer(4096)
        lib().bb_last_error(self._h, buf, 4096)
        return buf.value.decode()

    def _check(self, st, what):
        if st != BB_OK:
            raise BambooError(st, f"{what}: {self.last_error()}")

    def load_params(self, flat):
        flat = np.ascontiguousarray(flat, dtype=np.float32)
        self._check(lib().bb_load_params(self._h, flat.ctypes.data, flat.size), "bb_load_params")

    def _inputs(self, tokens, targets):
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        g = np.ascontiguousarray(targets, dtype=np.int32)
        if t.size != self._n_in or g.size != self._n_in:
            raise ValueError(f"tokens / targets: need {self._n_in} ids "
                             "(pipelines * microbatches * micro_batch * seq_len)")
        return t, g

    def stage_inputs(self, tokens, targets):
        t, g = self._inputs(tokens, targets)
        self._check(lib().bb_stage_inputs(self._h, t.ctypes.data, g.ctypes.data),
                    "bb_stage_inputs")

    def step(self, tokens=None, targets=None):
        """Returns ('ok' | 'preempted', BBStepStats). tokens=targets=None runs
        on the inputs staged with stage_inputs (resident in HBM)."""
        st = BBStepStats()
        if tokens is None:
            s = lib().bb_step(self._h, None, None, ctypes.byref(st))
        else:
            t, g = self._inputs(tokens, targets)
            s = lib().bb_step(self._h, t.ctypes.data, g.ctypes.data, ctypes.byref(st))
        if s == BB_E_PREEMPTED:
            return "preempted", st
        self._check(s, "bb_step")
        return "ok", st

    def preempt(self, stage, at_instr):
        self._check(lib().bb_preempt(self._h, stage, at_instr), "bb_preempt")

    def recover(self):
        r = BBRecoveryStats()
        self._check(lib().bb_recover(self._h, ctypes.byref(r)), "bb_recover")
        return r

    def rejoin(self):
        self._check(lib().bb_rejoin(self._h), "bb_rejoin")

    def stage_params(self, stage):
        off, cnt = ctypes.c_size_t(), ctypes.c_size_t()
        self._check(lib().bb_stage_params(self._h, stage, ctypes.byref(off), ctypes.byref(cnt)),
                    "bb_stage_params")
        return off.value, cnt.value

    def stage_memory(self, stage):
        """(bytes of one saved set, FRC saved sets the replica retains or -1)."""
        b, r = ctypes.c_size_t(), ctypes.c_int()
        self._check(lib().bb_stage_memory(self._h, stage, ctypes.byref(b), ctypes.byref(r)),
                    "bb_stage_memory")
        return b.value, r.value

    def read_state(self, stage, what="params", replica=False):
        """stage < stages, or d*stages + s for pipeline d's copy (D > 1)."""
        _, n = self.stage_params(stage % self.stages)
        out = np.empty(n, np.float32)
        self._check(lib().bb_read_state(self._h, stage, int(replica), STATE[what],
                                        out.ctypes.data, n), "bb_read_state")
        return out

    def write_state(self, stage, what, values):
        """Overwrite stage's fp32 params / adam_m / adam_v in every copy this
        process hosts (primary and replica), e.g. to start a step from an
        oracle state."""
        v = np.ascontiguousarray(values, dtype=np.float32)
        self._check(lib().bb_write_state(self._h, stage, STATE[what], v.ctypes.data, v.size),
                    "bb_write_state")

    def node_stats(self):
        arr = (BBNodeStat * 64)()
        n = ctypes.c_int()
        self._check(lib().bb_node_stats(self._h, arr, 64, ctypes.byref(n)), "bb_node_stats")
        return [{f: getattr(arr[i], f) for f, _ in BBNodeStat._fields_} for i in range(n.value)]

    def schedule_dump(self):
        return _text(lib().bb_schedule_dump, self._h)

    def recovery_dump(self):
        return _text(lib().bb_recovery_dump, self._h)

    def kernel_stats(self):
        arr = (BBKernelStat * 32)()
        n = ctypes.c_int()
        self._check(lib().bb_kernel_stats(self._h, arr, 32, ctypes.byref(n)), "bb_kernel_stats")
        return {arr[i].name.decode(): (arr[i].launches, arr[i].ms, arr[i].work)
                for i in range(n.value)}

    def close(self):
        if getattr(self, "_h", None):
            lib().bb_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- single ops
def _call(fn, *args):
    st = fn(*args)
    if st != BB_OK:
        raise BambooError(st, fn.__name__)


def op_gemm(prec, impl, M, N, K, A, lda, a_mn, B, ldb, b_mn, epi, C, ldc, bias=0, res=0, aux=0,
            stream=0):
    _call(lib().bb_op_gemm, PREC[prec], impl, M, N, K, A, lda, int(a_mn), B, ldb, int(b_mn), epi,
          C, ldc, bias or None, res or None, aux or None, stream or None)


def op_attention_fwd(prec, B, S, H, nh, causal, qkv, o, lse, stream=0):
    _call(lib().bb_op_attention_fwd, PREC[prec], B, S, H, nh, int(causal), qkv, o, lse,
          stream or None)


def op_attention_bwd(prec, B, S, H, nh, causal, qkv, o, lse, dout, dqkv, stream=0):
    _call(lib().bb_op_attention_bwd, PREC[prec], B, S, H, nh, int(causal), qkv, o, lse, dout,
          dqkv, stream or None)


def op_layernorm_fwd(prec, R, H, x, g, b, y, mean, rstd, stream=0):
    _call(lib().bb_op_layernorm_fwd, PREC[prec], R, H, x, g, b, y, mean, rstd, stream or None)


def op_layernorm_bwd(prec, R, H, dy, x, mean, rstd, g, dres, dx, dg, db, stream=0):
    _call(lib().bb_op_layernorm_bwd, PREC[prec], R, H, dy, x, mean, rstd, g, dres or None, dx, dg,
          db, stream or None)


def op_cross_entropy(prec, R, V, logits, targets, n_tok, loss_rows, stream=0):
    _call(lib().bb_op_cross_entropy, PREC[prec], R, V, logits, targets, float(n_tok), loss_rows,
          stream or None)


def op_adam(n, p, g, m, v, w16, t, lr, b1, b2, eps, stream=0):
    _call(lib().bb_op_adam, n, p, g, m, v, w16 or None, t, lr, b1, b2, eps, stream or None)
