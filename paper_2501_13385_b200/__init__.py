"""B200-native PRGD hot path for low-TT-rank tensor completion (arXiv 2501.13385).

Thin ctypes binding over the C-ABI in include/prgd.h (argument marshalling only:
every step of the path runs in the CUDA kernels of libprgd.so).  PyTorch, when
present, supplies device memory (caching allocator) and the CUDA stream.

There is no CPU fallback: if libprgd.so is missing, `load()` raises; if no
sm_100 device is visible, creating a context raises PRGDError(TT_ERR_CUDA).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PRGD_LIB_PATH") or os.path.join(HERE, "libprgd.so")   # override: experiments
HEADER = os.path.join(os.path.dirname(HERE), "include", "prgd.h")

TT_OK, TT_ERR_ARG, TT_ERR_RANK, TT_ERR_INDEX, TT_ERR_STATE = 0, -1, -2, -3, -4
TT_ERR_NUMERIC, TT_ERR_CUDA, TT_ERR_OOM, TT_ERR_UNSUPPORTED = -5, -6, -7, -8
STATUS_NAMES = {0: "TT_OK", -1: "TT_ERR_ARG", -2: "TT_ERR_RANK", -3: "TT_ERR_INDEX",
                -4: "TT_ERR_STATE", -5: "TT_ERR_NUMERIC", -6: "TT_ERR_CUDA", -7: "TT_ERR_OOM",
                -8: "TT_ERR_UNSUPPORTED"}
EPS_RULES = {"vee": 0, "fixed": 1, "none": 2}
STEP_RULES = {"theory": 0, "raw": 1, "adaptive": 2}
DBG = {"perm_pre": 1, "offs_l": 2, "perm_suf": 3, "offs_r": 4, "resid": 5, "h": 6, "phi": 7,
       "eps": 8, "u": 9, "p": 10, "y": 11, "ahat": 12, "perm_mode": 13, "offs_mode": 14}
PATHS = {"auto": 0, "tables": 1, "chains": 2}


class PRGDError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        self.code = code
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")


class _Stats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("steps", ctypes.c_int64),
                ("launches_per_step", ctypes.c_int64), ("K_L", ctypes.c_int32),
                ("graphs", ctypes.c_int32)]


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)
ALLREDUCE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p)

_lib = None


def load() -> ctypes.CDLL:
    """Load libprgd.so (built by `python -m paper_2501_13385_b200.build`)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() "
                          "(no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    i64p = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "tt_create": (ctypes.c_int, [ctypes.c_int, i64p, i64p, ctypes.POINTER(P)]),
        "tt_destroy": (ctypes.c_int, [P]),
        "tt_set_stream": (ctypes.c_int, [P, P]),
        "tt_set_allocator": (ctypes.c_int, [P, ALLOC_FN, FREE_FN, P]),
        "tt_set_observations": (ctypes.c_int, [P, P, P, ctypes.c_int64]),
        "tt_set_observations_u8": (ctypes.c_int, [P, P, P, ctypes.c_int64]),
        "tt_set_core": (ctypes.c_int, [P, ctypes.c_int, P]),
        "tt_get_core": (ctypes.c_int, [P, ctypes.c_int, P]),
        "tt_set_metric": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_double, ctypes.c_int]),
        "tt_prgd_step": (ctypes.c_int, [P, ctypes.c_double]),
        "tt_eval_at": (ctypes.c_int, [P, P, ctypes.c_int64, P]),
        "tt_residual_norm": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_double)]),
        "tt_sync": (ctypes.c_int, [P]),
        "tt_last_error": (ctypes.c_char_p, [P]),
        "tt_plan": (ctypes.c_int, [ctypes.c_int, i64p, i64p, ctypes.POINTER(ctypes.c_int),
                                   i64p, i64p]),
        "tt_set_path": (ctypes.c_int, [P, ctypes.c_int]),
        "tt_set_retraction": (ctypes.c_int, [P, ctypes.c_int]),
        "tt_get_path": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_int)]),
        "tt_spectral_init": (ctypes.c_int, [P]),
        "tt_set_allreduce": (ctypes.c_int, [P, ALLREDUCE_FN, P, ctypes.c_int64]),
        "tt_get_stats": (ctypes.c_int, [P, ctypes.POINTER(_Stats)]),
        "tt_set_profiling": (ctypes.c_int, [P, ctypes.c_int]),
        "tt_get_profile": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_int), i64p]),
        "tt_profile_name": (ctypes.c_char_p, [ctypes.c_int]),
        "tt_debug_get": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, ctypes.c_int64, i64p]),
        "tt_debug_round": (ctypes.c_int, [P, P, ctypes.c_int64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _i64(seq) -> ctypes.Array:
    return (ctypes.c_int64 * len(seq))(*[int(v) for v in seq])


def plan(n: Sequence[int], r: Sequence[int]):
    """Host-only split planning (tt_plan): returns (K_L, N_L, N_R)."""
    lib = load()
    kl = ctypes.c_int()
    nl, nr = ctypes.c_int64(), ctypes.c_int64()
    rc = lib.tt_plan(len(n), _i64(n), _i64(r), ctypes.byref(kl), ctypes.byref(nl), ctypes.byref(nr))
    if rc != TT_OK:
        raise PRGDError(rc, "tt_plan")
    return kl.value, nl.value, nr.value


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


_SHARED_STREAMS = {}


class TTContext:
    """One PRGD problem on the current CUDA device.

    use_torch: route device allocations through PyTorch's caching allocator and run on a
    torch.cuda.Stream (exposed as .stream): by default one library stream per device shared
    by all contexts, so the allocator's cached blocks (which belong to the stream they were
    allocated on) are reused by the next context instead of fresh cudaMalloc calls; pass
    stream= to give a context its own stream."""

    def __init__(self, n: Sequence[int], r: Sequence[int], use_torch: bool = True, stream=None,
                 path: str = "auto"):
        self.lib = load()
        self.n = tuple(int(v) for v in n)
        self.r = tuple(int(v) for v in r)
        self.d = len(self.n)
        self.m = 0
        self._h = ctypes.c_void_p()
        rc = self.lib.tt_create(self.d, _i64(self.n), _i64(self.r), ctypes.byref(self._h))
        if rc != TT_OK:
            raise PRGDError(rc, "tt_create")
        self.stream = None
        self._keep = []
        if path != "auto":
            self._check(self.lib.tt_set_path(self._h, PATHS[path]), "tt_set_path")
        if use_torch:
            self._attach_torch(stream)

    @property
    def path(self) -> str:
        """The path over Omega in use (tt_get_path): "tables" or "chains"."""
        v = ctypes.c_int()
        self._check(self.lib.tt_get_path(self._h, ctypes.byref(v)), "tt_get_path")
        return {1: "tables", 2: "chains"}[v.value]

    # -- plumbing: PyTorch device memory and stream
    def _attach_torch(self, stream=None):
        import torch
        if not torch.cuda.is_available():
            return
        dev = torch.cuda.current_device()
        if stream is None:
            stream = _SHARED_STREAMS.get(dev)
            if stream is None:
                stream = _SHARED_STREAMS[dev] = torch.cuda.Stream(device=dev)
        self.stream = stream

        alloc_fn = torch.cuda.caching_allocator_alloc
        delete_fn = torch.cuda.caching_allocator_delete

        def _alloc(nbytes, _user):
            try:
                return alloc_fn(int(nbytes), device=dev, stream=stream)
            except Exception:
                return None   # the library reports TT_ERR_OOM

        def _free(ptr, _user):
            try:
                delete_fn(ptr)
            except Exception:
                pass          # interpreter teardown: the process is exiting anyway

        fa, ff = ALLOC_FN(_alloc), FREE_FN(_free)
        self._keep += [fa, ff]
        self._check(self.lib.tt_set_allocator(self._h, fa, ff, None), "tt_set_allocator")
        self._check(self.lib.tt_set_stream(self._h, ctypes.c_void_p(stream.cuda_stream)),
                    "tt_set_stream")

    # -- sharded (multi-GPU) mode: Omega split over ranks, h and Y all-reduced (tt_set_allreduce)
    def set_allreduce(self, fn, m_global: int):
        """fn(buffer_ptr, count, stream_ptr): in-place fp64 sum over ranks of a device buffer,
        enqueued on the given CUDA stream.  fn=None returns to single-rank mode."""
        if fn is None:
            self._check(self.lib.tt_set_allreduce(self._h, ALLREDUCE_FN(), None, 0), "tt_set_allreduce")
            return
        cb = ALLREDUCE_FN(lambda buf, count, stream, _user: fn(buf, count, stream))
        self._keep.append(cb)
        self._check(self.lib.tt_set_allreduce(self._h, cb, None, int(m_global)), "tt_set_allreduce")

    def _check(self, rc, what):
        if rc != TT_OK:
            msg = self.lib.tt_last_error(self._h)
            raise PRGDError(rc, f"{what}: {msg.decode() if msg else ''}")

    def close(self):
        if self._h:
            self.lib.tt_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- data
    def set_observations(self, idx: np.ndarray, vals: np.ndarray):
        # uint8 multi-indices go through tt_set_observations_u8 (a quarter of the upload)
        u8 = isinstance(idx, np.ndarray) and idx.dtype == np.uint8
        idx = np.ascontiguousarray(idx, dtype=np.uint8 if u8 else np.int32)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        m = vals.shape[0]
        if m and idx.shape != (m, self.d):
            raise ValueError("idx must be [m, d]")
        self.m = 0
        if u8:
            self._check(self.lib.tt_set_observations_u8(self._h, _ptr(idx), _ptr(vals), m),
                        "tt_set_observations_u8")
        else:
            self._check(self.lib.tt_set_observations(self._h, _ptr(idx), _ptr(vals), m),
                        "tt_set_observations")
        self.m = int(m)

    def set_core(self, k: int, core: np.ndarray):
        core = np.ascontiguousarray(core, dtype=np.float64)
        if core.shape != (self.r[k], self.n[k], self.r[k + 1]):
            raise ValueError(f"core {k} must have shape {(self.r[k], self.n[k], self.r[k + 1])}")
        self._check(self.lib.tt_set_core(self._h, k, _ptr(core)), "tt_set_core")

    def set_cores(self, cores):
        for k, c in enumerate(cores):
            self.set_core(k, c)

    def get_core(self, k: int) -> np.ndarray:
        out = np.empty((self.r[k], self.n[k], self.r[k + 1]))
        self._check(self.lib.tt_get_core(self._h, k, _ptr(out)), "tt_get_core")
        return out

    def get_cores(self):
        return [self.get_core(k) for k in range(self.d)]

    def spectral_init(self):
        """Cores <- SVD_r^tt(p^{-1} P_Omega(y)) computed on the GPU (tt_spectral_init)."""
        self._check(self.lib.tt_spectral_init(self._h), "tt_spectral_init")

    def set_metric(self, eps_rule: str = "vee", eps: float = 0.0, step_rule: str = "theory"):
        self._check(self.lib.tt_set_metric(self._h, EPS_RULES[eps_rule], float(eps),
                                           STEP_RULES[step_rule]), "tt_set_metric")

    def set_retraction(self, kind: str = "plain"):
        """"plain": SVD_r^tt(W_l) (Alg. 2 line 5); "weighted": W^{-1/2} SVD_r^tt W^{1/2}."""
        self._check(self.lib.tt_set_retraction(self._h, {"plain": 0, "weighted": 1}[kind]),
                    "tt_set_retraction")

    # -- hot path
    def step(self, step_size: float = 1.0):
        self._check(self.lib.tt_prgd_step(self._h, float(step_size)), "tt_prgd_step")

    def eval_at(self, idx: np.ndarray) -> np.ndarray:
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        out = np.empty(idx.shape[0])
        self._check(self.lib.tt_eval_at(self._h, _ptr(idx), idx.shape[0], _ptr(out)), "tt_eval_at")
        return out

    def residual_norm(self) -> float:
        v = ctypes.c_double()
        self._check(self.lib.tt_residual_norm(self._h, ctypes.byref(v)), "tt_residual_norm")
        return v.value

    def sync(self):
        self._check(self.lib.tt_sync(self._h), "tt_sync")

    # -- introspection
    def stats(self) -> dict:
        s = _Stats()
        self._check(self.lib.tt_get_stats(self._h, ctypes.byref(s)), "tt_get_stats")
        return {f: getattr(s, f) for f, _ in _Stats._fields_}

    def set_profiling(self, on: bool):
        self._check(self.lib.tt_set_profiling(self._h, 1 if on else 0), "tt_set_profiling")

    def get_profile(self) -> dict:
        buf = (ctypes.c_double * 64)()
        ng, ns = ctypes.c_int(), ctypes.c_int64()
        self._check(self.lib.tt_get_profile(self._h, buf, 64, ctypes.byref(ng), ctypes.byref(ns)),
                    "tt_get_profile")
        names = [self.lib.tt_profile_name(i).decode() for i in range(ng.value)]
        return {"steps": ns.value, "ms": {nm: buf[i] for i, nm in enumerate(names)}}

    def debug(self, what: str, k: int = 0) -> np.ndarray:
        """Read back internal device state (tt_debug_get; tests only)."""
        code = DBG[what]
        dt = np.int32 if code in (1, 3, 13) else (np.int64 if code in (2, 4, 14) else np.float64)
        out = np.empty(max(self._debug_size(code, k), 4), dtype=dt)
        cnt = ctypes.c_int64()
        self._check(self.lib.tt_debug_get(self._h, code, k, _ptr(out), out.shape[0],
                                          ctypes.byref(cnt)), f"tt_debug_get({what})")
        return out[:cnt.value]

    def debug_round(self, blocks):
        """Round a rank-2r block TT (list of cores [R_k, n_k, R_{k+1}], R = 2r inside) with the
        library's A14 kernels into the context's cores (tt_debug_round; tests only)."""
        flat = np.ascontiguousarray(np.concatenate([np.ascontiguousarray(b, dtype=np.float64).ravel()
                                                    for b in blocks]))
        self._check(self.lib.tt_debug_round(self._h, _ptr(flat), flat.shape[0]), "tt_debug_round")

    def _debug_size(self, code, k):
        if code in (1, 3, 5, 13):
            return self.m
        if code in (2, 4):
            kl, nl, nr = plan(self.n, self.r)
            return (nl if code == 2 else nr) + 1
        if code == 14:
            return self.n[k] + 1
        if code in (6, 7):
            return self.n[k]
        if code == 8:
            return 29
        if code in (9, 11, 12):
            return self.r[k] * self.n[k] * self.r[k + 1]
        if code == 10:
            return self.r[k + 1] ** 2
        return 0


def torch_allreduce(group=None):
    """An all-reduce callback for TTContext.set_allreduce built on torch.distributed (NCCL on
    GPUs): wraps the library's device buffer as a tensor (zero copy) and sums it in place
    over the process group on the library's stream."""
    import torch
    import torch.distributed as dist

    class _Buf:
        def __init__(self, ptr, count):
            self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                             "data": (int(ptr), False), "version": 3,
                                             "strides": None}

    def fn(ptr, count, stream_ptr):
        if count <= 0:
            return
        t = torch.as_tensor(_Buf(ptr, count), device="cuda")
        with torch.cuda.stream(torch.cuda.ExternalStream(int(stream_ptr))):
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return fn
