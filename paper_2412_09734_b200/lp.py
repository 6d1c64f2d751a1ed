"""ctypes binding of include/lp.h.  Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.environ.get("MPAX_LIB") or os.path.join(_HERE, "libmpax_b200.so")
_lock = threading.Lock()
_lib = None

LP_HOST, LP_DEVICE = 0, 1
LP_OPTIMAL, LP_ITERATION_LIMIT, LP_NUMERICAL_ERROR, LP_PRIMAL_INFEASIBLE, LP_DUAL_INFEASIBLE = 1, 2, 3, 4, 5
RAPDHG, R2HPDHG = 0, 1
PATH_AUTO, PATH_INSTANCE, PATH_GRID, PATH_DMMA = 0, 1, 2, 3
STEP_ADAPTIVE, STEP_CONSTANT = 0, 1
FP64, FP32 = 0, 1
SHARD_ROWS, SHARD_COLS, SHARD_AUTO = 0, 1, 2

EXPORTED_SYMBOLS = [
    "lp_default_options", "lp_create", "lp_create_batch", "lp_update_batch", "lp_solve", "lp_solve_batch",
    "lp_get_solution", "lp_get_solutions", "lp_get_shape", "lp_get_scaling", "lp_spmv_scaled",
    "lp_kernel_launch_count", "lp_error_string", "lp_last_error_detail", "lp_destroy",
    "lp_create_sharded", "lp_create_sharded_virtual", "lp_nccl_unique_id", "lp_nccl_comm_init",
    "lp_nccl_comm_destroy", "lp_spo_plus", "lp_selftest_division", "lp_set_decision_log",
    "lp_shard_axis", "lp_create_sharded_cols", "lp_create_sharded_virtual_axis", "lp_set_decision_log_instance",
]


class LpError(RuntimeError):
    def __init__(self, code: int, where: str):
        L = lib()
        msg = L.lp_error_string(code).decode()
        detail = L.lp_last_error_detail().decode()
        super().__init__(f"{where}: {msg} ({code}){': ' + detail if detail else ''}")
        self.code = code


class ProblemDesc(C.Structure):
    _fields_ = [("n", C.c_int64), ("m1", C.c_int64), ("m2", C.c_int64), ("nnz", C.c_int64),
                ("dense", C.c_int32), ("memory", C.c_int32),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p),
                ("c", C.c_void_p), ("q", C.c_void_p), ("l", C.c_void_p), ("u", C.c_void_p)]


class Options(C.Structure):
    _fields_ = [("eps_abs", C.c_double), ("eps_rel", C.c_double), ("eps_primal_infeasible", C.c_double),
                ("eps_dual_infeasible", C.c_double), ("eps_feas_polish", C.c_double),
                ("iteration_limit", C.c_int64), ("check_frequency", C.c_int32), ("algorithm", C.c_int32),
                ("warm_start", C.c_int32), ("feasibility_polishing", C.c_int32), ("verbose", C.c_int32),
                ("display_frequency", C.c_int32), ("path", C.c_int32), ("step_rule", C.c_int32),
                ("reflection", C.c_double), ("precision", C.c_int32), ("sharded_exchange", C.c_int32)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("polish", C.c_int32), ("iterations", C.c_int64),
                ("attempts", C.c_int64), ("restarts", C.c_int64),
                ("primal_objective", C.c_double), ("dual_objective", C.c_double),
                ("primal_residual", C.c_double), ("dual_residual", C.c_double), ("gap", C.c_double),
                ("rel_kkt", C.c_double), ("omega", C.c_double), ("eta", C.c_double),
                ("solve_seconds", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


RESULT_DTYPE = np.dtype([(f, np.int32 if t is C.c_int32 else np.int64 if t is C.c_int64 else np.float64)
                         for f, t in Result._fields_], align=True)
assert RESULT_DTYPE.itemsize == C.sizeof(Result)


def library_path() -> str:
    return _LIBPATH


def lib():
    """Load libmpax_b200.so.  Raises if it has not been built (no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIBPATH):
                raise ImportError(f"{_LIBPATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = C.CDLL(_LIBPATH)
            P, V = C.POINTER, C.c_void_p
            L.lp_default_options.argtypes = [P(Options)]
            L.lp_create.argtypes = [P(ProblemDesc), V, P(V)]
            L.lp_create_batch.argtypes = [P(ProblemDesc), C.c_int64, V, V, C.c_int32, V, P(V)]
            L.lp_update_batch.argtypes = [V, V, V, C.c_int32]
            L.lp_solve.argtypes = [V, P(Options), V, V, C.c_int32, P(Result)]
            L.lp_solve_batch.argtypes = [V, P(Options), V, V, C.c_int32, V]
            L.lp_get_solution.argtypes = [V, C.c_int64, V, V, V, C.c_int32]
            L.lp_spo_plus.argtypes = [V, P(Options), V, V, V, V, C.c_int32, C.c_int32, V, V, V]
            L.lp_get_solutions.argtypes = [V, V, V, C.c_int32]
            L.lp_get_shape.argtypes = [V, P(C.c_int64), P(C.c_int64), P(C.c_int64), P(C.c_int64)]
            L.lp_get_scaling.argtypes = [V, V, V, C.c_int32]
            if hasattr(L, "lp_set_decision_log"):
                L.lp_set_decision_log.argtypes = [V, V, C.c_int64, V, C.c_int64]
            if hasattr(L, "lp_set_decision_log_instance"):
                L.lp_set_decision_log_instance.argtypes = [V, C.c_int64]
            L.lp_spmv_scaled.argtypes = [V, V, V, V, V, C.c_int32]
            L.lp_kernel_launch_count.restype = C.c_int64
            L.lp_create_sharded.argtypes = [P(ProblemDesc), C.c_int64, C.c_int64, C.c_int64, V, C.c_int, C.c_int,
                                            V, P(V)]
            L.lp_create_sharded_virtual.argtypes = [P(ProblemDesc), C.c_int32, V, P(V)]
            if hasattr(L, "lp_create_sharded_cols"):
                L.lp_shard_axis.argtypes = [C.c_int64, C.c_int64]
                L.lp_create_sharded_cols.argtypes = [P(ProblemDesc), C.c_int64, C.c_int64, V, C.c_int, C.c_int, V,
                                                     P(V)]
                L.lp_create_sharded_virtual_axis.argtypes = [P(ProblemDesc), C.c_int32, C.c_int32, V, P(V)]
            L.lp_nccl_unique_id.argtypes = [V]
            L.lp_nccl_comm_init.argtypes = [P(V), C.c_int, V, C.c_int]
            L.lp_nccl_comm_destroy.argtypes = [V]
            if hasattr(L, "lp_selftest_division"):  # (older builds, loaded for A/B timing, lack it)
                L.lp_selftest_division.argtypes = [C.c_int64, C.c_uint64, P(C.c_int64), P(C.c_int64)]
            L.lp_error_string.argtypes = [C.c_int]
            L.lp_error_string.restype = C.c_char_p
            L.lp_last_error_detail.restype = C.c_char_p
            L.lp_destroy.argtypes = [V]
            _lib = L
    return _lib


def selftest_division(count: int, seed: int = 1):
    """(mismatches, slow_path) of lp_selftest_division: the kernels' division fast path against
    IEEE a / b on `count` device-generated operand pairs."""
    m, sl = C.c_int64(), C.c_int64()
    _check(lib().lp_selftest_division(int(count), int(seed), C.byref(m), C.byref(sl)), "lp_selftest_division")
    return m.value, sl.value


def launch_count() -> int:
    return int(lib().lp_kernel_launch_count())


def _check(code, where):
    if code != 0:
        raise LpError(code, where)


# ------------------------------------------------------------ arrays --------

def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _mem_of(a):
    if a is None:
        return None
    if _is_torch(a):
        return LP_DEVICE if a.is_cuda else LP_HOST
    return LP_HOST


_TORCH_DT = {}


def _torch_dtype(dtype):
    if not _TORCH_DT:
        import torch
        _TORCH_DT.update({np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32})
    return _TORCH_DT[dtype]


class _Arr:
    """A contiguous array of a given dtype on host (numpy) or device (torch)."""

    __slots__ = ("src", "obj", "ptr")

    def __init__(self, a, dtype):
        self.src = a
        if a is None:
            self.obj, self.ptr = None, None
        elif _is_torch(a):
            tdt = _torch_dtype(dtype)
            # already the right dtype and contiguous (the common case): no torch op, just the pointer
            t = a if (a.dtype == tdt and a.is_contiguous()) else a.to(dtype=tdt).contiguous()
            self.obj, self.ptr = t, t.data_ptr()
        else:
            arr = np.ascontiguousarray(a, dtype=dtype)
            self.obj, self.ptr = arr, (arr.ctypes.data if arr.size else None)


def _same_mem(arrs):
    kinds = {_mem_of(a) for a in arrs if a is not None}
    if len(kinds) > 1:
        raise ValueError("mix of host and device arrays in one call")
    return kinds.pop() if kinds else LP_HOST


def _stream_handle(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ------------------------------------------------------------ problem -------

class Problem:
    """The LP of PAPER.md Eq. (1) stacked as K = [G; A] (CSR), q = (h; b)."""

    def __init__(self, n, m1, m2, row_ptr, col_idx, values, c, q, l, u, dense=False):
        self.n, self.m1, self.m2 = int(n), int(m1), int(m2)
        self.row_ptr, self.col_idx, self.values = row_ptr, col_idx, values
        self.c, self.q, self.l, self.u = c, q, l, u
        self.dense = bool(dense)

    @property
    def m(self):
        return self.m1 + self.m2

    @classmethod
    def from_lp(cls, lp):
        """From any object with n, m1, m2, row_ptr, col_idx, val, c, q, l, u (e.g. lpgen.LP)."""
        values = lp.val if hasattr(lp, "val") else lp.values
        return cls(lp.n, lp.m1, lp.m2, lp.row_ptr, lp.col_idx, values, lp.c, lp.q, lp.l, lp.u,
                   getattr(lp, "dense", False))

    def to(self, device):
        import torch
        f = lambda a, dt: None if a is None else torch.as_tensor(np.asarray(a) if not _is_torch(a) else a,
                                                                 dtype=dt, device=device)
        return Problem(self.n, self.m1, self.m2, f(self.row_ptr, torch.int64), f(self.col_idx, torch.int32),
                       f(self.values, torch.float64), f(self.c, torch.float64), f(self.q, torch.float64),
                       f(self.l, torch.float64), f(self.u, torch.float64), self.dense)

    def _desc(self):
        """The lp_problem_desc of this problem (and the arrays it points into, kept alive).  Cached
        while the problem's arrays are the same objects (a batch loop creates handles on one
        problem many times; the descriptor is pure marshalling)."""
        key = tuple(id(a) for a in (self.row_ptr, self.col_idx, self.values, self.c, self.q, self.l, self.u))
        cached = getattr(self, "_desc_cache", None)
        if cached is not None and cached[0] == key:
            return cached[1], cached[2]
        arrs = [_Arr(self.row_ptr, np.int64), _Arr(self.col_idx, np.int32), _Arr(self.values, np.float64),
                _Arr(self.c, np.float64), _Arr(self.q, np.float64), _Arr(self.l, np.float64),
                _Arr(self.u, np.float64)]
        mem = _same_mem([a.src for a in arrs])
        nnz = int(arrs[2].obj.numel() if _is_torch(arrs[2].obj) else arrs[2].obj.size)
        d = ProblemDesc(self.n, self.m1, self.m2, nnz, int(self.dense), mem, *[a.ptr for a in arrs])
        self._desc_cache = (key, d, arrs)
        return d, arrs


def create_lp(c, A=None, b=None, G=None, h=None, l=None, u=None, use_sparse_matrix=True) -> Problem:
    """PAPER.md P:121 `create_lp(c, A, b, G, h, l, u)`: stacks K = [G; A], q = (h; b).
    A and G may be dense arrays or scipy sparse matrices; l/u default to -inf/+inf."""
    c = np.asarray(c, np.float64)
    n = c.size
    try:
        import scipy.sparse as sp
    except Exception:  # pragma: no cover
        sp = None

    def as_csr(M):
        if M is None:
            return sp.csr_matrix((0, n)) if sp else None
        if sp is not None and sp.issparse(M):
            return sp.csr_matrix(M)
        return sp.csr_matrix(np.atleast_2d(np.asarray(M, np.float64)))

    Gm, Am = as_csr(G), as_csr(A)
    K = sp.vstack([Gm, Am]).tocsr()
    K.sum_duplicates()
    K.sort_indices()
    if use_sparse_matrix:
        K.eliminate_zeros()
        rp, ci, v = K.indptr.astype(np.int64), K.indices.astype(np.int32), K.data.astype(np.float64)
        dense = False
    else:
        Kd = K.toarray()
        m = Kd.shape[0]
        rp = (np.arange(m + 1) * n).astype(np.int64)
        ci = np.tile(np.arange(n, dtype=np.int32), m)
        v = Kd.ravel().astype(np.float64)
        dense = True
    hq = np.zeros(0) if h is None else np.atleast_1d(np.asarray(h, np.float64))
    bq = np.zeros(0) if b is None else np.atleast_1d(np.asarray(b, np.float64))
    if hq.size != Gm.shape[0] or bq.size != Am.shape[0] or Gm.shape[1] != n or Am.shape[1] != n:
        raise ValueError("dimension mismatch between c, G, h, A, b")
    l = np.full(n, -np.inf) if l is None else np.asarray(l, np.float64)
    u = np.full(n, np.inf) if u is None else np.asarray(u, np.float64)
    return Problem(n, Gm.shape[0], Am.shape[0], rp, ci, v, c, np.concatenate([hq, bq]), l, u, dense)


_DEFAULTS = None


def default_options(**kw) -> Options:
    global _DEFAULTS
    if _DEFAULTS is None:
        _DEFAULTS = Options()
        lib().lp_default_options(C.byref(_DEFAULTS))
    o = Options.from_buffer_copy(_DEFAULTS)
    rule = kw.pop("step_rule", None)
    if rule is not None:
        o.step_rule = STEP_CONSTANT if rule in ("constant", STEP_CONSTANT) else STEP_ADAPTIVE
    prec = kw.pop("precision", None)
    if prec is not None:
        o.precision = FP32 if prec in ("fp32", FP32) else FP64
    alg = kw.pop("algorithm", None)
    if alg is not None:
        o.algorithm = R2HPDHG if alg in ("r2", "r2hpdhg", "r2HPDHG", R2HPDHG) else RAPDHG
    for k, v in kw.items():
        if v is None:
            continue
        if not hasattr(o, k):
            raise TypeError(f"unknown option {k}")
        setattr(o, k, v)
    return o


def _new_out(shape, like_mem, device):
    if like_mem == LP_DEVICE:
        import torch
        return torch.empty(shape, dtype=torch.float64, device=device)
    return np.zeros(shape)


class Solver:
    """One LP handle: lp_create / lp_solve / lp_get_solution / lp_destroy."""

    def __init__(self, problem: Problem, stream=None):
        self.problem = problem
        d, keep = problem._desc()
        self._mem = d.memory
        self._device = problem.c.device if _is_torch(problem.c) else None
        h = C.c_void_p()
        _check(lib().lp_create(C.byref(d), _stream_handle(stream), C.byref(h)), "lp_create")
        self._h = h
        del keep

    def solve(self, x0=None, y0=None, **opts):
        o = default_options(**opts)
        a, b = _Arr(x0, np.float64), _Arr(y0, np.float64)
        mem = _same_mem([x0, y0])
        if getattr(self, "_alog", None) is not None:   # the decision log's rows start unwritten
            self._alog.fill_(float("nan"))
            self._clog.fill_(float("nan"))
            import torch
            torch.cuda.current_stream().synchronize()
        r = Result()
        _check(lib().lp_solve(self._h, C.byref(o), a.ptr, b.ptr, mem, C.byref(r)), "lp_solve")
        return r.as_dict()

    def solution(self, memory=LP_HOST):
        n, m = self.problem.n, self.problem.m
        x, y, lam = (_new_out(n, memory, self._device), _new_out(m, memory, self._device),
                     _new_out(n, memory, self._device))
        p = lambda t: t.data_ptr() if _is_torch(t) else (t.ctypes.data if t.size else None)
        _check(lib().lp_get_solution(self._h, 0, p(x), p(y) if m else None, p(lam), memory), "lp_get_solution")
        return x, y, lam

    def set_decision_log(self, att_cap=4096, chk_cap=256, device=None):
        """Record the grid path's or the sharded engine's decisions (lp_set_decision_log) into device buffers of the given
        capacities (NaN-filled before every solve); decision_log() returns the rows written.
        att_cap = 0 and chk_cap = 0 switch it off."""
        import torch
        dev = device or (self._device if self._device is not None else "cuda")
        self._alog = torch.full((max(att_cap, 1), 4), float("nan"), dtype=torch.float64, device=dev)
        self._clog = torch.full((max(chk_cap, 1), 6), float("nan"), dtype=torch.float64, device=dev)
        _check(lib().lp_set_decision_log(self._h, self._alog.data_ptr() if att_cap else None, att_cap,
                                         self._clog.data_ptr() if chk_cap else None, chk_cap),
               "lp_set_decision_log")
        if not att_cap and not chk_cap:
            self._alog = self._clog = None

    def decision_log(self):
        """(attempts, checks): numpy arrays of the rows the last solve wrote (the row layout of ora_log, include/lp.h)."""
        a = self._alog.cpu().numpy()
        c = self._clog.cpu().numpy()
        return a[~np.isnan(a[:, 0])], c[~np.isnan(c[:, 0])]

    def scaling(self):
        Dr, Dc = np.zeros(max(self.problem.m, 1)), np.zeros(self.problem.n)
        _check(lib().lp_get_scaling(self._h, Dr.ctypes.data, Dc.ctypes.data, LP_HOST), "lp_get_scaling")
        return Dr[: self.problem.m], Dc

    def spmv_scaled(self, v=None, w=None, out=None):
        """K~ v and K~' w with the solver's scaled matrices (lp_spmv_scaled).  Host (numpy) or
        device (torch) inputs; device calls may pass preallocated outputs (Kv, KTw)."""
        n, m = self.problem.n, self.problem.m
        mem = _same_mem([v, w])
        va, wa = _Arr(v, np.float64), _Arr(w, np.float64)
        if out is not None:
            Kv, KTw = out
        else:
            dev = (v.device if _is_torch(v) else w.device) if mem == LP_DEVICE else None
            Kv = _new_out((max(m, 1),), mem, dev) if v is not None else None
            KTw = _new_out((n,), mem, dev) if w is not None else None
        p = lambda t: None if t is None else (t.data_ptr() if _is_torch(t) else t.ctypes.data)
        _check(lib().lp_spmv_scaled(self._h, va.ptr, p(Kv), wa.ptr, p(KTw), mem), "lp_spmv_scaled")
        return (None if Kv is None else Kv[:m]), KTw

    def close(self):
        if getattr(self, "_h", None):
            lib().lp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class BatchSolver:
    """A batch sharing K, l, u: lp_create_batch / lp_solve_batch."""

    def __init__(self, problem: Problem, C_=None, Q=None, stream=None):
        self.problem = problem
        d, keep = problem._desc()
        ca, qa = _Arr(C_, np.float64), _Arr(Q, np.float64)
        mem = _same_mem([C_, Q])
        if C_ is not None:
            self.batch = int(C_.shape[0])
        elif Q is not None:
            self.batch = int(Q.shape[0])
        else:
            raise ValueError("a batch needs C or Q")
        self._device = problem.c.device if _is_torch(problem.c) else (C_.device if _is_torch(C_) else None)
        h = C.c_void_p()
        _check(lib().lp_create_batch(C.byref(d), self.batch, ca.ptr, qa.ptr, mem, _stream_handle(stream),
                                     C.byref(h)), "lp_create_batch")
        self._h = h
        del keep

    def update(self, C_=None, Q=None):
        ca, qa = _Arr(C_, np.float64), _Arr(Q, np.float64)
        _check(lib().lp_update_batch(self._h, ca.ptr, qa.ptr, _same_mem([C_, Q])), "lp_update_batch")

    def set_decision_log(self, att_cap=4096, chk_cap=256, instance=0, device=None):
        """Record the line-search and restart decisions of batch instance `instance` (register
        kernel, C2 shapes; lp_set_decision_log / lp_set_decision_log_instance)."""
        _check(lib().lp_set_decision_log_instance(self._h, int(instance)), "lp_set_decision_log_instance")
        Solver.set_decision_log(self, att_cap, chk_cap, device)

    decision_log = Solver.decision_log

    def solve(self, X0=None, Y0=None, **opts):
        """Returns a numpy structured array of `batch` results (fields as lp_result);
        res[b]["status"], res["iterations"], ... (no per-instance Python objects)."""
        o = default_options(**opts)
        if getattr(self, "_alog", None) is not None:   # the decision log's rows start unwritten
            self._alog.fill_(float("nan"))
            self._clog.fill_(float("nan"))
            import torch
            torch.cuda.current_stream().synchronize()
        a, b = _Arr(X0, np.float64), _Arr(Y0, np.float64)
        res = np.zeros(self.batch, dtype=RESULT_DTYPE)
        _check(lib().lp_solve_batch(self._h, C.byref(o), a.ptr, b.ptr, _same_mem([X0, Y0]), res.ctypes.data),
               "lp_solve_batch")
        return res

    def spo_plus(self, C_pred, C_true, X_true, obj_true, warm=False, **opts):
        """SPO+ loss and subgradient per instance (lp_spo_plus; Eq. spo+ loss P:76-78 and
        Eq. spo+ gradient P:80-82): returns (loss[B], grad[B, n], results).  Inputs all on
        the host (numpy) or all on the device (torch); outputs live where the inputs do."""
        o = default_options(**opts)
        mem = _same_mem([C_pred, C_true, X_true, obj_true])
        ins = [_Arr(a, np.float64) for a in (C_pred, C_true, X_true, obj_true)]
        B, n = self.batch, self.problem.n
        dev = C_pred.device if _is_torch(C_pred) else self._device
        loss = _new_out((B,), mem, dev)
        grad = _new_out((B, n), mem, dev)
        p = lambda t: t.data_ptr() if _is_torch(t) else t.ctypes.data
        res = np.zeros(B, dtype=RESULT_DTYPE)
        _check(lib().lp_spo_plus(self._h, C.byref(o), ins[0].ptr, ins[1].ptr, ins[2].ptr, ins[3].ptr,
                                 1 if warm else 0, mem, p(loss), p(grad), res.ctypes.data), "lp_spo_plus")
        return loss, grad, res

    def solutions(self, memory=LP_HOST, X=None, Y=None):
        n, m, B = self.problem.n, self.problem.m, self.batch
        X = _new_out((B, n), memory, self._device) if X is None else X
        Y = _new_out((B, m), memory, self._device) if Y is None else Y
        p = lambda t: t.data_ptr() if _is_torch(t) else (t.ctypes.data if t.size else None)
        _check(lib().lp_get_solutions(self._h, p(X), p(Y) if m else None, memory), "lp_get_solutions")
        return X, Y

    def close(self):
        if getattr(self, "_h", None):
            lib().lp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------- sharded ------

def row_partition(row_ptr, parts: int):
    """Contiguous row blocks balanced by nnz (a cut on the row_ptr prefix,
    SURVEY §8(e)); returns parts+1 cut points.  Same rule as the library's
    virtual shards."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    m = rp.size - 1
    cuts = [0]
    for g in range(1, parts):
        t = int(rp[-1]) * g // parts
        c = int(np.searchsorted(rp, t, side="left"))
        cuts.append(min(max(c, cuts[-1]), m))
    cuts.append(m)
    return cuts


def local_rows(problem: Problem, r0: int, r1: int) -> Problem:
    """Rows [r0, r1) of K = [G; A] as a local problem for lp_create_sharded:
    local m1 = the ">=" rows among them; full c, l, u."""
    rp = np.asarray(problem.row_ptr, dtype=np.int64)
    lrp = rp[r0:r1 + 1] - rp[r0]
    m1 = max(0, min(problem.m1 - r0, r1 - r0))
    sl = slice(int(rp[r0]), int(rp[r1]))
    return Problem(problem.n, m1, (r1 - r0) - m1, lrp, np.asarray(problem.col_idx)[sl],
                   np.asarray(problem.values)[sl], problem.c, np.asarray(problem.q)[r0:r1], problem.l, problem.u)


def shard_axis(m: int, n: int) -> int:
    """The axis whose exchanged vector is shorter (lp_shard_axis): columns iff m < n."""
    return int(lib().lp_shard_axis(int(m), int(n)))


def col_partition(problem: Problem, parts: int):
    """Contiguous column blocks balanced by nnz (a cut on the prefix of the column counts);
    returns parts+1 cut points.  Same rule as the library's virtual column shards."""
    n = problem.n
    cc = np.zeros(n + 1, np.int64)
    cc[1:] = np.bincount(np.asarray(problem.col_idx, np.int64), minlength=n)
    cc = np.cumsum(cc)
    nnz = int(cc[-1])
    cuts = [0]
    for g in range(1, parts):
        c = int(np.searchsorted(cc, nnz * g // parts, side="left"))
        cuts.append(min(max(c, cuts[-1]), n))
    cuts.append(n)
    return cuts


def local_cols(problem: Problem, c0: int, c1: int) -> Problem:
    """Columns [c0, c1) of K as a local problem for lp_create_sharded_cols: every row (global m1,
    m2), local column indices, the full q, and c, l, u of those columns."""
    rp = np.asarray(problem.row_ptr, dtype=np.int64)
    ci = np.asarray(problem.col_idx, dtype=np.int64)
    v = np.asarray(problem.values, dtype=np.float64)
    keep = (ci >= c0) & (ci < c1)
    rows = np.repeat(np.arange(rp.size - 1), np.diff(rp))[keep]
    lrp = np.zeros(rp.size, np.int64)
    lrp[1:] = np.bincount(rows, minlength=rp.size - 1)
    lrp = np.cumsum(lrp)
    sl = slice(c0, c1)
    return Problem(c1 - c0, problem.m1, problem.m2, lrp, (ci[keep] - c0).astype(np.int32), v[keep],
                   np.asarray(problem.c)[sl], problem.q, np.asarray(problem.l)[sl], np.asarray(problem.u)[sl])


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().lp_nccl_unique_id(buf), "lp_nccl_unique_id")
    return buf.raw


def nccl_comm_init(nranks: int, uid: bytes, rank: int) -> int:
    comm = C.c_void_p()
    buf = C.create_string_buffer(bytes(uid), 128)
    _check(lib().lp_nccl_comm_init(C.byref(comm), nranks, buf, rank), "lp_nccl_comm_init")
    return comm.value


def nccl_comm_destroy(comm: int):
    lib().lp_nccl_comm_destroy(comm)


class ShardedSolver(Solver):
    """One LP sharded across GPUs by rows (lp_create_sharded) or, axis="cols", by columns
    (lp_create_sharded_cols: `problem` is this rank's local_cols block), or across
    `virtual_shards` blocks on one GPU (lp_create_sharded_virtual_axis; axis "rows", "cols" or
    "auto" = the axis whose exchanged vector is shorter)."""

    def __init__(self, problem: Problem, global_row_offset=0, m1_global=None, m2_global=None, comm=None,
                 rank=0, nranks=1, virtual_shards=None, stream=None, axis="rows", global_col_offset=0,
                 n_global=None):
        self.problem = problem
        d, keep = problem._desc()
        self._device = problem.c.device if _is_torch(problem.c) else None
        h = C.c_void_p()
        ax = {"rows": SHARD_ROWS, "cols": SHARD_COLS, "auto": SHARD_AUTO}.get(axis, axis)
        if virtual_shards is not None and ax == SHARD_ROWS:
            _check(lib().lp_create_sharded_virtual(C.byref(d), int(virtual_shards), _stream_handle(stream),
                                                   C.byref(h)), "lp_create_sharded_virtual")
        elif virtual_shards is not None:
            _check(lib().lp_create_sharded_virtual_axis(C.byref(d), int(virtual_shards), int(ax),
                                                        _stream_handle(stream), C.byref(h)),
                   "lp_create_sharded_virtual_axis")
        elif ax == SHARD_COLS:
            ng = problem.n if n_global is None else n_global
            _check(lib().lp_create_sharded_cols(C.byref(d), int(global_col_offset), int(ng), comm, int(rank),
                                                int(nranks), _stream_handle(stream), C.byref(h)),
                   "lp_create_sharded_cols")
        else:
            m1g = problem.m1 if m1_global is None else m1_global
            m2g = problem.m2 if m2_global is None else m2_global
            _check(lib().lp_create_sharded(C.byref(d), int(global_row_offset), int(m1g), int(m2g), comm, int(rank),
                                           int(nranks), _stream_handle(stream), C.byref(h)), "lp_create_sharded")
        self._h = h
        del keep
