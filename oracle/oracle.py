"""ctypes wrapper of oracle/mpax_oracle.c (TEST INFRASTRUCTURE ONLY).

Argument marshalling only; all arithmetic is in the C file.  The library is
compiled on first use (gcc -O2 -fopenmp -ffp-contract=off), or by
``__graft_entry__.build()``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mpax_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# The same source compiled with FMA contraction (-ffp-contract=fast): an equally valid evaluation
# order of the same arithmetic (reading 27), used by the GPU parity tests only as a
# rounding-sensitivity probe -- how far the oracle's own trajectory moves when every step rounds
# differently.  Never a reference value.
_LIB_FMA = os.path.join(_HERE, "liboracle_fma.so")
# The same source compiled as the fp32 program (-DORA_FP32 -fsingle-precision-constant; DESIGN.md
# reading 39): MPAX's default single precision.  The reference of the fp32 GPU paths.
_LIB_F32 = os.path.join(_HERE, "liboracle_f32.so")
# tests/test_oracle_mutations.py points this at a deliberately mutated build
_LIB_OVERRIDE = os.environ.get("MPAX_ORACLE_LIB")
_lock = threading.Lock()
_lib = None
_lib_fma = None
_lib_f32 = None

OPTIMAL, ITERATION_LIMIT, NUMERICAL_ERROR, PRIMAL_INFEASIBLE, DUAL_INFEASIBLE = 1, 2, 3, 4, 5
RAPDHG, R2HPDHG = 0, 1


def build(force: bool = False, fma: bool = False, f32: bool = False) -> str:
    """Compile the oracle shared library (plain C, no FMA contraction; `fma`: the contracted
    rounding-sensitivity build; `f32`: the fp32 program, reading 39)."""
    out = _LIB_F32 if f32 else _LIB_FMA if fma else _LIB
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        tmp = out + f".tmp{os.getpid()}"
        contract = "-ffp-contract=fast" if fma else "-ffp-contract=off"
        flags = ["-march=x86-64-v3"] if fma else []   # hardware FMA so contraction really happens
        if f32:
            flags = ["-DORA_FP32", "-fsingle-precision-constant"]
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", contract, *flags,
                               "-fno-fast-math", "-fPIC", "-shared", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, out)
    return out


class Problem(C.Structure):
    _fields_ = [("n", C.c_int64), ("m1", C.c_int64), ("m2", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("val", C.c_void_p),
                ("c", C.c_void_p), ("q", C.c_void_p), ("l", C.c_void_p), ("u", C.c_void_p)]


class Options(C.Structure):
    _fields_ = [("eps_abs", C.c_double), ("eps_rel", C.c_double), ("iteration_limit", C.c_int64),
                ("check_frequency", C.c_int32), ("algorithm", C.c_int32),
                ("ruiz_iters", C.c_int32), ("pock_chambolle", C.c_int32),
                ("step_rule", C.c_int32), ("power_iters", C.c_int32),
                ("eps_primal_infeasible", C.c_double), ("eps_dual_infeasible", C.c_double),
                ("eps_feas_polish", C.c_double), ("feasibility_polishing", C.c_int32), ("polish_mode", C.c_int32),
                ("reflection", C.c_double)]


class Options32(C.Structure):
    """ora_options of the fp32 build (every double field is a float there)."""
    _fields_ = [(f, C.c_float if t is C.c_double else t) for f, t in Options._fields_]


class Certificate(C.Structure):
    _fields_ = [("primal_infeasible", C.c_int32), ("dual_infeasible", C.c_int32),
                ("norm_dy", C.c_double), ("dual_ray_objective", C.c_double), ("dual_ray_violation", C.c_double),
                ("norm_dx", C.c_double), ("primal_ray_objective", C.c_double),
                ("primal_ray_violation", C.c_double)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("polish", C.c_int32), ("iterations", C.c_int64),
                ("attempts", C.c_int64), ("restarts", C.c_int64),
                ("primal_objective", C.c_double), ("dual_objective", C.c_double),
                ("primal_residual", C.c_double), ("dual_residual", C.c_double),
                ("gap", C.c_double), ("rel_kkt", C.c_double), ("omega", C.c_double),
                ("eta", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Result32(C.Structure):
    _fields_ = [(f, C.c_float if t is C.c_double else t) for f, t in Result._fields_]

    def as_dict(self):
        return {f: float(getattr(self, f)) if t is C.c_float else getattr(self, f) for f, t in self._fields_}


class Log(C.Structure):
    _fields_ = [("att_cap", C.c_int64), ("att_len", C.c_int64), ("att", C.c_void_p),
                ("chk_cap", C.c_int64), ("chk_len", C.c_int64), ("chk", C.c_void_p)]


class Kkt(C.Structure):
    _fields_ = [("pres", C.c_double), ("dres", C.c_double), ("pobj", C.c_double),
                ("dobj", C.c_double), ("gap", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def lib(fma: bool = False):
    global _lib, _lib_fma
    with _lock:
        if fma and _lib_fma is not None:
            return _lib_fma
        if (fma and _lib_fma is None) or (not fma and _lib is None):
            L = C.CDLL(build(fma=True) if fma else (_LIB_OVERRIDE or build()))
            P = C.POINTER
            L.ora_validate.argtypes = [P(Problem)]
            L.ora_solve.argtypes = [P(Problem), P(Options), C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, P(Result), P(Log)]
            L.ora_solve_batch.argtypes = [P(Problem), C.c_int64, C.c_void_p, C.c_void_p, P(Options),
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, P(Result)]
            L.ora_precondition.argtypes = [P(Problem), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
            L.ora_scaled_problem.argtypes = [P(Problem), C.c_int32, C.c_int32] + [C.c_void_p] * 10
            L.ora_spmv_pair.argtypes = [P(Problem)] + [C.c_void_p] * 4
            L.ora_pdhg_step.argtypes = [P(Problem), C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                        C.c_void_p, C.c_void_p]
            L.ora_step_size.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                        C.c_int64, P(C.c_double), P(C.c_int32), P(C.c_double)]
            L.ora_halpern.argtypes = [C.c_int64, C.c_int64] + [C.c_void_p] * 4
            L.ora_average_update.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_double, C.c_double]
            L.ora_average_update.restype = C.c_double
            L.ora_restart_test.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double]
            L.ora_restart_test.restype = C.c_int32
            L.ora_primal_weight.argtypes = [C.c_double, C.c_double, C.c_double]
            L.ora_primal_weight.restype = C.c_double
            L.ora_termination.argtypes = [P(Kkt), C.c_double, C.c_double, C.c_double, C.c_double]
            L.ora_termination.restype = C.c_int32
            L.ora_rel_kkt.argtypes = [P(Kkt), C.c_double, C.c_double]
            L.ora_rel_kkt.restype = C.c_double
            L.ora_kkt_original.argtypes = [P(Problem), C.c_void_p, C.c_void_p, P(Kkt)]
            L.ora_project_box.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
            L.ora_project_dual.argtypes = [C.c_int64, C.c_void_p]
            L.ora_default_options.argtypes = [P(Options)]
            L.ora_num_threads.restype = C.c_int
            L.ora_set_threads.argtypes = [C.c_int]
            L.ora_spectral_norm.argtypes = [P(Problem), C.c_int32, P(C.c_double)]
            L.ora_halpern_rho.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
            L.ora_certificate_test.argtypes = [P(Problem), C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                               P(Certificate)]
            L.ora_kkt_omega.argtypes = [P(Problem), C.c_double, C.c_void_p, C.c_void_p, P(C.c_double)]
            L.ora_initial_steps.argtypes = [P(Problem), P(Options), P(C.c_double), P(C.c_double)]
            L.ora_restart_candidate.argtypes = [C.c_double, C.c_double]
            L.ora_restart_candidate.restype = C.c_int32
            L.ora_last_timing.argtypes = [P(C.c_double), P(C.c_double)]
            if fma:
                _lib_fma = L
                return L
            _lib = L
    return _lib


def lib32():
    """The fp32 build (reading 39): solve / solve_batch / default options only."""
    global _lib_f32
    with _lock:
        if _lib_f32 is None:
            L = C.CDLL(build(f32=True))
            P = C.POINTER
            L.ora_solve.argtypes = [P(Problem), P(Options32), C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, P(Result32), P(Log)]
            L.ora_solve_batch.argtypes = [P(Problem), C.c_int64, C.c_void_p, C.c_void_p, P(Options32),
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, P(Result32)]
            L.ora_default_options.argtypes = [P(Options32)]
            L.ora_set_threads.argtypes = [C.c_int]
            _lib_f32 = L
    return _lib_f32


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return None if a is None else a.ctypes.data


class _Bound:
    """Keeps the numpy buffers a Problem struct points into alive."""

    def __init__(self, lp, dtype=np.float64):
        self.row_ptr = np.ascontiguousarray(lp.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(lp.col_idx, dtype=np.int32)
        f = lambda a: np.ascontiguousarray(a, dtype=dtype)  # noqa: E731
        self.val = f(lp.val)
        self.c, self.q, self.l, self.u = f(lp.c), f(lp.q), f(lp.l), f(lp.u)
        self.s = Problem(int(lp.n), int(lp.m1), int(lp.m2), int(self.val.size),
                         self.row_ptr.ctypes.data, self.col_idx.ctypes.data, self.val.ctypes.data,
                         self.c.ctypes.data, self.q.ctypes.data if self.q.size else None,
                         self.l.ctypes.data, self.u.ctypes.data)


def options(algorithm="r2", eps_abs=1e-4, eps_rel=1e-4, iteration_limit=None, check_frequency=64,
            step_rule=0, power_iters=200, eps_primal_infeasible=1e-8,
            eps_dual_infeasible=1e-8, feasibility_polishing=False, eps_feas_polish=1e-6, reflection=1.0,
            ruiz_iters=10, pock_chambolle=1):
    o = Options()
    lib().ora_default_options(C.byref(o))
    o.algorithm = R2HPDHG if algorithm in ("r2", "r2hpdhg", R2HPDHG) else RAPDHG
    o.eps_abs, o.eps_rel = eps_abs, eps_rel
    if iteration_limit is not None:
        o.iteration_limit = int(iteration_limit)
    o.check_frequency = check_frequency
    o.ruiz_iters, o.pock_chambolle = ruiz_iters, pock_chambolle
    o.step_rule = 1 if step_rule in (1, "constant") else 0
    o.power_iters = power_iters
    o.eps_primal_infeasible, o.eps_dual_infeasible = eps_primal_infeasible, eps_dual_infeasible
    o.feasibility_polishing, o.eps_feas_polish = int(bool(feasibility_polishing)), eps_feas_polish
    o.reflection = reflection
    return o


def validate(lp) -> int:
    b = _Bound(lp)
    return lib().ora_validate(C.byref(b.s))


def solve(lp, algorithm="r2", eps_abs=1e-4, eps_rel=1e-4, iteration_limit=None, x0=None, y0=None,
          check_frequency=64, log_capacity=0, step_rule=0, eps_primal_infeasible=1e-8, eps_dual_infeasible=1e-8,
          feasibility_polishing=False, eps_feas_polish=1e-6, reflection=1.0, ruiz_iters=10, pock_chambolle=1,
          fma=False, precision="fp64"):
    """Full solve (contract steps 0-6).  Returns a dict with x, y, lam, the
    result fields, and (if log_capacity) the attempt/check decision logs.
    precision="fp32": the fp32 build (reading 39); inputs rounded to single, outputs as float64
    arrays holding the single-precision results."""
    if precision == "fp32":
        return _solve32(lp, algorithm, eps_abs, eps_rel, iteration_limit, x0, y0, check_frequency, step_rule,
                        eps_primal_infeasible, eps_dual_infeasible, feasibility_polishing, eps_feas_polish,
                        reflection, ruiz_iters, pock_chambolle, log_capacity)
    b = _Bound(lp)
    m = lp.m1 + lp.m2
    o = options(algorithm, eps_abs, eps_rel, iteration_limit, check_frequency, step_rule=step_rule,
                eps_primal_infeasible=eps_primal_infeasible, eps_dual_infeasible=eps_dual_infeasible,
                feasibility_polishing=feasibility_polishing, eps_feas_polish=eps_feas_polish,
                reflection=reflection, ruiz_iters=ruiz_iters, pock_chambolle=pock_chambolle)
    x = np.zeros(lp.n)
    y = np.zeros(m)
    lam = np.zeros(lp.n)
    r = Result()
    g = None
    if log_capacity:
        att = np.zeros((log_capacity, 4))
        chk = np.zeros((log_capacity, 6))
        g = Log(log_capacity, 0, att.ctypes.data, log_capacity, 0, chk.ctypes.data)
    x0a = None if x0 is None else _f64(x0)
    y0a = None if y0 is None else _f64(y0)
    e = lib(fma).ora_solve(C.byref(b.s), C.byref(o), _ptr(x0a), _ptr(y0a), x.ctypes.data,
                        y.ctypes.data if m else None, lam.ctypes.data, C.byref(r),
                        C.byref(g) if g is not None else None)
    if e != 0:
        raise ValueError(f"oracle error {e}")
    out = r.as_dict()
    out.update(x=x, y=y, lam=lam)
    if g is not None:
        out["att_log"] = att[: g.att_len].copy()
        out["chk_log"] = chk[: g.chk_len].copy()
    return out


def _options32(o):
    return Options32(*[getattr(o, f) for f, _ in Options._fields_])


def _solve32(lp, algorithm, eps_abs, eps_rel, iteration_limit, x0, y0, check_frequency, step_rule,
             eps_primal_infeasible, eps_dual_infeasible, feasibility_polishing, eps_feas_polish, reflection,
             ruiz_iters, pock_chambolle, log_capacity=0):
    b = _Bound(lp, np.float32)
    m = lp.m1 + lp.m2
    o = _options32(options(algorithm, eps_abs, eps_rel, iteration_limit, check_frequency, step_rule=step_rule,
                           eps_primal_infeasible=eps_primal_infeasible, eps_dual_infeasible=eps_dual_infeasible,
                           feasibility_polishing=feasibility_polishing, eps_feas_polish=eps_feas_polish,
                           reflection=reflection, ruiz_iters=ruiz_iters, pock_chambolle=pock_chambolle))
    x, y, lam = np.zeros(lp.n, np.float32), np.zeros(max(m, 1), np.float32), np.zeros(lp.n, np.float32)
    x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float32)
    y0a = None if y0 is None else np.ascontiguousarray(y0, dtype=np.float32)
    r = Result32()
    g = None
    if log_capacity:   # the decision logs, in the build's precision (float32 records)
        att = np.zeros((log_capacity, 4), np.float32)
        chk = np.zeros((log_capacity, 6), np.float32)
        g = Log(log_capacity, 0, att.ctypes.data, log_capacity, 0, chk.ctypes.data)
    e = lib32().ora_solve(C.byref(b.s), C.byref(o), _ptr(x0a), _ptr(y0a), x.ctypes.data,
                          y.ctypes.data if m else None, lam.ctypes.data, C.byref(r),
                          C.byref(g) if g is not None else None)
    if e != 0:
        raise ValueError(f"oracle error {e}")
    out = r.as_dict()
    out.update(x=x.astype(np.float64), y=y[:m].astype(np.float64), lam=lam.astype(np.float64))
    if g is not None:
        out["att_log"] = att[: g.att_len].astype(np.float64)
        out["chk_log"] = chk[: g.chk_len].astype(np.float64)
    return out


def solve_batch(lp, C_=None, Q=None, algorithm="r2", eps_abs=1e-4, eps_rel=1e-4, iteration_limit=None,
                X0=None, Y0=None, check_frequency=64, threads=None, step_rule=0, eps_primal_infeasible=1e-8,
                eps_dual_infeasible=1e-8, feasibility_polishing=False, eps_feas_polish=1e-6, reflection=1.0,
                fma=False, precision="fp64"):
    """Batch solve sharing K, l, u; one instance per OpenMP thread.  precision="fp32": the fp32
    build (reading 39)."""
    f32 = precision == "fp32"
    dt = np.float32 if f32 else np.float64
    b = _Bound(lp, dt)
    m = lp.m1 + lp.m2
    Cm = None if C_ is None else np.ascontiguousarray(C_, dtype=dt)
    Qm = None if Q is None else np.ascontiguousarray(Q, dtype=dt)
    B = Cm.shape[0] if Cm is not None else Qm.shape[0]
    o = options(algorithm, eps_abs, eps_rel, iteration_limit, check_frequency, step_rule=step_rule,
                eps_primal_infeasible=eps_primal_infeasible, eps_dual_infeasible=eps_dual_infeasible,
                feasibility_polishing=feasibility_polishing, eps_feas_polish=eps_feas_polish,
                reflection=reflection)
    X = np.zeros((B, lp.n), dt)
    Y = np.zeros((B, m), dt)
    res = ((Result32 if f32 else Result) * B)()
    L = lib32() if f32 else lib(fma)
    if f32:
        o = _options32(o)
    if threads:
        L.ora_set_threads(int(threads))
    X0a = None if X0 is None else np.ascontiguousarray(X0, dtype=dt)
    Y0a = None if Y0 is None else np.ascontiguousarray(Y0, dtype=dt)
    e = L.ora_solve_batch(C.byref(b.s), B, _ptr(Cm), _ptr(Qm), C.byref(o), _ptr(X0a), _ptr(Y0a),
                          X.ctypes.data, Y.ctypes.data if m else None, res)
    if e != 0:
        raise ValueError(f"oracle error {e}")
    return X.astype(np.float64), Y.astype(np.float64), [r.as_dict() for r in res]


def num_threads() -> int:
    return int(lib().ora_num_threads())


def set_threads(t: int):
    """t > 0: that many OpenMP threads; t <= 0: every core this process may use."""
    import os
    lib().ora_set_threads(int(t) if t > 0 else len(os.sched_getaffinity(0)))


def precondition(lp, ruiz_iters=10, pock_chambolle=1):
    b = _Bound(lp)
    Dr = np.zeros(max(lp.m1 + lp.m2, 1))
    Dc = np.zeros(lp.n)
    lib().ora_precondition(C.byref(b.s), ruiz_iters, pock_chambolle, Dr.ctypes.data, Dc.ctypes.data)
    return Dr[: lp.m1 + lp.m2], Dc


def scaled_problem(lp, ruiz_iters=10, pock_chambolle=1):
    """Step 1 outputs: dict(Dr, Dc, Kv, KT_row_ptr, KT_col_idx, KTv, c, q, l, u)."""
    b = _Bound(lp)
    n, m, nnz = lp.n, lp.m1 + lp.m2, b.val.size
    out = dict(Dr=np.zeros(max(m, 1)), Dc=np.zeros(n), Kv=np.zeros(max(nnz, 1)),
               KT_row_ptr=np.zeros(n + 1, np.int64), KT_col_idx=np.zeros(max(nnz, 1), np.int32),
               KTv=np.zeros(max(nnz, 1)), c=np.zeros(n), q=np.zeros(max(m, 1)), l=np.zeros(n),
               u=np.zeros(n))
    e = lib().ora_scaled_problem(C.byref(b.s), ruiz_iters, pock_chambolle, out["Dr"].ctypes.data,
                                 out["Dc"].ctypes.data, out["Kv"].ctypes.data,
                                 out["KT_row_ptr"].ctypes.data, out["KT_col_idx"].ctypes.data,
                                 out["KTv"].ctypes.data, out["c"].ctypes.data, out["q"].ctypes.data,
                                 out["l"].ctypes.data, out["u"].ctypes.data)
    if e != 0:
        raise ValueError(f"oracle error {e}")
    for k in ("Dr", "q"):
        out[k] = out[k][:m]
    for k in ("Kv", "KT_col_idx", "KTv"):
        out[k] = out[k][:nnz]
    return out


def spmv_pair(lp, x=None, w=None):
    b = _Bound(lp)
    m = lp.m1 + lp.m2
    xa = None if x is None else _f64(x)
    wa = None if w is None else _f64(w)
    Kx = np.zeros(max(m, 1)) if x is not None else None
    KTw = np.zeros(lp.n) if w is not None else None
    lib().ora_spmv_pair(C.byref(b.s), _ptr(xa), _ptr(Kx), _ptr(wa), _ptr(KTw))
    return (None if Kx is None else Kx[:m]), KTw


def pdhg_step(lp, x, y, tau, sigma):
    b = _Bound(lp)
    m = lp.m1 + lp.m2
    xo, yo = np.zeros(lp.n), np.zeros(max(m, 1))
    xa, ya = _f64(x), _f64(y) if m else np.zeros(1)
    lib().ora_pdhg_step(C.byref(b.s), xa.ctypes.data, ya.ctypes.data, tau, sigma, xo.ctypes.data,
                        yo.ctypes.data)
    return xo, yo[:m]


def step_size(eta, omega, dx2, dy2, interaction, j):
    eb, acc, en = C.c_double(), C.c_int32(), C.c_double()
    lib().ora_step_size(eta, omega, dx2, dy2, interaction, j, C.byref(eb), C.byref(acc), C.byref(en))
    return eb.value, bool(acc.value), en.value


def halpern(k, z, w, z0):
    z, w, z0 = _f64(z), _f64(w), _f64(z0)
    out = np.zeros_like(z)
    lib().ora_halpern(z.size, k, z.ctypes.data, w.ctypes.data, z0.ctypes.data, out.ctypes.data)
    return out


def halpern_rho(k, z, w, z0, rho):
    """Partial reflection step a((1 + rho) w - rho z) + b z0 (reading 38)."""
    z, w, z0 = _f64(z), _f64(w), _f64(z0)
    out = np.zeros_like(z)
    lib().ora_halpern_rho(z.size, k, rho, z.ctypes.data, w.ctypes.data, z0.ctypes.data, out.ctypes.data)
    return out


def average_update(avg, z, W, eta):
    avg = _f64(avg).copy()
    z = _f64(z)
    W1 = lib().ora_average_update(avg.size, avg.ctypes.data, z.ctypes.data, W, eta)
    return avg, W1


def restart_test(k_in, k, metric, ref, last):
    return bool(lib().ora_restart_test(k_in, k, metric, ref, last))


def primal_weight(omega, dx, dy):
    return lib().ora_primal_weight(omega, dx, dy)


def termination(kkt: dict, norm_q, norm_c, eps_abs, eps_rel):
    k = Kkt(kkt["pres"], kkt["dres"], kkt["pobj"], kkt["dobj"], kkt["gap"])
    return bool(lib().ora_termination(C.byref(k), norm_q, norm_c, eps_abs, eps_rel))


def rel_kkt(kkt: dict, norm_q, norm_c):
    k = Kkt(kkt["pres"], kkt["dres"], kkt["pobj"], kkt["dobj"], kkt["gap"])
    return lib().ora_rel_kkt(C.byref(k), norm_q, norm_c)


def kkt_original(lp, x, y):
    b = _Bound(lp)
    xa = _f64(x)
    ya = _f64(y) if (lp.m1 + lp.m2) else np.zeros(1)
    k = Kkt()
    lib().ora_kkt_original(C.byref(b.s), xa.ctypes.data, ya.ctypes.data, C.byref(k))
    return k.as_dict()


def project_box(x, l, u):
    x, l, u = _f64(x).copy(), _f64(l), _f64(u)
    lib().ora_project_box(x.size, l.ctypes.data, u.ctypes.data, x.ctypes.data)
    return x


def project_dual(y, m1):
    y = _f64(y).copy()
    lib().ora_project_dual(m1, y.ctypes.data)
    return y


def spectral_norm(lp, iters=200):
    """sigma_max(K) of the problem's (unscaled) K by the oracle's power iteration."""
    b = _Bound(lp)
    s = C.c_double()
    lib().ora_spectral_norm(C.byref(b.s), iters, C.byref(s))
    return s.value


def certificate_test(lp, dx, dy, eps_primal_infeasible=1e-8, eps_dual_infeasible=1e-8):
    """Reading 35's certificate test on original-space rays (d_x, d_y)."""
    b = _Bound(lp)
    dxa, dya = _f64(dx), _f64(dy)
    r = Certificate()
    e = lib().ora_certificate_test(C.byref(b.s), dxa.ctypes.data, dya.ctypes.data if dya.size else None,
                                   eps_primal_infeasible, eps_dual_infeasible, C.byref(r))
    if e != 0:
        raise ValueError(f"oracle error {e}")
    return {f: getattr(r, f) for f, _ in r._fields_}


def kkt_omega(lp, omega, x, y):
    """The raPDHG restart metric sqrt(omega pres^2 + dres^2/omega + gap^2) of (x, y) on the
    problem as given (contract step 5)."""
    b = _Bound(lp)
    xa = _f64(x)
    ya = _f64(y) if (lp.m1 + lp.m2) else np.zeros(1)
    out = C.c_double()
    lib().ora_kkt_omega(C.byref(b.s), omega, xa.ctypes.data, ya.ctypes.data, C.byref(out))
    return out.value


def initial_steps(lp, step_rule=0, ruiz_iters=10, pock_chambolle=1):
    """(omega0, eta0) of contract step 2 on the problem scaled with the given rounds."""
    b = _Bound(lp)
    o = options("ra", step_rule=step_rule, ruiz_iters=ruiz_iters, pock_chambolle=pock_chambolle)
    om, et = C.c_double(), C.c_double()
    e = lib().ora_initial_steps(C.byref(b.s), C.byref(o), C.byref(om), C.byref(et))
    if e != 0:
        raise ValueError(f"oracle error {e}")
    return om.value, et.value


def restart_candidate(kkt_omega_avg, kkt_omega_cur):
    """'avg' if the average's KKT_omega is strictly smaller, else 'cur' (reading c.3 #10)."""
    return "avg" if lib().ora_restart_candidate(kkt_omega_avg, kkt_omega_cur) else "cur"


def last_timing():
    """(setup_s, solve_s) of this thread's last oracle.solve: validation + preconditioning +
    scaled copies, then steps 2-6 (wall clock; timing only)."""
    a, b = C.c_double(), C.c_double()
    lib().ora_last_timing(C.byref(a), C.byref(b))
    return a.value, b.value
