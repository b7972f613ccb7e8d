"""ctypes front-end for the two CPU checkers (see oracle/__init__.py)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2407_16144_b200 import abi
from paper_2407_16144_b200.abi import dptr, i32ptr, i64ptr

HERE = Path(__file__).resolve().parent
LIBS = {"port": (HERE / "liboracle.so", "orc_"), "reference": (HERE / "_ref" / "libhplp_ref.so", "ref_"),
        # the same reference sources built -O3 / AVX2 + FMA: timing only (bench.py)
        "reference_fast": (HERE / "_ref" / "libhplp_ref_fast.so", "ref_")}
REF_SRC = Path(os.environ.get("HPLP_REFERENCE", "/root/reference/proj"))

_cache: dict[str, C.CDLL] = {}


def build(kinds=("port", "reference"), quiet=True) -> None:
    """Compile the checkers with oracle/Makefile.  The reference build needs
    /root/reference (present in the build container, absent on GPU boxes,
    where the prebuilt .so travels with the repo snapshot)."""
    out = subprocess.DEVNULL if quiet else None
    if "port" in kinds:
        subprocess.run(["make", "-s", "liboracle.so"], cwd=HERE, check=True, stdout=out)
    if "reference" in kinds and (REF_SRC / "src").is_dir():
        subprocess.run(["make", "-s", "ref", "ref_fast", f"REF={REF_SRC}"], cwd=HERE, check=True, stdout=out)


def available(kind: str) -> bool:
    return LIBS[kind][0].exists()


def load(kind: str = "port") -> C.CDLL:
    if kind in _cache:
        return _cache[kind]
    path, p = LIBS[kind]
    if not path.exists():
        if kind == "port":
            build(("port",))
        else:
            raise FileNotFoundError(f"{path} not built (run make -C oracle ref)")
    lib = C.CDLL(str(path))
    V, I64, I32, D = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    PD, PI64, PI32 = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32)

    def sig(name, res, *args):
        f = getattr(lib, p + name)
        f.restype, f.argtypes = res, list(args)

    sig("last_error", C.c_char_p)
    sig("lp_create", C.c_int, I64, I64, PI64, PI32, PD, PD, PD, C.POINTER(V))
    sig("lp_free", None, V)
    if hasattr(lib, p + "power_start"):  # the restatement only
        sig("power_start", C.c_int, I64, C.c_uint64, PD)
    sig("spmv", C.c_int, V, PD, PD)
    sig("spmv_transpose", C.c_int, V, PD, PD)
    sig("power_iteration", C.c_int, V, D, I64, C.c_uint64, PD, PI64, PI32, PD)
    sig("pdhg_step", C.c_int, V, D, PD, PD, PD, PD, PD, PD, PD)
    sig("kkt_error", C.c_int, V, PD, PD, C.POINTER(abi.Kkt))
    sig("canonical_norm_with_product", C.c_int, I64, I64, PD, PD, PD, D, PD)
    sig("validate_primal", C.c_int, V, PD, D, D, PD)
    sig("validate_dual", C.c_int, V, PD, D, D, PD)
    sig("should_restart", C.c_int, I32, I64, D, I64, I64, I64, D, D)
    sig("lp_solve", C.c_int, V, C.POINTER(abi.Config), C.POINTER(abi.IO), C.POINTER(abi.Result))
    sig("lp_solve_baseline", C.c_int, V, C.c_int32, C.POINTER(abi.Config), C.POINTER(abi.IO), C.POINTER(abi.Result))
    sig("to_standard_form", C.c_int, C.POINTER(abi.General), C.POINTER(V), PI64, PI64, PI64)
    sig("std_export", C.c_int, V, PI64, PI32, PD, PD, PD)
    sig("std_recover", C.c_int, V, PD, PD, D, PD)
    sig("std_lp", C.c_int, V, C.POINTER(V))
    sig("std_free", None, V)
    lib._prefix = p
    _cache[kind] = lib
    return lib


class CheckerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _chk(lib, rc):
    if rc != 0:
        msg = getattr(lib, lib._prefix + "last_error")().decode()
        exc = {abi.HPLP_EINVAL: ValueError, abi.HPLP_EDOMAIN: ArithmeticError}.get(rc)
        if exc:
            raise exc(msg)
        raise CheckerError(rc, msg)


def _f(lib, name):
    return getattr(lib, lib._prefix + name)


class CpuLp:
    """A StandardFormLP held by one of the CPU checkers."""

    def __init__(self, kind, m, n, row_ptr, col_idx, val, b, c, _handle=None):
        self.kind = kind
        self.lib = load(kind)
        self.m, self.n = int(m), int(n)
        if _handle is not None:
            self.h = _handle
            return
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col_idx = np.ascontiguousarray(col_idx, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        c = np.ascontiguousarray(c, np.float64)
        h = C.c_void_p()
        _chk(self.lib, _f(self.lib, "lp_create")(self.m, self.n, i64ptr(row_ptr), i32ptr(col_idx),
                                                 dptr(val), dptr(b), dptr(c), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            _f(self.lib, "lp_free")(self.h)
        except Exception:
            pass

    def set_box(self, u):
        """Box form (port only; no reference counterpart): column upper bounds u
        (+inf = none) enforced by the primal projection; None clears."""
        if self.kind != "port":
            raise ValueError("the box form exists only in the port (the reference has no counterpart)")
        if u is None:
            _chk(self.lib, _f(self.lib, "lp_set_box")(self.h, None))
            return self
        self._box_u = np.ascontiguousarray(u, np.float64)
        _chk(self.lib, _f(self.lib, "lp_set_box")(self.h, dptr(self._box_u)))
        return self

    def spmv(self, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(self.m)
        _chk(self.lib, _f(self.lib, "spmv")(self.h, dptr(x), dptr(out)))
        return out

    def spmv_transpose(self, y):
        y = np.ascontiguousarray(y, np.float64)
        out = np.empty(self.n)
        _chk(self.lib, _f(self.lib, "spmv_transpose")(self.h, dptr(y), dptr(out)))
        return out

    def power_iteration(self, tol=1e-4, max_iters=5000, seed=12345):
        s, it, cv, sec = C.c_double(), C.c_int64(), C.c_int32(), C.c_double()
        _chk(self.lib, _f(self.lib, "power_iteration")(self.h, tol, max_iters, seed, C.byref(s),
                                                       C.byref(it), C.byref(cv), C.byref(sec)))
        return s.value, it.value, bool(cv.value), sec.value

    def pdhg_step(self, eta, x, y, a_x):
        x, y, a_x = (np.ascontiguousarray(v, np.float64) for v in (x, y, a_x))
        xn, yn, axn, aty = np.empty(self.n), np.empty(self.m), np.empty(self.m), np.empty(self.n)
        _chk(self.lib, _f(self.lib, "pdhg_step")(self.h, eta, dptr(x), dptr(y), dptr(a_x), dptr(xn),
                                                 dptr(yn), dptr(axn), dptr(aty)))
        return xn, yn, axn, aty

    def kkt_error(self, x, y):
        x, y = np.ascontiguousarray(x, np.float64), np.ascontiguousarray(y, np.float64)
        k = abi.Kkt()
        _chk(self.lib, _f(self.lib, "kkt_error")(self.h, dptr(x), dptr(y), C.byref(k)))
        return k.as_tuple()

    def canonical_norm_with_product(self, dx, dy, a_dx, eta):
        dx, dy, a_dx = (np.ascontiguousarray(v, np.float64) for v in (dx, dy, a_dx))
        out = C.c_double()
        _chk(self.lib, _f(self.lib, "canonical_norm_with_product")(len(dx), len(dy), dptr(dx), dptr(dy),
                                                                   dptr(a_dx), eta, C.byref(out)))
        return out.value

    def validate_primal(self, v_y, tol, sigma):
        v_y = np.ascontiguousarray(v_y, np.float64)
        r = np.empty(4)
        _chk(self.lib, _f(self.lib, "validate_primal")(self.h, dptr(v_y), tol, sigma, dptr(r)))
        return dict(residual=r[0], margin=r[1], orientation=int(r[2]), valid=bool(r[3]))

    def validate_dual(self, v_x, tol, sigma):
        v_x = np.ascontiguousarray(v_x, np.float64)
        r = np.empty(4)
        _chk(self.lib, _f(self.lib, "validate_dual")(self.h, dptr(v_x), tol, sigma, dptr(r)))
        return dict(residual=r[0], margin=r[1], orientation=int(r[2]), valid=bool(r[3]))

    def should_restart(self, kind, n, k, res_now, res_start, k_star=0, beta=0.36787944117144233, tau0=32):
        return bool(_f(self.lib, "should_restart")(kind, k_star, beta, tau0, n, k, res_now, res_start))

    def solve_baseline(self, mode, config=None, init=None, trace=False, epochs_capacity=4096, **kw):
        """solve_baseline() (src/solver.cpp:344-509): mode 0 vanilla PDHG, 1
        averaged, 2 restarted average.  Same result dict as solve()."""
        return self.solve(config, init, trace, epochs_capacity, _baseline=int(mode), **kw)

    def solve(self, config=None, init=None, trace=False, epochs_capacity=4096, _baseline=-1, sink=None, **kw):
        """solve() (src/solver.cpp:206-342).  Returns a dict with the result
        fields, final x/y, certificates, epochs and (trace=True) the per-
        iteration trace records with their iterates.  sink(record, x, y):
        called per trace record instead of keeping copies (x, y are views
        valid during the call) -- for instances too large to keep 100
        iterates of."""
        cfg = config if config is not None else abi.Config.default(**kw)
        x, y = np.empty(self.n), np.empty(self.m)
        pc, dc = np.zeros(self.m), np.zeros(self.n)
        eps = (abi.Epoch * epochs_capacity)()
        recs = []

        def record(rec, xp, n, yp, m, user):
            r = rec.contents
            d = dict(epoch=r.epoch, inner=r.inner, iteration=r.iteration,
                     res=r.fixed_point_residual, kkt=r.kkt.as_tuple(),
                     cand_norm_normalized=r.candidate_norm_normalized,
                     cand_norm_difference=r.candidate_norm_difference,
                     partition=abi.trace_partition(r))
            if sink is not None:
                sink(d, np.ctypeslib.as_array(xp, (n,)), np.ctypeslib.as_array(yp, (m,)))
                return
            d["x"] = np.ctypeslib.as_array(xp, (n,)).copy()
            d["y"] = np.ctypeslib.as_array(yp, (m,)).copy()
            recs.append(d)

        cb = abi.TRACE_FN(record) if trace else abi.TRACE_FN()
        if trace and cfg.trace_period == 0:
            cfg.trace_period = 1
        ix = iy = None
        if init is not None:
            ix = np.ascontiguousarray(init[0], np.float64)
            iy = np.ascontiguousarray(init[1], np.float64)
        io = abi.IO(dptr(ix), dptr(iy), dptr(x), dptr(y), dptr(pc), dptr(dc), eps, epochs_capacity, cb, None)
        res = abi.Result()
        if _baseline < 0:
            _chk(self.lib, _f(self.lib, "lp_solve")(self.h, C.byref(cfg), C.byref(io), C.byref(res)))
        else:
            _chk(self.lib, _f(self.lib, "lp_solve_baseline")(self.h, _baseline, C.byref(cfg), C.byref(io),
                                                            C.byref(res)))
        ne = min(res.n_epochs, epochs_capacity)
        return dict(
            status=abi.STATUS_NAMES[res.status], status_code=res.status, iterations=res.iterations,
            spmv_count=res.spmv_count, wall_seconds=res.wall_seconds, eta=res.eta,
            sigma_estimate=res.sigma_estimate, kkt=res.final_kkt.as_tuple(), n_epochs=res.n_epochs,
            epochs=[(e.epoch, e.restart_length, e.residual_at_start, e.kkt_at_start.as_tuple())
                    for e in eps[:ne]],
            x=x, y=y,
            primal_cert=(pc, _meta(res.primal_cert)) if res.primal_cert.present else None,
            dual_cert=(dc, _meta(res.dual_cert)) if res.dual_cert.present else None,
            trace=recs,
        )


def _meta(m):
    return dict(source=m.source, orientation=m.orientation, at_iteration=m.at_iteration,
                residual=m.residual, margin=m.margin)


class CpuStd:
    """to_standard_form output held by a checker: CSR arrays + VariableMap."""

    def __init__(self, kind, general: abi.General):
        self.kind = kind
        self.lib = load(kind)
        h = C.c_void_p()
        ms, ns, nz = C.c_int64(), C.c_int64(), C.c_int64()
        _chk(self.lib, _f(self.lib, "to_standard_form")(C.byref(general), C.byref(h), C.byref(ms),
                                                        C.byref(ns), C.byref(nz)))
        self.h = h
        self.m, self.n, self.nnz = ms.value, ns.value, nz.value
        self.row_ptr = np.empty(self.m + 1, np.int64)
        self.col_idx = np.empty(self.nnz, np.int32)
        self.val = np.empty(self.nnz)
        self.b, self.c = np.empty(self.m), np.empty(self.n)
        _chk(self.lib, _f(self.lib, "std_export")(h, i64ptr(self.row_ptr), i32ptr(self.col_idx),
                                                  dptr(self.val), dptr(self.b), dptr(self.c)))

    def lp(self) -> CpuLp:
        h = C.c_void_p()
        _chk(self.lib, _f(self.lib, "std_lp")(self.h, C.byref(h)))
        return CpuLp(self.kind, self.m, self.n, None, None, None, None, None, _handle=h)

    def recover(self, x_std, std_objective, n_orig):
        x_std = np.ascontiguousarray(x_std, np.float64)
        xo = np.empty(n_orig)
        obj = C.c_double()
        _chk(self.lib, _f(self.lib, "std_recover")(self.h, dptr(x_std), dptr(xo), std_objective, C.byref(obj)))
        return xo, obj.value

    def __del__(self):
        try:
            _f(self.lib, "std_free")(self.h)
        except Exception:
            pass
