"""Python front-end of the B200 rHPDHG solver (ctypes over include/hplp_gpu.h
and include/hx.h).

Names mirror the reference API (/root/reference/proj/include/hplp):
``to_standard_form``, ``Solver.solve`` / ``solve`` (SolverConfig fields as
keyword arguments), status strings of ``to_string(SolveStatus)``.  There is
no CPU path: if libhplp_gpu.so cannot be loaded, or no B200 is visible, every
call raises.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import abi
from .abi import dptr, i32ptr, i64ptr
from .build import GPU_LIB, ensure_built


class HplpError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class HxProgress(C.Structure):
    """hx_progress_t (include/hx.h)."""

    _fields_ = [
        ("it", C.c_int64), ("n", C.c_int64), ("k", C.c_int64), ("spmv_count", C.c_int64),
        ("status", C.c_int32), ("error", C.c_int32), ("paused", C.c_int32), ("best_valid", C.c_int32),
        ("res_epoch_start", C.c_double), ("best_kkt", C.c_double), ("best_err", abi.Kkt),
        ("trace_it", C.c_int64), ("trace_n", C.c_int64), ("trace_k", C.c_int64),
        ("trace_res", C.c_double), ("trace_kkt", abi.Kkt), ("final_kkt", abi.Kkt),
        ("n_epochs", C.c_int64), ("primal_cert", abi.CertMeta), ("dual_cert", abi.CertMeta),
        ("device_ms", C.c_double), ("launches", C.c_int64), ("trace_res_diff", C.c_double),
    ]


_lib = None


def lib() -> C.CDLL:
    """Load libhplp_gpu.so (building it in-tree if needed)."""
    global _lib
    if _lib is not None:
        return _lib
    ensure_built()
    if not GPU_LIB.exists():
        raise HplpError(abi.HPLP_ECUDA, f"{GPU_LIB} missing: the B200 path has no CPU fallback")
    L = C.CDLL(str(GPU_LIB))
    V, I64, I32, D = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    PD, PI64, PI32, PV = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_void_p)

    def sig(name, res, *args):
        f = getattr(L, name)
        f.restype, f.argtypes = res, list(args)

    sig("hplp_last_error", C.c_char_p)
    sig("hplp_status_string", C.c_char_p, I32)
    sig("hplp_validate_config", C.c_int, C.POINTER(abi.Config))
    sig("hplp_power_start", C.c_int, I64, C.c_uint64, PD)
    sig("hplp_solve_csr", C.c_int, I32, I64, I64, PI64, PI32, PD, PD, PD, C.POINTER(abi.Config),
        C.POINTER(abi.IO), C.POINTER(abi.Result))
    sig("hplp_solver_create", C.c_int, I32, I64, I64, PI64, PI32, PD, PD, PD, PV)
    sig("hplp_solver_solve", C.c_int, V, C.POINTER(abi.Config), C.POINTER(abi.IO), C.POINTER(abi.Result))
    sig("hplp_solver_create_team", C.c_int, PI32, I32, I32, I32, I64, I64, PI64, PI32, PD, PD, PD, PV)
    sig("hplp_solver_rank_hx", V, V, I32)
    sig("hplp_solver_create_rank", C.c_int, I32, I32, I32, I64, I64, PI64, PI32, PD, PD, PD, PV)
    sig("hplp_solver_team_export", C.c_int, V, C.c_char_p, I64, PI64)
    sig("hplp_solver_team_import", C.c_int, V, C.c_char_p, I64)
    sig("hplp_plan_partition", C.c_int, I64, I64, PI64, PI32, I32, PI64, PI64)
    sig("hplp_solver_create_box", C.c_int, I32, I64, I64, PI64, PI32, PD, PD, PD, PV)
    sig("hplp_box_form_dims", C.c_int, I64, I64, PI64, PI32, PD, PD, PD, PI64, PI64, PD)
    # MPS ingestion + reports (inc/hplp/mps_io.hpp)
    sig("hplp_mps_parse", C.c_int, C.c_char_p, PV, PI64, PI64, PI64)
    sig("hplp_mps_view", C.c_int, V, C.POINTER(abi.General))
    sig("hplp_mps_names", C.c_int, V, I32, C.c_char_p, I64, PI64)
    sig("hplp_mps_write", C.c_int, V, C.c_char_p, I64, PI64)
    sig("hplp_mps_from_general", C.c_int, C.POINTER(abi.General), C.c_char_p, I64, PI64)
    sig("hplp_mps_free", None, V)
    sig("hplp_solve_mps", C.c_int, I32, C.c_char_p, C.POINTER(abi.Config), C.c_char_p, I64, C.c_char_p, I64, PI64,
        C.c_char_p, I64, PI64, PI32)
    sig("hplp_json_normalize", C.c_int, C.c_char_p, I32, C.c_char_p, I64, PI64)
    sig("hplp_solver_hx", V, V)
    sig("hplp_solver_free", None, V)
    sig("hplp_to_standard_form", C.c_int, C.POINTER(abi.General), PV, PI64, PI64, PI64)
    sig("hplp_std_export", C.c_int, V, PI64, PI32, PD, PD, PD)
    sig("hplp_std_recover", C.c_int, V, PD, PD, D, PD)
    sig("hplp_std_free", None, V)
    sig("hplp_solve_general", C.c_int, I32, C.POINTER(abi.General), C.POINTER(abi.Config), C.POINTER(abi.IO),
        C.POINTER(abi.Result), PD, PD)
    # hx layer
    sig("hx_create", C.c_int, I32, PV)
    sig("hx_destroy", None, V)
    sig("hx_last_error", C.c_char_p, V)
    sig("hx_device_info", C.c_int, V, PI32, PI32, PI32)
    sig("hx_stream", V, V)
    sig("hx_launch_count", I64, V)
    sig("hx_upload_csr", C.c_int, V, I64, I64, PI64, PI32, PD, PD, PD)
    sig("hx_dims", C.c_int, V, PI64, PI64, PI64)
    sig("hx_loop_variant", I32, V)
    sig("hx_spmv", C.c_int, V, PD, PD)
    sig("hx_spmv_transpose", C.c_int, V, PD, PD)
    sig("hx_power_iteration", C.c_int, V, PD, D, I64, I64, D, PD, PI64, PI32, PI32)
    sig("hx_setup", C.c_int, V, C.POINTER(abi.Config), D, D, PD, PD)
    sig("hx_run", C.c_int, V, I64, C.POINTER(HxProgress))
    sig("hx_progress", C.c_int, V, C.POINTER(HxProgress))
    sig("hx_epochs", C.c_int, V, I64, I64, C.POINTER(abi.Epoch))
    sig("hx_get_iterate", C.c_int, V, I32, PD, PD)
    sig("hx_get_certificate", C.c_int, V, I32, PD)
    sig("hx_kkt_current", C.c_int, V, C.POINTER(abi.Kkt))
    sig("hx_sizeof", I64, I32)
    sig("hx_profile", C.c_int, V, C.POINTER(C.c_uint64), I32)
    sig("hx_sched_tasks", C.c_int, V, I32, C.POINTER(C.c_int32), I64, C.POINTER(C.c_int64))
    sig("hx_precondition", C.c_int, V, I32, D, PD, PD)
    sig("hx_set_sum_order", C.c_int, V, I32)
    sig("hx_stored_nonzeros", C.c_int, V, C.POINTER(C.c_int64), C.POINTER(C.c_int64))
    sig("hx_schedule_info", C.c_int, C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.c_double, C.POINTER(C.c_int32),
        C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_double))
    sig("hx_trace_reduced_costs", C.c_int, V, PD)
    sig("hx_sum_order", I32, V)
    sig("hx_set_default_sum_order", C.c_int, I32)
    sig("hx_download_problem", C.c_int, V, PI64, PI32, PD, PD, PD)
    sig("hx_set_partition", C.c_int, V, I32, I32, PI64, PI64, I32)
    sig("hx_team_bind", C.c_int, PV, I32)
    sig("hx_team_export", C.c_int, V, C.c_char_p, I64, PI64)
    sig("hx_team_import", C.c_int, V, C.c_char_p, I64)
    sig("hx_team_run", C.c_int, PV, I32, I64, C.POINTER(HxProgress))
    _lib = L
    return L


class MpsParseError(ValueError):
    """MpsParseError of inc/hplp/mps_io.hpp:29-39 (message starts "line N: ")."""

    def __init__(self, msg: str):
        super().__init__(msg)
        try:
            self.line = int(msg.split(":", 1)[0].split()[1])
        except (IndexError, ValueError):
            self.line = -1


def _check(rc: int, ctx=None) -> None:
    if rc == 0:
        return
    L = lib()
    msg = (L.hx_last_error(ctx) if ctx is not None else L.hplp_last_error()).decode()
    if rc == abi.HPLP_EPARSE:
        raise MpsParseError(msg)
    if rc == abi.HPLP_EINVAL:
        raise ValueError(msg)
    if rc == abi.HPLP_EDOMAIN:
        raise ArithmeticError(msg)
    raise HplpError(rc, msg)


def to_string(status: int) -> str:
    """to_string(SolveStatus), src/solver.cpp:176-192."""
    return lib().hplp_status_string(status).decode()


class StdForm:
    """to_standard_form output: standard-form CSR + VariableMap handle."""

    def __init__(self, general):
        L = lib()
        self._g = general
        ga = general.as_abi()
        h = C.c_void_p()
        m, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        _check(L.hplp_to_standard_form(C.byref(ga), C.byref(h), C.byref(m), C.byref(n), C.byref(nnz)))
        self.h = h
        self.m, self.n, self.nnz = m.value, n.value, nnz.value
        self.row_ptr = np.empty(self.m + 1, np.int64)
        self.col_idx = np.empty(self.nnz, np.int32)
        self.val = np.empty(self.nnz)
        self.b, self.c = np.empty(self.m), np.empty(self.n)
        _check(L.hplp_std_export(h, i64ptr(self.row_ptr), i32ptr(self.col_idx), dptr(self.val), dptr(self.b),
                                 dptr(self.c)))

    def csr(self):
        return self.m, self.n, self.row_ptr, self.col_idx, self.val, self.b, self.c

    def recover(self, x_std, std_objective=None):
        """(x_original, objective_original) -- VariableMap recovery."""
        x_std = np.ascontiguousarray(x_std, np.float64)
        if std_objective is None:
            std_objective = float(self.c @ x_std)
        xo = np.empty(self._g.n)
        obj = C.c_double()
        _check(lib().hplp_std_recover(self.h, dptr(x_std), dptr(xo), std_objective, C.byref(obj)))
        return xo, obj.value

    def __del__(self):
        try:
            lib().hplp_std_free(self.h)
        except Exception:
            pass


def to_standard_form(general) -> StdForm:
    return StdForm(general)


def _result(res: abi.Result, x, y, pc, dc, eps, recs) -> dict:
    ne = min(res.n_epochs, len(eps))
    meta = lambda m: dict(source=m.source, orientation=m.orientation, at_iteration=m.at_iteration,  # noqa: E731
                          residual=m.residual, margin=m.margin)
    return dict(
        status=abi.STATUS_NAMES[res.status], status_code=res.status, iterations=res.iterations,
        spmv_count=res.spmv_count, wall_seconds=res.wall_seconds, eta=res.eta, sigma_estimate=res.sigma_estimate,
        kkt=res.final_kkt.as_tuple(), n_epochs=res.n_epochs,
        epochs=[(e.epoch, e.restart_length, e.residual_at_start, e.kkt_at_start.as_tuple()) for e in eps[:ne]],
        x=x, y=y,
        primal_cert=(pc, meta(res.primal_cert)) if res.primal_cert.present else None,
        dual_cert=(dc, meta(res.dual_cert)) if res.dual_cert.present else None,
        trace=recs,
    )


def _io(m, n, init, trace, epochs_capacity, sink=None):
    x, y = np.empty(n), np.empty(m)
    pc, dc = np.zeros(m), np.zeros(n)
    eps = (abi.Epoch * epochs_capacity)()
    recs = []

    def record(rec, xp, nn, yp, mm, user):
        r = rec.contents
        d = dict(epoch=r.epoch, inner=r.inner, iteration=r.iteration, res=r.fixed_point_residual,
                 kkt=r.kkt.as_tuple(), cand_norm_normalized=r.candidate_norm_normalized,
                 cand_norm_difference=r.candidate_norm_difference, partition=abi.trace_partition(r))
        if sink is not None:  # per-record callback instead of kept copies (large instances)
            sink(d, np.ctypeslib.as_array(xp, (nn,)), np.ctypeslib.as_array(yp, (mm,)))
            return
        d["x"] = np.ctypeslib.as_array(xp, (nn,)).copy()
        d["y"] = np.ctypeslib.as_array(yp, (mm,)).copy()
        recs.append(d)

    cb = abi.TRACE_FN(record) if trace else abi.TRACE_FN()
    ix = iy = None
    if init is not None:
        ix = np.ascontiguousarray(init[0], np.float64)
        iy = np.ascontiguousarray(init[1], np.float64)
    io = abi.IO(dptr(ix), dptr(iy), dptr(x), dptr(y), dptr(pc), dptr(dc), eps, epochs_capacity, cb, None)
    keep = (ix, iy, cb)
    return io, x, y, pc, dc, eps, recs, keep


def _config(config, trace, kw):
    cfg = config if config is not None else abi.Config.default(**kw)
    if trace and cfg.trace_period == 0:
        cfg.trace_period = 1
    return cfg


class Solver:
    """A device-resident standard-form LP (hplp_solver_create): upload once,
    solve many times.  ``solve`` mirrors hplp::solve (src/solver.cpp:206)."""

    def __init__(self, m, n, row_ptr, col_idx, val, b, c, device: int = 0):
        L = lib()
        self.m, self.n = int(m), int(n)
        self._keep = [np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int32),
                      np.ascontiguousarray(val, np.float64), np.ascontiguousarray(b, np.float64),
                      np.ascontiguousarray(c, np.float64)]
        rp, ci, v, bb, cc = self._keep
        h = C.c_void_p()
        _check(L.hplp_solver_create(device, self.m, self.n, i64ptr(rp), i32ptr(ci), dptr(v), dptr(bb), dptr(cc),
                                    C.byref(h)))
        self.h = h
        self._keep = None
        self.hx = HX(L.hplp_solver_hx(h), owned=False)

    @classmethod
    def from_std(cls, std: StdForm, device: int = 0) -> "Solver":
        return cls(*std.csr(), device=device)

    @classmethod
    def team(cls, m, n, row_ptr, col_idx, val, b, c, nranks: int, devices=(0,), ctas_per_rank: int = 0) -> "Solver":
        """The LP row-partitioned across `nranks` contexts of this process
        (hplp_solver_create_team): rank r on devices[r % len(devices)]; ranks
        sharing a device are emulated as CTA groups of one launch."""
        self = cls.__new__(cls)
        L = lib()
        self.m, self.n = int(m), int(n)
        rp, ci, v, bb, cc = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int32),
                             np.ascontiguousarray(val, np.float64), np.ascontiguousarray(b, np.float64),
                             np.ascontiguousarray(c, np.float64))
        devs = np.ascontiguousarray(devices, np.int32)
        h = C.c_void_p()
        _check(L.hplp_solver_create_team(i32ptr(devs), len(devs), int(nranks), int(ctas_per_rank), self.m, self.n,
                                         i64ptr(rp), i32ptr(ci), dptr(v), dptr(bb), dptr(cc), C.byref(h)))
        self.h = h
        self._keep = None
        self.nranks = int(nranks)
        self.hx = HX(L.hplp_solver_hx(h), owned=False)
        return self

    @classmethod
    def box(cls, m, n, row_ptr, col_idx, val, b, c, device: int = 0) -> "Solver":
        """The box form of a standard-form LP (hplp_solver_create_box; no
        reference counterpart): bound rows become the
        projection x in [0, u].  solve() returns standard-form x, y; no
        infeasibility scan; final KKT of the box form."""
        self = cls.__new__(cls)
        L = lib()
        self.m, self.n = int(m), int(n)
        rp, ci, v, bb, cc = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int32),
                             np.ascontiguousarray(val, np.float64), np.ascontiguousarray(b, np.float64),
                             np.ascontiguousarray(c, np.float64))
        h = C.c_void_p()
        _check(L.hplp_solver_create_box(int(device), self.m, self.n, i64ptr(rp), i32ptr(ci), dptr(v), dptr(bb),
                                        dptr(cc), C.byref(h)))
        self.h = h
        self._keep = None
        self.hx = HX(L.hplp_solver_hx(h), owned=False)
        return self

    @classmethod
    def rank(cls, m, n, row_ptr, col_idx, val, b, c, nranks: int, rank: int, device: int = 0) -> "Solver":
        """One rank of a team spread over processes (hplp_solver_create_rank):
        exchange team_export() blobs between the processes (see
        paper_2407_16144_b200.team.join) before the first solve()."""
        self = cls.__new__(cls)
        L = lib()
        self.m, self.n = int(m), int(n)
        rp, ci, v, bb, cc = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int32),
                             np.ascontiguousarray(val, np.float64), np.ascontiguousarray(b, np.float64),
                             np.ascontiguousarray(c, np.float64))
        h = C.c_void_p()
        _check(L.hplp_solver_create_rank(int(device), int(nranks), int(rank), self.m, self.n, i64ptr(rp), i32ptr(ci),
                                         dptr(v), dptr(bb), dptr(cc), C.byref(h)))
        self.h = h
        self._keep = None
        self.nranks = int(nranks)
        self.hx = HX(L.hplp_solver_hx(h), owned=False)
        return self

    def team_export(self) -> bytes:
        size = C.c_int64()
        _check(lib().hplp_solver_team_export(self.h, None, 0, C.byref(size)))
        buf = C.create_string_buffer(size.value)
        _check(lib().hplp_solver_team_export(self.h, buf, size.value, C.byref(size)))
        return buf.raw[: size.value]

    def team_import(self, blob: bytes):
        _check(lib().hplp_solver_team_import(self.h, blob, len(blob)))

    def rank_hx(self, r: int) -> "HX":
        """hx context of rank r of a team (rank 0 = self.hx)."""
        return HX(lib().hplp_solver_rank_hx(self.h, int(r)), owned=False)

    def solve(self, config=None, init=None, trace=False, epochs_capacity=1 << 16, sink=None, **kw) -> dict:
        """sink(record, x, y): per-trace-record callback instead of kept copies."""
        cfg = _config(config, trace, kw)
        io, x, y, pc, dc, eps, recs, keep = _io(self.m, self.n, init, trace, epochs_capacity, sink)
        res = abi.Result()
        _check(lib().hplp_solver_solve(self.h, C.byref(cfg), C.byref(io), C.byref(res)))
        del keep
        return _result(res, x, y, pc, dc, eps, recs)

    def close(self):
        if getattr(self, "h", None):
            lib().hplp_solver_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


SUM_FAST, SUM_REFERENCE = 0, 1


class sum_order:
    """Context manager: solvers created inside start with this SpMV summation
    order (hx_set_default_sum_order) -- "reference" gives row sums
    bit-identical to the reference's sequential loops (include/hx.h)."""

    def __init__(self, order):
        self.order = {"fast": SUM_FAST, "reference": SUM_REFERENCE}.get(order, order)

    def __enter__(self):
        _check(lib().hx_set_default_sum_order(int(self.order)))
        return self

    def __exit__(self, *exc):
        lib().hx_set_default_sum_order(-1)


def solve(m, n, row_ptr, col_idx, val, b, c, config=None, init=None, trace=False, device=0,
          epochs_capacity=1 << 16, **kw) -> dict:
    """One-shot solve() through the C ABI with host buffers (hplp_solve_csr)."""
    cfg = _config(config, trace, kw)
    rp, ci, v, bb, cc = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int32),
                         np.ascontiguousarray(val, np.float64), np.ascontiguousarray(b, np.float64),
                         np.ascontiguousarray(c, np.float64))
    io, x, y, pc, dc, eps, recs, keep = _io(int(m), int(n), init, trace, epochs_capacity)
    res = abi.Result()
    _check(lib().hplp_solve_csr(device, int(m), int(n), i64ptr(rp), i32ptr(ci), dptr(v), dptr(bb), dptr(cc),
                                C.byref(cfg), C.byref(io), C.byref(res)))
    del keep
    return _result(res, x, y, pc, dc, eps, recs)


def schedule_info(row_ptr, ctas: int = 148, lead: float = 0.0):
    """The loop kernels' warp schedule for a CSR row-pointer array (host
    only, hx_schedule_info): (tasks int32[slots, 4] in the kernels' layout,
    stats dict W / max_warp / mean_warp / max_cta / mean_cta)."""
    rp = np.ascontiguousarray(row_ptr, np.int32)
    rows = len(rp) - 1
    n = C.c_int64()
    st = (C.c_double * 5)()
    L = lib()
    p = rp.ctypes.data_as(C.POINTER(C.c_int32))
    rc = L.hx_schedule_info(p, rows, ctas, lead, None, 0, C.byref(n), st)  # sizes first
    if rc and not (rc == abi.HPLP_EINVAL and n.value > 0):
        raise ValueError(L.hx_last_error(None).decode())
    tasks = np.zeros((n.value, 4), np.int32)
    if n.value and L.hx_schedule_info(p, rows, ctas, lead, tasks.ctypes.data_as(C.POINTER(C.c_int32)), n.value,
                                      C.byref(n), st):
        raise ValueError(L.hx_last_error(None).decode())
    return tasks, dict(W=int(st[0]), max_warp=st[1], mean_warp=st[2], max_cta=st[3], mean_cta=st[4])


def solve_general(general, config=None, device=0, **kw):
    """Problem load in CSR with bounds -> to_standard_form -> solve -> recovery
    (hplp_solve_general).  Returns (result dict, x_original, objective)."""
    cfg = _config(config, False, kw)
    L = lib()
    ga = general.as_abi()
    std_m, std_n = _std_dims(general)
    io, x, y, pc, dc, eps, recs, keep = _io(std_m, std_n, None, False, 1 << 16)
    res = abi.Result()
    xo = np.empty(general.n)
    obj = C.c_double()
    _check(L.hplp_solve_general(device, C.byref(ga), C.byref(cfg), C.byref(io), C.byref(res), dptr(xo),
                                C.byref(obj)))
    del keep
    return _result(res, x, y, pc, dc, eps, recs), xo, obj.value


def _std_dims(general):
    s = StdForm(general)
    return s.m, s.n


class HX:
    """The hx C-ABI CUDA layer (include/hx.h), for kernel-level tests/bench."""

    def __init__(self, handle=None, device: int = 0, owned: bool = True):
        L = lib()
        if handle is None:
            h = C.c_void_p()
            rc = L.hx_create(device, C.byref(h))
            if rc:
                raise HplpError(rc, L.hx_last_error(None).decode())
            handle = h.value
        self.h = C.c_void_p(handle)
        self.owned = owned
        self.m = self.n = self.nnz = 0
        if not owned:
            m, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
            if L.hx_dims(self.h, C.byref(m), C.byref(n), C.byref(nnz)) == 0:
                self.m, self.n, self.nnz = m.value, n.value, nnz.value

    def _c(self, rc):
        _check(rc, self.h)

    def info(self):
        sm, g, t = C.c_int32(), C.c_int32(), C.c_int32()
        lib().hx_device_info(self.h, C.byref(sm), C.byref(g), C.byref(t))
        return dict(sm_count=sm.value, grid=g.value, threads=t.value)

    LOOP_KERNELS = ("hx::loop_kernel", "hx::loop_kernel_stream", "hx::loop_kernel_box", "hx::loop_kernel_stream_cb",
                    "hx::loop_kernel_exact", "hx::loop_kernel_team", "hx::loop_kernel_team_stream")

    def loop_kernel(self) -> str:
        """Name of the loop kernel hx_run launches for this problem."""
        v = lib().hx_loop_variant(self.h)
        return self.LOOP_KERNELS[v] if v >= 0 else ""

    def stored_nonzeros(self):
        """(nnz of A, nnz of A^T) this context keeps on its device (a rank: its blocks)."""
        a, t = C.c_int64(), C.c_int64()
        self._c(lib().hx_stored_nonzeros(self.h, C.byref(a), C.byref(t)))
        return a.value, t.value

    def sum_order(self) -> int:
        """hx_sum_order: SUM_FAST or SUM_REFERENCE."""
        return int(lib().hx_sum_order(self.h))

    def set_sum_order(self, order):
        """hx_set_sum_order (before upload)."""
        self._c(lib().hx_set_sum_order(self.h, int(order)))

    def stream(self) -> int:
        return lib().hx_stream(self.h) or 0

    def launches(self) -> int:
        return lib().hx_launch_count(self.h)

    def upload(self, m, n, row_ptr, col_idx, val, b, c):
        rp, ci, v, bb, cc = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int32),
                             np.ascontiguousarray(val, np.float64), np.ascontiguousarray(b, np.float64),
                             np.ascontiguousarray(c, np.float64))
        self._c(lib().hx_upload_csr(self.h, int(m), int(n), i64ptr(rp), i32ptr(ci), dptr(v), dptr(bb), dptr(cc)))
        self.m, self.n, self.nnz = int(m), int(n), int(rp[-1])

    def spmv(self, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(self.m)
        self._c(lib().hx_spmv(self.h, dptr(x), dptr(out)))
        return out

    def spmv_transpose(self, y):
        y = np.ascontiguousarray(y, np.float64)
        out = np.empty(self.n)
        self._c(lib().hx_spmv_transpose(self.h, dptr(y), dptr(out)))
        return out

    def power_iteration(self, x0, tol=1e-4, k0=0, max_iters=5000, sigma_prev=0.0):
        x0 = np.ascontiguousarray(x0, np.float64)
        s, it, cv, rd = C.c_double(), C.c_int64(), C.c_int32(), C.c_int32()
        self._c(lib().hx_power_iteration(self.h, dptr(x0), tol, k0, max_iters, sigma_prev, C.byref(s),
                                         C.byref(it), C.byref(cv), C.byref(rd)))
        return s.value, it.value, bool(cv.value), bool(rd.value)

    def setup(self, config, sigma_used, eta, x0=None, y0=None):
        x0 = None if x0 is None else np.ascontiguousarray(x0, np.float64)
        y0 = None if y0 is None else np.ascontiguousarray(y0, np.float64)
        self._c(lib().hx_setup(self.h, C.byref(config), sigma_used, eta, dptr(x0), dptr(y0)))

    def run(self, max_iters) -> HxProgress:
        p = HxProgress()
        self._c(lib().hx_run(self.h, int(max_iters), C.byref(p)))
        return p

    def progress(self) -> HxProgress:
        p = HxProgress()
        self._c(lib().hx_progress(self.h, C.byref(p)))
        return p

    def epochs(self, first, count):
        out = (abi.Epoch * max(count, 1))()
        self._c(lib().hx_epochs(self.h, first, count, out))
        return [(e.epoch, e.restart_length, e.residual_at_start, e.kkt_at_start.as_tuple()) for e in out[:count]]

    def precondition(self, ruiz_iters=10, pc_alpha=1.0):
        """Ruiz + Pock-Chambolle scaling of the uploaded problem in place;
        returns the accumulated (row_scale R, col_scale C)."""
        R, Cs = np.empty(self.m), np.empty(self.n)
        self._c(lib().hx_precondition(self.h, int(ruiz_iters), float(pc_alpha), dptr(R), dptr(Cs)))
        return R, Cs

    def download_problem(self):
        """(row_ptr, col_idx, val, b, c) of the device problem."""
        rp = np.empty(self.m + 1, np.int64)
        ci, v = np.empty(self.nnz, np.int32), np.empty(self.nnz)
        b, c = np.empty(self.m), np.empty(self.n)
        self._c(lib().hx_download_problem(self.h, i64ptr(rp), i32ptr(ci), dptr(v), dptr(b), dptr(c)))
        return rp, ci, v, b, c

    # ---- row-partitioned team (include/hx.h) ----
    def set_partition(self, nranks, rank, row_bounds, col_bounds, ctas=0):
        """hx_set_partition: this context is rank `rank` of the partition given
        by row_bounds / col_bounds (nranks + 1 entries each)."""
        rb = np.ascontiguousarray(row_bounds, np.int64)
        cb = np.ascontiguousarray(col_bounds, np.int64)
        self._c(lib().hx_set_partition(self.h, int(nranks), int(rank), i64ptr(rb), i64ptr(cb), int(ctas)))

    def team_export(self) -> bytes:
        size = C.c_int64()
        self._c(lib().hx_team_export(self.h, None, 0, C.byref(size)))
        buf = C.create_string_buffer(size.value)
        self._c(lib().hx_team_export(self.h, buf, size.value, C.byref(size)))
        return buf.raw[: size.value]

    def team_import(self, blob: bytes):
        self._c(lib().hx_team_import(self.h, blob, len(blob)))

    def get_iterate(self, which=0):
        x, y = np.empty(self.n), np.empty(self.m)
        self._c(lib().hx_get_iterate(self.h, which, dptr(x), dptr(y)))
        return x, y

    def phase_profile(self, reset=True, sm_mhz=1965.0):
        """Per-CTA phase timers (HX_PROFILE=1, SM cycles): mean/max/min us per iteration."""
        g = self.info()["grid"]
        buf = (C.c_uint64 * (g * (16 + 2 * self.WARPS)))()
        self._c(lib().hx_profile(self.h, buf, int(reset)))
        a = np.array(buf[: g * 16], dtype=np.float64).reshape(g, 16)
        its = max(a[0, 5], 1.0)
        # phase_A: the (speculative) phase A after warp 0's controller; controller:
        # warp 0's totals + logic (its split: ctl_totals / ctl_scalar);
        # scan_or_redo: certificate scans and redone phases A
        names = {"phase_A": 0, "barrier1": 1, "phase_B": 2, "barrier2": 3, "controller": 4, "scan_or_redo": 7,
                 "ctl_totals": 8, "ctl_scalar": 9}
        k = 1.0 / its / sm_mhz  # cycles -> us per iteration
        return {nm: dict(mean_us=float(a[:, i].mean() * k), max_us=float(a[:, i].max() * k),
                         min_us=float(a[:, i].min() * k)) for nm, i in names.items()}

    WARPS = 16  # warps per CTA (csrc/hx_internal.cuh kWarps)

    def warp_profile(self, reset=True):
        """Per-warp SpMV cycles of phases A and B (a -DHX_WPROF build with
        HX_PROFILE=1), shape (2, grid * WARPS); plus the per-CTA counters."""
        g = self.info()["grid"]
        buf = (C.c_uint64 * (g * (16 + 2 * self.WARPS)))()
        self._c(lib().hx_profile(self.h, buf, int(reset)))
        a = np.array(buf[:], dtype=np.float64)
        return a[g * 16:].reshape(2, g * self.WARPS), a[: g * 16].reshape(g, 16)

    def sched_tasks(self, which):
        """Warp task list (0: rows of A, 1: rows of A^T) as an (n_tasks, 4) int32 array."""
        cnt = C.c_int64()
        self._c(lib().hx_sched_tasks(self.h, which, None, 0, C.byref(cnt)))
        out = np.empty((cnt.value, 4), np.int32)
        self._c(lib().hx_sched_tasks(self.h, which, out.ctypes.data_as(C.POINTER(C.c_int32)), cnt.value,
                                     C.byref(cnt)))
        return out

    def kkt_current(self):
        k = abi.Kkt()
        self._c(lib().hx_kkt_current(self.h, C.byref(k)))
        return k.as_tuple()

    def close(self):
        if self.owned and getattr(self, "h", None):
            lib().hx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def box_form(m, n, row_ptr, col_idx, val, b, c):
    """hplp_box_form_dims: (m_box, n_box, upper[n_box]) of a standard-form LP."""
    rp, ci, v, bb, cc = (np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int32),
                         np.ascontiguousarray(val, np.float64), np.ascontiguousarray(b, np.float64),
                         np.ascontiguousarray(c, np.float64))
    mb, nb = C.c_int64(), C.c_int64()
    up = np.empty(int(n))
    _check(lib().hplp_box_form_dims(int(m), int(n), i64ptr(rp), i32ptr(ci), dptr(v), dptr(bb), dptr(cc),
                                    C.byref(mb), C.byref(nb), dptr(up)))
    return mb.value, nb.value, up[: nb.value].copy()


def power_start(n, seed=12345):
    """hplp_power_start: the normalised power-iteration start vector (host)."""
    x = np.empty(int(n))
    _check(lib().hplp_power_start(int(n), C.c_uint64(seed), dptr(x)))
    return x


def plan_partition(m, n, row_ptr, col_idx, parts):
    """hplp_plan_partition: (row_bounds, col_bounds), parts + 1 entries each."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx, np.int32)
    rb, cb = np.empty(parts + 1, np.int64), np.empty(parts + 1, np.int64)
    _check(lib().hplp_plan_partition(int(m), int(n), i64ptr(rp), i32ptr(ci), int(parts), i64ptr(rb), i64ptr(cb)))
    return rb, cb


def team_run(hxs, max_iters):
    """hx_team_run over contexts bound by hx_team_bind; one progress per context."""
    arr = (C.c_void_p * len(hxs))(*[h.h.value for h in hxs])
    prog = (HxProgress * len(hxs))()
    _check(lib().hx_team_run(arr, len(hxs), int(max_iters), prog), hxs[0].h)
    return list(prog)


def team_bind(hxs):
    arr = (C.c_void_p * len(hxs))(*[h.h.value for h in hxs])
    _check(lib().hx_team_bind(arr, len(hxs)), hxs[0].h)


def _text(call) -> str:
    """Two-call text protocol of the C ABI: size, then fill."""
    size = C.c_int64()
    _check(call(None, 0, C.byref(size)))
    buf = C.create_string_buffer(size.value + 1)
    _check(call(buf, size.value + 1, C.byref(size)))
    return buf.value.decode()


class MpsProblem:
    """parse_mps result (inc/hplp/mps_io.hpp:54-57): the GeneralFormLP as a
    CSR-with-bounds problem plus the document metadata."""

    def __init__(self, text: str):
        L = lib()
        h, m, n, nnz = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int64()
        _check(L.hplp_mps_parse(text.encode(), C.byref(h), C.byref(m), C.byref(n), C.byref(nnz)))
        self.h = h
        self.m, self.n, self.nnz = m.value, n.value, nnz.value

    def _names(self, what):
        return _text(lambda b, c, sz: lib().hplp_mps_names(self.h, what, b, c, sz))

    @property
    def name(self) -> str:
        return self._names(0)

    @property
    def objective_name(self) -> str:
        return self._names(1)

    @property
    def warnings(self) -> list:
        return [w for w in self._names(2).split("\n") if w]

    @property
    def row_names(self) -> list:
        return self._names(3).split("\n")[: self.m]

    @property
    def col_names(self) -> list:
        return self._names(4).split("\n")[: self.n]

    def general(self):
        """The problem as gen.GeneralLP (numpy copies)."""
        from .gen import GeneralLP

        v = abi.General()
        _check(lib().hplp_mps_view(self.h, C.byref(v)))
        arr = lambda p, k, dt: np.ctypeslib.as_array(p, (k,)).astype(dt, copy=True) if k else np.zeros(0, dt)  # noqa
        return GeneralLP(m=v.m, n=v.n, row_ptr=arr(v.row_ptr, v.m + 1, np.int64), col_idx=arr(v.col_idx, v.nnz, np.int32),
                         val=arr(v.val, v.nnz, np.float64), row_relation=arr(v.row_relation, v.m, np.int32),
                         row_rhs=arr(v.row_rhs, v.m, np.float64), col_lower=arr(v.col_lower, v.n, np.float64),
                         col_upper=arr(v.col_upper, v.n, np.float64), objective=arr(v.objective, v.n, np.float64),
                         row_range=arr(v.row_range, v.m, np.float64), maximize=bool(v.maximize),
                         objective_constant=v.objective_constant)

    def write(self) -> str:
        """write_mps: normalized free MPS."""
        return _text(lambda b, c, sz: lib().hplp_mps_write(self.h, b, c, sz))

    def __del__(self):
        try:
            lib().hplp_mps_free(self.h)
        except Exception:
            pass


def parse_mps(text: str) -> MpsProblem:
    return MpsProblem(text)


def mps_from_general(general) -> str:
    """write_mps of a gen.GeneralLP (rows R<i>, columns C<j>)."""
    ga = general.as_abi()
    return _text(lambda b, c, sz: lib().hplp_mps_from_general(C.byref(ga), b, c, sz))


def solve_mps(text: str, config=None, device: int = 0, instance: str | None = None, elide_above: int = -1, **kw):
    """cmd_solve (SPEC.md [MODULE] cli): MPS text -> GPU solve -> (report
    JSON text, trace CSV text, status string)."""
    cfg = _config(config, False, kw)
    L = lib()
    args = [device, text.encode(), C.byref(cfg), instance.encode() if instance else None, int(elide_above)]
    js, ts, st = C.c_int64(), C.c_int64(), C.c_int32()
    jcap, tcap = 1 << 16, 1 << 12
    n_guess = text.count("\n")
    jcap += 64 * n_guess
    if cfg.trace_period > 0:
        tcap += 400 * (cfg.iteration_limit // cfg.trace_period + 2)
    while True:  # report sizes are known only after the solve: retry once if too small
        jb, tb = C.create_string_buffer(jcap), C.create_string_buffer(tcap)
        rc = L.hplp_solve_mps(*args, jb, jcap, C.byref(js), tb, tcap, C.byref(ts), C.byref(st))
        if rc == abi.HPLP_EINVAL and (js.value + 1 > jcap or ts.value + 1 > tcap):
            jcap, tcap = max(jcap, js.value + 1), max(tcap, ts.value + 1)
            continue
        _check(rc)
        return jb.value.decode(), tb.value.decode(), abi.STATUS_NAMES[st.value]


def json_normalize(text: str, include_timing: bool = True) -> str:
    """parse_solution_json then write_solution_json."""
    return _text(lambda b, c, sz: lib().hplp_json_normalize(text.encode(), int(include_timing), b, c, sz))


ITERATE_CURRENT, ITERATE_BEST, ITERATE_NEXT, ITERATE_LAST = range(4)
INF = math.inf
