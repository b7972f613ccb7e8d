"""ctypes mirrors of include/hplp_types.h (the POD types of every C ABI here).

Field order and widths must match the header exactly; tests/test_abi.py
checks the sizes against the compiled library's own ``sizeof`` exports.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

HPLP_OK, HPLP_EINVAL, HPLP_EDOMAIN, HPLP_ECUDA, HPLP_ENOMEM, HPLP_ESTATE, HPLP_ETIMEOUT, HPLP_EPARSE = range(8)

RESTART_FIXED, RESTART_ADAPTIVE, RESTART_NONE = range(3)

STATUS_NAMES = (
    "optimal",
    "primal_infeasible",
    "dual_infeasible",
    "primal_dual_infeasible",
    "iteration_limit",
    "time_limit",
)
(STATUS_OPTIMAL, STATUS_PRIMAL_INFEASIBLE, STATUS_DUAL_INFEASIBLE,
 STATUS_PRIMAL_DUAL_INFEASIBLE, STATUS_ITERATION_LIMIT, STATUS_TIME_LIMIT) = range(6)

SOURCE_NORMALIZED_ITERATE, SOURCE_ITERATE_DIFFERENCE = range(2)
ORIENT_AS_IS, ORIENT_NEGATED = range(2)
ROW_LE, ROW_EQ, ROW_GE = range(3)
SCHEME_RHPDHG, SCHEME_VANILLA, SCHEME_AVERAGED, SCHEME_RESTARTED_AVERAGE = range(4)


class Config(C.Structure):
    """SolverConfig, inc/solver.hpp:62-80."""

    _fields_ = [
        ("restart_kind", C.c_int32),
        ("has_eta_override", C.c_int32),
        ("k_star", C.c_int64),
        ("beta", C.c_double),
        ("tau0", C.c_int64),
        ("tolerance", C.c_double),
        ("iteration_limit", C.c_int64),
        ("time_limit_seconds", C.c_double),
        ("eta_override", C.c_double),
        ("infeasibility_check_period", C.c_int64),
        ("trace_period", C.c_int64),
        ("certificate_tolerance", C.c_double),
        ("tol_active", C.c_double),
        ("adaptive_stall_cap", C.c_int64),
        ("seed", C.c_uint64),
        ("precondition_ruiz_iters", C.c_int32),
        ("scheme", C.c_int32),
        ("precondition_pc_alpha", C.c_double),
    ]

    @classmethod
    def default(cls, **kw) -> "Config":
        c = cls(
            restart_kind=RESTART_ADAPTIVE,
            has_eta_override=0,
            k_star=0,
            beta=0.36787944117144233,
            tau0=32,
            tolerance=1e-8,
            iteration_limit=1000000,
            time_limit_seconds=math.inf,
            eta_override=0.0,
            infeasibility_check_period=100,
            trace_period=0,
            certificate_tolerance=1e-6,
            tol_active=1e-6,
            adaptive_stall_cap=2000,
            seed=12345,
            precondition_ruiz_iters=0,
            scheme=0,
            precondition_pc_alpha=-1.0,
        )
        for k, v in kw.items():
            if k == "eta_override" and v is not None:
                c.has_eta_override = 1
            if not hasattr(c, k):
                raise AttributeError(k)
            setattr(c, k, v)
        return c


class Kkt(C.Structure):
    """KktError, inc/pdhg_core.hpp:82-87."""

    _fields_ = [
        ("primal_residual", C.c_double),
        ("dual_residual", C.c_double),
        ("gap_residual", C.c_double),
        ("max_relative", C.c_double),
    ]

    def as_tuple(self):
        return (self.primal_residual, self.dual_residual, self.gap_residual, self.max_relative)


class Epoch(C.Structure):
    """EpochStats, inc/solver.hpp:82-87."""

    _fields_ = [
        ("epoch", C.c_int64),
        ("restart_length", C.c_int64),
        ("residual_at_start", C.c_double),
        ("kkt_at_start", Kkt),
    ]


class CertMeta(C.Structure):
    """Certificate metadata, inc/solver.hpp:91-98."""

    _fields_ = [
        ("present", C.c_int32),
        ("source", C.c_int32),
        ("orientation", C.c_int32),
        ("reserved", C.c_int32),
        ("at_iteration", C.c_int64),
        ("residual", C.c_double),
        ("margin", C.c_double),
    ]


class Result(C.Structure):
    """SolveResult + SolveTotals, inc/solver.hpp:100-116."""

    _fields_ = [
        ("status", C.c_int32),
        ("reserved", C.c_int32),
        ("iterations", C.c_int64),
        ("spmv_count", C.c_int64),
        ("wall_seconds", C.c_double),
        ("eta", C.c_double),
        ("sigma_estimate", C.c_double),
        ("final_kkt", Kkt),
        ("n_epochs", C.c_int64),
        ("primal_cert", CertMeta),
        ("dual_cert", CertMeta),
    ]


class Trace(C.Structure):
    """TraceRecord subset, inc/diagnostics.hpp:72-84."""

    _fields_ = [
        ("epoch", C.c_int64),
        ("inner", C.c_int64),
        ("iteration", C.c_int64),
        ("fixed_point_residual", C.c_double),
        ("kkt", Kkt),
        ("candidate_norm_normalized", C.c_double),
        ("candidate_norm_difference", C.c_double),
        ("wall_seconds", C.c_double),
        ("partition_n", C.c_int64),
        ("partition_b1", C.c_int64),
        ("partition_b2", C.c_int64),
        ("partition_sets", C.POINTER(C.c_int64)),
    ]


def trace_partition(r):
    """(N, B1, B2) index arrays of a Trace record (PartitionEstimate)."""
    k = r.partition_n + r.partition_b1 + r.partition_b2
    a = np.ctypeslib.as_array(r.partition_sets, (k,)).copy() if k else np.zeros(0, np.int64)
    return a[: r.partition_n], a[r.partition_n: r.partition_n + r.partition_b1], a[r.partition_n + r.partition_b1:]


TRACE_FN = C.CFUNCTYPE(None, C.POINTER(Trace), C.POINTER(C.c_double), C.c_int64,
                       C.POINTER(C.c_double), C.c_int64, C.c_void_p)


class IO(C.Structure):
    _fields_ = [
        ("init_x", C.POINTER(C.c_double)),
        ("init_y", C.POINTER(C.c_double)),
        ("x", C.POINTER(C.c_double)),
        ("y", C.POINTER(C.c_double)),
        ("primal_cert", C.POINTER(C.c_double)),
        ("dual_cert", C.POINTER(C.c_double)),
        ("epochs", C.POINTER(Epoch)),
        ("epochs_capacity", C.c_int64),
        ("trace_fn", TRACE_FN),
        ("trace_user", C.c_void_p),
    ]


class General(C.Structure):
    """GeneralFormLP in CSR with relations and bounds (inc/lp_model.hpp:60-74)."""

    _fields_ = [
        ("m", C.c_int64),
        ("n", C.c_int64),
        ("nnz", C.c_int64),
        ("row_ptr", C.POINTER(C.c_int64)),
        ("col_idx", C.POINTER(C.c_int32)),
        ("val", C.POINTER(C.c_double)),
        ("row_relation", C.POINTER(C.c_int32)),
        ("row_rhs", C.POINTER(C.c_double)),
        ("row_range", C.POINTER(C.c_double)),
        ("col_lower", C.POINTER(C.c_double)),
        ("col_upper", C.POINTER(C.c_double)),
        ("objective", C.POINTER(C.c_double)),
        ("maximize", C.c_int32),
        ("reserved", C.c_int32),
        ("objective_constant", C.c_double),
    ]


def dptr(a):
    """double* of a C-contiguous float64 array (or NULL for None)."""
    if a is None:
        return C.POINTER(C.c_double)()
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], (a.dtype, a.flags)
    return a.ctypes.data_as(C.POINTER(C.c_double))


def i32ptr(a):
    if a is None:
        return C.POINTER(C.c_int32)()
    assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def i64ptr(a):
    if a is None:
        return C.POINTER(C.c_int64)()
    assert a.dtype == np.int64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(C.c_int64))
