"""Seeded synthetic LPs for the BASELINE.json configs (include/hplp_gen.h).

The paper's MIPLIB-2017 relaxations are not in this container; these planted
and transportation instances stand in for them with the shapes, sizes and
value distributions BASELINE.json states.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import abi
from .abi import dptr, i32ptr, i64ptr
from .build import GEN_LIB, ensure_built


class GenParams(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("zipf", C.c_int32),
        ("m", C.c_int64),
        ("n", C.c_int64),
        ("nnz_per_row", C.c_int64),
        ("eq_frac", C.c_double),
        ("row_scale_log10", C.c_double),
        ("zipf_s", C.c_double),
        ("zipf_cap", C.c_int64),
        ("zipf_target_nnz", C.c_int64),
        ("zipf_force_cap", C.c_int64),
        ("infeasible_rows", C.c_int64),
        ("ub_lo", C.c_double),
        ("ub_hi", C.c_double),
        ("sources", C.c_int64),
        ("sinks", C.c_int64),
        ("seed", C.c_uint64),
    ]


_lib = None


def _load():
    global _lib
    if _lib is None:
        ensure_built()
        lib = C.CDLL(str(GEN_LIB))
        lib.hplp_gen_preset.argtypes = [C.c_int32, C.POINTER(GenParams)]
        lib.hplp_gen_create.argtypes = [C.POINTER(GenParams), C.POINTER(C.c_void_p)]
        lib.hplp_gen_dims.argtypes = [C.c_void_p] + [C.POINTER(C.c_int64)] * 3
        lib.hplp_gen_dims.restype = None
        PD = C.POINTER(C.c_double)
        lib.hplp_gen_export.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int32), PD,
                                        C.POINTER(C.c_int32), PD, PD, PD, PD, PD]
        lib.hplp_gen_planted_x.argtypes = [C.c_void_p, PD]
        lib.hplp_gen_free.argtypes = [C.c_void_p]
        lib.hplp_gen_free.restype = None
        lib.hplp_gen_last_error.restype = C.c_char_p
        _lib = lib
    return _lib


@dataclass
class GeneralLP:
    """General-form LP: CSR rows with relations, column bounds, objective."""

    m: int
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    val: np.ndarray
    row_relation: np.ndarray
    row_rhs: np.ndarray
    col_lower: np.ndarray
    col_upper: np.ndarray
    objective: np.ndarray
    planted_objective: float = float("nan")
    x_star: np.ndarray | None = None
    row_range: np.ndarray | None = None
    maximize: bool = False
    objective_constant: float = 0.0

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def as_abi(self) -> abi.General:
        """hplp_general_t view (keep self alive while it is used)."""
        return abi.General(self.m, self.n, self.nnz, i64ptr(self.row_ptr), i32ptr(self.col_idx), dptr(self.val),
                           i32ptr(self.row_relation), dptr(self.row_rhs), dptr(self.row_range),
                           dptr(self.col_lower), dptr(self.col_upper), dptr(self.objective),
                           int(self.maximize), 0, self.objective_constant)


def preset(cfg: int) -> GenParams:
    p = GenParams()
    if _load().hplp_gen_preset(cfg, C.byref(p)) != 0:
        raise ValueError(f"unknown config {cfg}")
    return p


def scaled(cfg: int, **over) -> GenParams:
    """A preset with some fields overridden (reduced-size parity variants)."""
    p = preset(cfg)
    for k, v in over.items():
        setattr(p, k, v)
    return p


def generate(params: GenParams | int) -> GeneralLP:
    lib = _load()
    if isinstance(params, int):
        params = preset(params)
    h = C.c_void_p()
    if lib.hplp_gen_create(C.byref(params), C.byref(h)) != 0:
        raise ValueError(lib.hplp_gen_last_error().decode())
    try:
        m, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        lib.hplp_gen_dims(h, C.byref(m), C.byref(n), C.byref(nnz))
        m, n, nnz = m.value, n.value, nnz.value
        g = GeneralLP(m, n, np.empty(m + 1, np.int64), np.empty(nnz, np.int32), np.empty(nnz),
                      np.empty(m, np.int32), np.empty(m), np.empty(n), np.empty(n), np.empty(n))
        po = C.c_double()
        lib.hplp_gen_export(h, i64ptr(g.row_ptr), i32ptr(g.col_idx), dptr(g.val), i32ptr(g.row_relation),
                            dptr(g.row_rhs), dptr(g.col_lower), dptr(g.col_upper), dptr(g.objective), C.byref(po))
        g.planted_objective = po.value
        xs = np.empty(n)
        lib.hplp_gen_planted_x(h, dptr(xs))
        g.x_star = xs
        return g
    finally:
        lib.hplp_gen_free(h)


__all__ = ["GenParams", "GeneralLP", "generate", "preset", "scaled", "replace"]
