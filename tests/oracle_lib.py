"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the CPU checkers.

* ``Oracle("port")``      -> oracle/libndg_oracle.so (plain-C restatement)
* ``Oracle("reference")`` -> oracle/_ref/libndg_ref.so (the reference itself,
  compiled from /root/reference/proj/src by oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module.  The product (paper_2510_05254_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
PORT_SO = os.path.join(ORACLE_DIR, "libndg_oracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libndg_ref.so")

ADVECTION, EULER = 0, 1
RK3, RK4, RK6 = 0, 1, 2
RK_STAGES = {RK3: 3, RK4: 4, RK6: 7}


class NdgoConfig(C.Structure):
    _fields_ = [
        ("dim", C.c_int),
        ("cells", C.c_int * 3),
        ("length", C.c_double * 3),
        ("order", C.c_int),
        ("kind", C.c_int),
        ("velocity", C.c_double * 3),
        ("sound_speed", C.c_double),
        ("rk", C.c_int),
        ("cfl", C.c_double),
        ("t_end", C.c_double),
    ]


class NdgoStats(C.Structure):
    _fields_ = [("steps", C.c_long), ("dt_min", C.c_double), ("dt_max", C.c_double),
                ("wall_seconds", C.c_double)]


class NdgoError(C.Structure):
    _fields_ = [("code", C.c_int), ("step", C.c_long), ("worker", C.c_int),
                ("message", C.c_char * 256)]


@dataclass
class Problem:
    """Plain description of one solver configuration (Mesh+EquationModel+SolverConfig)."""
    dim: int
    cells: tuple
    order: int
    kind: int = EULER
    rk: int = RK4
    velocity: tuple = (1.0, 0.0, 0.0)
    sound_speed: float = 1.0
    cfl: float = 0.4
    t_end: float = 1.0
    length: tuple = (1.0, 1.0, 1.0)

    @property
    def n_var(self) -> int:
        return 1 if self.kind == ADVECTION else self.dim + 1

    @property
    def cells3(self):
        c = list(self.cells) + [1] * (3 - len(self.cells))
        return tuple(c[a] if a < self.dim else 1 for a in range(3))

    @property
    def size(self) -> int:
        s = self.n_var
        for a in range(self.dim):
            s *= self.cells3[a] * self.order
        return s

    def ndgo(self) -> NdgoConfig:
        c = NdgoConfig()
        c.dim = self.dim
        for a in range(3):
            c.cells[a] = self.cells3[a]
            c.length[a] = self.length[a]
            c.velocity[a] = self.velocity[a]
        c.order = self.order
        c.kind = self.kind
        c.sound_speed = self.sound_speed
        c.rk = self.rk
        c.cfl = self.cfl
        c.t_end = self.t_end
        return c


def build_port() -> None:
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class CheckerError(Exception):
    def __init__(self, code, step, worker, message):
        super().__init__(message)
        self.code, self.step, self.worker, self.message = code, step, worker, message


class Oracle:
    """Uniform interface over the C restatement ("port") and the reference ("reference")."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if kind == "port" and not os.path.exists(path):
            build_port()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        L = self.lib
        P = C.POINTER
        cfg = P(NdgoConfig)
        if kind == "port":
            self._advance = L.ndgo_advance
            self._advance.argtypes = [cfg, P(C.c_double), C.c_long, C.c_int, P(NdgoStats), P(NdgoError)]
            self._rhs = L.ndgo_serial_rhs
            self._rhs.argtypes = [cfg, P(C.c_double), P(C.c_double), P(NdgoError)]
            L.ndgo_l2_error.restype = C.c_double
            L.ndgo_l2_error.argtypes = [cfg, P(C.c_double), P(C.c_double), C.c_int]
            L.ndgo_l1_norm.restype = C.c_double
            L.ndgo_l1_norm.argtypes = [cfg, P(C.c_double), C.c_int]
            L.ndgo_conserved_totals.argtypes = [cfg, P(C.c_double), P(C.c_double)]
            L.ndgo_init_multisine.argtypes = [cfg, P(C.c_double), C.c_int, P(C.c_double)]
            L.ndgo_init_euler_subsonic.argtypes = [cfg, P(C.c_double)]
            L.ndgo_multisine_amplitudes.argtypes = [C.c_int, C.c_uint64, P(C.c_double)]
            L.ndgo_gauss_lobatto.argtypes = [C.c_int, P(C.c_double), P(C.c_double)]
            L.ndgo_differentiation_matrix.argtypes = [C.c_int, P(C.c_double), P(C.c_double)]
            L.ndgo_decompose.argtypes = [cfg, C.c_int, P(C.c_int), P(C.c_int), P(C.c_int), P(C.c_int), P(NdgoError)]
            L.ndgo_fnv1a64.restype = C.c_uint64
            L.ndgo_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
            L.ndgo_index.restype = C.c_size_t
            L.ndgo_index.argtypes = [cfg, P(C.c_int), P(C.c_int), C.c_int]
            L.ndgo_face_trace_size.restype = C.c_size_t
            L.ndgo_face_trace_size.argtypes = [cfg, P(C.c_int), C.c_int]
            L.ndgo_pack_face_trace.argtypes = [cfg, P(C.c_int), P(C.c_double), C.c_int, C.c_int, C.c_int, P(C.c_double)]
            L.ndgo_max_wavespeed_bound.restype = C.c_double
            L.ndgo_max_wavespeed_bound.argtypes = [cfg, P(C.c_double), C.c_size_t, P(NdgoError)]
            L.ndgo_dt_from_alpha.restype = C.c_double
            L.ndgo_dt_from_alpha.argtypes = [cfg, C.c_double]
        else:
            self._advance = L.ref_advance
            self._advance.argtypes = [cfg, P(C.c_double), C.c_long, C.c_int, P(NdgoStats), P(NdgoError)]
            self._rhs = L.ref_serial_rhs
            self._rhs.argtypes = [cfg, P(C.c_double), P(C.c_double), P(NdgoError)]
            L.ref_run_partitioned.argtypes = [cfg, P(C.c_double), C.c_int, C.c_long, C.c_int, P(NdgoStats), P(NdgoError)]
            L.ref_l2_error.restype = C.c_double
            L.ref_l2_error.argtypes = [cfg, P(C.c_double), P(C.c_double), C.c_int]
            L.ref_conserved_totals.argtypes = [cfg, P(C.c_double), P(C.c_double)]
            L.ref_init_multisine.argtypes = [cfg, P(C.c_double), C.c_int, P(C.c_double)]
            L.ref_init_multisine_seed.argtypes = [cfg, C.c_int, C.c_ulonglong, P(C.c_double)]
            L.ref_init_euler_subsonic.argtypes = [cfg, P(C.c_double)]
            L.ref_gauss_lobatto.argtypes = [C.c_int, P(C.c_double), P(C.c_double), P(C.c_double)]
            L.ref_decompose.argtypes = [cfg, C.c_int, P(C.c_int), P(C.c_int), P(C.c_int), P(C.c_int), P(NdgoError)]
            L.ref_pack_face_trace.argtypes = [cfg, P(C.c_int), P(C.c_double), C.c_int, C.c_int, C.c_int, P(C.c_double)]
            L.ref_max_wavespeed_bound.restype = C.c_double
            L.ref_max_wavespeed_bound.argtypes = [cfg, P(C.c_double), P(NdgoError)]

    # ------------------------------------------------------------------ ICs
    def amplitudes(self, n_modes: int, seed: int) -> np.ndarray:
        out = np.zeros(n_modes)
        if self.kind == "port":
            self.lib.ndgo_multisine_amplitudes(n_modes, seed, _dp(out))
        else:
            raise NotImplementedError
        return out

    def init_multisine(self, p: Problem, amps=None, n_modes=None, seed=None) -> np.ndarray:
        out = np.zeros(p.size)
        c = p.ndgo()
        if amps is None:
            if self.kind == "port":
                amps = self.amplitudes(n_modes, seed)
            else:
                self.lib.ref_init_multisine_seed(C.byref(c), n_modes, seed, _dp(out))
                return out
        amps = np.ascontiguousarray(amps, dtype=np.float64)
        fn = self.lib.ndgo_init_multisine if self.kind == "port" else self.lib.ref_init_multisine
        fn(C.byref(c), _dp(amps), len(amps), _dp(out))
        return out

    def init_euler(self, p: Problem) -> np.ndarray:
        out = np.zeros(p.size)
        fn = self.lib.ndgo_init_euler_subsonic if self.kind == "port" else self.lib.ref_init_euler_subsonic
        fn(C.byref(p.ndgo()), _dp(out))
        return out

    def initial(self, p: Problem, n_modes=40, seed=42) -> np.ndarray:
        if p.kind == EULER:
            return self.init_euler(p)
        return self.init_multisine(p, n_modes=n_modes, seed=seed)

    # --------------------------------------------------------------- solver
    def rhs(self, p: Problem, u: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros_like(u)
        err = NdgoError()
        rc = self._rhs(C.byref(p.ndgo()), _dp(u), _dp(out), C.byref(err))
        if rc:
            raise CheckerError(err.code, err.step, err.worker, err.message.decode())
        return out

    def advance(self, p: Problem, u: np.ndarray, fixed_steps: int = -1, warmup: bool = False):
        u = np.array(u, dtype=np.float64, copy=True)
        st, err = NdgoStats(), NdgoError()
        rc = self._advance(C.byref(p.ndgo()), _dp(u), fixed_steps, int(warmup), C.byref(st), C.byref(err))
        if rc:
            raise CheckerError(err.code, err.step, err.worker, err.message.decode())
        return u, st

    def run_partitioned(self, p: Problem, u: np.ndarray, workers: int, fixed_steps: int = -1,
                        warmup: bool = False):
        assert self.kind == "reference"
        u = np.array(u, dtype=np.float64, copy=True)
        st, err = NdgoStats(), NdgoError()
        rc = self.lib.ref_run_partitioned(C.byref(p.ndgo()), _dp(u), workers, fixed_steps,
                                          int(warmup), C.byref(st), C.byref(err))
        if rc:
            raise CheckerError(err.code, err.step, err.worker, err.message.decode())
        return u, st

    def l2_error(self, p: Problem, a: np.ndarray, b: np.ndarray, var: int) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        fn = self.lib.ndgo_l2_error if self.kind == "port" else self.lib.ref_l2_error
        return fn(C.byref(p.ndgo()), _dp(a), _dp(b), var)

    def conserved_totals(self, p: Problem, u: np.ndarray) -> np.ndarray:
        assert self.kind == "reference"
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros(p.n_var)
        self.lib.ref_conserved_totals(C.byref(p.ndgo()), _dp(u), _dp(out))
        return out

    def basis(self, order: int):
        nodes, w, d = np.zeros(order), np.zeros(order), np.zeros(order * order)
        if self.kind == "port":
            self.lib.ndgo_gauss_lobatto(order, _dp(nodes), _dp(w))
            self.lib.ndgo_differentiation_matrix(order, _dp(nodes), _dp(d))
        else:
            self.lib.ref_gauss_lobatto(order, _dp(nodes), _dp(w), _dp(d))
        return nodes, w, d

    def decompose(self, p: Problem, workers: int):
        grid = (C.c_int * 3)()
        lo = (C.c_int * (3 * workers))()
        hi = (C.c_int * (3 * workers))()
        nbr = (C.c_int * (6 * workers))()
        err = NdgoError()
        fn = self.lib.ndgo_decompose if self.kind == "port" else self.lib.ref_decompose
        rc = fn(C.byref(p.ndgo()), workers, grid, lo, hi, nbr, C.byref(err))
        if rc:
            raise CheckerError(err.code, err.step, err.worker, err.message.decode())
        return (tuple(grid), np.array(lo).reshape(workers, 3), np.array(hi).reshape(workers, 3),
                np.array(nbr).reshape(workers, 3, 2))

    def pack_face_trace(self, p: Problem, cells, u, axis, cell_d, node_d) -> np.ndarray:
        cl = (C.c_int * 3)(*cells)
        n = p.n_var
        for a in range(p.dim):
            if a != axis:
                n *= cells[a] * p.order
        out = np.zeros(n)
        u = np.ascontiguousarray(u, dtype=np.float64)
        fn = self.lib.ndgo_pack_face_trace if self.kind == "port" else self.lib.ref_pack_face_trace
        fn(C.byref(p.ndgo()), cl, _dp(u), axis, cell_d, node_d, _dp(out))
        return out


def fnv1a64(a: np.ndarray) -> str:
    """FNV-1a 64 of the raw little-endian bytes (report.cpp:284-293 over the state)."""
    b = np.ascontiguousarray(a, dtype="<f8").tobytes()
    h = 0xCBF29CE484222325
    mask = (1 << 64) - 1
    # vectorised FNV is sequential; do it in C via the port when available
    try:
        lib = Oracle("port").lib
        return "%016x" % lib.ndgo_fnv1a64(b, len(b))
    except Exception:  # pragma: no cover
        for ch in b:
            h ^= ch
            h = (h * 0x100000001B3) & mask
        return "%016x" % h


def rel_l2(checker: Oracle, p: Problem, got: np.ndarray, want: np.ndarray):
    """Per-variable relative GL-L2 (SURVEY.md §8d correctness gate)."""
    zero = np.zeros_like(want)
    out = []
    for v in range(p.n_var):
        num = checker.l2_error(p, got, want, v)
        den = checker.l2_error(p, want, zero, v)
        out.append(num / max(den, 1e-300) if den > 1e-14 else num)
    return out
