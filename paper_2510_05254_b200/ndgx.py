"""Host-side mirror of the reference solver API over the ndgx C ABI.

The names, argument meaning and error behaviour follow the reference's C++
interface (/root/reference/proj, paths below relative to it):

    Mesh, EquationModel          include/ndg/grid.hpp:18-37, models.hpp:43-73
    SolverConfig, StepPlan       include/ndg/solver.hpp:142-171
    advance                      src/solver.cpp:372-440
    serial_rhs                   src/solver.cpp:442-456
    decompose                    src/partition.cpp:44-106
    gauss_lobatto, differentiation_matrix   src/basis.cpp:32-118
    init_multisine, init_euler_subsonic     src/grid.cpp:135-188
    ConfigError ... RunError     include/ndg/errors.hpp:13-56

States are numpy float64 arrays in the reference's AoS layout
(FieldShape::index).  Every compute call goes through libndgx.so (sm_100a
kernels); there is no CPU fallback -- a missing library or a missing GPU
raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NDGX_LIB") or os.path.join(_PKG, "libndgx.so")  # NDGX_LIB: tuning builds

ADVECTION, EULER_ISOTHERMAL = 0, 1
RK3, RK4, RK6 = 0, 1, 2
RK_NAMES = {"rk3": RK3, "rk4": RK4, "rk6": RK6}
RK_STAGES = {RK3: 3, RK4: 4, RK6: 7}
ARITH_EXACT, ARITH_FAST = 0, 1
IC_MULTISINE, IC_EULER_SUBSONIC = 0, 1  # ndgx_ic: device initial conditions


# ----------------------------------------------------------------- errors
class NdgError(Exception):
    """Base of the mirrored exception taxonomy."""


class ConfigError(NdgError, ValueError):
    pass


class PhysicsError(NdgError, RuntimeError):
    pass


class InstabilityError(NdgError, RuntimeError):
    def __init__(self, what: str, step: int):
        super().__init__(what)
        self.step = step


class DecompositionError(NdgError, RuntimeError):
    pass


class TransportError(NdgError, RuntimeError):
    pass


class RunError(NdgError, RuntimeError):
    def __init__(self, what: str, worker: int):
        super().__init__(what)
        self.worker = worker


class CudaError(NdgError, RuntimeError):
    pass


# ------------------------------------------------------------------ ABI
class Problem(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("cells", C.c_int * 3), ("length", C.c_double * 3), ("order", C.c_int),
        ("equation", C.c_int), ("velocity", C.c_double * 3), ("sound_speed", C.c_double),
        ("rk", C.c_int), ("cfl", C.c_double), ("t_end", C.c_double),
        ("nodes", C.POINTER(C.c_double)), ("weights", C.POINTER(C.c_double)),
        ("diff", C.POINTER(C.c_double)), ("device", C.c_int), ("arith", C.c_int),
    ]


class Stats(C.Structure):
    _fields_ = [("steps", C.c_long), ("dt_min", C.c_double), ("dt_max", C.c_double),
                ("wall_seconds", C.c_double)]


class Error(C.Structure):
    _fields_ = [("code", C.c_int), ("step", C.c_long), ("stage", C.c_int), ("worker", C.c_int),
                ("cell", C.c_int * 3), ("message", C.c_char * 256)]


class RankPlan(C.Structure):
    """ndgx_rank_plan: one rank's block of decompose()'s tiling (include/ndgx.h)."""
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("grid", C.c_int * 3), ("lo", C.c_int * 3),
                ("hi", C.c_int * 3), ("split", C.c_int * 3), ("nbr", (C.c_int * 2) * 3),
                ("plane", C.c_longlong * 3)]

    def cells(self):
        return tuple(self.hi[a] - self.lo[a] for a in range(3))


_lib = None


def lib() -> C.CDLL:
    """Load libndgx.so (built in-tree by paper_2510_05254_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2510_05254_b200.build` "
                          "(the ndgx path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    D = P(C.c_double)
    L.ndgx_create.argtypes = [P(Problem), P(C.c_void_p), P(Error)]
    L.ndgx_destroy.argtypes = [C.c_void_p]
    L.ndgx_destroy.restype = None
    L.ndgx_upload.argtypes = [C.c_void_p, C.c_void_p, P(Error)]
    L.ndgx_download.argtypes = [C.c_void_p, C.c_void_p, P(Error)]
    L.ndgx_rhs.argtypes = [C.c_void_p, C.c_void_p, P(Error)]
    L.ndgx_advance.argtypes = [C.c_void_p, C.c_long, C.c_int, P(Stats), P(Error)]
    L.ndgx_launch_steps.argtypes = [C.c_void_p, C.c_long, P(Error)]
    L.ndgx_sync.argtypes = [C.c_void_p, P(Stats), P(Error)]
    L.ndgx_profile_step.argtypes = [C.c_void_p, P(C.c_float), C.c_int, P(Error)]
    L.ndgx_stream.argtypes = [C.c_void_p]
    L.ndgx_stream.restype = C.c_void_p
    L.ndgx_dof.argtypes = [C.c_void_p]
    L.ndgx_dof.restype = C.c_int64
    L.ndgx_state_size.argtypes = [C.c_void_p]
    L.ndgx_state_size.restype = C.c_size_t
    L.ndgx_stages.argtypes = [C.c_void_p]
    L.ndgx_gauss_lobatto.argtypes = [C.c_int, D, D]
    L.ndgx_differentiation_matrix.argtypes = [C.c_int, D, D]
    L.ndgx_init_multisine.argtypes = [P(Problem), D, C.c_int, D]
    L.ndgx_multisine_amplitudes.argtypes = [C.c_int, C.c_uint64, D]
    L.ndgx_multisine_amplitudes.restype = None
    L.ndgx_init_euler_subsonic.argtypes = [P(Problem), D]
    L.ndgx_decompose.argtypes = [C.c_int, P(C.c_int), C.c_int, P(C.c_int), P(C.c_int), P(C.c_int),
                                 P(C.c_int), P(Error)]
    L.ndgx_version.restype = C.c_char_p
    L.ndgx_plan_rank.argtypes = [P(Problem), C.c_int, C.c_int, C.c_int, P(RankPlan), P(Error)]
    L.ndgx_nccl_unique_id.argtypes = [C.c_char_p, P(Error)]
    L.ndgx_create_rank.argtypes = [P(Problem), C.c_int, C.c_int, C.c_char_p, C.c_int, P(C.c_void_p), P(Error)]
    L.ndgx_get_plan.argtypes = [C.c_void_p, P(RankPlan)]
    L.ndgx_create_partitioned.argtypes = [P(Problem), C.c_int, C.c_int, P(C.c_int), C.c_int, P(C.c_void_p),
                                          P(Error)]
    L.ndgx_workers.argtypes = [C.c_void_p]
    L.ndgx_get_block.argtypes = [C.c_void_p, C.c_int, P(RankPlan)]
    L.ndgx_dump_field.argtypes = [C.c_void_p, C.c_char_p, P(Error)]
    L.ndgx_load_field.argtypes = [C.c_void_p, C.c_char_p, P(Error)]
    L.ndgx_init_multisine_block.argtypes = [P(Problem), D, C.c_int, P(C.c_int), P(C.c_int), D]
    L.ndgx_init_euler_subsonic_block.argtypes = [P(Problem), P(C.c_int), P(C.c_int), D]
    L.ndgx_init_device.argtypes = [C.c_void_p, C.c_int, D, C.c_int, P(Error)]
    L.ndgx_conserved_totals_device.argtypes = [C.c_void_p, D, P(Error)]
    L.ndgx_l2_error_ic_device.argtypes = [C.c_void_p, C.c_int, D, C.c_int, C.c_int, D, P(Error)]
    L.ndgx_l1_norm_device.argtypes = [C.c_void_p, C.c_int, D, P(Error)]
    _lib = L
    return L


def _raise(err: Error, rc: int):
    msg = err.message.decode(errors="replace")
    code = err.code or rc
    if code == 1:
        raise ConfigError(msg)
    if code == 2:
        raise PhysicsError(msg)
    if code == 3:
        raise InstabilityError(msg, int(err.step))
    if code == 4:
        raise DecompositionError(msg)
    if code == 5:
        raise TransportError(msg)
    if code == 6:
        raise RunError(msg, int(err.worker))
    raise CudaError(msg or f"ndgx call failed with status {rc}")


def _check(rc: int, err: Error):
    if rc != 0:
        _raise(err, rc)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# --------------------------------------------------------- mirrored types
@dataclass
class Mesh:
    """Mesh(dim, cells, order, length) -- include/ndg/grid.hpp:18-37."""
    dim: int
    cells: Sequence[int]
    order: int
    length: Sequence[float] = (1.0, 1.0, 1.0)

    def __post_init__(self):
        if self.dim < 1 or self.dim > 3:
            raise ConfigError("mesh dimension must be 1..3")
        if self.order < 2 or self.order > 16:
            raise ConfigError("mesh order must lie in 2..16")
        c = list(self.cells) + [1] * (3 - len(self.cells))
        ln = list(self.length) + [1.0] * (3 - len(self.length))
        for a in range(self.dim):
            if c[a] < 1:
                raise ConfigError("cell count must be >= 1 on every axis")
            if not ln[a] > 0.0:
                raise ConfigError("domain length must be positive")
        self.cells = tuple(c[a] if a < self.dim else 1 for a in range(3))
        self.length = tuple(float(ln[a]) if a < self.dim else 1.0 for a in range(3))

    def cell_size(self, axis: int) -> float:
        return self.length[axis] / self.cells[axis]

    def cell_count(self) -> int:
        return self.cells[0] * self.cells[1] * self.cells[2]

    def nodes_per_cell(self) -> int:
        return self.order ** self.dim

    def dof(self, model: "EquationModel") -> int:
        return self.cell_count() * self.nodes_per_cell() * model.n_var()

    def wrap_cell(self, axis: int, cell: int, offset: int) -> int:
        n = self.cells[axis]
        c = (cell + offset) % n  # python % is already non-negative
        return c


@dataclass
class EquationModel:
    """EquationModel::advection / ::isothermal_euler -- include/ndg/models.hpp:43-73."""
    kind: int
    spatial_dim: int
    velocity: tuple = (0.0, 0.0, 0.0)
    sound_speed: float = 0.0

    @staticmethod
    def advection(spatial_dim: int, velocity) -> "EquationModel":
        if spatial_dim < 1 or spatial_dim > 3:
            raise ConfigError("advection: spatial_dim must be 1..3")
        v = tuple(float(x) for x in (list(velocity) + [0.0, 0.0, 0.0])[:3])
        return EquationModel(ADVECTION, spatial_dim, v, 0.0)

    @staticmethod
    def isothermal_euler(spatial_dim: int, sound_speed: float) -> "EquationModel":
        if spatial_dim < 2 or spatial_dim > 3:
            raise ConfigError("isothermal_euler: spatial_dim must be 2 or 3")
        if not sound_speed > 0.0:
            raise ConfigError("isothermal_euler: sound speed must be positive")
        return EquationModel(EULER_ISOTHERMAL, spatial_dim, (0.0, 0.0, 0.0), float(sound_speed))

    def n_var(self) -> int:
        return 1 if self.kind == ADVECTION else self.spatial_dim + 1


@dataclass
class SolverConfig:
    """SolverConfig -- include/ndg/solver.hpp:142-148."""
    mesh: Mesh
    model: EquationModel
    rk: int = RK4
    cfl: float = 0.4
    t_end: float = 1.0


@dataclass
class StepPlan:
    """StepPlan -- include/ndg/solver.hpp:168-171."""
    fixed_steps: int = -1
    warmup: bool = False


@dataclass
class StepStats:
    """StepStats -- include/ndg/solver.hpp:153-158 (wall_seconds from CUDA events)."""
    steps: int = 0
    dt_min: float = float("inf")
    dt_max: float = 0.0
    wall_seconds: float = 0.0


@dataclass
class AdvanceResult:
    state: np.ndarray
    stats: StepStats


def rk_from_name(name: str) -> int:
    if name not in RK_NAMES:
        raise ConfigError(f"unknown Runge-Kutta scheme '{name}' (expected rk3, rk4 or rk6)")
    return RK_NAMES[name]


def validate(config: SolverConfig) -> None:
    """validate (src/solver.cpp:349-357)."""
    if not config.cfl > 0.0 or config.cfl > 1.0:
        raise ConfigError("cfl must lie in (0, 1]")
    if not config.t_end > 0.0:
        raise ConfigError("t_end must be positive")
    if config.model.spatial_dim != config.mesh.dim:
        raise ConfigError("model dimension does not match mesh dimension")


def make_problem(config: SolverConfig, device: int = 0, arith: int = ARITH_EXACT,
                 basis=None) -> Problem:
    m, mod = config.mesh, config.model
    p = Problem()
    p.dim = m.dim
    for a in range(3):
        p.cells[a] = m.cells[a]
        p.length[a] = m.length[a]
        p.velocity[a] = mod.velocity[a]
    p.order = m.order
    p.equation = mod.kind
    p.sound_speed = mod.sound_speed
    p.rk = config.rk
    p.cfl = config.cfl
    p.t_end = config.t_end
    p.device = device
    p.arith = arith
    if basis is not None:
        nodes, weights, diff = (np.ascontiguousarray(x, dtype=np.float64) for x in basis)
        p._keep = (nodes, weights, diff)  # keep alive
        p.nodes, p.weights, p.diff = _dptr(nodes), _dptr(weights), _dptr(diff)
    return p


class Solver:
    """A device-resident solver handle (one ndgx_solver)."""

    def __init__(self, config: SolverConfig, device: int = 0, arith: int = ARITH_EXACT, basis=None,
                 _rank=None, _part=None):
        validate(config)
        self.config = config
        self.problem = make_problem(config, device, arith, basis)
        self._h = C.c_void_p()
        err = Error()
        if _part is not None:
            workers, devices, force = _part
            devs = (C.c_int * max(1, len(devices)))(*devices) if devices else None
            _check(lib().ndgx_create_partitioned(C.byref(self.problem), workers, len(devices) if devices else 0,
                                                 devs, int(force), C.byref(self._h), C.byref(err)), err)
        elif _rank is None:
            _check(lib().ndgx_create(C.byref(self.problem), C.byref(self._h), C.byref(err)), err)
        else:
            nranks, rank, nccl_id, force = _rank
            _check(lib().ndgx_create_rank(C.byref(self.problem), nranks, rank, nccl_id, int(force),
                                          C.byref(self._h), C.byref(err)), err)
        self.size = int(lib().ndgx_state_size(self._h))
        self.dof = int(lib().ndgx_dof(self._h))
        self.stages = int(lib().ndgx_stages(self._h))
        self.plan = RankPlan()
        lib().ndgx_get_plan(self._h, C.byref(self.plan))
        self.workers = int(lib().ndgx_workers(self._h))

    @classmethod
    def partitioned(cls, config: SolverConfig, workers: int, devices: Optional[Sequence[int]] = None,
                    arith: int = ARITH_EXACT, force_exchange: bool = False) -> "Solver":
        """run_partitioned's `workers` blocks (src/partition.cpp:186-333) in one
        handle, block w on devices[w % len(devices)] (default: device 0).  Halo
        planes move by peer stores; states in and out are the GLOBAL field;
        failures raise RunError("worker w: ...")."""
        devices = list(devices) if devices else [0]
        return cls(config, devices[0], arith, None, _part=(workers, devices, force_exchange))

    def block(self, worker: int) -> RankPlan:
        """The Block of `worker` (lo/hi, neighbours, split axes) in this handle."""
        pl = RankPlan()
        if lib().ndgx_get_block(self._h, worker, C.byref(pl)) != 0:
            raise ConfigError(f"no worker {worker} in this handle")
        return pl

    @classmethod
    def for_rank(cls, config: SolverConfig, nranks: int, rank: int, nccl_id: bytes, device: int = 0,
                 arith: int = ARITH_EXACT, force_exchange: bool = False) -> "Solver":
        """This rank's block of `config.mesh` (the GLOBAL mesh), exchanging face
        halos over NCCL with the other ranks (run_partitioned, src/partition.cpp:186-333)."""
        if len(nccl_id) != 128:
            raise TransportError("an NCCL unique id is 128 bytes")
        _preload_nccl()
        return cls(config, device, arith, None, _rank=(nranks, rank, nccl_id, force_exchange))

    def close(self):
        if self._h:
            lib().ndgx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _arr(self, u) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        if u.size != self.size:
            raise ConfigError(f"state has {u.size} values, expected {self.size}")
        return u

    def upload(self, u) -> None:
        u = self._arr(u)
        err = Error()
        _check(lib().ndgx_upload(self._h, u.ctypes.data, C.byref(err)), err)

    def upload_ptr(self, host_ptr: int) -> None:
        err = Error()
        _check(lib().ndgx_upload(self._h, C.c_void_p(host_ptr), C.byref(err)), err)

    def download(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.size, dtype=np.float64)
        err = Error()
        _check(lib().ndgx_download(self._h, out.ctypes.data, C.byref(err)), err)
        return out

    def download_ptr(self, host_ptr: int) -> None:
        err = Error()
        _check(lib().ndgx_download(self._h, C.c_void_p(host_ptr), C.byref(err)), err)

    def rhs(self) -> np.ndarray:
        out = np.empty(self.size, dtype=np.float64)
        err = Error()
        _check(lib().ndgx_rhs(self._h, out.ctypes.data, C.byref(err)), err)
        return out

    def advance(self, plan: StepPlan = StepPlan()) -> StepStats:
        st, err = Stats(), Error()
        _check(lib().ndgx_advance(self._h, plan.fixed_steps, int(plan.warmup), C.byref(st),
                                  C.byref(err)), err)
        return StepStats(st.steps, st.dt_min, st.dt_max, st.wall_seconds)

    def launch_steps(self, steps: int) -> None:
        err = Error()
        _check(lib().ndgx_launch_steps(self._h, steps, C.byref(err)), err)

    def sync(self) -> StepStats:
        st, err = Stats(), Error()
        _check(lib().ndgx_sync(self._h, C.byref(st), C.byref(err)), err)
        return StepStats(st.steps, st.dt_min, st.dt_max, st.wall_seconds)

    def profile_step(self):
        ms = (C.c_float * 16)()
        err = Error()
        _check(lib().ndgx_profile_step(self._h, ms, 16, C.byref(err)), err)
        return [ms[i] for i in range(self.stages)], ms[self.stages]

    def dump_field(self, path: str) -> None:
        """Checkpoint the device state in the reference's ndgfield format
        (dump_field, src/field_io.cpp:18-34)."""
        err = Error()
        _check(lib().ndgx_dump_field(self._h, os.fsencode(path), C.byref(err)), err)

    def load_field(self, path: str) -> None:
        """Restart from an ndgfield dump (load_field, src/field_io.cpp:36-72)."""
        err = Error()
        _check(lib().ndgx_load_field(self._h, os.fsencode(path), C.byref(err)), err)

    # ------------------------------------------------ f4: device ICs and diagnostics
    def init_device(self, ic: int, amplitudes=None) -> None:
        """Generate the initial condition straight into HBM (init_multisine /
        init_euler_subsonic, src/grid.cpp:135-188, + upload): no host field,
        no H2D copy.  `amplitudes` (multisine) as from multisine_amplitudes."""
        amps = None if amplitudes is None else np.ascontiguousarray(amplitudes, dtype=np.float64)
        err = Error()
        _check(lib().ndgx_init_device(self._h, ic, None if amps is None else _dptr(amps),
                                      0 if amps is None else len(amps), C.byref(err)), err)

    def conserved_totals_device(self) -> np.ndarray:
        """conserved_totals of the device state (src/grid.cpp:205-213)."""
        out = np.zeros(4)
        err = Error()
        _check(lib().ndgx_conserved_totals_device(self._h, _dptr(out), C.byref(err)), err)
        return out[:self.config.model.n_var()].copy()

    def l2_error_ic_device(self, ic: int, amplitudes=None, var: int = 0) -> float:
        """l2_error(state, init_*(...), var) with the IC evaluated on the fly
        (src/grid.cpp:190-203; the experiments' error, src/experiments.cpp:112)."""
        amps = None if amplitudes is None else np.ascontiguousarray(amplitudes, dtype=np.float64)
        out = np.zeros(1)
        err = Error()
        _check(lib().ndgx_l2_error_ic_device(self._h, ic, None if amps is None else _dptr(amps),
                                             0 if amps is None else len(amps), var, _dptr(out),
                                             C.byref(err)), err)
        return float(out[0])

    def l1_norm_device(self, var: int = 0) -> float:
        """l1_norm of the device state (src/grid.cpp:215-223)."""
        out = np.zeros(1)
        err = Error()
        _check(lib().ndgx_l1_norm_device(self._h, var, _dptr(out), C.byref(err)), err)
        return float(out[0])

    @property
    def stream(self) -> int:
        return int(lib().ndgx_stream(self._h) or 0)


# ------------------------------------------------------- reference API
def advance(config: SolverConfig, initial, plan: StepPlan = StepPlan(), device: int = 0,
            arith: int = ARITH_EXACT) -> AdvanceResult:
    """advance(config, initial, plan) -- src/solver.cpp:372-440, on the GPU."""
    with Solver(config, device, arith) as s:
        s.upload(initial)
        stats = s.advance(plan)
        return AdvanceResult(s.download(), stats)


@dataclass
class WorkerTiming:
    """WorkerTiming (include/ndg/partition.hpp:49-52).  The device path overlaps
    the halo exchange with interior elements, so the whole stepping time of the
    handle is reported as compute and the exchange as 0."""
    compute_seconds: float = 0.0
    exchange_seconds: float = 0.0


@dataclass
class PartitionedResult:
    """PartitionedResult (include/ndg/partition.hpp:54-60)."""
    state: np.ndarray
    stats: StepStats
    worker_timings: list
    decomposition: "BlockDecomposition"


def run_partitioned(config: SolverConfig, initial, worker_count: int, plan: StepPlan = StepPlan(),
                    devices: Optional[Sequence[int]] = None, arith: int = ARITH_EXACT) -> PartitionedResult:
    """run_partitioned(config, initial, workers, plan) -- src/partition.cpp:186-333,
    on the GPU: worker_count blocks of decompose()'s tiling in one handle (block w
    on devices[w % len(devices)]).  Bit-identical to advance() in either
    arithmetic mode; failures raise RunError("worker w: ...", w)."""
    validate(config)
    decomposition = decompose(config.mesh, worker_count)
    with Solver.partitioned(config, worker_count, devices, arith) as s:
        s.upload(initial)
        stats = s.advance(plan)
        state = s.download()
    timings = [WorkerTiming(stats.wall_seconds, 0.0) for _ in range(worker_count)]
    return PartitionedResult(state, stats, timings, decomposition)


def serial_rhs(mesh: Mesh, model: EquationModel, field, basis=None, device: int = 0,
               arith: int = ARITH_EXACT) -> np.ndarray:
    """serial_rhs(mesh, basis, model, field) -- src/solver.cpp:442-456, on the GPU."""
    with Solver(SolverConfig(mesh, model), device, arith, basis) as s:
        s.upload(field)
        return s.rhs()


def gauss_lobatto(order: int):
    nodes, w = np.zeros(order), np.zeros(order)
    if lib().ndgx_gauss_lobatto(order, _dptr(nodes), _dptr(w)) != 0:
        raise ConfigError(f"gauss_lobatto: order must lie in 2..16, got {order}")
    return nodes, w


def differentiation_matrix(order: int, nodes) -> np.ndarray:
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    d = np.zeros(order * order)
    lib().ndgx_differentiation_matrix(order, _dptr(nodes), _dptr(d))
    return d


def multisine_amplitudes(n_modes: int, seed: int) -> np.ndarray:
    if n_modes < 1:
        raise ConfigError("multisine: need at least one mode")
    out = np.zeros(n_modes)
    lib().ndgx_multisine_amplitudes(n_modes, seed, _dptr(out))
    return out


def init_multisine(mesh: Mesh, model: EquationModel, amplitudes=None, n_modes=None, seed=None,
                   out: Optional[np.ndarray] = None) -> np.ndarray:
    if amplitudes is None:
        amplitudes = multisine_amplitudes(n_modes, seed)
    amps = np.ascontiguousarray(amplitudes, dtype=np.float64)
    p = make_problem(SolverConfig(mesh, model))
    if out is None:
        out = np.zeros(mesh.dof(model))
    if lib().ndgx_init_multisine(C.byref(p), _dptr(amps), len(amps), _dptr(out)) != 0:
        raise ConfigError("init_multisine applies to the advection scalar only")
    return out


def init_euler_subsonic(mesh: Mesh, model: EquationModel, out: Optional[np.ndarray] = None) -> np.ndarray:
    p = make_problem(SolverConfig(mesh, model))
    if out is None:
        out = np.zeros(mesh.dof(model))
    if lib().ndgx_init_euler_subsonic(C.byref(p), _dptr(out)) != 0:
        raise ConfigError("init_euler_subsonic requires an isothermal Euler model on a 2D/3D mesh")
    return out


def l2_error(mesh: Mesh, model: EquationModel, a, b, var: int = 0) -> float:
    """l2_error (src/grid.cpp:190-203), summed in the reference's order (bit-identical)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.size != mesh.dof(model) or b.size != a.size:
        raise ConfigError("l2_error: field shapes do not match")
    if not 0 <= var < model.n_var():
        raise IndexError("l2_error: bad variable")
    p = make_problem(SolverConfig(mesh, model))
    out = C.c_double()
    if lib().ndgx_l2_error(C.byref(p), _dptr(a), _dptr(b), var, C.byref(out)) != 0:
        raise ConfigError("l2_error: invalid problem")
    return out.value


def conserved_totals(mesh: Mesh, model: EquationModel, u) -> np.ndarray:
    """conserved_totals (src/grid.cpp:205-213), summed in the reference's order."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    if u.size != mesh.dof(model):
        raise ConfigError("conserved_totals: field shape does not match")
    p = make_problem(SolverConfig(mesh, model))
    out = np.zeros(model.n_var())
    if lib().ndgx_conserved_totals(C.byref(p), _dptr(u), _dptr(out)) != 0:
        raise ConfigError("conserved_totals: invalid problem")
    return out


@dataclass
class Block:
    coord: tuple
    lo: tuple
    hi: tuple
    neighbor: tuple  # [axis][0 low, 1 high]

    def cells(self):
        return tuple(self.hi[a] - self.lo[a] for a in range(3))


@dataclass
class BlockDecomposition:
    worker_count: int
    grid: tuple
    blocks: list = field(default_factory=list)


def decompose(mesh: Mesh, worker_count: int) -> BlockDecomposition:
    """decompose (src/partition.cpp:44-106)."""
    w = max(worker_count, 1)
    cells = (C.c_int * 3)(*mesh.cells)
    grid = (C.c_int * 3)()
    lo, hi = (C.c_int * (3 * w))(), (C.c_int * (3 * w))()
    nbr = (C.c_int * (6 * w))()
    err = Error()
    _check(lib().ndgx_decompose(mesh.dim, cells, worker_count, grid, lo, hi, nbr, C.byref(err)), err)
    g = tuple(grid)
    blocks = []
    for k in range(worker_count):
        coord = (k // (g[1] * g[2]), (k // g[2]) % g[1], k % g[2])
        blocks.append(Block(coord, tuple(lo[3 * k:3 * k + 3]), tuple(hi[3 * k:3 * k + 3]),
                            tuple((nbr[6 * k + 2 * a], nbr[6 * k + 2 * a + 1]) for a in range(3))))
    return BlockDecomposition(worker_count, g, blocks)


def plan_rank(config: SolverConfig, nranks: int, rank: int, force_exchange: bool = False) -> RankPlan:
    """The block of `rank` in decompose()'s tiling of the global mesh (no GPU needed)."""
    p = make_problem(config)
    plan, err = RankPlan(), Error()
    _check(lib().ndgx_plan_rank(C.byref(p), nranks, rank, int(force_exchange), C.byref(plan), C.byref(err)), err)
    return plan


_nccl_preloaded = False


def _preload_nccl() -> None:
    """Make libndgx's dlopen("libnccl.so.2") resolve to PyTorch's bundled NCCL
    (the one torch.distributed already uses in the same process), not a
    second, older system copy."""
    global _nccl_preloaded
    if _nccl_preloaded:
        return
    _nccl_preloaded = True
    try:
        import nvidia.nccl  # the wheel torch links against
        path = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        if os.path.exists(path):
            C.CDLL(path, mode=C.RTLD_GLOBAL)
    except Exception:  # noqa: BLE001 -- fall back to the system libnccl.so.2
        pass


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 creates it; broadcast it to every rank)."""
    _preload_nccl()
    buf = C.create_string_buffer(128)
    err = Error()
    _check(lib().ndgx_nccl_unique_id(buf, C.byref(err)), err)
    return buf.raw


def init_block(config: SolverConfig, lo, hi, n_modes: int = 40, seed: int = 42,
               out: Optional[np.ndarray] = None) -> np.ndarray:
    """The reference's initial condition (init_euler_subsonic for Euler,
    init_multisine otherwise) on the block [lo, hi) of the global mesh, in the
    block's own AoS layout -- exactly the slice of the global field."""
    p = make_problem(config)
    lo3 = (C.c_int * 3)(*(list(lo) + [0, 0, 0])[:3])
    hi3 = (C.c_int * 3)(*(list(hi) + [1, 1, 1])[:3])
    n = config.model.n_var() * config.mesh.nodes_per_cell()
    for a in range(config.mesh.dim):
        n *= hi3[a] - lo3[a]
    if out is None:
        out = np.zeros(n)
    if config.model.kind == EULER_ISOTHERMAL:
        rc = lib().ndgx_init_euler_subsonic_block(C.byref(p), lo3, hi3, _dptr(out))
    else:
        amps = multisine_amplitudes(n_modes, seed)
        rc = lib().ndgx_init_multisine_block(C.byref(p), _dptr(amps), len(amps), lo3, hi3, _dptr(out))
    if rc != 0:
        raise ConfigError("init_block: invalid block or model")
    return out


def dump_field(path: str, mesh: Mesh, field) -> None:
    """dump_field(path, mesh, field) (src/field_io.cpp:18-34) for a host field."""
    f = np.ascontiguousarray(field, dtype="<f8")
    lines = ["ndgfield 1", f"dim {mesh.dim}", "cells " + " ".join(str(mesh.cells[a]) for a in range(mesh.dim)),
             f"order {mesh.order}", f"nvar {f.size // (mesh.cell_count() * mesh.nodes_per_cell())}",
             "length " + " ".join(_fmt_g6(mesh.length[a]) for a in range(mesh.dim)), "data"]
    with open(path, "wb") as fh:
        fh.write(("\n".join(lines) + "\n").encode())
        fh.write(f.tobytes())


def load_field(path: str):
    """load_field(path) (src/field_io.cpp:36-72) -> (dim, cells, order, nvar, length, field)."""
    with open(path, "rb") as fh:
        if fh.readline() != b"ndgfield 1\n":
            raise RuntimeError(f"{path}: not an ndgfield dump")
        hdr = {}
        while True:
            line = fh.readline()
            if not line:
                raise RuntimeError(f"{path}: missing data section")
            line = line.decode().rstrip("\n")
            if line == "data":
                break
            key, *vals = line.split()
            if key not in ("dim", "cells", "order", "nvar", "length"):
                raise RuntimeError(f"{path}: unknown header key '{key}'")
            hdr[key] = vals
        payload = fh.read()
    dim = int(hdr["dim"][0])
    cells = tuple(int(x) for x in hdr["cells"][:dim])
    order, nvar = int(hdr["order"][0]), int(hdr["nvar"][0])
    n = nvar * order ** dim * int(np.prod(cells))
    if len(payload) < 8 * n:
        raise RuntimeError(f"{path}: truncated payload")
    return dim, cells, order, nvar, tuple(float(x) for x in hdr["length"][:dim]), \
        np.frombuffer(payload[:8 * n], dtype="<f8").copy()


def _fmt_g6(x: float) -> str:
    """std::ostream's default double formatting (precision 6, %g)."""
    return f"{x:g}"


def version() -> str:
    return lib().ndgx_version().decode()
