"""Python mirror of the reference's BA / LM API over the C ABI.

Names, argument meaning and error behaviour follow traceopt
(/root/reference/proj/include/traceopt):

* ``make_ba_problem(poses, points, intrinsics, observations)`` -- problems.hpp:87-136
* ``TracedProblem.{set_parameters, evaluate, jacobian, residual_rows, num_poses, num_points}``
  -- problems.hpp:36-82
* ``LmConfig`` / ``LmIterationRecord`` / ``LmReport`` / ``TerminationReason`` / ``SolverChoice``
  -- lm.hpp:20-77
* ``optimize(model, init_poses, init_points, config, final_state=None)`` -- lm.hpp:205-255
* ``stop_on_plateau(history, config)`` -- lm.hpp:104-108
* exceptions ``IndexError`` (with ``position``), ``CheiralityError`` (``observation``),
  ``NotSpdError``, ``NumericalBreakdownError``, ``UnsupportedOperationError`` -- errors.hpp:10-57;
  ``std::invalid_argument`` maps to ``ValueError``.

Arrays: poses (C, 7) = [tx, ty, tz, qx, qy, qz, qw] world->camera, points (P, 3),
BAL intrinsics (C, 3) = [f, k1, k2], observations = (cam_idx (N,), pt_idx (N,), pixels (N, 2)).
"""
from __future__ import annotations

import builtins
import ctypes
import dataclasses
import enum
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import CreateOptionsC, IterRecordC, LmConfigC, LmReportC, ptr


class IndexError(builtins.IndexError):  # noqa: A001 - mirrors traceopt::IndexError
    def __init__(self, msg, position):
        super().__init__(msg)
        self.position = position


class CheiralityError(RuntimeError):
    def __init__(self, msg, observation):
        super().__init__(msg)
        self.observation = observation


class NotSpdError(RuntimeError):
    def __init__(self, msg, pivot=-1):
        super().__init__(msg)
        self.pivot = pivot


class NumericalBreakdownError(RuntimeError):
    pass


class UnsupportedOperationError(RuntimeError):
    pass


class ParseError(RuntimeError):  # mirrors traceopt::ParseError (errors.hpp:60-69)
    def __init__(self, msg, line):
        super().__init__(msg)
        self.line = line


class DeviceError(RuntimeError):
    """CUDA / NCCL failure (no reference counterpart)."""


def _raise(code: int):
    lib = _lib.load()
    msg = (lib.bae_last_error() or b"").decode()
    idx = int(lib.bae_last_error_index())
    if code == 1:
        raise ValueError(msg)
    if code == 2:
        raise IndexError(msg, idx)
    if code == 3:
        raise CheiralityError(msg, idx)
    if code == 4:
        raise NotSpdError(msg, idx)
    if code == 5:
        raise NumericalBreakdownError(msg)
    if code == 6:
        raise UnsupportedOperationError(msg)
    if code == 9:
        raise ParseError(msg, idx)
    if code == 10:
        raise OSError(msg)
    raise DeviceError(f"[{code}] {msg}")


def _check(code: int):
    if code != 0:
        _raise(code)


class SolverChoice(enum.IntEnum):
    cholesky = 0
    pcg = 1


class TerminationReason(enum.IntEnum):
    plateau = 0
    max_iters = 1
    solver_failure = 2


@dataclasses.dataclass
class LmConfig:
    initial_damping: float = 1e-6
    damping_min: float = 1e-16
    damping_max: float = 1e16
    damping_up: float = 2.0
    damping_down: float = 0.5
    clamp_min: float = 1e-6
    clamp_max: float = 1e32
    max_iterations: int = 10
    plateau_patience: int = 3
    plateau_rel_tol: float = 1e-6
    solver: SolverChoice = SolverChoice.cholesky
    pcg_tol: float = 1e-8
    pcg_max_iters: int = 0
    use_caches: bool = True

    def to_c(self) -> LmConfigC:
        c = LmConfigC()
        for f in ("initial_damping", "damping_min", "damping_max", "damping_up", "damping_down", "clamp_min",
                  "clamp_max", "plateau_rel_tol", "pcg_tol"):
            setattr(c, f, float(getattr(self, f)))
        c.pcg_max_iters = int(self.pcg_max_iters)
        c.max_iterations = int(self.max_iterations)
        c.plateau_patience = int(self.plateau_patience)
        c.solver = int(self.solver)
        c.use_caches = 1 if self.use_caches else 0
        return c


@dataclasses.dataclass
class LmIterationRecord:
    iteration: int
    cost: float
    mse: float
    lmbda: float
    accepted: bool
    cum_time_s: float
    pcg_iters: int = 0
    grad_norm: float = 0.0
    trial_cost: float = float("nan")


@dataclasses.dataclass
class LmReport:
    final_cost: float
    final_mse: float
    iterations: int
    trajectory: List[LmIterationRecord]
    reason: TerminationReason
    accepted_steps: int = 0
    rejected_steps: int = 0
    final_lambda: float = 0.0
    solve_seconds: float = 0.0
    total_pcg_iters: int = 0
    device_seconds: float = 0.0


@dataclasses.dataclass
class LmState:
    poses: np.ndarray
    points: np.ndarray
    lmbda: float
    iterations: int
    accepted_steps: int
    rejected_steps: int


@dataclasses.dataclass
class BsrMatrix:
    """One Jacobian half (bsr.hpp:42-93): one br x bc block per residual row."""
    block_rows: int
    block_cols: int
    br: int
    bc: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray  # (nnz, br, bc)


@dataclasses.dataclass
class JacobianPair:
    j_pose: BsrMatrix
    j_point: BsrMatrix


@dataclasses.dataclass
class TransposePlan:
    row_ptr: np.ndarray
    col_idx: np.ndarray
    src_block: np.ndarray


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class TracedProblem:
    """Device-resident BA problem (the TracedProblem of problems.hpp:36-82)."""

    def __init__(self, handle, C, P, N):
        self._h = handle
        self._C, self._P, self._N = C, P, N

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.load().bae_destroy(h)
            self._h = None

    def num_poses(self) -> int:
        return self._C

    def num_points(self) -> int:
        return self._P

    def residual_rows(self) -> int:
        return self._N

    def residual_width(self) -> int:
        return 2

    def set_parameters(self, poses, points):
        p7 = _f64(poses, (self._C, 7))
        p3 = _f64(points, (self._P, 3))
        _check(_lib.load().bae_set_parameters(self._h, ptr(p7), ptr(p3)))

    def get_parameters(self):
        p7 = np.empty((self._C, 7))
        p3 = np.empty((self._P, 3))
        _check(_lib.load().bae_get_parameters(self._h, ptr(p7), ptr(p3)))
        return p7, p3

    def evaluate(self) -> np.ndarray:
        r = np.empty(2 * self._N)
        cost = ctypes.c_double()
        _check(_lib.load().bae_evaluate(self._h, ptr(r), ctypes.byref(cost)))
        return r

    def cost(self) -> float:
        cost = ctypes.c_double()
        _check(_lib.load().bae_evaluate(self._h, None, ctypes.byref(cost)))
        return cost.value

    def jacobian(self) -> JacobianPair:
        N = self._N
        jp = np.empty((N, 2, 6))
        jl = np.empty((N, 2, 3))
        prp = np.empty(N + 1, np.int64)
        lrp = np.empty(N + 1, np.int64)
        pc = np.empty(N, np.int32)
        lc = np.empty(N, np.int32)
        _check(_lib.load().bae_jacobian(self._h, ptr(jp), ptr(jl), ptr(prp, ctypes.c_int64), ptr(pc, ctypes.c_int32),
                                        ptr(lrp, ctypes.c_int64), ptr(lc, ctypes.c_int32)))
        return JacobianPair(BsrMatrix(N, self._C, 2, 6, prp, pc, jp), BsrMatrix(N, self._P, 2, 3, lrp, lc, jl))

    def transpose_plan(self, which: int) -> TransposePlan:
        cols = self._C if which == 0 else self._P
        rp = np.empty(cols + 1, np.int64)
        ci = np.empty(self._N, np.int32)
        sb = np.empty(self._N, np.int64)
        _check(_lib.load().bae_transpose_plan(self._h, which, ptr(rp, ctypes.c_int64), ptr(ci, ctypes.c_int32),
                                              ptr(sb, ctypes.c_int64)))
        return TransposePlan(rp, ci, sb)

    def normal_pattern(self, which: int):
        """(row_ptr, col_idx) of quadrant `which` of A = J^T J (0 CC, 1 CL,
        2 LC, 3 LL; spgemm_symbolic) or of the scalar CSR matrix A (4), from
        the device's observation decomposition."""
        lib = _lib.load()
        rows, nnz = ctypes.c_int64(), ctypes.c_int64()
        _check(lib.bae_normal_pattern(self._h, int(which), ctypes.byref(rows), ctypes.byref(nnz), None, None))
        rp = np.empty(rows.value + 1, np.int64)
        ci = np.empty(nnz.value, np.int32)
        _check(lib.bae_normal_pattern(self._h, int(which), ctypes.byref(rows), ctypes.byref(nnz),
                                      ptr(rp, ctypes.c_int64), ptr(ci, ctypes.c_int32)))
        return rp, ci

    def block_diagonals(self):
        hcc = np.empty((self._C, 6, 6))
        gc = np.empty((self._C, 6))
        hpp = np.empty((self._P, 3, 3))
        gp = np.empty((self._P, 3))
        _check(_lib.load().bae_block_diagonals(self._h, ptr(hcc), ptr(gc), ptr(hpp), ptr(gp)))
        return hcc, gc, hpp, gp

    def solve_step(self, lmbda: float, config: Optional[LmConfig] = None):
        cfg = (config or LmConfig(solver=SolverChoice.pcg)).to_c()
        delta = np.empty(6 * self._C + 3 * self._P)
        iters = ctypes.c_int64()
        rel = ctypes.c_double()
        _check(_lib.load().bae_solve_step(self._h, float(lmbda), ctypes.byref(cfg), ptr(delta), ctypes.byref(iters),
                                          ctypes.byref(rel)))
        return delta, iters.value, rel.value

    def time_kernel(self, kind: int, reps: int) -> float:
        ms = ctypes.c_double()
        _check(_lib.load().bae_time_kernel(self._h, int(kind), int(reps), ctypes.byref(ms)))
        return ms.value

    PHASES = ("linearize", "prep", "assemble", "factor", "pcg", "trial", "commit")

    def phase_times(self, reset: bool = False) -> dict:
        """Device ms per LM phase accumulated since the last reset."""
        out = np.zeros(7)
        _check(_lib.load().bae_phase_times(self._h, ptr(out), 1 if reset else 0))
        return dict(zip(self.PHASES, (float(v) for v in out)))

    def launch_count(self) -> int:
        return int(_lib.load().bae_launch_count(self._h))

    def shard(self):
        """(rank, world, local points, local observations) of this handle."""
        r, w, lp = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        lo = ctypes.c_int64()
        _check(_lib.load().bae_problem_shard(self._h, ctypes.byref(r), ctypes.byref(w), ctypes.byref(lp),
                                             ctypes.byref(lo)))
        return r.value, w.value, lp.value, lo.value

    def plan_array(self, which: int) -> np.ndarray:
        """One of the plan's device arrays (bae_plan_array), for planner parity tests."""
        lib = _lib.load()
        n, eb = ctypes.c_int64(), ctypes.c_int32()
        _check(lib.bae_plan_array(self._h, int(which), None, 0, ctypes.byref(n), ctypes.byref(eb)))
        dt = {1: np.uint8, 2: np.uint16, 4: np.int32, 8: np.float64}[eb.value]
        out = np.zeros(max(n.value, 1), dt)
        _check(lib.bae_plan_array(self._h, int(which), out.ctypes.data_as(ctypes.c_void_p), n.value, ctypes.byref(n),
                                  ctypes.byref(eb)))
        return out[:n.value]

    def direct_stats(self):
        """Tile Cholesky structure of the direct solver (zeros before its first use)."""
        out = np.zeros(5, np.int64)
        _check(_lib.load().bae_direct_stats(self._h, ptr(out, ctypes.c_int64)))
        keys = ("tile_columns", "tiles", "tile_updates", "nd_groups", "positions")
        st = dict(zip(keys, (int(v) for v in out)))
        npairs, nblocks = ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.load().bae_direct_pairs(self._h, ctypes.byref(npairs), ctypes.byref(nblocks)))
        st.update(pairs=int(npairs.value), camera_blocks=int(nblocks.value))
        return st

    def stats(self):
        out = np.empty(6, np.int64)
        _check(_lib.load().bae_problem_stats(self._h, ptr(out, ctypes.c_int64)))
        keys = ("observations", "points", "cameras", "tiles", "entries", "max_tile_obs")
        return dict(zip(keys, (int(v) for v in out)))


class PoseGraphProblem(TracedProblem):
    """make_pgo_problem (problems.hpp:141-188): one 6-row residual per edge,
    Log(z_i^-1 z_j T^-1) whitened by L^T of the edge information."""

    def residual_width(self) -> int:
        return 6

    def evaluate(self) -> np.ndarray:
        r = np.empty(6 * self._N)
        cost = ctypes.c_double()
        _check(_lib.load().bae_evaluate(self._h, ptr(r), ctypes.byref(cost)))
        return r

    def get_parameters(self):
        p7 = np.empty((self._C, 7))
        _check(_lib.load().bae_get_parameters(self._h, ptr(p7), None))
        return p7, np.zeros((0, 3))

    def set_parameters(self, poses, points=None):
        p7 = _f64(poses, (self._C, 7))
        _check(_lib.load().bae_set_parameters(self._h, ptr(p7), None))

    def edge_jacobians(self):
        """Per edge d r_w / d pose_i and d r_w / d pose_j (6 x 6 each)."""
        ji, jj = np.empty((self._N, 6, 6)), np.empty((self._N, 6, 6))
        _check(_lib.load().bae_pgo_jacobian(self._h, ptr(ji), ptr(jj)))
        return ji, jj


def make_pgo_problem(poses, edge_i=None, edge_j=None, measurements=None, information=None, has_information=None,
                     anchor_first: bool = True, *, device: int = 0) -> PoseGraphProblem:
    """make_pgo_problem (problems.hpp:141-188). ``information`` is E x 6 x 6
    (or None: unwhitened), ``has_information`` flags the edges that carry one.
    ``make_pgo_problem(graph)`` takes a PoseGraph (io/g2o.hpp:82-84)."""
    if isinstance(poses, PoseGraph):
        g = poses
        return make_pgo_problem(g.vertices, g.edge_i, g.edge_j, g.measurements, g.information,
                                g.has_information, anchor_first if edge_i is None else bool(edge_i), device=device)
    p7 = _f64(poses).reshape(-1, 7)
    ei, ej = _i32(edge_i), _i32(edge_j)
    meas = _f64(measurements).reshape(-1, 7)
    info = None if information is None else _f64(information).reshape(-1, 36)
    has = None if has_information is None else _i32(has_information)
    lib = _lib.load()
    opt = CreateOptionsC()
    lib.bae_create_options_default(ctypes.byref(opt))
    opt.device = device
    h = ctypes.c_void_p()
    _check(lib.bae_create_pgo(ptr(p7), p7.shape[0], ptr(ei, ctypes.c_int32), ptr(ej, ctypes.c_int32), ptr(meas),
                              ptr(info), ptr(has, ctypes.c_int32), ei.size, 1 if anchor_first else 0,
                              ctypes.byref(opt), ctypes.byref(h)))
    return PoseGraphProblem(h, p7.shape[0], 0, ei.size)


class RankGroup:
    """In-process rank group: ``world`` ranks in one process, one host thread
    per rank (bae_group_create). Its problems keep the native group alive
    after this handle is dropped."""

    def __init__(self, world: int):
        self._h = ctypes.c_void_p()
        _check(_lib.load().bae_group_create(int(world), ctypes.byref(self._h)))
        self.world = int(world)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.load().bae_group_destroy(h)
            self._h = None


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it and broadcasts it)."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.load().bae_nccl_unique_id(buf))
    return buf.raw


def make_ba_problem(poses, points, intrinsics, observations, *, device: int = 0, tile_obs: int = 0,
                    rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                    group: Optional[RankGroup] = None) -> TracedProblem:
    """make_ba_problem (problems.hpp:87-136) for BAL cameras.

    ``observations`` is ``(cam_idx, pt_idx, pixels)``; ``intrinsics`` is C x 3
    (BAL: f, k1, k2) or C x 4 (pinhole: fx, fy, cx, cy). Raises ValueError for a
    wrong intrinsics count or no observations, IndexError(position) for an
    out-of-range index, CheiralityError(observation) when an initial point
    lies on a camera plane (the reference's eager forward at construction).

    Landmark-sharded: with ``world > 1`` and an ``nccl_id``
    (one process per GPU) or a ``group`` (one thread per rank), every rank
    passes the whole problem and keeps its point partition; all later calls
    on the handle are collective."""
    cam_idx, pt_idx, pixels = observations
    p7 = _f64(poses).reshape(-1, 7)
    p3 = _f64(points).reshape(-1, 3)
    kk = _f64(intrinsics)
    # the CameraIntrinsics variant (camera.hpp:17-27): rows of 3 = BalIntrinsics
    # [f, k1, k2], rows of 4 = PinholeIntrinsics [fx, fy, cx, cy]
    pinhole = kk.ndim == 2 and kk.shape[1] == 4
    k3 = kk.reshape(-1, 4 if pinhole else 3)
    ci, pi = _i32(cam_idx), _i32(pt_idx)
    px = _f64(pixels).reshape(-1, 2)
    C, P, N = p7.shape[0], p3.shape[0], ci.shape[0]
    if k3.shape[0] != C:
        raise ValueError("make_ba_problem: one intrinsics entry per camera required")
    if N == 0:
        raise ValueError("make_ba_problem: no observations")
    lib = _lib.load()
    opt = CreateOptionsC()
    lib.bae_create_options_default(ctypes.byref(opt))
    opt.device = device
    opt.tile_obs = tile_obs
    opt.camera_model = 1 if pinhole else 0
    opt.rank = rank
    opt.world = world
    idbuf = None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        opt.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
    if group is not None:
        opt.group = group._h
    h = ctypes.c_void_p()
    _check(lib.bae_create_ba(ptr(p7), C, ptr(p3), P, ptr(k3), ptr(ci, ctypes.c_int32), ptr(pi, ctypes.c_int32),
                             ptr(px), N, ctypes.byref(opt), ctypes.byref(h)))
    tp = TracedProblem(h, C, P, N)
    tp._group = group  # the group also outlives its handle on the C side (reference counted)
    return tp


def optimize(model: TracedProblem, init_poses, init_points, config: LmConfig,
             final_state: Optional[dict] = None) -> LmReport:
    """optimize (lm.hpp:205-255); the model keeps the optimised parameters."""
    lib = _lib.load()
    cfg = config.to_c()
    cap = int(config.max_iterations) + 1
    recs = (IterRecordC * cap)()
    rep = LmReportC()
    # init_poses / init_points = None: start from the parameters already on the device
    p7 = None if init_poses is None else _f64(init_poses, (model.num_poses(), 7))
    p3 = None if init_points is None else _f64(init_points, (model.num_points(), 3))
    out7 = np.empty((model.num_poses(), 7))
    out3 = np.empty((model.num_points(), 3))
    _check(lib.bae_optimize(model._h, ptr(p7), ptr(p3), ctypes.byref(cfg), recs, cap, ctypes.byref(rep), ptr(out7),
                            ptr(out3)))
    n = min(cap, rep.iterations + 1)
    traj = [LmIterationRecord(r.iteration, r.cost, r.mse, r.lmbda, bool(r.accepted), r.cum_time_s, r.pcg_iters,
                              r.grad_norm, r.trial_cost) for r in recs[:n]]
    report = LmReport(rep.final_cost, rep.final_mse, rep.iterations, traj, TerminationReason(rep.reason),
                      rep.accepted_steps, rep.rejected_steps, rep.final_lambda, rep.solve_seconds,
                      rep.total_pcg_iters, rep.device_seconds)
    if final_state is not None:
        final_state.update(dict(poses=out7, points=out3, lmbda=rep.final_lambda, iterations=rep.iterations,
                                accepted_steps=rep.accepted_steps, rejected_steps=rep.rejected_steps))
    return report


def stop_on_plateau(history, config: LmConfig) -> bool:
    h = _f64(history)
    cfg = config.to_c()
    stop = ctypes.c_int32()
    _check(_lib.load().bae_stop_on_plateau(ptr(h), h.size, ctypes.byref(cfg), ctypes.byref(stop)))
    return bool(stop.value)


def partition_points(num_cameras: int, num_points: int, observations, world: int) -> np.ndarray:
    """Landmark partition used by the multi-GPU path (host only)."""
    cam_idx, pt_idx, _ = observations
    ci, pi = _i32(cam_idx), _i32(pt_idx)
    out = np.empty(num_points, np.int32)
    _check(_lib.load().bae_partition_points(num_cameras, num_points, ptr(ci, ctypes.c_int32), ptr(pi, ctypes.c_int32),
                                            ci.size, world, ptr(out, ctypes.c_int32)))
    return out


def write_csv(path: str, report: LmReport):
    """CSV trajectory with the reference CLI's schema (cli.hpp:69-79), written by the library."""
    recs = (IterRecordC * len(report.trajectory))()
    for i, r in enumerate(report.trajectory):
        recs[i].iteration, recs[i].cost, recs[i].mse = r.iteration, r.cost, r.mse
        recs[i].lmbda, recs[i].accepted, recs[i].cum_time_s = r.lmbda, 1 if r.accepted else 0, r.cum_time_s
    _check(_lib.load().bae_write_csv(path.encode(), recs, len(recs)))


@dataclasses.dataclass
class BalProblem:
    """BalProblem (io/bal.hpp:29-47): cameras as the 9 BAL scalars
    [rodrigues3, translation3, f, k1, k2]; poses / intrinsics through
    BalCamera::pose / intrinsics (io/bal.hpp:24-27)."""
    cameras: np.ndarray
    points: np.ndarray
    cam_idx: np.ndarray
    pt_idx: np.ndarray
    pixels: np.ndarray
    poses: np.ndarray
    intrinsics: np.ndarray

    @property
    def observations(self):
        return self.cam_idx, self.pt_idx, self.pixels


def _bal_from_handle(h) -> BalProblem:
    lib = _lib.load()
    C, P, N = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
    try:
        _check(lib.bae_bal_counts(h, ctypes.byref(C), ctypes.byref(P), ctypes.byref(N)))
        C, P, N = C.value, P.value, N.value
        cams, pts, px = np.empty((C, 9)), np.empty((P, 3)), np.empty((N, 2))
        poses, intr = np.empty((C, 7)), np.empty((C, 3))
        ci, pi = np.empty(N, np.int32), np.empty(N, np.int32)
        _check(lib.bae_bal_arrays(h, ptr(poses), ptr(intr), ptr(pts), ptr(ci, ctypes.c_int32),
                                  ptr(pi, ctypes.c_int32), ptr(px), ptr(cams)))
    finally:
        lib.bae_bal_free(h)
    return BalProblem(cams, pts, ci, pi, px, poses, intr)


def read_bal(path: str) -> BalProblem:
    """parse_bal (io/bal.hpp:103-142) of a file; ParseError carries the line (ParseError.line)."""
    h = ctypes.c_void_p()
    _check(_lib.load().bae_bal_read(str(path).encode(), ctypes.byref(h)))
    return _bal_from_handle(h)


def parse_bal(text) -> BalProblem:
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = ctypes.c_void_p()
    _check(_lib.load().bae_bal_parse(data, len(data), ctypes.byref(h)))
    return _bal_from_handle(h)


@dataclasses.dataclass
class PoseGraph:
    """PoseGraph (io/g2o.hpp:16-23): vertices as pose7 [t, q(x,y,z,w)] in file
    order with their g2o ids; edges remapped to vertex positions; identity
    information elided (has_information 0); skipped-tag warnings."""
    vertex_ids: np.ndarray
    vertices: np.ndarray
    edge_i: np.ndarray
    edge_j: np.ndarray
    measurements: np.ndarray
    information: np.ndarray
    has_information: np.ndarray
    warnings: list


def _g2o_from_handle(h) -> PoseGraph:
    lib = _lib.load()
    n, m, w = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32()
    try:
        _check(lib.bae_g2o_counts(h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(w)))
        n, m = n.value, m.value
        ids, poses = np.empty(n, np.int64), np.empty((n, 7))
        ei, ej, has = np.empty(m, np.int32), np.empty(m, np.int32), np.empty(m, np.int32)
        meas, info = np.empty((m, 7)), np.empty((m, 6, 6))
        _check(lib.bae_g2o_arrays(h, ptr(poses), ptr(ids, ctypes.c_int64), ptr(ei, ctypes.c_int32),
                                  ptr(ej, ctypes.c_int32), ptr(meas), ptr(info), ptr(has, ctypes.c_int32)))
        warnings = [lib.bae_g2o_warning(h, k).decode() for k in range(w.value)]
    finally:
        lib.bae_g2o_free(h)
    return PoseGraph(ids, poses, ei, ej, meas, info, has, warnings)


def read_g2o(path: str) -> PoseGraph:
    """parse_g2o (io/g2o.hpp:30-80) of a file; ParseError carries the line."""
    h = ctypes.c_void_p()
    _check(_lib.load().bae_g2o_read(str(path).encode(), ctypes.byref(h)))
    return _g2o_from_handle(h)


def parse_g2o(text) -> PoseGraph:
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = ctypes.c_void_p()
    _check(_lib.load().bae_g2o_parse(data, len(data), ctypes.byref(h)))
    return _g2o_from_handle(h)


def synth_ba(num_cameras: int, num_points: int, pixel_noise: float, pose_noise: float, seed: int) -> BalProblem:
    """synth_ba (io/synthetic.hpp:46-91): every camera sees every point."""
    h = ctypes.c_void_p()
    _check(_lib.load().bae_bal_synthetic(num_cameras, num_points, pixel_noise, pose_noise, seed, ctypes.byref(h)))
    return _bal_from_handle(h)


def write_bal(path: str, problem: BalProblem, binary: bool = False):
    """serialize_bal (io/bal.hpp:145-157), %.17g; ``binary=True`` writes the
    binary problem cache instead (read back by read_bal and the CLI)."""
    lib = _lib.load()
    cams, pts = _f64(problem.cameras).reshape(-1, 9), _f64(problem.points).reshape(-1, 3)
    ci, pi, px = _i32(problem.cam_idx), _i32(problem.pt_idx), _f64(problem.pixels).reshape(-1, 2)
    h = ctypes.c_void_p()
    _check(lib.bae_bal_from_arrays(cams.shape[0], pts.shape[0], ci.size, ptr(cams), ptr(pts), ptr(ci, ctypes.c_int32),
                                   ptr(pi, ctypes.c_int32), ptr(px), ctypes.byref(h)))
    try:
        _check((lib.bae_bal_write_binary if binary else lib.bae_bal_write)(h, str(path).encode()))
    finally:
        lib.bae_bal_free(h)


def cli_main(argv) -> int:
    """cli_main (cli.hpp:116-200) in-process; argv without the program name."""
    args = [b"traceopt_bench"] + [str(a).encode() for a in argv]
    arr = (ctypes.c_char_p * len(args))(*args)
    return int(_lib.load().bae_cli_main(len(args), arr))
