"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the CPU restatement of the
reference hot path (oracle/bae_oracle.cpp -> oracle/liboracle_bae.so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU arms may import this,
and only as the checker / CPU baseline. See bae_oracle.cpp's header for what
pins it (reference unit-test KATs + the reference RNG golden stream)."""
from __future__ import annotations

import ctypes
import dataclasses
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle_bae.so")


# The plain C structs of include/bae_b200.h (bae_lm_config, bae_iter_record,
# bae_lm_report), declared here so the oracle never imports the product
# package: bench.py's reference arm loads liboracle_bae.so only.
class LmConfigC(ctypes.Structure):
    _fields_ = [("initial_damping", ctypes.c_double), ("damping_min", ctypes.c_double),
                ("damping_max", ctypes.c_double), ("damping_up", ctypes.c_double), ("damping_down", ctypes.c_double),
                ("clamp_min", ctypes.c_double), ("clamp_max", ctypes.c_double), ("plateau_rel_tol", ctypes.c_double),
                ("pcg_tol", ctypes.c_double), ("pcg_max_iters", ctypes.c_int64), ("max_iterations", ctypes.c_int32),
                ("plateau_patience", ctypes.c_int32), ("solver", ctypes.c_int32), ("use_caches", ctypes.c_int32)]


class IterRecordC(ctypes.Structure):
    _fields_ = [("iteration", ctypes.c_int32), ("accepted", ctypes.c_int32), ("cost", ctypes.c_double),
                ("mse", ctypes.c_double), ("lmbda", ctypes.c_double), ("cum_time_s", ctypes.c_double),
                ("pcg_iters", ctypes.c_int64), ("grad_norm", ctypes.c_double), ("trial_cost", ctypes.c_double)]


class LmReportC(ctypes.Structure):
    _fields_ = [("final_cost", ctypes.c_double), ("final_mse", ctypes.c_double), ("iterations", ctypes.c_int32),
                ("reason", ctypes.c_int32), ("accepted_steps", ctypes.c_int32), ("rejected_steps", ctypes.c_int32),
                ("final_lambda", ctypes.c_double), ("solve_seconds", ctypes.c_double),
                ("total_pcg_iters", ctypes.c_int64), ("device_seconds", ctypes.c_double)]


@dataclasses.dataclass
class LmConfig:
    """LmConfig (lm.hpp:23-46) defaults; solver 0 = cholesky, 1 = pcg."""
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
    solver: int = 0
    pcg_tol: float = 1e-8
    pcg_max_iters: int = 0
    use_caches: bool = True


def _cfg(config) -> LmConfigC:
    """Any LmConfig-shaped object (this module's or the product binding's)."""
    c = LmConfigC()
    for f in ("initial_damping", "damping_min", "damping_max", "damping_up", "damping_down", "clamp_min",
              "clamp_max", "plateau_rel_tol", "pcg_tol"):
        setattr(c, f, float(getattr(config, f)))
    c.pcg_max_iters = int(config.pcg_max_iters)
    c.max_iterations = int(config.max_iterations)
    c.plateau_patience = int(config.plateau_patience)
    c.solver = int(config.solver)
    c.use_caches = 1 if config.use_caches else 0
    return c

D = ctypes.POINTER(ctypes.c_double)
I32 = ctypes.POINTER(ctypes.c_int32)
I64 = ctypes.POINTER(ctypes.c_int64)
VP = ctypes.c_void_p

_SIG = {
    "or_last_error": (ctypes.c_char_p, []),
    "or_last_error_index": (ctypes.c_int64, []),
    "or_set_threads": (None, [ctypes.c_int]),
    "or_symbolic_count": (ctypes.c_int64, []),
    "or_rng_new": (VP, [ctypes.c_uint64]),
    "or_rng_free": (None, [VP]),
    "or_rng_uniform": (ctypes.c_double, [VP]),
    "or_rng_uniform_range": (ctypes.c_double, [VP, ctypes.c_double, ctypes.c_double]),
    "or_rng_normal": (ctypes.c_double, [VP]),
    "or_rng_index": (ctypes.c_uint64, [VP, ctypes.c_uint64]),
    "or_se3_exp": (ctypes.c_int, [D, D]),
    "or_se3_log": (ctypes.c_int, [D, D]),
    "or_se3_compose": (ctypes.c_int, [D, D, D]),
    "or_se3_retract": (ctypes.c_int, [D, D, D]),
    "or_quat_make": (ctypes.c_int, [D, D]),
    "or_quat_matrix": (None, [D, D]),
    "or_bal_project": (ctypes.c_int, [D, D, D, D]),
    "or_pinhole_project": (ctypes.c_int, [D, D, D, D]),
    "or_bal_project_cam": (ctypes.c_int, [D, D, D]),
    "or_pinhole_project_cam": (ctypes.c_int, [D, D, D]),
    "or_bal_camera_pose": (ctypes.c_int, [D, D, D]),
    "or_make_random_ba": (ctypes.c_int, [VP, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, D, D, D, I32,
                                         I32, D, I64]),
    "or_synth_ba": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, D,
                                   D, D, I32, I32, D, D]),
    "or_synth_bal_shaped_philox": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64,
                                                  ctypes.c_double, ctypes.c_double, ctypes.c_double, D, D, D, I32, I32,
                                                  D, D, D]),
    "or_synth_bal_shaped": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, D, D, D, I32, I32, D, D, D]),
    "or_philox4x32_10": (ctypes.c_uint32, [ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32),
                                           ctypes.POINTER(ctypes.c_uint32)]),
    "or_ba_problem_new": (VP, [ctypes.c_int, ctypes.c_int, D, ctypes.c_int, D, D, ctypes.c_int64, I32, I32, D,
                               ctypes.POINTER(ctypes.c_int)]),
    "or_scalar_problem_new": (VP, [ctypes.c_int, D]),
    "or_pgo_problem_new": (VP, [D, ctypes.c_int, I32, I32, D, D, I32, ctypes.c_int64, ctypes.c_int]),
    "or_make_random_pgo": (ctypes.c_int, [VP, ctypes.c_int, ctypes.c_int, ctypes.c_double, D, I32, I32, D, D, I32,
                                          I64]),
    "or_problem_jacobian_dense": (ctypes.c_int, [VP, D, ctypes.c_int64, ctypes.c_int64]),
    "or_problem_free": (None, [VP]),
    "or_problem_evaluate": (ctypes.c_int, [VP, D, D, D, D]),
    "or_problem_jacobian": (ctypes.c_int, [VP, D, D, I64, I32, I64, I32]),
    "or_transpose_plan": (ctypes.c_int, [VP, ctypes.c_int, I64, I32, I64]),
    "or_normal_size": (ctypes.c_int, [VP, I64, I64]),
    "or_normal_pattern": (ctypes.c_int, [VP, ctypes.c_int, I64, I64, I64, I32]),
    "or_normal_dense": (ctypes.c_int, [VP, ctypes.c_double, ctypes.c_double, ctypes.c_double, D, D]),
    "or_solve_step": (ctypes.c_int, [VP, ctypes.c_double, ctypes.POINTER(LmConfigC), D, I64]),
    "or_lm_begin": (ctypes.c_int, [VP, D, D, ctypes.c_double]),
    "or_lm_step": (ctypes.c_int, [VP, ctypes.POINTER(LmConfigC), ctypes.POINTER(ctypes.c_int)]),
    "or_lm_state": (ctypes.c_int, [VP, D, D, D, ctypes.POINTER(ctypes.c_int), D, ctypes.c_int,
                                   ctypes.POINTER(ctypes.c_int)]),
    "or_optimize": (ctypes.c_int, [VP, D, D, ctypes.POINTER(LmConfigC), ctypes.POINTER(IterRecordC), ctypes.c_int,
                                   ctypes.POINTER(ctypes.c_int), ctypes.POINTER(LmReportC), D, D]),
    "or_stop_on_plateau": (ctypes.c_int, [D, ctypes.c_int64, ctypes.POINTER(LmConfigC), ctypes.POINTER(ctypes.c_int)]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C oracle`")
        L = ctypes.CDLL(LIB_PATH)
        for n, (r, a) in _SIG.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


class OracleError(Exception):
    def __init__(self, code, msg, index):
        super().__init__(f"[{code}] {msg} (index {index})")
        self.code, self.msg, self.index = code, msg, index


def _chk(code):
    if code != 0:
        L = lib()
        raise OracleError(code, (L.or_last_error() or b"").decode(), int(L.or_last_error_index()))


def p(a, t=ctypes.c_double):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(t))


def set_threads(n: int):
    lib().or_set_threads(int(n))


class Rng:
    def __init__(self, seed):
        self.h = lib().or_rng_new(int(seed))

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_rng_free(self.h)

    def uniform(self, lo=None, hi=None):
        if lo is None:
            return lib().or_rng_uniform(self.h)
        return lib().or_rng_uniform_range(self.h, lo, hi)

    def normal(self):
        return lib().or_rng_normal(self.h)

    def index(self, n):
        return int(lib().or_rng_index(self.h, int(n)))


def make_random_ba(rng: Rng, C: int, P: int, pinhole: bool, keep: float = 0.8):
    """tests/oracles.hpp:26-61."""
    kw = 4 if pinhole else 3
    poses = np.empty((C, 7))
    pts = np.empty((P, 3))
    intr = np.empty((C, kw))
    ci = np.empty(C * P, np.int32)
    pi = np.empty(C * P, np.int32)
    px = np.empty((C * P, 2))
    n = ctypes.c_int64()
    _chk(lib().or_make_random_ba(rng.h, C, P, 1 if pinhole else 0, keep, p(poses), p(pts), p(intr),
                                 p(ci, ctypes.c_int32), p(pi, ctypes.c_int32), p(px), ctypes.byref(n)))
    N = n.value
    return dict(poses=poses, points=pts, intrinsics=intr, cam_idx=ci[:N].copy(), pt_idx=pi[:N].copy(),
                pixels=px[:N].copy(), pinhole=pinhole)


def synth_ba(C, P, pix_sigma, pose_sigma, seed):
    """io/synthetic.hpp:46-91 (dense visibility), poses via BalCamera::pose."""
    N = C * P
    poses = np.empty((C, 7))
    intr = np.empty((C, 3))
    pts = np.empty((P, 3))
    ci = np.empty(N, np.int32)
    pi = np.empty(N, np.int32)
    px = np.empty((N, 2))
    tp = np.empty((C, 7))
    _chk(lib().or_synth_ba(C, P, pix_sigma, pose_sigma, seed, p(poses), p(intr), p(pts), p(ci, ctypes.c_int32),
                           p(pi, ctypes.c_int32), p(px), p(tp)))
    return dict(poses=poses, points=pts, intrinsics=intr, cam_idx=ci, pt_idx=pi, pixels=px, true_poses=tp,
                pinhole=False)


def synth_bal_shaped_philox(C, P, N, seed, pixel_sigma=1.0, pose_sigma=0.05, point_sigma=0.01):
    """The on-device generator's algorithm (row f4) restated on the host."""
    out = dict(poses=np.empty((C, 7)), points=np.empty((P, 3)), intrinsics=np.empty((C, 3)),
               cam_idx=np.empty(N, np.int32), pt_idx=np.empty(N, np.int32), pixels=np.empty((N, 2)),
               true_poses=np.empty((C, 7)), true_points=np.empty((P, 3)))
    _chk(lib().or_synth_bal_shaped_philox(C, P, N, seed, pixel_sigma, pose_sigma, point_sigma, p(out["poses"]),
                                          p(out["points"]), p(out["intrinsics"]), p(out["cam_idx"], ctypes.c_int32),
                                          p(out["pt_idx"], ctypes.c_int32), p(out["pixels"]), p(out["true_poses"]),
                                          p(out["true_points"])))
    return out


def synth_bal_shaped(C, P, N, seed=None, pixel_sigma=1.0, pose_sigma=0.05, point_sigma=0.01):
    """SURVEY.md 8d's host generator restated on the reference Rng (independent
    of the product's csrc/synth.cpp; the CPU baseline's inputs)."""
    seed = C if seed is None else seed
    out = dict(poses=np.empty((C, 7)), points=np.empty((P, 3)), intrinsics=np.empty((C, 3)),
               cam_idx=np.empty(N, np.int32), pt_idx=np.empty(N, np.int32), pixels=np.empty((N, 2)),
               true_poses=np.empty((C, 7)), true_points=np.empty((P, 3)))
    _chk(lib().or_synth_bal_shaped(C, P, N, seed, pixel_sigma, pose_sigma, point_sigma, p(out["poses"]),
                                   p(out["points"]), p(out["intrinsics"]), p(out["cam_idx"], ctypes.c_int32),
                                   p(out["pt_idx"], ctypes.c_int32), p(out["pixels"]), p(out["true_poses"]),
                                   p(out["true_points"])))
    return out


def philox4x32_10(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return list(o)


class Problem:
    """make_ba_problem restated (problems.hpp:87-136) + LM driver."""

    def __init__(self, poses, points, intrinsics, cam_idx, pt_idx, pixels, pinhole=False):
        self.poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 7)
        self.points = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        self.kw = 4 if pinhole else 3
        intr = np.ascontiguousarray(intrinsics, dtype=np.float64).reshape(-1, self.kw)
        ci = np.ascontiguousarray(cam_idx, dtype=np.int32)
        pi = np.ascontiguousarray(pt_idx, dtype=np.int32)
        px = np.ascontiguousarray(pixels, dtype=np.float64).reshape(-1, 2)
        self.C, self.P, self.N = self.poses.shape[0], self.points.shape[0], ci.shape[0]
        err = ctypes.c_int()
        self.h = lib().or_ba_problem_new(1 if pinhole else 0, self.C, p(self.poses), self.P, p(self.points), p(intr),
                                         self.N, p(ci, ctypes.c_int32), p(pi, ctypes.c_int32), p(px),
                                         ctypes.byref(err))
        _chk(err.value)

    @classmethod
    def from_dict(cls, d):
        return cls(d["poses"], d["points"], d["intrinsics"], d["cam_idx"], d["pt_idx"], d["pixels"],
                   d.get("pinhole", False))

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_problem_free(self.h)

    def evaluate(self, poses=None, points=None):
        r = np.empty(2 * self.N)
        c = ctypes.c_double()
        p7 = None if poses is None else np.ascontiguousarray(poses, dtype=np.float64)
        p3 = None if points is None else np.ascontiguousarray(points, dtype=np.float64)
        _chk(lib().or_problem_evaluate(self.h, p(p7), p(p3), p(r), ctypes.byref(c)))
        return r, c.value

    def jacobian(self):
        N = self.N
        jp = np.empty((N, 2, 6))
        jl = np.empty((N, 2, 3))
        prp = np.empty(N + 1, np.int64)
        lrp = np.empty(N + 1, np.int64)
        pc = np.empty(N, np.int32)
        lc = np.empty(N, np.int32)
        _chk(lib().or_problem_jacobian(self.h, p(jp), p(jl), p(prp, ctypes.c_int64), p(pc, ctypes.c_int32),
                                       p(lrp, ctypes.c_int64), p(lc, ctypes.c_int32)))
        return dict(j_pose=jp, j_point=jl, pose_row_ptr=prp, pose_col=pc, point_row_ptr=lrp, point_col=lc)

    def transpose_plan(self, which):
        cols = self.C if which == 0 else self.P
        rp = np.empty(cols + 1, np.int64)
        ci = np.empty(self.N, np.int32)
        sb = np.empty(self.N, np.int64)
        _chk(lib().or_transpose_plan(self.h, which, p(rp, ctypes.c_int64), p(ci, ctypes.c_int32),
                                     p(sb, ctypes.c_int64)))
        return rp, ci, sb

    def normal_pattern(self, which):
        """(row_ptr, col_idx) of quadrant `which` (0 CC, 1 CL, 2 LC, 3 LL,
        spgemm_symbolic) or of the scalar CSR matrix A (4)."""
        rows, nnz = ctypes.c_int64(), ctypes.c_int64()
        _chk(lib().or_normal_pattern(self.h, which, ctypes.byref(rows), ctypes.byref(nnz), None, None))
        rp = np.empty(rows.value + 1, np.int64)
        ci = np.empty(nnz.value, np.int32)
        _chk(lib().or_normal_pattern(self.h, which, ctypes.byref(rows), ctypes.byref(nnz), p(rp, ctypes.c_int64),
                                     p(ci, ctypes.c_int32)))
        return rp, ci

    def normal_dense(self, lmbda, cmin=1e-6, cmax=1e32):
        n = ctypes.c_int64()
        nnz = ctypes.c_int64()
        _chk(lib().or_normal_size(self.h, ctypes.byref(n), ctypes.byref(nnz)))
        A = np.empty((n.value, n.value))
        b = np.empty(n.value)
        _chk(lib().or_normal_dense(self.h, lmbda, cmin, cmax, p(A), p(b)))
        return A, b

    def solve_step(self, lmbda, config):
        n = 6 * self.C + 3 * self.P
        x = np.empty(n)
        it = ctypes.c_int64()
        cfg = _cfg(config)
        _chk(lib().or_solve_step(self.h, lmbda, ctypes.byref(cfg), p(x), ctypes.byref(it)))
        return x, it.value

    def optimize(self, config, poses=None, points=None):
        cfg = _cfg(config)
        cap = int(config.max_iterations) + 1
        recs = (IterRecordC * cap)()
        n = ctypes.c_int()
        rep = LmReportC()
        p7 = np.ascontiguousarray(self.poses if poses is None else poses, dtype=np.float64)
        p3 = np.ascontiguousarray(self.points if points is None else points, dtype=np.float64)
        o7 = np.empty_like(p7)
        o3 = np.empty_like(p3)
        _chk(lib().or_optimize(self.h, p(p7), p(p3), ctypes.byref(cfg), recs, cap, ctypes.byref(n),
                               ctypes.byref(rep), p(o7), p(o3)))
        traj = [dict(iteration=r.iteration, accepted=bool(r.accepted), cost=r.cost, mse=r.mse, lmbda=r.lmbda,
                     cum_time_s=r.cum_time_s, pcg_iters=r.pcg_iters, grad_norm=r.grad_norm, trial_cost=r.trial_cost)
                for r in recs[:min(cap, n.value)]]
        return dict(final_cost=rep.final_cost, final_mse=rep.final_mse, iterations=rep.iterations,
                    reason=rep.reason, trajectory=traj, poses=o7, points=o3, solve_seconds=rep.solve_seconds,
                    accepted_steps=rep.accepted_steps, rejected_steps=rep.rejected_steps)


def make_random_pgo(rng: Rng, n: int, with_information: bool, noise: float = 0.05):
    """tests/oracles.hpp:120-152: a chain of poses plus n/2 random extra edges."""
    cap = n - 1 + n // 2
    poses = np.empty((n, 7))
    ei, ej = np.empty(cap, np.int32), np.empty(cap, np.int32)
    meas, info = np.empty((cap, 7)), np.zeros((cap, 6, 6))
    has = np.zeros(cap, np.int32)
    m = ctypes.c_int64()
    _chk(lib().or_make_random_pgo(rng.h, n, 1 if with_information else 0, noise, p(poses), p(ei, ctypes.c_int32),
                                  p(ej, ctypes.c_int32), p(meas), p(info), p(has, ctypes.c_int32), ctypes.byref(m)))
    k = m.value
    return dict(poses=poses, edge_i=ei[:k].copy(), edge_j=ej[:k].copy(), measurements=meas[:k].copy(),
                information=info[:k].copy(), has_information=has[:k].copy())


class PgoProblem(Problem):
    """make_pgo_problem restated (problems.hpp:141-188) + the generic LM driver."""

    def __init__(self, poses, edge_i, edge_j, measurements, information=None, has_information=None,
                 anchor_first=True):
        self.poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 7)
        self.points = np.zeros((0, 3))
        ei = np.ascontiguousarray(edge_i, dtype=np.int32)
        ej = np.ascontiguousarray(edge_j, dtype=np.int32)
        meas = np.ascontiguousarray(measurements, dtype=np.float64).reshape(-1, 7)
        self.C, self.P, self.M = self.poses.shape[0], 0, ei.shape[0]
        self.anchor = bool(anchor_first)
        info = None if information is None else np.ascontiguousarray(information, dtype=np.float64).reshape(-1, 36)
        has = None if has_information is None else np.ascontiguousarray(has_information, dtype=np.int32)
        self.h = lib().or_pgo_problem_new(p(self.poses), self.C, p(ei, ctypes.c_int32), p(ej, ctypes.c_int32),
                                          p(meas), p(info), p(has, ctypes.c_int32), self.M, 1 if anchor_first else 0)
        if not self.h:
            _chk(7 if not lib().or_last_error() else 1)

    @classmethod
    def from_dict(cls, d, anchor_first=True):
        return cls(d["poses"], d["edge_i"], d["edge_j"], d["measurements"], d["information"], d["has_information"],
                   anchor_first)

    def evaluate(self, poses=None, points=None):
        r = np.empty(6 * self.M)
        c = ctypes.c_double()
        p7 = None if poses is None else np.ascontiguousarray(poses, dtype=np.float64)
        _chk(lib().or_problem_evaluate(self.h, p(p7), None, p(r), ctypes.byref(c)))
        return r, c.value

    def jacobian_dense(self):
        cols = 6 * (self.C - (1 if self.anchor else 0))
        out = np.empty((6 * self.M, cols))
        _chk(lib().or_problem_jacobian_dense(self.h, p(out), out.shape[0], cols))
        return out


class ScalarProblem:
    """Points-only LM KAT models (test_optim.cpp:15-32): kind 0 r = theta,
    1 r = theta^2 - 2, 2 r = theta^2 + 1."""

    def __init__(self, kind, theta):
        th = np.ascontiguousarray(theta, dtype=np.float64)
        self.h = lib().or_scalar_problem_new(kind, p(th))

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_problem_free(self.h)

    def begin(self, theta, lmbda):
        th = np.ascontiguousarray(theta, dtype=np.float64).reshape(1, 3)
        _chk(lib().or_lm_begin(self.h, None, p(th), lmbda))

    def step(self, config):
        cfg = _cfg(config)
        acc = ctypes.c_int()
        _chk(lib().or_lm_step(self.h, ctypes.byref(cfg), ctypes.byref(acc)))
        return bool(acc.value)

    def state(self):
        pts = np.empty((1, 3))
        lam = ctypes.c_double()
        cnt = (ctypes.c_int * 3)()
        hist = np.empty(4096)
        nh = ctypes.c_int()
        _chk(lib().or_lm_state(self.h, None, p(pts), ctypes.byref(lam), cnt, p(hist), 4096, ctypes.byref(nh)))
        return dict(points=pts, lmbda=lam.value, iterations=cnt[0], accepted=cnt[1], rejected=cnt[2],
                    history=hist[:nh.value].copy())

    def optimize(self, config, theta):
        cfg = _cfg(config)
        cap = int(config.max_iterations) + 1
        recs = (IterRecordC * cap)()
        n = ctypes.c_int()
        rep = LmReportC()
        th = np.ascontiguousarray(theta, dtype=np.float64).reshape(1, 3)
        o3 = np.empty((1, 3))
        _chk(lib().or_optimize(self.h, None, p(th), ctypes.byref(cfg), recs, cap, ctypes.byref(n), ctypes.byref(rep),
                               None, p(o3)))
        return dict(final_cost=rep.final_cost, iterations=rep.iterations, reason=rep.reason,
                    trajectory=[dict(cost=r.cost, accepted=bool(r.accepted)) for r in recs[:min(cap, n.value)]],
                    points=o3)


def stop_on_plateau(history, config):
    h = np.ascontiguousarray(history, dtype=np.float64)
    cfg = _cfg(config)
    s = ctypes.c_int()
    _chk(lib().or_stop_on_plateau(p(h), h.size, ctypes.byref(cfg), ctypes.byref(s)))
    return bool(s.value)


def se3_exp(tau):
    out = np.empty(7)
    _chk(lib().or_se3_exp(p(np.ascontiguousarray(tau, dtype=np.float64)), p(out)))
    return out


def se3_retract(pose, tau):
    out = np.empty(7)
    _chk(lib().or_se3_retract(p(np.ascontiguousarray(pose, dtype=np.float64)),
                              p(np.ascontiguousarray(tau, dtype=np.float64)), p(out)))
    return out


def se3_compose(a, b):
    out = np.empty(7)
    _chk(lib().or_se3_compose(p(np.ascontiguousarray(a, dtype=np.float64)), p(np.ascontiguousarray(b, dtype=np.float64)),
                              p(out)))
    return out


def quat_matrix(q):
    out = np.empty(9)
    lib().or_quat_matrix(p(np.ascontiguousarray(q, dtype=np.float64)), p(out))
    return out.reshape(3, 3)


def bal_project(pose, point, k3):
    out = np.empty(2)
    _chk(lib().or_bal_project(p(np.ascontiguousarray(pose, dtype=np.float64)),
                              p(np.ascontiguousarray(point, dtype=np.float64)),
                              p(np.ascontiguousarray(k3, dtype=np.float64)), p(out)))
    return out


def pinhole_project(pose, point, k4):
    out = np.empty(2)
    _chk(lib().or_pinhole_project(p(np.ascontiguousarray(pose, dtype=np.float64)),
                                  p(np.ascontiguousarray(point, dtype=np.float64)),
                                  p(np.ascontiguousarray(k4, dtype=np.float64)), p(out)))
    return out


def camera_window_slice(scene, cameras):
    """A bounded CPU sample of a BAL-shaped scene (bench.py's CPU baseline):
    cameras 0..cameras-1 of the ring and every point all of whose cameras lie
    among them, re-indexed. The generator's visibility is banded (windows of
    min(C, 16) ring neighbours), so the slice keeps the scene's
    per-camera density, per-point track lengths and band structure; the
    reference's per-iteration work is linear in the observations at fixed
    band width, which is what makes the sample's time scale to the full
    scene by N / N_slice."""
    ci = np.asarray(scene["cam_idx"])
    pi = np.asarray(scene["pt_idx"])
    P = len(scene["points"])
    outside = np.bincount(pi, weights=(ci >= cameras).astype(np.float64), minlength=P) > 0
    seen = np.bincount(pi, minlength=P) > 0
    keep_pt = seen & ~outside
    new_id = np.cumsum(keep_pt) - 1
    keep = keep_pt[pi]
    out = dict(poses=np.ascontiguousarray(scene["poses"][:cameras]),
               intrinsics=np.ascontiguousarray(scene["intrinsics"][:cameras]),
               points=np.ascontiguousarray(scene["points"][keep_pt]),
               cam_idx=np.ascontiguousarray(ci[keep], dtype=np.int32),
               pt_idx=np.ascontiguousarray(new_id[pi[keep]], dtype=np.int32),
               pixels=np.ascontiguousarray(np.asarray(scene["pixels"])[keep]))
    return out
