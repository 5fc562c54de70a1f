"""Synthetic BAL-shaped scenes for the BASELINE.json configs."""
from __future__ import annotations

import ctypes
import dataclasses

import numpy as np

from . import _lib
from ._lib import ptr

# name -> (cameras, points, observations); seed = camera count
CONFIGS = {
    "ladybug-49": (49, 7776, 31843),
    "trafalgar-257": (257, 65132, 225911),
    "dubrovnik-356": (356, 226730, 1255268),
    "venice-1778": (1778, 993923, 5001946),
    "final-13682": (13682, 4456117, 28987644),
}


@dataclasses.dataclass
class Scene:
    poses: np.ndarray        # (C, 7) initial
    points: np.ndarray       # (P, 3) initial
    intrinsics: np.ndarray   # (C, 3)
    cam_idx: np.ndarray      # (N,)
    pt_idx: np.ndarray       # (N,)
    pixels: np.ndarray       # (N, 2)
    true_poses: np.ndarray
    true_points: np.ndarray

    @property
    def observations(self):
        return (self.cam_idx, self.pt_idx, self.pixels)


def bal_shaped(C: int, P: int, N: int, seed: int | None = None, pixel_sigma: float = 1.0,
               pose_sigma: float = 0.05, point_sigma: float = 0.01) -> Scene:
    lib = _lib.load()
    seed = C if seed is None else seed
    poses = np.empty((C, 7))
    points = np.empty((P, 3))
    intr = np.empty((C, 3))
    ci = np.empty(N, np.int32)
    pi = np.empty(N, np.int32)
    px = np.empty((N, 2))
    tp = np.empty((C, 7))
    tl = np.empty((P, 3))
    code = lib.bae_synth_bal_shaped(C, P, N, seed, pixel_sigma, pose_sigma, point_sigma, ptr(poses), ptr(points),
                                    ptr(intr), ptr(ci, ctypes.c_int32), ptr(pi, ctypes.c_int32), ptr(px), ptr(tp),
                                    ptr(tl))
    if code != 0:
        raise ValueError((lib.bae_last_error() or b"").decode())
    return Scene(poses, points, intr, ci, pi, px, tp, tl)


def bal_shaped_device(C: int, P: int, N: int, seed: int | None = None, pixel_sigma: float = 1.0,
                      pose_sigma: float = 0.05, point_sigma: float = 0.01, device: int = 0) -> Scene:
    """The same scene family generated on the GPU from Philox streams (row f4,
    csrc/synth_device.cu): seconds less setup at Final-13682 size; not the
    host generator's values."""
    lib = _lib.load()
    seed = C if seed is None else seed
    out = [np.empty((C, 7)), np.empty((P, 3)), np.empty((C, 3)), np.empty(N, np.int32), np.empty(N, np.int32),
           np.empty((N, 2)), np.empty((C, 7)), np.empty((P, 3))]
    code = lib.bae_synth_bal_shaped_device(C, P, N, seed, pixel_sigma, pose_sigma, point_sigma, device, ptr(out[0]),
                                           ptr(out[1]), ptr(out[2]), ptr(out[3], ctypes.c_int32),
                                           ptr(out[4], ctypes.c_int32), ptr(out[5]), ptr(out[6]), ptr(out[7]))
    if code != 0:
        raise ValueError((lib.bae_last_error() or b"").decode())
    return Scene(*out)


def config_scene(name: str, **kw) -> Scene:
    C, P, N = CONFIGS[name]
    return bal_shaped(C, P, N, **kw)
