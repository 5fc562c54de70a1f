"""ctypes binding of the C ABI in include/bae_b200.h (libbae_b200.so, built in-tree).

There is no fallback: if the shared library is missing or a GPU is absent the
calls fail loudly (the B200 path has no CPU implementation)."""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbae_b200.so")

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_int64_p = ctypes.POINTER(ctypes.c_int64)


class LmConfigC(ctypes.Structure):
    _fields_ = [
        ("initial_damping", ctypes.c_double),
        ("damping_min", ctypes.c_double),
        ("damping_max", ctypes.c_double),
        ("damping_up", ctypes.c_double),
        ("damping_down", ctypes.c_double),
        ("clamp_min", ctypes.c_double),
        ("clamp_max", ctypes.c_double),
        ("plateau_rel_tol", ctypes.c_double),
        ("pcg_tol", ctypes.c_double),
        ("pcg_max_iters", ctypes.c_int64),
        ("max_iterations", ctypes.c_int32),
        ("plateau_patience", ctypes.c_int32),
        ("solver", ctypes.c_int32),
        ("use_caches", ctypes.c_int32),
    ]


class IterRecordC(ctypes.Structure):
    _fields_ = [
        ("iteration", ctypes.c_int32),
        ("accepted", ctypes.c_int32),
        ("cost", ctypes.c_double),
        ("mse", ctypes.c_double),
        ("lmbda", ctypes.c_double),
        ("cum_time_s", ctypes.c_double),
        ("pcg_iters", ctypes.c_int64),
        ("grad_norm", ctypes.c_double),
        ("trial_cost", ctypes.c_double),
    ]


class LmReportC(ctypes.Structure):
    _fields_ = [
        ("final_cost", ctypes.c_double),
        ("final_mse", ctypes.c_double),
        ("iterations", ctypes.c_int32),
        ("reason", ctypes.c_int32),
        ("accepted_steps", ctypes.c_int32),
        ("rejected_steps", ctypes.c_int32),
        ("final_lambda", ctypes.c_double),
        ("solve_seconds", ctypes.c_double),
        ("total_pcg_iters", ctypes.c_int64),
        ("device_seconds", ctypes.c_double),
    ]


class CreateOptionsC(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int32),
        ("tile_obs", ctypes.c_int32),
        ("jacobian", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("camera_model", ctypes.c_int32),
        ("nccl_id", ctypes.c_void_p),
        ("group", ctypes.c_void_p),
    ]


# name -> (restype, argtypes); must cover every function declared in the header
SIGNATURES = {
    "bae_version": (ctypes.c_char_p, []),
    "bae_lm_config_default": (None, [ctypes.POINTER(LmConfigC)]),
    "bae_create_options_default": (None, [ctypes.POINTER(CreateOptionsC)]),
    "bae_last_error": (ctypes.c_char_p, []),
    "bae_last_error_index": (ctypes.c_int64, []),
    "bae_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "bae_group_create": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]),
    "bae_group_destroy": (None, [ctypes.c_void_p]),
    "bae_create_ba": (ctypes.c_int, [c_double_p, ctypes.c_int32, c_double_p, ctypes.c_int32, c_double_p,
                                     c_int32_p, c_int32_p, c_double_p, ctypes.c_int64,
                                     ctypes.POINTER(CreateOptionsC), ctypes.POINTER(ctypes.c_void_p)]),
    "bae_destroy": (None, [ctypes.c_void_p]),
    "bae_num_poses": (ctypes.c_int32, [ctypes.c_void_p]),
    "bae_num_points": (ctypes.c_int32, [ctypes.c_void_p]),
    "bae_residual_rows": (ctypes.c_int64, [ctypes.c_void_p]),
    "bae_set_parameters": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_double_p]),
    "bae_get_parameters": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_double_p]),
    "bae_evaluate": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_double_p]),
    "bae_jacobian": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_double_p, c_int64_p, c_int32_p,
                                    c_int64_p, c_int32_p]),
    "bae_transpose_plan": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, c_int64_p, c_int32_p, c_int64_p]),
    "bae_normal_pattern": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, c_int64_p, c_int64_p, c_int64_p,
                                          c_int32_p]),
    "bae_block_diagonals": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_double_p, c_double_p, c_double_p]),
    "bae_optimize": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_double_p, ctypes.POINTER(LmConfigC),
                                    ctypes.POINTER(IterRecordC), ctypes.c_int32, ctypes.POINTER(LmReportC),
                                    c_double_p, c_double_p]),
    "bae_solve_step": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.POINTER(LmConfigC), c_double_p,
                                      c_int64_p, c_double_p]),
    "bae_stop_on_plateau": (ctypes.c_int, [c_double_p, ctypes.c_int64, ctypes.POINTER(LmConfigC), c_int32_p]),
    "bae_synth_bal_shaped": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                            ctypes.c_double, ctypes.c_double, ctypes.c_double, c_double_p,
                                            c_double_p, c_double_p, c_int32_p, c_int32_p, c_double_p,
                                            c_double_p, c_double_p]),
    "bae_synth_bal_shaped_device": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                            ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int32, c_double_p,
                                            c_double_p, c_double_p, c_int32_p, c_int32_p, c_double_p,
                                            c_double_p, c_double_p]),
    "bae_partition_points": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, c_int32_p, c_int32_p, ctypes.c_int64,
                                            ctypes.c_int32, c_int32_p]),
    "bae_time_kernel": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, c_double_p]),
    "bae_launch_count": (ctypes.c_int64, [ctypes.c_void_p]),
    "bae_phase_times": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_int32]),
    "bae_direct_pairs": (ctypes.c_int, [ctypes.c_void_p, c_int64_p, c_int64_p]),
    "bae_problem_stats": (ctypes.c_int, [ctypes.c_void_p, c_int64_p]),
    "bae_problem_shard": (ctypes.c_int, [ctypes.c_void_p, c_int32_p, c_int32_p, c_int32_p, c_int64_p]),
    "bae_direct_stats": (ctypes.c_int, [ctypes.c_void_p, c_int64_p]),
    "bae_plan_array": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64,
                                      c_int64_p, ctypes.POINTER(ctypes.c_int32)]),
    "bae_create_pgo": (ctypes.c_int, [c_double_p, ctypes.c_int32, c_int32_p, c_int32_p, c_double_p, c_double_p,
                                      c_int32_p, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(CreateOptionsC),
                                      ctypes.POINTER(ctypes.c_void_p)]),
    "bae_pgo_jacobian": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_double_p]),
    "bae_nd_order": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, c_int32_p, ctypes.c_int32, c_int32_p, c_int32_p,
                                     c_int32_p]),
    "bae_tile_symbolic": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, c_int32_p, c_int32_p, c_int32_p,
                                          ctypes.c_int64, c_int64_p]),
    "bae_chol_tasks": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, c_int32_p, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int64, c_int32_p, c_int32_p, c_int32_p, c_int32_p, c_int32_p,
                                       c_int32_p, ctypes.POINTER(ctypes.c_uint32)]),
    "bae_bal_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "bae_bal_parse": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]),
    "bae_bal_synthetic": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]),
    "bae_bal_from_arrays": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, c_double_p, c_double_p,
                                           c_int32_p, c_int32_p, c_double_p, ctypes.POINTER(ctypes.c_void_p)]),
    "bae_bal_counts": (ctypes.c_int, [ctypes.c_void_p, c_int32_p, c_int32_p, c_int64_p]),
    "bae_bal_arrays": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_double_p, c_double_p, c_int32_p, c_int32_p,
                                      c_double_p, c_double_p]),
    "bae_bal_write": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p]),
    "bae_bal_write_binary": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p]),
    "bae_bal_free": (None, [ctypes.c_void_p]),
    "bae_g2o_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "bae_g2o_parse": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]),
    "bae_g2o_counts": (ctypes.c_int, [ctypes.c_void_p, c_int32_p, c_int64_p, c_int32_p]),
    "bae_g2o_arrays": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_int64_p, c_int32_p, c_int32_p, c_double_p,
                                      c_double_p, c_int32_p]),
    "bae_g2o_warning": (ctypes.c_char_p, [ctypes.c_void_p, ctypes.c_int32]),
    "bae_g2o_free": (None, [ctypes.c_void_p]),
    "bae_write_csv": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(IterRecordC), ctypes.c_int32]),
    "bae_cli_main": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_char_p)]),
}

_lib = None


def load():
    """Load libbae_b200.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing; build it with __graft_entry__.build() "
                               "(the B200 path has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def ptr(a, ctype=ctypes.c_double):
    """Pointer to a contiguous numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctype))
