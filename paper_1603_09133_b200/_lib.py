"""ctypes binding of libce_gpu.so (include/ce_gpu.h).

The library is built in-tree (``make -C paper_1603_09133_b200/csrc`` or
``__graft_entry__.build()``).  A missing library is a hard error: the product
path has no CPU fallback.
"""

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CE_LIB_OVERRIDE") or os.path.join(_HERE, "libce_gpu.so")  # override: development A/B builds


class LibraryMissing(ImportError):
    pass


i64 = C.c_int64
i64p = C.POINTER(C.c_int64)
dblp = C.POINTER(C.c_double)
vp = C.c_void_p


class CsbHost(C.Structure):
    _fields_ = [("n", i64), ("m", i64), ("offsets", i64p), ("row_ptr", i64p), ("col_idx", i64p),
                ("val_ptr", i64p), ("values", dblp)]


class PlanHost(C.Structure):
    _fields_ = [("join", i64), ("n_levels", i64), ("level_blocks", i64p), ("assign", i64p)]


class Strategy(C.Structure):
    _fields_ = [("mode", C.c_int), ("eps", C.c_double), ("absolute", C.c_int), ("rank", i64)]


class FactorOpts(C.Structure):
    _fields_ = [("dense_threshold", i64), ("max_levels", i64), ("n_forced_levels", i64),
                ("forced_counts", i64p), ("forced", i64p)]


class Status(C.Structure):
    _fields_ = [("code", C.c_int), ("level", C.c_int), ("block", i64), ("shift_retries", i64),
                ("message", C.c_char * 256)]


BcastFn = C.CFUNCTYPE(C.c_int, vp, vp, i64, C.c_int)  # ce_bcast_fn(user, dev_ptr, bytes, root)


class Shard(C.Structure):
    _fields_ = [("rank", C.c_int), ("n_ranks", C.c_int), ("n_boxes", i64), ("box_of_block", i64p),
                ("bcast", BcastFn), ("user", vp)]


class PcgOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("maxit", i64), ("track_true_residual", C.c_int)]


class Report(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", i64), ("final_recurrence_residual", C.c_double),
                ("final_true_residual", C.c_double), ("seconds", C.c_double)]


class FactorStats(C.Structure):
    _fields_ = [("n_levels", i64), ("tail_dim", i64), ("factor_blocks", C.c_double),
                ("predicted_factor_blocks", C.c_double), ("l_scalar_nnz", i64), ("l_payload_bytes", i64),
                ("q_payload_bytes", i64), ("tail_bytes", i64), ("shift_retries", i64),
                ("total_seconds", C.c_double), ("device_seconds", C.c_double),
                ("sweep_kernel_seconds", C.c_double), ("algorithmic_bytes", C.c_double),
                ("algorithmic_flops", C.c_double), ("validate_seconds", C.c_double), ("max_orth_error", C.c_double),
                ("apply_algorithmic_bytes", C.c_double), ("shard_phase1_rows", i64), ("shard_own_rows", i64),
                ("shard_phase3_rows", i64), ("shard_exchange_bytes", C.c_double),
                ("shard_exchange_seconds", C.c_double)]


class LevelStats(C.Structure):
    _fields_ = [("block_count", i64), ("pattern_blocks", i64), ("factor_blocks", i64), ("eliminated", i64),
                ("retained", i64), ("max_rank", i64), ("mean_rank", C.c_double), ("seconds", C.c_double),
                ("l_bytes", i64), ("q_bytes", i64), ("shift_retries", i64), ("max_block", i64),
                ("max_far_cols", i64), ("max_close", i64), ("sweep_seconds", C.c_double),
                ("algorithmic_bytes", C.c_double), ("algorithmic_flops", C.c_double), ("n_waves", i64),
                ("n_items", i64)]


# name -> (restype, argtypes); every symbol include/ce_gpu.h declares
SIGNATURES = {
    "ce_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "ce_ctx_destroy": (None, [vp]),
    "ce_last_error": (C.c_char_p, []),
    "ce_device_count": (C.c_int, []),
    "ce_ctx_stream": (C.c_int, [vp, C.POINTER(vp)]),
    "ce_launch_count": (i64, []),
    "ce_matrix_upload": (C.c_int, [vp, C.POINTER(CsbHost), C.POINTER(vp)]),
    "ce_matrix_free": (None, [vp]),
    "ce_matrix_dim": (i64, [vp]),
    "ce_matvec": (C.c_int, [vp, vp, vp, i64, C.c_int, vp]),
    "ce_matrix_from_triplets": (C.c_int, [vp, i64, i64, vp, vp, vp, i64, i64p, C.c_int, C.c_int, C.POINTER(vp)]),
    "ce_matrix_csb": (C.c_int, [vp, C.POINTER(CsbHost), C.POINTER(C.c_double)]),
    "ce_pattern_square": (C.c_int, [vp, i64, i64p, i64p, i64p, i64p, i64, i64p]),
    "ce_pattern_coarsen": (C.c_int, [vp, i64, i64p, i64p, i64, i64p, i64p, i64p, i64, i64p]),
    "ce_factorize": (C.c_int, [vp, vp, C.POINTER(PlanHost), C.POINTER(Strategy), C.POINTER(FactorOpts),
                               C.POINTER(vp), C.POINTER(Status)]),
    "ce_factor_free": (None, [vp]),
    "ce_factor_dim": (i64, [vp]),
    "ce_apply_precond": (C.c_int, [vp, vp, vp, i64, C.c_int, vp]),
    "ce_factor_apply_tool": (C.c_int, [vp, C.c_int, vp, vp, i64]),
    "ce_factor_get_stats": (C.c_int, [vp, C.POINTER(FactorStats)]),
    "ce_factor_get_level_stats": (C.c_int, [vp, i64, C.POINTER(LevelStats)]),
    "ce_factor_level_rows": (C.c_int, [vp, i64, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
    "ce_factor_row_sigma": (i64, [vp, i64, i64, C.POINTER(C.c_double), i64]),
    "ce_factor_dump": (C.c_int, [vp, C.c_char_p]),
    "ce_pcg": (C.c_int, [vp, vp, vp, vp, vp, i64, C.c_int, C.POINTER(PcgOpts), C.POINTER(Report), vp]),
    "ce_minres": (C.c_int, [vp, vp, vp, vp, vp, i64, C.c_int, C.POINTER(PcgOpts), C.POINTER(Report), vp]),
    "ce_fmt_double": (C.c_int, [C.c_double, C.c_char_p, C.c_int]),
    "ce_strategy_describe": (C.c_int, [C.POINTER(Strategy), C.c_char_p, C.c_int]),
    "ce_factor_stats_csv": (i64, [vp, C.c_char_p, i64]),
    "ce_factor_summary_csv": (i64, [vp, i64, C.POINTER(Strategy), C.c_double, C.c_char_p, C.c_char_p, i64]),
    "ce_solve_report_csv": (i64, [i64, C.c_char_p, C.POINTER(Strategy), C.c_int, C.POINTER(Report), C.c_double,
                                  C.c_double, C.c_char_p, i64]),
    "ce_trace_csv": (i64, [i64, i64p, dblp, dblp, dblp, C.c_char_p, i64]),
    "ce_ctx_last_trace": (i64, [vp, i64p, dblp, dblp, dblp, i64]),
    "ce_problem_create": (C.c_int, [C.c_int, i64, i64, i64, C.POINTER(vp)]),
    "ce_problem_create_plan": (C.c_int, [C.c_int, i64, i64, i64, C.c_int, C.POINTER(vp)]),
    "ce_problem_free": (None, [vp]),
    "ce_problem_load": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, i64, C.POINTER(vp)]),
    "ce_problem_save": (C.c_int, [vp, C.c_char_p, C.c_char_p, C.c_char_p]),
    "ce_problem_csb": (C.c_int, [vp, C.POINTER(CsbHost)]),
    "ce_problem_plan": (C.c_int, [vp, C.POINTER(PlanHost)]),
    "ce_problem_boxes": (C.c_int, [vp, C.POINTER(C.POINTER(i64)), C.POINTER(i64)]),
    "ce_factorize_sharded": (C.c_int, [vp, vp, C.POINTER(PlanHost), C.POINTER(Strategy), C.POINTER(FactorOpts),
                                       C.POINTER(Shard), C.POINTER(vp), C.POINTER(Status)]),
    "ce_shard_plan_summary": (C.c_int, [vp, C.c_int, i64, i64p, i64p]),
    "ce_problem_rhs": (dblp, [vp]),
    "ce_problem_perm": (i64p, [vp]),
    "ce_problem_params": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_double), i64p]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} is not built; run `make -C {os.path.join(_HERE, 'csrc')}` "
            "(or __graft_entry__.build()). There is no CPU fallback.")
    handle = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    return handle


lib = _load()


def last_error():
    msg = lib.ce_last_error()
    return msg.decode() if msg else ""
