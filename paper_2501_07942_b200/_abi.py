"""ctypes / numpy mirror of ``include/ttgbf.h`` and the product library loader.

The product library is ``paper_2501_07942_b200/_lib/libttgbf.so`` (sm_100a,
built in-tree by :func:`paper_2501_07942_b200.build.build`).  There is no CPU
fallback: :func:`load_library` raises if the library or a CUDA device is
missing.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

MAXD = 16
MAXB = 16
NMOM = 1 + MAXD + MAXD * (MAXD + 1) // 2

STATUS = {
    0: "ok", 1: "invalid argument / shape", 2: "evaluator returned a non-finite value",
    3: "TT weights carry no probability mass", 4: "per-filter workspace exhausted",
    5: "evaluator cache capacity exhausted", 6: "CUDA error", 7: "singular matrix",
    8: "dense guard exceeded",
}
E_ARG, E_NONFINITE, E_DEGENERATE, E_WORKSPACE, E_CACHE = 1, 2, 3, 4, 5
E_STATE_CAP = 9

AXIS = np.dtype([("base", "f8"), ("step", "f8"), ("off", "i4"), ("n", "i4")], align=True)
TT = np.dtype([("d", "i4"), ("n", "i4", MAXD), ("r", "i4", MAXD + 1), ("pad", "i4"),
               ("off", "i8", MAXD)], align=True)
CROSS_INFO = np.dtype([("achieved", "f8"), ("calls", "i8"), ("sweeps", "i4"), ("converged", "i4")],
                      align=True)
DIAG = np.dtype([("status", "i4"), ("outlier", "i4"), ("mass_before_norm", "f8"),
                 ("clipped_mass", "f8"), ("cross", CROSS_INFO, 3), ("raw_moments", "f8", NMOM),
                 ("ws_peak", "i8"), ("ranks", "i4", (10, MAXD + 1)), ("cycles", "i8", 8),
                 ("prof", "i8", 32), ("big_used", "i8"), ("big_peak", "i8"),
                 ("big_wait", "i8")], align=True)
MODEL = np.dtype([("d", "i4"), ("b", "i4"), ("hkind", "i4"), ("nang", "i4"), ("ang", "i4", MAXB),
                  ("F", "f8", MAXD * MAXD), ("Finv", "f8", MAXD * MAXD), ("LUq", "f8", MAXD * MAXD),
                  ("pivq", "i4", MAXD), ("invq", "f8", MAXD), ("logn_q", "f8"),
                  ("LUr", "f8", MAXB * MAXB), ("pivr", "i4", MAXB), ("invr", "f8", MAXB), ("logn_r", "f8"),
                  ("H", "f8", MAXB * MAXD), ("Q", "f8", MAXD * MAXD)], align=True)
GAUSS = np.dtype([("mean", "f8", MAXD), ("LU", "f8", MAXD * MAXD), ("piv", "i4", MAXD), ("inv", "f8", MAXD),
                  ("logn", "f8")], align=True)
RUN_CFG_FIELDS = None
STEP_REC = np.dtype([("status", "i4"), ("k", "i4"), ("spd_fixed", "i4"), ("outlier", "i4"), ("mean", "f8", MAXD),
                     ("cov", "f8", MAXD * (MAXD + 1) // 2), ("mass_before_norm", "f8"), ("clipped_mass", "f8"),
                     ("calls", "i8", 3), ("ranks", "i4", (10, MAXD + 1)), ("cycles", "i8")], align=True)


def rec_cov(rec, d: int) -> np.ndarray:
    """Unpack STEP_REC covariances (upper triangle, row-major) to (..., d, d)."""
    packed = np.asarray(rec["cov"])
    out = np.zeros(packed.shape[:-1] + (d, d))
    iu = np.triu_indices(d)
    out[(...,) + iu] = packed[..., : len(iu[0])]
    out[(...,) + (iu[1], iu[0])] = packed[..., : len(iu[0])]
    return out


FILTER_IO = np.dtype([("cur", AXIS, MAXD), ("filt", AXIS, MAXD), ("pred", AXIS, MAXD),
                      ("z", "f8", MAXB), ("has_z", "i4"), ("active", "i4")], align=True)


class GridCfg(ctypes.Structure):
    _fields_ = [("round_tol", ctypes.c_double), ("round_max_rank", ctypes.c_int32),
                ("normalize_before_round", ctypes.c_int32), ("densify_guard", ctypes.c_int64)]


class Axis(ctypes.Structure):
    _fields_ = [("base", ctypes.c_double), ("step", ctypes.c_double), ("off", ctypes.c_int32),
                ("n", ctypes.c_int32)]


class RunCfg(ctypes.Structure):
    _fields_ = [("n_per_axis", ctypes.c_int32), ("kf", ctypes.c_int32), ("steps", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("sigma_mult", ctypes.c_double), ("prior_grid", Axis * MAXD),
                ("nbig", ctypes.c_int32), ("pad2", ctypes.c_int32), ("big_bytes", ctypes.c_int64),
                ("big_ws", ctypes.c_void_p), ("big_locks", ctypes.c_void_p),
                ("nbig2", ctypes.c_int32), ("pad3", ctypes.c_int32), ("big2_bytes", ctypes.c_int64),
                ("big2_ws", ctypes.c_void_p), ("big2_locks", ctypes.c_void_p)]


class CrossCfg(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_rank", ctypes.c_int32),
                ("max_sweeps", ctypes.c_int32), ("validation_count", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("rng_state", ctypes.c_uint64 * 6),
                ("cache_cap", ctypes.c_int64)]


P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
F64 = ctypes.c_double

SIGNATURES = {
    "ttgbf_filter_prior": [P, P, GridCfg, CrossCfg, P, I32, P, I32, P, P, I64, P, I64, P, P],
    "ttgbf_filter_measure": [P, GridCfg, CrossCfg, P, I32, P, I32, P, I32, P, P, I64, P, I64, P, P],
    "ttgbf_filter_time_update": [P, GridCfg, CrossCfg, P, I32, P, I32, P, I32, P, P, I64, P, I64, P, P],
    "ttgbf_filter_time_update_std": [P, GridCfg, CrossCfg, P, I32, P, I32, P, P, I64, P, I64, P, P],
    "ttgbf_filter_run": [P, P, GridCfg, CrossCfg, RunCfg, P, P, P, I32, P, I32, P, I32, P, P, I64, P, I64, P, I32,
                         P, P, P],
    "ttgbf_tt_round": [P, P, I64, I32, F64, I32, P, P, I64, P, I64, P, P],
    "ttgbf_tt_hadamard": [P, P, I64, P, P, I64, I32, P, P, I64, P, I64, P, P],
    "ttgbf_tt_fft_convolve": [P, P, I64, P, P, I64, I32, F64, I32, P, P, I64, P, I64, P, P],
    "ttgbf_tt_interpolate": [P, P, I64, I32, P, P, P, P, I64, P, I64, P, P],
    "ttgbf_tt_eval_many": [P, P, I64, I32, P, I64, P, P, I64, P, P],
    "ttgbf_tt_eval_at_points": [P, P, I64, I32, P, P, I64, P, P, I64, P, P],
    "ttgbf_tt_sum_moments": [P, P, I64, I32, P, P, P, I64, P, P],
    "ttgbf_greedy_cross": [I32, P, P, CrossCfg, P, I32, P, I32, P, P, I64, P, I64, P, P],
    "ttgbf_negative_mass": [P, P, I64, I32, P, I64, P, I32, P, P, I64, P, P],
    "ttgbf_eval_blackbox": [I32, P, P, P, P, P, I64, I32, P, I64, P, P, I64, P, P],
    "ttgbf_rng_draws": [I32, P, P, I32, I64, I64, I64, P, P, I64, P, P],
    "ttgbf_sizeof": [I32],
    "ttgbf_version": [],
    "ttgbf_block_threads": [],
    "ttgbf_smem_bytes": [],
    "ttgbf_ctas_per_sm": [],
    "ttgbf_status_string": [I32],
    # dense grid filter (csrc/dense.cu)
    "ttgbf_dense_prior": [P, P, I32, P, P],
    "ttgbf_dense_likelihood": [P, P, P, I32, P, P],
    "ttgbf_dense_reduce": [P, P, I32, I32, F64, P, P, P, P],
    "ttgbf_dense_reduce_blocks": [],
    "ttgbf_dense_finalize": [P, I64, F64, P],
    "ttgbf_dense_interp": [P, P, P, I32, P, P, P],
    "ttgbf_dense_kernel": [P, P, I32, P, F64, F64, P, P],
    "ttgbf_dense_dft": [P, P, I32, I32, I32, P, P],
    "ttgbf_dense_cmul": [P, P, I64, P],
    "ttgbf_dense_real": [P, P, I64, P],
}
DENSE = frozenset(n for n in SIGNATURES if n.startswith("ttgbf_dense_"))
RESTYPES = {"ttgbf_smem_bytes": I64, "ttgbf_status_string": ctypes.c_char_p, "ttgbf_sizeof": I64}

BB_GAUSS, BB_LIKELIHOOD, BB_KERNEL, BB_REALIGN = 0, 1, 2, 3


def struct_sizes() -> dict:
    """numpy / ctypes mirrors of the ABI structs, indexed like ttgbf_sizeof()."""
    return {0: AXIS.itemsize, 1: TT.itemsize, 2: ctypes.sizeof(CrossCfg), 3: ctypes.sizeof(GridCfg),
            4: DIAG.itemsize, 5: MODEL.itemsize, 6: GAUSS.itemsize, 7: FILTER_IO.itemsize,
            8: ctypes.sizeof(RunCfg), 9: STEP_REC.itemsize}

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "_lib")
# TTGBF_LIB_VARIANT=<tag> loads _lib/libttgbf_<tag>.so (a build of the same
# sources with other compile-time tuning, e.g. CTAs per SM; tools/build_variant.sh)
PRODUCT_LIB = os.path.join(LIB_DIR, "libttgbf%s.so" % (("_" + os.environ["TTGBF_LIB_VARIANT"])
                                                       if os.environ.get("TTGBF_LIB_VARIANT") else ""))


def bind(lib, dense: bool = True):
    """Set ctypes signatures; every declared symbol must exist (the test-only
    host emulation of the TT engine passes dense=False: it has no dense TU)."""
    for name, args in SIGNATURES.items():
        if not dense and name in DENSE:
            continue
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = RESTYPES.get(name, I32)
    return lib


_LIB = None


def load_library():
    """Load the sm_100a product library; raise loudly if it cannot run here."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(PRODUCT_LIB):
        raise RuntimeError(
            f"{PRODUCT_LIB} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the TT-GBF hot path needs a CUDA device (B200, sm_100a); none is visible")
    torch.cuda.init()
    _LIB = bind(ctypes.CDLL(PRODUCT_LIB))
    return _LIB


def status_text(code: int) -> str:
    return STATUS.get(int(code), f"status {int(code)}")
