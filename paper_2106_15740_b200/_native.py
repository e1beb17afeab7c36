"""ctypes binding of the in-tree C-ABI library `libqtn_b200.so`.

The boundary is plain C (include/qtn_b200.h); this module only declares
argument types and maps return codes onto the reference's exceptions:
QTN_EINVAL -> ValueError (contraction.py:61-62), QTN_ERANKCAP ->
RankCapExceeded (contraction.py:32-39), everything else -> RuntimeError.
There is no CPU fallback: if the library is missing the import fails.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QTN_LIB") or os.path.join(_HERE, "libqtn_b200.so")

QTN_OK, QTN_EINVAL, QTN_ERANKCAP, QTN_ENOMEM, QTN_ECUDA, QTN_ENODEV = range(6)
DTYPE_C128, DTYPE_C64 = 0, 1
EXEC_SMEM, EXEC_HBM = 0, 1

GATE_INIT, GATE_H, GATE_ZPOW, GATE_XPOW, GATE_CNOT, GATE_ZZ = range(6)
GATE_ZPOW_DIAG, GATE_ZZ_DIAG, GATE_SCALAR = 6, 7, 8


class NetworkDesc(C.Structure):
    _fields_ = [
        ("n_tensors", C.c_int32),
        ("ranks", C.POINTER(C.c_int32)),
        ("var_offsets", C.POINTER(C.c_int32)),
        ("vars", C.POINTER(C.c_int32)),
        ("n_vars", C.c_int32),
        ("is_fixed", C.POINTER(C.c_uint8)),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("executor", C.c_int32),
        ("n_buckets", C.c_int32),
        ("n_empty_buckets", C.c_int32),
        ("width", C.c_int32),
        ("input_elems", C.c_int64),
        ("workspace_bytes", C.c_int64),
        ("smem_bytes", C.c_int64),
        ("program_bytes", C.c_int64),
        ("alg_bytes", C.c_double),
        ("flops_sum", C.c_double),
        ("n_levels", C.c_int32),
        ("n_fused_chains", C.c_int32),
        ("exec_bytes", C.c_double),
        ("n_pairs", C.c_int32),
        ("n_tails", C.c_int32),
    ]


# numpy dtype matching qtn_tensor_recipe (include/qtn_b200.h)
import numpy as np  # noqa: E402

RECIPE_DTYPE = np.dtype(
    [
        ("out_offset", np.int64),
        ("scale", np.float64),
        ("offset", np.float64),
        ("angle", np.int32),
        ("kind", np.uint8),
        ("full_rank", np.uint8),
        ("keep_mask", np.uint8),
        ("fixed_bits", np.uint8),
    ],
    align=True,
)
assert RECIPE_DTYPE.itemsize == 32

_p = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)

_SIGNATURES = {
    "qtn_order_pass": [C.c_int32, C.c_int32, _i32p, _i32p, _f64p, _f64p, C.c_int32, _i32p, _i32p],
    "qtn_rgreedy": [C.c_int32, C.c_int32, _i32p, _i32p, C.c_int32, _f64p, _f64p, C.c_int32,
                    _i32p, _i32p, _i32p],
    "qtn_order_ranks": [C.c_int32, C.c_int32, _i32p, _i32p, _i32p, _i32p],
    "qtn_plan_create": [C.POINTER(NetworkDesc), _i32p, C.c_int32, C.c_int32, C.c_int32,
                        C.c_int32, C.c_int64, C.POINTER(_p), _i32p],
    "qtn_plan_info": [_p, C.POINTER(PlanInfo)],
    "qtn_plan_step_ranks": [_p, _i32p],
    "qtn_plan_input_offsets": [_p, _i64p],
    "qtn_plan_destroy": [_p],
    "qtn_plan_execute": [_p, _p, _p, _p, _p],
    "qtn_batch_create": [C.POINTER(_p), C.c_int32, C.POINTER(_p)],
    "qtn_batch_input_elems": [_p, _i64p],
    "qtn_batch_input_offsets": [_p, _i64p],
    "qtn_batch_workspace_bytes": [_p, C.c_int32, _i64p],
    "qtn_batch_launches": [_p, C.c_int32, _i32p],
    "qtn_batch_uses_setmajor": [_p, C.c_int32, _i32p],
    "qtn_batch_setmajor_elem_bytes": [_p, C.c_int32, _i32p],
    "qtn_batch_execute_host": [_p, _p, C.c_int64, _p, _p, _p, _p, _p],
    "qtn_batch_energies_host": [_p, _p, C.c_int32, C.c_int32, _p, _p, _p, _p, _p, _p, _p, _p],
    "qtn_batch_execute": [_p, _p, C.c_int64, C.c_int32, _p, _p, _p],
    "qtn_batch_destroy": [_p],
    "qtn_batch_set_recipes": [_p, _p, _i64p],
    "qtn_batch_execute_angles": [_p, _p, C.c_int32, C.c_int32, _p, _p, _p, _p],
    "qtn_tensorgen": [_p, C.c_int64, _p, C.c_int32, C.c_int32, C.c_int64, _p, _p],
    "qtn_energy_reduce": [_p, _p, C.c_int32, C.c_int32, _p, _p, _p],
    "qtn_bucket_contract": [C.c_int32, _i32p, _i32p, _i32p, C.POINTER(_p), _u8p, C.c_int32,
                            C.c_int32, _i32p, C.c_int32, _p, _p],
    "qtn_bucket_layout": [C.c_int32, _i32p, _i32p, _i32p, C.c_int32, _i32p, _i32p],
    "qtn_last_error": [],
    "qtn_version": [],
}

EXPORTED = tuple(_SIGNATURES)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback for the B200 backend)"
        )
    lib = C.CDLL(LIB_PATH)
    for name, args in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_char_p if name == "qtn_last_error" else C.c_int
    return lib


lib = _load()


class NativeError(RuntimeError):
    pass


def last_error() -> str:
    msg = lib.qtn_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Raise the Python exception matching a C-ABI return code."""
    if rc == QTN_OK:
        return
    msg = last_error() or what
    if rc == QTN_EINVAL:
        raise ValueError(msg)
    raise NativeError(f"{what}: {msg} (code {rc})" if what else msg)


def i32(a: np.ndarray):
    return a.ctypes.data_as(_i32p)


def i64(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


def f64(a: np.ndarray):
    return a.ctypes.data_as(_f64p)


def u8(a: np.ndarray):
    return a.ctypes.data_as(_u8p)
