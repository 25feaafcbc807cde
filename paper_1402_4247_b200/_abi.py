"""ctypes mirror of include/kbgrid.h and include/kbgsynth.h.

The C-ABI is the product boundary; this module only declares
its structs and function prototypes and loads the in-tree shared libraries.
There is no fallback: a missing library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBDIR = os.path.join(HERE, "lib")
# KBG_LIBKBGRID: alternative build of the same library (tools/ kernel variants)
KBGRID_SO = os.environ.get("KBG_LIBKBGRID") or os.path.join(LIBDIR, "libkbgrid.so")
KBGSYNTH_SO = os.path.join(LIBDIR, "libkbgsynth.so")

KBG_OK = 0
KBG_ERR_CONFIG = 1
KBG_ERR_DIMENSION = 2
KBG_ERR_CONSISTENCY = 3
KBG_ERR_NONFINITE = 4
KBG_ERR_CUDA = 5
KBG_ERR_NCCL = 6
KBG_OPT_WARPS = 1
KBG_OPT_FAULT_SIGN = 2
KBG_OPT_SCATTER_STORE = 3
KBG_OPT_PERSIST = 4
KBG_OPT_DEBUG_COUNTERS = 5
KBG_OPT_SCHEDULE = 6
KBG_OPT_BLOCK_ORDER = 7
KBG_OPT_XC = 8
KBG_OPT_DETERMINISTIC = 9
KBG_OPT_SHARD_IO = 10
KBG_OPT_SPARSE_DFMA = 11
KBG_OPT_EXCHANGE_SMS = 12
KBG_OPT_FUSED_PASS = 13
KBG_COMM_HANDLE_BYTES = 96
KBG_CELL_PRIMITIVE = 0
KBG_CELL_CUBIC = 1


class kbg_species(C.Structure):
    _fields_ = [
        ("nrad", C.c_int),
        ("l", C.POINTER(C.c_int)),
        ("rc", C.c_double),
        ("ntab", C.c_int),
        ("table", C.POINTER(C.c_double)),
    ]


class kbg_system(C.Structure):
    _fields_ = [
        ("lattice", C.c_double * 9),
        ("grid", C.c_int * 3),
        ("natom", C.c_int),
        ("species", C.POINTER(C.c_int)),
        ("tau", C.POINTER(C.c_double)),
        ("nspecies", C.c_int),
        ("spec", C.POINTER(kbg_species)),
    ]


class kbg_index(C.Structure):
    _fields_ = [
        ("npts", C.c_int64),
        ("nblk", C.c_int * 3),
        ("nblock", C.c_int64),
        ("ncover", C.c_int64),
        ("blk_ptr", C.POINTER(C.c_int32)),
        ("cov_atom", C.POINTER(C.c_int32)),
        ("cov_R", C.POINTER(C.c_int32)),
        ("cov_mask", C.POINTER(C.c_uint64)),
        ("npair", C.c_int64),
        ("pair_a", C.POINTER(C.c_int32)),
        ("pair_b", C.POINTER(C.c_int32)),
        ("pair_R", C.POINTER(C.c_int32)),
        ("pair_off", C.POINTER(C.c_int64)),
        ("pair_mirror", C.POINTER(C.c_int32)),
        ("nnz", C.c_int64),
        ("nbpair", C.c_int64),
        ("natompt", C.c_int64),
        ("sum_m", C.c_double),
        ("sum_m2", C.c_double),
    ]


class kbg_tally(C.Structure):
    _fields_ = [("flops", C.c_double), ("bytes", C.c_double)]


_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_D = C.c_double
_DP = C.POINTER(C.c_double)

# (name, restype, argtypes) of every symbol declared in include/kbgrid.h.
KBGRID_SYMBOLS = [
    ("kbg_create", _I, [C.POINTER(kbg_system), _I, C.POINTER(_P)]),
    ("kbg_create_sharded", _I, [C.POINTER(kbg_system), _I, _I, _I, C.POINTER(_P)]),
    ("kbg_build_index", _I, [_P]),
    ("kbg_index_view", _I, [_P, C.POINTER(kbg_index)]),
    ("kbg_shard_range", _I, [_P, C.POINTER(_I64), C.POINTER(_I64)]),
    ("kbg_plan_info", _I, [_P, C.POINTER(_I64)]),
    ("kbg_density", _I, [_P, _I, _DP, _DP]),
    ("kbg_hamiltonian", _I, [_P, _I, _DP, _D, _DP]),
    ("kbg_grid_pass", _I, [_P, _I, _DP, _DP, _D, _DP, _DP]),
    ("kbg_density_dev", _I, [_P, _I, _P, _P, _P]),
    ("kbg_hamiltonian_dev", _I, [_P, _I, _P, _D, _P, _P]),
    ("kbg_hamiltonian_accumulate_dev", _I, [_P, _I, _P, _D, _P, _P]),
    ("kbg_hamiltonian_mirror_dev", _I, [_P, _I, _P, _P]),
    ("kbg_grid_pass_dev", _I, [_P, _I, _P, _P, C.c_double, _P, _P, _P]),
    ("kbg_block_orbitals", _I, [_P, _I64, _DP, _I64, C.POINTER(_I)]),
    ("kbg_last_launches", _I, [_P]),
    ("kbg_last_tally", _I, [_P, C.POINTER(kbg_tally)]),
    ("kbg_debug_counters", _I, [_P, C.POINTER(C.c_int64), _I]),
    ("kbg_set_option", _I, [_P, _I, _I64]),
    ("kbg_last_error", C.c_char_p, [_P]),
    ("kbg_status_string", C.c_char_p, [_I]),
    ("kbg_destroy", None, [_P]),
    ("kbg_version", C.c_char_p, []),
    ("kbg_veff", _I, [_P, _I, _DP, _DP, _DP, _DP]),
    ("kbg_veff_dev", _I, [_P, _I, _P, _P, _P, _P, _P]),
    ("kbg_comm_handle", _I, [_P, _P]),
    ("kbg_comm_open", _I, [_P, _P]),
    ("kbg_comm_check", _I, [_P]),
    ("kbg_shard_io", _I, [_P, C.POINTER(C.c_int64)]),
    ("kbg_comm_timing", _I, [_P, _DP]),
    ("kbg_hamiltonian_allreduce_dev", _I, [_P, _I, _P, _D, _P, _P]),
    ("kbg_hamiltonian_partial_dev", _I, [_P, _I, _P, _D, _P]),
    ("kbg_hamiltonian_exchange_dev", _I, [_P, _I, _P, _P]),
    ("kbg_offsets", _I, [_P, C.POINTER(_I), C.POINTER(C.c_int32)]),
    ("kbg_to_realspace", _I, [_P, _DP, _DP]),
    ("kbg_from_realspace", _I, [_P, _DP, _DP]),
    ("kbg_to_realspace_dev", _I, [_P, _P, _P, _P]),
    ("kbg_from_realspace_dev", _I, [_P, _P, _P, _P]),
    ("kbg_bloch", _I, [_P, _DP, _I, _DP, _DP]),
    ("kbg_bloch_dev", _I, [_P, _P, _I, _DP, _P, _P]),
    ("kbg_fold", _I, [_P, _I, _DP, _DP, _DP, _DP, _DP]),
    ("kbg_fold_dev", _I, [_P, _I, _DP, _DP, _P, _P, _P]),
    ("kbg_density_matrix_k", _I, [_P, _I, _DP, _DP, _DP]),
    ("kbg_density_matrix_k_dev", _I, [_P, _I, _P, _P, _P, _P]),
    ("kbg_normalize_rows_dev", _I, [_P, _I64, _I64, _P]),
    ("kbg_normalize_rows", _I, [_DP, _I64, _I64]),
    ("kbg_hh_tridiagonalize", _I, [_I64, _DP, _I, _DP, _DP, _DP, _DP, _DP, _DP]),
    ("kbg_hh_tridiagonalize_dev", _I, [_I64, _P, _I, _P, _P, _P, _P, _P, _P, _P]),
    ("kbg_hh_back_transform", _I, [_I64, _I64, _DP, _DP, _DP, _DP, _DP]),
    ("kbg_hh_back_transform_dev", _I, [_I64, _I64, _P, _P, _P, _P, _P, _P]),
    ("kbg_hh_normalize_columns", _I, [_I64, _I64, _DP]),
    ("kbg_hh_normalize_columns_dev", _I, [_I64, _I64, _P, _P]),
    ("kbg_hh_triple_product", _I, [_I64, _I64, _DP, _DP, _DP]),
    ("kbg_hh_eigen", _I, [_I64, _DP, _I, _DP, _DP]),
    ("kbg_tridiag_solve", _I, [_I64, _DP, _DP, _I, _DP, _DP]),
    ("kbg_tridiag_solve_dev", _I, [_I64, C.c_void_p, C.c_void_p, _I, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("kbg_hh_last_error", C.c_char_p, []),
]

KBGSYNTH_SYMBOLS = [
    ("kbg_synth_create", _I, [_I, _I, _D, C.c_uint64, _I, C.POINTER(_P)]),
    ("kbg_synth_system", C.POINTER(kbg_system), [_P]),
    ("kbg_synth_dV", _D, [_P]),
    ("kbg_synth_veff", _I, [_P, _I, C.c_uint64, _DP]),
    ("kbg_synth_dm", _I, [_P, C.POINTER(kbg_index), _I, C.c_uint64, _DP]),
    ("kbg_synth_free", None, [_P]),
    ("kbg_synth_radial_table", _D, [_I, _D, _D, _I, _DP]),
    ("kbg_synth_good_size", _I, [_I]),
]


def _bind(lib, symbols):
    for name, res, args in symbols:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_cache: dict[str, C.CDLL] = {}


def load(path: str, symbols) -> C.CDLL:
    if path in _cache:
        return _cache[path]
    if not os.path.exists(path):
        raise OSError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the grid pass)")
    lib = _bind(C.CDLL(path, mode=C.RTLD_GLOBAL), symbols)
    _cache[path] = lib
    return lib


def kbgrid() -> C.CDLL:
    return load(KBGRID_SO, KBGRID_SYMBOLS)


def kbgsynth() -> C.CDLL:
    return load(KBGSYNTH_SO, KBGSYNTH_SYMBOLS)


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_DP)


def index_to_numpy(ix: kbg_index) -> dict:
    """Copy a kbg_index view into owned numpy arrays."""

    def arr(ptr, n, dt):
        if n == 0:
            return np.zeros(0, dtype=dt)
        return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)

    return {
        "npts": int(ix.npts),
        "nblk": tuple(ix.nblk),
        "nblock": int(ix.nblock),
        "blk_ptr": arr(ix.blk_ptr, ix.nblock + 1, np.int32),
        "cov_atom": arr(ix.cov_atom, ix.ncover, np.int32),
        "cov_R": arr(ix.cov_R, 3 * ix.ncover, np.int32).reshape(-1, 3),
        "cov_mask": arr(ix.cov_mask, ix.ncover, np.uint64),
        "pair_a": arr(ix.pair_a, ix.npair, np.int32),
        "pair_b": arr(ix.pair_b, ix.npair, np.int32),
        "pair_R": arr(ix.pair_R, 3 * ix.npair, np.int32).reshape(-1, 3),
        "pair_off": arr(ix.pair_off, ix.npair + 1, np.int64),
        "pair_mirror": arr(ix.pair_mirror, ix.npair, np.int32),
        "nnz": int(ix.nnz),
        "nbpair": int(ix.nbpair),
        "natompt": int(ix.natompt),
        "sum_m": float(ix.sum_m),
        "sum_m2": float(ix.sum_m2),
    }


def index_from_numpy(d: dict):
    """Build a kbg_index struct pointing at numpy arrays (keep `d` alive)."""
    ix = kbg_index()
    ix.npts = d["npts"]
    for c in range(3):
        ix.nblk[c] = d["nblk"][c]
    ix.nblock = d["nblock"]
    keep = {}

    def p(name, ct):
        a = np.ascontiguousarray(d[name]).reshape(-1)
        keep[name] = a
        return a.ctypes.data_as(C.POINTER(ct))

    ix.ncover = len(d["cov_atom"])
    ix.blk_ptr = p("blk_ptr", C.c_int32)
    ix.cov_atom = p("cov_atom", C.c_int32)
    ix.cov_R = p("cov_R", C.c_int32)
    ix.cov_mask = p("cov_mask", C.c_uint64)
    ix.npair = len(d["pair_a"])
    ix.pair_a = p("pair_a", C.c_int32)
    ix.pair_b = p("pair_b", C.c_int32)
    ix.pair_R = p("pair_R", C.c_int32)
    ix.pair_off = p("pair_off", C.c_int64)
    ix.pair_mirror = p("pair_mirror", C.c_int32)
    ix.nnz = d["nnz"]
    ix.nbpair = d["nbpair"]
    ix.natompt = d["natompt"]
    ix.sum_m = d["sum_m"]
    ix.sum_m2 = d["sum_m2"]
    ix._keep = keep
    return ix
