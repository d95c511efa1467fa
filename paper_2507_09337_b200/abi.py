"""ctypes binding of liborcha.so (include/orcha.h) -- argument marshalling only.

Every function here has the name of the C entry point it calls and does no
arithmetic of the method: all device work happens in the CUDA kernels of the
library.  A missing library is an error (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {False: os.path.join(HERE, "liborcha.so"), True: os.path.join(HERE, "liborcha_parity.so")}

ORCHA_OK = 0
STATUS = {0: "ORCHA_OK", -1: "ORCHA_E_ARG", -2: "ORCHA_E_RANGE", -3: "ORCHA_E_HALO", -4: "ORCHA_E_NONPHYSICAL",
          -5: "ORCHA_E_LAYOUT", -6: "ORCHA_E_CUDA", -7: "ORCHA_E_NCCL", -8: "ORCHA_E_STATE"}
BC_OUTFLOW, BC_PERIODIC, BC_REFLECT = 0, 1, 2
RIEMANN_HLL, RIEMANN_HLLC = 0, 1
LIMITER_MINMOD, LIMITER_MC = 0, 1
EOS_GAMMA_LAW, EOS_GAS_RADIATION = 0, 1
DT_CFL, DT_CLAMP = 0, 1
FNV1A64_OFFSET = 0xcbf29ce484222325
PHASES = ("fill", "exchange", "dt", "dt_allgather", "stage1", "stage2")

EXPORTS = [
    "orcha_grid_create", "orcha_grid_destroy", "orcha_grid_nblocks", "orcha_packet_bytes", "orcha_packet_create",
    "orcha_packet_destroy", "orcha_packet_nblocks", "orcha_packet_layout", "orcha_packet_pack",
    "orcha_packet_unpack", "orcha_packet_pack_device", "orcha_packet_unpack_device", "orcha_fill_guardcells",
    "orcha_compute_dt", "orcha_hydro_advance", "orcha_hydro_advance_devdt", "orcha_packet_counters",
    "orcha_build_is_parity", "orcha_launch_count", "orcha_last_error", "orcha_comm_unique_id",
    "orcha_comm_create", "orcha_comm_destroy", "orcha_set_kernel_variant", "orcha_get_kernel_variant",
    "orcha_comm_create_local", "orcha_comm_push", "orcha_comm_plan", "orcha_hydro_stage",
    "orcha_hydro_stage_devdt", "orcha_fill_guardcells_stage", "orcha_set_guard_push", "orcha_set_fill_mode",
    "orcha_packet_unpack_async", "orcha_fill_guardcells_packet", "orcha_packet_dt_records",
    "orcha_compute_dt_device", "orcha_unit_eos", "orcha_unit_face_flux", "orcha_unit_riemann",
    "orcha_comm_push_dt", "orcha_set_phase_timing", "orcha_phase_times", "orcha_probe_fp64",
    "orcha_fnv1a64", "orcha_comm_peer_register", "orcha_comm_check",
    "orcha_fill_prepare", "orcha_hydro_step_overlap", "orcha_comm_create_ipc", "orcha_comm_ipc_export",
    "orcha_comm_ipc_attach", "orcha_set_ring_mode", "orcha_get_ring_mode", "orcha_ring_classify",
]


class OrchaError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class orcha_grid_desc(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int32),
        ("nb", ctypes.c_int32 * 3),
        ("ng", ctypes.c_int32),
        ("nblk", ctypes.c_int32 * 3),
        ("xmin", ctypes.c_double * 3),
        ("xmax", ctypes.c_double * 3),
        ("bc", (ctypes.c_int32 * 2) * 3),
        ("gamma", ctypes.c_double),
        ("cfl", ctypes.c_double),
        ("smallp", ctypes.c_double),
        ("riemann", ctypes.c_int32),
        ("limiter", ctypes.c_int32),
        ("eos", ctypes.c_int32),
        ("eos_work", ctypes.c_int32),
        ("arad", ctypes.c_double),
    ]


class orcha_dt_info(ctypes.Structure):
    _fields_ = [
        ("dt", ctypes.c_double),
        ("smax", ctypes.c_double),
        ("argmax", ctypes.c_int64),
        ("tag", ctypes.c_int32),
        ("nonphysical", ctypes.c_int32),
    ]


class orcha_dev_clock(ctypes.Structure):
    _fields_ = [
        ("t", ctypes.c_double),
        ("t_end", ctypes.c_double),
        ("dt", ctypes.c_double),
        ("smax", ctypes.c_double),
        ("argmax", ctypes.c_int64),
        ("tag", ctypes.c_int32),
        ("nonphysical", ctypes.c_int32),
        ("steps", ctypes.c_int64),
        ("reserved", ctypes.c_int64),
    ]


_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_sz = ctypes.c_size_t
_dbl = ctypes.c_double
_P = ctypes.POINTER

_SIGS = {
    "orcha_grid_create": (_i32, [_P(orcha_grid_desc), _P(_vp)]),
    "orcha_grid_destroy": (_i32, [_vp]),
    "orcha_grid_nblocks": (_i64, [_vp]),
    "orcha_packet_bytes": (_i32, [_vp, _i32, _P(_sz), _P(_sz)]),
    "orcha_packet_create": (_i32, [_vp, _i32, _P(_i64), _vp, _vp, _P(_vp)]),
    "orcha_packet_destroy": (_i32, [_vp]),
    "orcha_packet_nblocks": (_i32, [_vp]),
    "orcha_packet_layout": (_i32, [_vp, _P(_vp), _P(_sz), _P(_i32)]),
    "orcha_packet_pack": (_i32, [_vp, _vp, _vp]),
    "orcha_packet_unpack": (_i32, [_vp, _vp, _vp]),
    "orcha_packet_pack_device": (_i32, [_vp, _vp, _vp]),
    "orcha_packet_unpack_device": (_i32, [_vp, _vp, _vp]),
    "orcha_packet_unpack_async": (_i32, [_vp, _vp, _vp]),
    "orcha_fill_guardcells": (_i32, [_P(_vp), _i32, _vp, _vp]),
    "orcha_fill_guardcells_packet": (_i32, [_P(_vp), _i32, _i32, _vp]),
    "orcha_packet_dt_records": (_i32, [_vp, _vp]),
    "orcha_compute_dt": (_i32, [_P(_vp), _i32, _vp, _dbl, _P(orcha_dt_info), _vp]),
    "orcha_hydro_advance": (_i32, [_vp, _dbl, _vp]),
    "orcha_hydro_advance_devdt": (_i32, [_vp, _vp, _vp]),
    "orcha_compute_dt_device": (_i32, [_P(_vp), _i32, _vp, _vp, _vp]),
    "orcha_packet_counters": (_i32, [_vp, _P(_i64), _P(_i64), _vp]),
    "orcha_build_is_parity": (_i32, []),
    "orcha_launch_count": (_i64, []),
    "orcha_last_error": (ctypes.c_char_p, []),
    "orcha_set_kernel_variant": (_i32, [_i32]),
    "orcha_get_kernel_variant": (_i32, []),
    "orcha_comm_unique_id": (_i32, [_vp]),
    "orcha_comm_create": (_i32, [_vp, _vp, _i32, _i32, _P(_i32), _P(_vp)]),
    "orcha_comm_destroy": (_i32, [_vp]),
    "orcha_comm_create_local": (_i32, [_vp, _i32, _P(_i32), _P(_vp)]),
    "orcha_comm_push": (_i32, [_vp, _P(_vp), _i32, _i32, _vp]),
    "orcha_hydro_stage": (_i32, [_vp, _i32, _dbl, _vp]),
    "orcha_set_guard_push": (_i32, [_i32]),
    "orcha_set_fill_mode": (_i32, [_i32]),
    "orcha_set_ring_mode": (_i32, [_i32]),
    "orcha_get_ring_mode": (_i32, []),
    "orcha_ring_classify": (_i32, [_vp, _i32, _P(_i64), _P(_i32), _P(_i32)]),
    "orcha_hydro_stage_devdt": (_i32, [_vp, _i32, _vp, _vp]),
    "orcha_fill_guardcells_stage": (_i32, [_P(_vp), _i32, _vp, _i32, _vp]),
    "orcha_comm_plan": (_i32, [_vp, _i32, _i32, _P(_i32), _i32, _i32, _P(_i64), _i64, _P(_i64)]),
    "orcha_set_phase_timing": (_i32, [_i32]),
    "orcha_phase_times": (_i32, [_P(_dbl), _P(_i64), _i32]),
    "orcha_comm_create_ipc": (_i32, [_vp, _i32, _i32, _P(_i32), _P(_vp)]),
    "orcha_comm_ipc_export": (_i32, [_vp, _vp, _vp, _sz, _P(_sz)]),
    "orcha_comm_ipc_attach": (_i32, [_vp, _vp, _sz]),
    "orcha_hydro_step_overlap": (_i32, [_vp, _vp, _vp, _vp]),
    "orcha_fill_prepare": (_i32, [_P(_vp), _i32, _vp]),
    "orcha_comm_peer_register": (_i32, [_vp, _vp, _vp]),
    "orcha_comm_check": (_i32, [_vp]),
    "orcha_fnv1a64": (_i32, [_vp, _sz, _P(ctypes.c_uint64)]),
    "orcha_probe_fp64": (_i32, [_i32, _P(_dbl), _P(_dbl), _vp]),
    "orcha_comm_push_dt": (_i32, [_vp, _P(_vp), _i32, _vp]),
    "orcha_unit_eos": (_i32, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "orcha_unit_face_flux": (_i32, [_vp, _i32, _i64, _vp, _vp, _vp]),
    "orcha_unit_riemann": (_i32, [_vp, _i32, _i64, _vp, _vp, _vp, _vp]),
}

_loaded = {}


def library_path(parity: bool = False) -> str:
    return LIBS[bool(parity)]


def load(parity: bool = False) -> ctypes.CDLL:
    """Load liborcha.so (or the parity build).  Raises if it is not built."""
    parity = bool(parity)
    if parity not in _loaded:
        path = LIBS[parity]
        if not parity and os.environ.get("ORCHA_LIB"):  # experiments: an alternative production build
            path = os.environ["ORCHA_LIB"]
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python -m paper_2507_09337_b200.build` "
                              "(the CUDA extension is required; there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _loaded[parity] = lib
    return _loaded[parity]


def check(lib, rc: int, where: str) -> None:
    if rc != ORCHA_OK:
        raise OrchaError(rc, where, lib.orcha_last_error().decode())


def call(lib, name: str, *args) -> None:
    """Call a status-returning entry point and raise OrchaError on failure."""
    check(lib, getattr(lib, name)(*args), name)
