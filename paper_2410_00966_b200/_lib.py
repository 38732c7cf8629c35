"""ctypes binding of libmcq.so (include/mcq.h).  Argument marshalling only: every step of the
hot path runs in the library's CUDA kernels.  There is no fallback: if the shared library is
missing or fails to load, importing this module raises."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCQ_LIB_PATH") or os.path.join(HERE, "libmcq.so")  # override: tuning variants

MCQ_OK, MCQ_EINVAL, MCQ_ESTATE, MCQ_ENOMEM, MCQ_ECUDA, MCQ_ENCCL = 0, -1, -2, -3, -4, -5
TERM_ZEEMAN, TERM_EXCHANGE, TERM_ANIS, TERM_DEMAG, TERM_CAVITY, TERM_EXCITATION = 1, 2, 4, 8, 16, 32
TERM_DMI = 64
TERM_ALL = 127
TERM_THERM = 128
K_YFWD, K_ZCONV, K_YINV, K_Y2D, K_UPDATE, K_CAVITY = range(6)
NKCLASS = 6
KCLASS_NAMES = ("yfwd", "zconv", "yinv", "y2d", "update", "cavity")


class mcq_aniso(C.Structure):
    _fields_ = [("ku1", C.c_double), ("u", C.c_double * 3), ("kc1", C.c_double),
                ("c1", C.c_double * 3), ("c2", C.c_double * 3)]


class mcq_dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("device", C.c_int),
                ("nccl_id", C.c_void_p), ("cuda_stream", C.c_void_p)]


class mcq_cavity_state(C.Structure):
    _fields_ = [("t", C.c_double), ("re_alpha", C.c_double), ("im_alpha", C.c_double),
                ("gamma", C.c_double), ("W", C.c_double), ("S", C.c_double), ("C", C.c_double),
                ("n_photon", C.c_double), ("step", C.c_longlong), ("S_resc", C.c_double), ("C_resc", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class MCQError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"mcq error {code}: {msg}")
        self.code = code


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2410_00966_b200.build` "
                      "(there is no CPU fallback)")
lib = C.CDLL(LIB_PATH)

_P = C.c_void_p
_sig = {
    "mcq_nccl_get_unique_id": (C.c_int, [_P]),
    "mcq_create": (C.c_int, [C.POINTER(_P), C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_double, C.c_double,
                             C.c_double, C.POINTER(mcq_aniso), C.POINTER(mcq_dist)]),
    "mcq_set_stream": (C.c_int, [_P, _P]),
    "mcq_set_slab_overlap": (C.c_int, [_P, C.c_int]),
    "mcq_set_persistent_2d": (C.c_int, [_P, C.c_int]),
    "mcq_set_geometry": (C.c_int, [_P, _P]),
    "mcq_set_m": (C.c_int, [_P, _P]),
    "mcq_set_m_device": (C.c_int, [_P, _P]),
    "mcq_set_bext": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "mcq_set_brms": (C.c_int, [_P, _P, C.POINTER(C.c_double)]),
    "mcq_set_cavity": (C.c_int, [_P, C.c_double, C.c_double, C.c_double, C.c_double]),
    "mcq_set_excitation": (C.c_int, [_P, C.c_double, C.c_double]),
    "mcq_set_dmi": (C.c_int, [_P, C.c_double]),
    "mcq_set_temperature": (C.c_int, [_P, C.c_double, C.c_ulonglong]),
    "mcq_get_thermal_step": (C.c_int, [_P, C.POINTER(C.c_longlong)]),
    "mcq_set_thermal_step": (C.c_int, [_P, C.c_longlong]),
    "mcq_reset_memory": (C.c_int, [_P]),
    "mcq_set_modes": (C.c_int, [_P, C.c_int]),
    "mcq_set_brms_mode": (C.c_int, [_P, C.c_int, _P, C.POINTER(C.c_double)]),
    "mcq_set_cavity_mode": (C.c_int, [_P, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double]),
    "mcq_set_excitation_mode": (C.c_int, [_P, C.c_int, C.c_double, C.c_double]),
    "mcq_get_cavity_mode": (C.c_int, [_P, C.c_int, C.POINTER(mcq_cavity_state)]),
    "mcq_set_cavity_state_mode": (C.c_int, [_P, C.c_int, C.POINTER(mcq_cavity_state)]),
    "mcq_relax": (C.c_int, [_P, C.c_double, C.c_double, C.c_longlong, C.POINTER(C.c_longlong)]),
    "mcq_run": (C.c_int, [_P, C.c_double, C.c_longlong]),
    "mcq_run_dp": (C.c_int, [_P, C.c_double, C.c_longlong]),
    "mcq_run_adaptive": (C.c_int, [_P, C.c_double, C.c_double, C.c_double, C.c_longlong, C.POINTER(C.c_longlong),
                                   C.POINTER(C.c_longlong), C.POINTER(C.c_double)]),
    "mcq_synchronize": (C.c_int, [_P]),
    "mcq_get_m": (C.c_int, [_P, _P]),
    "mcq_get_m_device": (C.c_int, [_P, _P]),
    "mcq_get_field": (C.c_int, [_P, _P, C.c_uint]),
    "mcq_get_cavity": (C.c_int, [_P, C.POINTER(mcq_cavity_state)]),
    "mcq_cavity_state_bytes": (C.c_longlong, []),
    "mcq_set_cavity_state": (C.c_int, [_P, C.POINTER(mcq_cavity_state)]),
    "mcq_cavity_status": (C.c_int, [_P]),
    "mcq_kernel_launches": (C.c_longlong, [_P]),
    "mcq_set_trace": (C.c_int, [_P, C.c_longlong, C.c_int]),
    "mcq_get_trace": (C.c_int, [_P, _P, C.c_longlong, C.POINTER(C.c_longlong)]),
    "mcq_trace_peaks": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _P, _P, _P]),
    "mcq_trace_peaks_batch": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _P, _P, _P]),
    "mcq_spectrum_peaks": (C.c_int, [_P, C.c_longlong, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int, _P, _P, _P]),
    "mcq_fit_anticrossing": (C.c_int, [C.c_int, _P, _P, _P, C.c_double, C.c_double, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]),
    "mcq_profile_run": (C.c_int, [_P, C.c_double, C.c_longlong, C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    "mcq_debug_layout": (C.c_int, [_P, C.POINTER(C.c_longlong)]),
    "mcq_debug_tensor_octant": (C.c_int, [_P, _P]),
    "mcq_debug_khat": (C.c_int, [_P, _P]),
    "mcq_last_error": (C.c_char_p, [_P]),
    "mcq_ovf_read": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_double), _P, C.c_longlong]),
    "mcq_ovf_write": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_double), _P, C.c_int]),
    "mcq_ovf_last_error": (C.c_char_p, []),
    "mcq_destroy": (None, [_P]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sig)
