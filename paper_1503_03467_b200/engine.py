"""ctypes mirror of gb_level_engine_args (csrc/gb_engine.h)."""

import ctypes

_P = ctypes.c_void_p
_D = ctypes.c_double


class LevelEngineArgs(ctypes.Structure):
    _fields_ = [
        ("L", ctypes.c_int), ("w", ctypes.c_int), ("max_chunk", ctypes.c_int),
        ("max_outer", ctypes.c_int),
        ("BsT", _P),
        ("inv", _P), ("xa", _P), ("ra", _P), ("pa", _P), ("apa", _P), ("za", _P),
        ("sta", _P), ("parta", _P), ("hsta", _P),
        ("xb", _P), ("yb", _P), ("x2", _P), ("xn", _P), ("ax", _P), ("cx", _P), ("cr", _P),
        ("cp", _P), ("cap", _P), ("stb", _P), ("partb", _P), ("hstb", _P),
        ("dots", _P), ("hdots", _P),
        ("tol", _D), ("inner_tol", _D), ("inner_max_iter", ctypes.c_int64),
        ("lam_min", _D), ("lam_max", _D), ("calls", ctypes.c_int64),
        ("power_its", ctypes.c_int), ("n_outer", ctypes.c_int), ("breakdown", ctypes.c_int),
        ("inner_pcg", ctypes.c_int), ("inner_its", ctypes.c_int * 64),
        ("cz", _P), ("layout", ctypes.c_int),
        ("spectral_mode", ctypes.c_int), ("lz_cap", ctypes.c_int), ("lz", _P), ("hlz", _P),
        ("lz_tol", _D), ("lz_its", ctypes.c_int), ("lz_rc", ctypes.c_int),
        ("n_dual", ctypes.c_int64), ("n_single", ctypes.c_int64),
        ("ev_cap", ctypes.c_int), ("ev_n", ctypes.c_int), ("ev_ms", _P), ("ev_events", _P),
    ]
