"""ctypes binding of libgamblets_b200.so (the C ABI in include/gamblets_b200.h).

There is no fallback: if the library is missing or no CUDA device is present
every entry point raises.  Device buffers are torch tensors (ownership and
the caching allocator only); the kernels see raw pointers.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import InvalidArgumentError, NumericalError

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libgamblets_b200.so"

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
_D = ctypes.c_double
_Z = ctypes.c_size_t

# name -> (argtypes, restype)
_SIGS = {
    "gb_abi_version": ([], _I),
    "gb_launch_count": ([], ctypes.c_ulonglong),
    "gb_last_error": ([], ctypes.c_char_p),
    "gb_device_count": ([], _I),
    "gb_csr_halfwidth": ([_I, _P, _P, _P, _P], _I),
    "gb_csr_to_box": ([_I, _I, _P, _P, _P, _P, _P, _P], _I),
    "gb_box_scale": ([_L, _I, _I, _P, _P, _P, _P], _I),
    "gb_box_diag_min": ([_L, _I, _I, _P, _P, _P], _I),
    "gb_box_sym_drop": ([_I, _I, _I, _P, _P, _P, _P, _P], _I),
    "gb_row_tail_drop": ([_L, _L, _P, _P], _I),
    "gb_mass_patch_workspace": ([_I, _I], _Z),
    "gb_mass_patches": ([_I, _I, _P, _P, _I, _I, _P, _P, _P, _I, _P], _I),
    "gb_mass_patches_v2": ([_I, _I, _P, _P, _I, _I, _P, _P, _P], _I),
    "gb_correction_patches_workspace": ([_I, _I, _I, _I], _Z),
    "gb_correction_patches_v2": ([_I, _I, _P, _P, _I, _P, _I, _P, _P, _P, _Z, _P], _I),
    "gb_mass_patches_rows": ([_I, _I, _P, _P, _I, _I, _P, _P, _I, _I, _P], _I),
    "gb_correction_patches_rows": ([_I, _I, _P, _P, _I, _P, _I, _P, _P, _I, _I, _P, _Z, _P],
                                   _I),
    "gb_psi_stencil": ([_I, _I, _I, _I, _P, _I, _P, _I, _P, _P], _I),
    "gb_psi_galerkin": ([_I, _I, _I, _I, _P, _I, _P, _I, _P, _P], _I),
    "gb_psi_galerkin_workspace": ([_I, _I, _I], _Z),
    "gb_psi_galerkin_t": ([_I, _I, _I, _I, _P, _I, _P, _I, _P, _P, _P], _I),
    "gb_level_diag": ([_I, _I, _P, _P, _P, _P, _P], _I),
    "gb_level_blocks": ([_I, _I, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P], _I),
    "gb_correction_workspace": ([_I, _I], _Z),
    "gb_correction_patches": ([_I, _I, _P, _P, _I, _P, _I, _P, _P, _P, _I, _P], _I),
    "gb_restriction": ([_I, _I, _P, _P, _P, _P], _I),
    "gb_bd": ([_I, _I, _P, _I, _P, _I, _P, _P], _I),
    "gb_gtd": ([_I, _I, _P, _I, _P, _I, _P, _P], _I),
    "gb_coarse_raw": ([_I, _I, _P, _I, _P, _I, _P, _I, _P, _I, _P, _P], _I),
    "gb_wpsi": ([_I, _I, _I, _I, _P, _P, _I, _P, _P], _I),
    "gb_psi_next": ([_I, _I, _I, _I, _I, _P, _I, _P, _I, _P, _I, _I, _P, _P, _P], _I),
    "gb_psi_next_rows": ([_I, _I, _I, _I, _I, _P, _I, _P, _I, _P, _I, _I, _P, _P, _I, _I, _P],
                         _I),
    "gb_products_mode": ([_I], _I),
    "gb_tune": ([_I, _I], _I),
    "gb_kstate_bytes": ([], _Z),
    "gb_red_blocks": ([], _I),
    "gb_state_reset": ([_P, _I, _P], _I),
    "gb_cg_init": ([_L, _P, _P, _P, _P, _P, _P, _D, _I, _P, _P, _P], _I),
    "gb_cg_iterations": ([_I, _I, _I, _P, _P, _I, _P, _P, _P, _P, _I, _P, _P, _P], _I),
    "gb_pow_iterations": ([_I, _I, _I, _P, _P, _I, _P, _P, _D, _I, _P, _P, _P], _I),
    "gb_scale_box": ([_I, _I, _I, _P, _P, _P, _P], _I),
    "gb_pad": ([_I, _I, _I, _P, _P, _P, _P], _I),
    "gb_unpad": ([_I, _I, _I, _P, _P, _P, _P], _I),
    "gb_pcg_iterations": ([_I, _I, _I, _P, _P, _P, _P, _P, _I, _P, _P, _P], _I),
    "gb_ppow_iterations": ([_I, _I, _I, _P, _P, _P, _D, _I, _P, _P, _P], _I),
    "gb_pbox_apply": ([_I, _I, _I, _P, _P, _P, _P], _I),
    "gb_boxT_elems": ([_I, _I, _I], _Z),
    "gb_scale_box_T": ([_I, _I, _I, _P, _P, _P, _P], _I),
    "gb_tcg_iterations": ([_I, _I, _I, _P, _P, _P, _P, _P, _I, _P, _P, _P, _I], _I),
    "gb_tpow_iterations": ([_I, _I, _I, _P, _P, _P, _D, _I, _P, _P, _P, _I], _I),
    "gb_tbox_apply": ([_I, _I, _I, _P, _P, _P, _P, _I], _I),
    "gb_boxsym_elems": ([_I, _I], _Z),
    "gb_sym_overflow_elems": ([_I, _I], _Z),
    "gb_sym_supported": ([_I, _I, _I], _I),
    "gb_scale_box_symT": ([_I, _I, _P, _P, _P, _P], _I),
    "gb_bj_setup": ([_I, _I, _P, _P, _P, _P], _I),
    "gb_bjcg_init": ([_I, _I, _P, _P, _P, _D, _P, _P, _P, _P, _P, _D, _I, _P, _P, _P], _I),
    "gb_bjcg_iterations": ([_I, _I, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _I], _I),
    "gb_sync_read": ([_P, _P, _Z, _P], _I),
    "gb_tcg_solve": ([_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _I], _I),
    "gb_bjcg_solve": ([_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _I], _I),
    "gb_bjcg_solve2": ([_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P], _I),
    "gb_tpow_solve": ([_I, _I, _I, _P, _P, _P, _D, _P, _P, _P, _I, _P, _I], _I),
    "gb_csr_apply": ([_L, _P, _P, _P, _P, _P, _P], _I),
    "gb_csr_cg_solve": ([_L, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P], _I),
    "gb_csr_pow_solve": ([_L, _P, _P, _P, _P, _P, _D, _P, _P, _P, _I, _P], _I),
    "gb_level_engine": ([_P, _P], _I),
    "gb_cell_energies": ([_I, _P, _P, _P, _P, _P], _I),
    "gb_decay_part_elems": ([_I], _Z),
    "gb_decay_sums": ([_I, _D, _P, _D, _D, _P, _I, _P, _P, _P], _I),
    "gb_box_diag_spectrum": ([_L, _I, _I, _P, _P, _P, _P], _I),
    "gb_topk_mask": ([_L, _P, _L, _P, _P, _P, _P], _I),
    "gb_quad_part_elems": ([], _Z),
    "gb_box_quadform": ([_I, _I, _P, _P, _P, _P, _P], _I),
    "gb_max_abs": ([_L, _P, _P, _P, _P], _I),
    "gb_h2d_staged": ([_P, _P, _L, _I, _P], _I),
    "gb_h2d_staged_i64_i32": ([_P, _P, _L, _I, _P], _I),
    "gb_assemble_q1": ([_I, _P, _D, _P, _P, _P], _I),
    "gb_box1_matvec": ([_I, _P, _P, _P, _P], _I),
    "gb_lanczos_emulate": ([_P, _I, _D, _I, _P, _P, _P, _P], _I),
    "gb_lanczos_check": ([_P, _I, _D, _I, _D, _P, _P, _P], _I),
    "gb_dot2": ([_L, _P, _P, _P, _P, _P, _P, _P], _I),
    "gb_scale_by_norm": ([_L, _P, _P, _I, _P, _P, _P], _I),
    "gb_box_apply": ([_I, _I, _I, _P, _P, _I, _P, _P, _P], _I),
    "gb_apply_w": ([_I, _P, _P, _P, _P, _P], _I),
    "gb_apply_wt": ([_I, _P, _P, _P, _P], _I),
    "gb_apply_r": ([_I, _I, _P, _P, _P, _P], _I),
    "gb_psi_t_apply": ([_I, _I, _I, _I, _P, _P, _P, _P], _I),
    "gb_psi_apply": ([_I, _I, _I, _I, _P, _P, _P, _P], _I),
    "gb_axpby": ([_L, _D, _P, _D, _P, _P, _P], _I),
    "gb_vmul": ([_L, _P, _P, _P, _P], _I),
    "gb_vadd": ([_L, _P, _P, _P, _P], _I),
    "gb_export_count": ([_I, _I, _I, _I, _I, _I, _I, _I, _P, _L, _L, _P, _P], _I),
    "gb_exclusive_scan": ([_P, _P, _L, _P, _P, _P], _I),
    "gb_export_emit": ([_I, _I, _I, _I, _I, _I, _I, _I, _P, _L, _L, _P, _P, _P, _P], _I),
    "gb_dense_gemm": ([_I, _I, _I, _D, _P, _I, _I, _P, _I, _I, _D, _P, _I, _P], _I),
    "gb_dense_potrf": ([_I, _P, _I, _P, _P], _I),
    "gb_dense_potrs": ([_I, _I, _P, _I, _P, _I, _P], _I),
    "gb_dense_sym": ([_I, _P, _I, _P, _P, _P], _I),
    "gb_dense_build_w": ([_I, _P, _P, _P], _I),
    "gb_dense_build_p": ([_I, _P, _D, _P], _I),
    "gb_csr_to_dense": ([_I, _I, _P, _P, _P, _P, _P], _I),
    "gb_eye": ([_I, _P, _P], _I),
    "gb_fp64_peak_probe": ([_I, _I, _P, _P], _I),
    # config 4: 3-D box stencils (csrc/gb_3d.cu)
    "gb3_csr_to_box": ([_I, _I, _P, _P, _P, _P, _P, _P], _I),
    "gb3_box_scale": ([_L, _I, _I, _P, _P, _P, _P], _I),
    "gb3_box_sym_drop": ([_I, _I, _I, _P, _P, _P, _P, _P], _I),
    "gb3_mass_patches": ([_I, _P, _P, _I, _I, _P, _P, _P], _I),
    "gb3_psi_galerkin": ([_I, _I, _I, _P, _P, _I, _P, _I, _P, _P], _I),
    "gb3_level_blocks": ([_I, _I, _P, _P, _I, _P, _P, _P, _P], _I),
    "gb3_correction_workspace": ([_I, _I, _I], _Z),
    "gb3_correction_patches": ([_I, _I, _P, _P, _P, _I, _P, _P, _P, _I, _P], _I),
    "gb3_restriction": ([_I, _I, _P, _P, _P, _P], _I),
    "gb3_triple": ([_I, _I, _P, _P, _P, _I, _P, _I, _P, _I, _P, _I, _P, _P], _I),
    "gb3_apply_w": ([_I, _P, _P, _P, _P, _P], _I),
    "gb3_apply_wt": ([_I, _P, _P, _P, _P], _I),
    "gb3_apply_r": ([_I, _I, _P, _P, _P, _P], _I),
    "gb3_apply_rt": ([_I, _I, _P, _P, _P, _P], _I),
    "gb3_psi_t_apply": ([_I, _I, _I, _P, _P, _P, _P], _I),
    "gb3_apply": ([_I, _I, _I, _P, _P, _P, _P, _P], _I),
    "gb3_cg_solve": ([_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P], _I),
    "gb3_lanczos_min": ([_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _D, _I, _D,
                         _P, _P, _P, _P], _I),
    "gb3_pow_solve": ([_I, _I, _I, _P, _P, _P, _P, _D, _P, _P, _P, _I, _P], _I),
    # row strips and the distributed Krylov pieces (multi-GPU partition)
    "gb_psi_galerkin_workspace_rows": ([_I, _I, _I, _I, _I, _I], _Z),
    "gb_csr_to_box_rows": ([_I, _I, _P, _P, _P, _P, _P, _I, _I, _P], _I),
    "gb_box_sym_drop_rows": ([_I, _I, _I, _P, _P, _P, _P, _I, _I, _P], _I),
    "gb_psi_stencil_rows": ([_I, _I, _I, _I, _P, _I, _P, _I, _P, _I, _I, _P], _I),
    "gb_psi_galerkin_t_rows": ([_I, _I, _I, _I, _P, _I, _P, _I, _P, _P, _I, _I, _P], _I),
    "gb_level_diag_rows": ([_I, _I, _P, _P, _P, _P, _I, _I, _P], _I),
    "gb_level_blocks_rows": ([_I, _I, _P, _P, _I, _P, _P, _P, _P, _P, _P, _I, _I, _P], _I),
    "gb_restriction_rows": ([_I, _I, _P, _P, _P, _I, _I, _P], _I),
    "gb_bd_rows": ([_I, _I, _P, _I, _P, _I, _P, _I, _I, _P], _I),
    "gb_gtd_rows": ([_I, _I, _P, _I, _P, _I, _P, _I, _I, _P], _I),
    "gb_coarse_raw_rows": ([_I, _I, _P, _I, _P, _I, _P, _I, _P, _I, _P, _I, _I, _P], _I),
    "gb_wpsi_rows": ([_I, _I, _I, _I, _P, _P, _I, _P, _I, _I, _I, _I, _P], _I),
    "gb_psi_next_raw_rows": ([_I, _I, _I, _I, _I, _P, _I, _P, _I, _P, _I, _I, _P, _P, _I, _I, _I, _I, _P], _I),
    "gb_psi_drop_rows": ([_I, _I, _I, _I, _P, _P, _I, _I, _I, _I, _P], _I),
    "gb_pad_rows": ([_I, _I, _I, _P, _P, _P, _I, _I, _P], _I),
    "gb_unpad_rows": ([_I, _I, _I, _P, _P, _P, _I, _I, _P], _I),
    "gb_apply_w_rows": ([_I, _P, _P, _P, _P, _I, _I, _P], _I),
    "gb_apply_wt_rows": ([_I, _P, _P, _P, _I, _I, _P], _I),
    "gb_apply_r_rows": ([_I, _I, _P, _P, _P, _I, _I, _P], _I),
    "gb_psi_t_apply_rows": ([_I, _I, _I, _I, _P, _P, _P, _I, _I, _I, _I, _P], _I),
    "gb_bj_setup_rows": ([_I, _I, _P, _P, _P, _I, _I, _P], _I),
    "gb_scale_box_symT_rows": ([_I, _I, _P, _P, _P, _I, _I, _P], _I),
    "gb_dist_apply": ([_I, _I, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P], _I),
    "gb_dist_pcg_init": ([_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P], _I),
    "gb_dist_pcg_init_commit": ([_P, _P, _D, _I, _P], _I),
    "gb_dist_pcg_update": ([_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P], _I),
    "gb_dist_pcg_commit_dir": ([_I, _I, _P, _P, _P, _P, _P, _I, _I, _P], _I),
    "gb_dist_fix_yy": ([_I, _I, _P, _P, _P, _P, _I, _I, _P], _I),
    "gb_dist_pow_step": ([_I, _I, _P, _P, _P, _P, _P, _P, _P, _D, _I, _I, _I, _P], _I),
    "gb_dist_lz_update": ([_I, _I, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P], _I),
    "gb_dist_lz_commit": ([_P, _P, _P, _P, _P], _I),
    "gb_dist_lz_begin": ([_P, _I, _P], _I),
    "gb_dist_dot": ([_L, _P, _P, _P, _P, _P, _P], _I),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path=None):
    """Load (once) and return the ctypes library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    import os
    # GB_LIB: an alternative build of the same library (tools/build_variant.sh)
    p = Path(path) if path else Path(os.environ.get("GB_LIB", LIB_PATH))
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = ctypes.CDLL(str(p), mode=ctypes.RTLD_GLOBAL)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def last_error():
    msg = load().gb_last_error()
    return msg.decode() if msg else ""


def call(name, *args):
    """Invoke one C entry point and map its status to the API exceptions."""
    rc = getattr(load(), name)(*args)
    if rc == 0:
        return 0
    if rc == 1:
        raise InvalidArgumentError(f"{name}: {last_error()}")
    if rc == 2:
        raise NumericalError(f"{name}: {last_error()}")
    raise RuntimeError(f"{name} failed: {last_error()}")


def query(name, *args):
    """Entry points that return a value instead of a status."""
    return getattr(load(), name)(*args)
