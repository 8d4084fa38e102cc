"""ctypes binding of libhga.so (the C ABI declared in include/hga.h).

This is the only way the package reaches the GPU.  There is no CPU
fallback: if the shared library is missing or a CUDA device is absent, the
calls that need it raise instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libhga.so"
if os.environ.get("HGA_LIB_VARIANT"):  # experiments: an A/B build next to the product library
    LIB_PATH = HERE / f"libhga_{os.environ['HGA_LIB_VARIANT']}.so"

# return codes / flags (include/hga.h)
HGA_OK = 0
HGA_E_INVALID = 1
HGA_E_UNSUPPORTED = 2
HGA_E_WORKSPACE = 3
HGA_E_CUDA_BASE = 1000

VAR_F1, VAR_F2, VAR_ORTH, VAR_SQ = 1, 2, 4, 8
VAR_ALL = 15
VARIANT_BITS = {"f1": VAR_F1, "f2": VAR_F2, "orth": VAR_ORTH, "sq": VAR_SQ}

FLAG_NOT_SIGN, FLAG_POINT_RANGE, FLAG_PLAN_RANGE, FLAG_FIT_RANGE, FLAG_NOT_GA = 1, 2, 4, 8, 16

RUN_FORCE = 1
RUN_TIMING = 2
RUN_ONE_BARRIER = 4  # HGA_RUN_ONE_BARRIER: opt-in one-barrier generation loop (identical runs)

MUT_CODES = {"shared": 0, "per-matrix": 1, "multi": 2}

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_u32 = ctypes.c_uint32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_sz = ctypes.c_size_t
_int = ctypes.c_int


class RunArgs(ctypes.Structure):
    """Mirror of `hga_run_args` (include/hga.h)."""

    _fields_ = [
        ("pop", _vp * 2),
        ("fit", _vp * 2),
        ("n_pairs", _i64),
        ("m", _i32),
        ("nc", _i32),
        ("nr", _i32),
        ("strategy", _i32),
        ("fit_var", _u32),
        ("stall_window", _i32),
        ("seed", _u64),
        ("max_generation", _i64),
        ("gens_this_call", _i64),
        ("state", _vp),
        ("trace", _vp),
        ("trace_capacity", _i64),
        ("best_matrix", _vp),
        ("ws", _vp),
        ("ws_bytes", _sz),
        ("flags", _u32),
    ]


# name -> (restype, argtypes); every symbol include/hga.h declares.
SIGNATURES = {
    "hga_abi_version": (_int, []),
    "hga_probe": (_int, [_i32, _i64, _i32, _i32, _vp, _vp]),
    "hga_strerror": (ctypes.c_char_p, [_int]),
    "hga_sm_count": (_int, [_int]),
    "hga_clear_last_error": (_int, []),
    "hga_fitness_i8_ws_bytes": (_sz, [_i64, _i32]),
    "hga_fitness_i8": (_int, [_vp, _i64, _i32, _u32, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "hga_fitness_packed": (_int, [_vp, _i64, _i32, _u32, _vp, _vp, _vp, _vp, _vp]),
    "hga_pack_i8": (_int, [_vp, _i64, _i32, _vp, _vp, _vp]),
    "hga_unpack_i8": (_int, [_vp, _i64, _i32, _vp, _vp]),
    "hga_ref_words": (_int, [_u64, _u64, _u64, _i64, _vp, _vp]),
    "hga_ref_uniform": (_int, [_u64, _u64, _u64, _i64, _i64, _i64, _vp, _vp]),
    "hga_ref_permutation_ws_bytes": (_sz, [_i64]),
    "hga_ref_permutation": (_int, [_u64, _u64, _u64, _i64, _vp, _vp, _sz, _vp]),
    "hga_ref_init_packed": (_int, [_u64, _u64, _u64, _i64, _i64, _i32, _vp, _vp]),
    "hga_ref_init_i8": (_int, [_u64, _u64, _u64, _i64, _i64, _i32, _vp, _vp]),
    "hga_crossover_i8": (_int, [_vp, _i64, _i32, _vp, _vp, _vp]),
    "hga_mutate_i8": (_int, [_vp, _i64, _i32, _vp, _vp, _vp, _i32, _i32, _vp, _vp]),
    "hga_select_max_range": (_i64, []),
    "hga_select_ws_bytes": (_sz, [_i64]),
    "hga_select_radix_ws_bytes": (_sz, [_i64]),
    "hga_select_smallest_radix": (_int, [_vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    "hga_select_order": (_int, [_vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "hga_select_smallest": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "hga_compose_gather": (_int, [_vp, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "hga_generation_explicit": (_int, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _i32, _i32, _u32, _vp, _vp]),
    "hga_argmin_key": (_int, [_vp, _i64, _vp, _int, _vp]),
    "hga_check_invariants_ws_bytes": (_sz, [_i64]),
    "hga_check_invariants": (_int, [_vp, _vp, _i64, _i32, _u32, _vp, _vp, _sz, _vp]),
    "hga_philox_init_packed": (_int, [_u64, _u64, _u64, _i64, _i64, _i32, _vp, _vp]),
    "hga_run_ws_bytes": (_sz, [_i64, _i32]),
    "hga_run_timing_offset": (_i64, [_i32]),
    "hga_run_init": (_int, [ctypes.POINTER(RunArgs), _vp]),
    "hga_run_prepare": (_int, [ctypes.POINTER(RunArgs), _vp]),
    "hga_run": (_int, [ctypes.POINTER(RunArgs), _vp]),
    "hga_step_host": (_int, [ctypes.POINTER(RunArgs), _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int32, _vp, _vp]),
    "hga_bits_to_cols": (_int, [_vp, ctypes.c_int64, ctypes.c_int32, _vp, _vp, _vp]),
    "hga_cols_to_bits": (_int, [_vp, ctypes.c_int64, ctypes.c_int32, _vp, _vp]),
    "hga_host_pack_bits": (_int, [_vp, ctypes.c_int64, _vp]),
    "hga_host_unpack_bits": (None, [_vp, ctypes.c_int64, _vp]),
    "hga_step_host_bits_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int32]),
    "hga_step_host_bits": (_int, [ctypes.POINTER(RunArgs), _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int32, _vp,
                                  _vp]),
}


class HgaError(RuntimeError):
    pass


class _Lib:
    def __init__(self) -> None:
        self._dll = None

    def dll(self) -> ctypes.CDLL:
        if self._dll is None:
            if not LIB_PATH.exists():
                raise HgaError(
                    f"{LIB_PATH} is missing: build it with `make -C {HERE}` (or __graft_entry__.build()); "
                    "there is no CPU fallback")
            dll = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                if os.environ.get("HGA_LIB_VARIANT") and not hasattr(dll, name):
                    continue  # fitness-only A/B build
                fn = getattr(dll, name)
                fn.restype = res
                fn.argtypes = args
            self._dll = dll
        return self._dll

    def __getattr__(self, name: str):
        if not name.startswith("hga_"):
            raise AttributeError(name)
        return getattr(self.dll(), name)


lib = _Lib()


def check(rc: int, what: str = "") -> None:
    if rc != HGA_OK:
        msg = lib.hga_strerror(rc).decode()
        raise HgaError(f"{what or 'libhga'} failed: {msg} (rc={rc})")
