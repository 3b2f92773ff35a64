"""ctypes binding of csrc/libckks_b200.so (C ABI: include/ckks_b200.h).

There is no CPU fallback: if the shared library is missing the import of any
device operation raises, and ``ckks_ctx_create`` itself fails without a CUDA
device.
"""
from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

CSRC = Path(__file__).resolve().parent / "csrc"
LIB_PATH = CSRC / "libckks_b200.so"

ABI_VERSION = 1

# every symbol include/ckks_b200.h declares (checked by tests/test_abi.py)
SYMBOLS = (
    "ckks_abi_version", "ckks_last_error", "ckks_profile_enable", "ckks_profile_read", "ckks_ctx_create", "ckks_ctx_destroy", "ckks_set_lanes", "ckks_select_lane", "ckks_arena_generation", "ckks_arena_reserve",
    "ckks_modulus_register", "ckks_modulus_register_tables", "ckks_modulus_tables", "ckks_ntt", "ckks_ntt_policy", "ckks_ntt_stages",
    "ckks_elementwise", "ckks_automorphism_eval", "ckks_automorphism_coeff", "ckks_lift2_centered", "ckks_pmult_accumulate", "ckks_fused_terms", "ckks_fused_terms_halves", "ckks_fused_terms_multi", "ckks_tensor", "ckks_tensor_halves",
    "ckks_bconv_table_create", "ckks_bconv_table_read", "ckks_bconv",
    "ckks_ks_plan_create", "ckks_moddown_plan_create", "ckks_ks_stage1", "ckks_ks_stage2", "ckks_ks_stage3", "ckks_ks_stage3_batch", "ckks_ks_stage3_batch_a", "ckks_keyswitch", "ckks_ks_hoisted", "ckks_ks_hoisted_raw", "ckks_bsgs_inner", "ckks_bsgs_inner_batch", "ckks_ks_relin_rescale", "ckks_hmult_relin_rescale", "ckks_ks_accumulate", "ckks_ks_accumulate_rot", "ckks_ks_accumulate_rot_qp", "ckks_ks_finish", "ckks_ks_finish_rescale",
)


class EngineUnavailable(RuntimeError):
    """libckks_b200.so is not built, or no CUDA device is present."""


def build(verbose: bool = False) -> Path:
    """Compile the library in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    proc = subprocess.run(["make", "-C", str(CSRC), "-j8", "libckks_b200.so"],
                          capture_output=True, text=True)
    if verbose or proc.returncode:
        print(proc.stdout[-4000:])
        print(proc.stderr[-4000:])
    if proc.returncode:
        raise RuntimeError("building libckks_b200.so failed")
    return LIB_PATH


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise EngineUnavailable(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    L = ctypes.CDLL(str(LIB_PATH))
    vp, i32, u32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_size_t
    pi32, pu32 = ctypes.POINTER(i32), ctypes.POINTER(u32)
    L.ckks_abi_version.restype = ctypes.c_int
    L.ckks_last_error.restype = ctypes.c_char_p
    L.ckks_profile_enable.argtypes = [ctypes.c_int]
    L.ckks_profile_read.argtypes = [ctypes.c_char_p, sz]
    L.ckks_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
    L.ckks_ctx_destroy.argtypes = [vp]
    L.ckks_ctx_destroy.restype = None
    L.ckks_set_lanes.argtypes = [vp, ctypes.c_int]
    L.ckks_select_lane.argtypes = [vp, ctypes.c_int]
    L.ckks_arena_generation.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64)]
    L.ckks_arena_reserve.argtypes = [vp, sz]
    L.ckks_modulus_register.argtypes = [vp, u32, u32, u32, pi32]
    L.ckks_modulus_register_tables.argtypes = [vp, u32, u32, vp, vp, u32, pi32]
    L.ckks_modulus_tables.argtypes = [vp, i32, vp, vp, pu32]
    L.ckks_ntt.argtypes = [vp, vp, vp, vp, ctypes.c_int, u32, ctypes.c_int, vp]
    L.ckks_ntt_policy.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp]
    L.ckks_ntt_stages.argtypes = [vp, vp, vp, vp, ctypes.c_int, u32, ctypes.c_int, u32, u32, vp]
    L.ckks_elementwise.argtypes = [vp, vp, vp, vp, vp, ctypes.c_int, sz, ctypes.c_int, vp]
    L.ckks_automorphism_eval.argtypes = [vp, vp, vp, ctypes.c_int, u32, u32, vp]
    L.ckks_automorphism_coeff.argtypes = [vp, vp, vp, vp, ctypes.c_int, u32, u32, vp]
    L.ckks_lift2_centered.argtypes = [vp, vp, i32, i32, vp, vp, ctypes.c_int, sz, vp]
    L.ckks_pmult_accumulate.argtypes = [vp, vp, vp, vp, vp, ctypes.c_int, sz, ctypes.c_int, vp]
    L.ckks_fused_terms.argtypes = [vp, ctypes.c_int, vp, vp, vp, vp, ctypes.c_int, sz, vp]
    L.ckks_fused_terms_halves.argtypes = [vp, ctypes.c_int, vp, vp, vp, vp, vp, ctypes.c_int, sz, vp]
    L.ckks_fused_terms_multi.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp, ctypes.c_int, sz, vp]
    L.ckks_tensor.argtypes = [vp, vp, vp, vp, vp, ctypes.c_int, sz, vp]
    L.ckks_tensor_halves.argtypes = [vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, sz, vp]
    L.ckks_bconv_table_create.argtypes = [vp, vp, ctypes.c_int, vp, ctypes.c_int, pi32]
    L.ckks_bconv_table_read.argtypes = [vp, i32, vp, vp]
    L.ckks_bconv.argtypes = [vp, i32, vp, vp, sz, vp]
    L.ckks_ks_plan_create.argtypes = [vp, u32, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int,
                                      ctypes.c_int, pi32]
    L.ckks_moddown_plan_create.argtypes = [vp, u32, ctypes.c_int, ctypes.c_int, vp, vp, pi32]
    L.ckks_ks_stage1.argtypes = [vp, i32, vp, vp, vp]
    L.ckks_ks_stage2.argtypes = [vp, i32, vp, vp, ctypes.c_int, ctypes.c_int, vp, vp, vp]
    L.ckks_ks_stage3.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp]
    L.ckks_keyswitch.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp]
    L.ckks_ks_hoisted.argtypes = [vp, i32, vp, u32, vp, vp, vp, vp, vp]
    L.ckks_ks_hoisted_raw.argtypes = [vp, i32, vp, u32, vp, vp, vp, vp]
    L.ckks_ks_relin_rescale.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, vp, vp]
    L.ckks_ks_stage3_batch.argtypes = [vp, i32, ctypes.c_int, vp, vp, vp]
    L.ckks_ks_stage3_batch_a.argtypes = [vp, i32, ctypes.c_int, vp, vp, vp]
    L.ckks_hmult_relin_rescale.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.ckks_bsgs_inner.argtypes = [vp, i32, vp, vp, vp, ctypes.c_int, vp, vp, ctypes.c_int, vp, vp, vp, vp]
    L.ckks_bsgs_inner_batch.argtypes = [vp, i32, ctypes.c_int, vp, vp, vp, ctypes.c_int, vp, vp, ctypes.c_int, vp, vp, vp, vp]
    L.ckks_ks_accumulate.argtypes = [vp, i32, vp, vp, ctypes.c_int, vp]
    L.ckks_ks_accumulate_rot.argtypes = [vp, i32, vp, vp, ctypes.c_uint32, vp, ctypes.c_int, vp]
    L.ckks_ks_accumulate_rot_qp.argtypes = [vp, i32, vp, vp, ctypes.c_uint32, vp, ctypes.c_int, vp]
    L.ckks_ks_finish.argtypes = [vp, i32, ctypes.c_int, vp, vp, vp, vp, vp]
    L.ckks_ks_finish_rescale.argtypes = [vp, i32, i32, ctypes.c_int, vp, vp, vp, vp, vp, vp]
    for name in SYMBOLS:
        fn = getattr(L, name)
        if name not in ("ckks_last_error", "ckks_ctx_destroy"):
            fn.restype = ctypes.c_int
    if L.ckks_abi_version() != ABI_VERSION:
        raise EngineUnavailable(
            f"libckks_b200.so has ABI {L.ckks_abi_version()}, binding expects {ABI_VERSION}: rebuild"
        )
    _lib = L
    return L


def check(status: int) -> None:
    if status:
        msg = load().ckks_last_error().decode("utf-8", "replace")
        if status == 3:
            raise NotImplementedError(msg)
        if status == 1:
            raise ValueError(msg)
        raise RuntimeError(f"libckks_b200 error {status}: {msg}")
