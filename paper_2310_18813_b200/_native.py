"""ctypes binding of the C-ABI in ``include/specbatch_b200.h``.

This is the only bridge between the Python host and the sm_100a kernels.
There is no fallback: if ``libspecbatch_b200.so`` is missing or fails to load,
every engine entry point raises :class:`NativeError` instead of silently
computing on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import NativeError

LIB_PATH = Path(__file__).resolve().parent / "libspecbatch_b200.so"

SB_EINVAL = 1001
SB_EWORKSPACE = 1002
SB_EUNSUPPORTED = 1003

SB_BF16, SB_F32 = 0, 1
ARCH_LLAMA, ARCH_OPT = 0, 1
LOGITS_ALL, LOGITS_LAST, LOGITS_NONE = 0, 1, 2
ACCEPT_GREEDY, ACCEPT_STOCHASTIC, ACCEPT_INJECTED = 0, 1, 2
SELECT_ARGMAX, SELECT_SAMPLE = 0, 1
EPI_STORE, EPI_STORE_F32, EPI_RESID_ADD, EPI_SILU_MUL = 0, 1, 2, 3
GEMM_AUTO, GEMM_SIMT, GEMM_TC, GEMM_SMALL = 0, 1, 2, 3

_P = C.c_void_p
_I = C.c_int32
_PP = C.POINTER(C.c_void_p)


_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p)
_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p)


class SbCollectives(C.Structure):
    """Mirror of ``sb_collectives_t`` (tensor-parallel exchange of a sharded target)."""

    _fields_ = [("ctx", _P), ("all_reduce_sum", _ALLREDUCE_FN), ("all_gather", _ALLGATHER_FN), ("world", _I),
                ("rank", _I)]


class SbDecoder(C.Structure):
    """Mirror of ``sb_decoder_t``."""

    _fields_ = [
        ("n_layers", _I), ("hidden", _I), ("n_heads", _I), ("n_kv_heads", _I), ("head_dim", _I),
        ("ffn", _I), ("vocab", _I), ("dtype", _I), ("max_pos", _I), ("rms_eps", C.c_float),
        ("embed", _P), ("final_norm", _P), ("lm_head", _P),
        ("attn_norm", _PP), ("w_qkv", _PP), ("w_o", _PP), ("mlp_norm", _PP), ("w_gu", _PP), ("w_down", _PP),
        ("rope_cos", _P), ("rope_sin", _P), ("tp", C.POINTER(SbCollectives)),
        ("arch", _I), ("pos_offset", _I), ("pos_embed", _P), ("final_norm_b", _P), ("attn_norm_b", _PP),
        ("mlp_norm_b", _PP), ("b_qkv", _PP), ("b_o", _PP), ("b_fc1", _PP), ("b_fc2", _PP),
        ("ln_qkv_c1", _PP), ("ln_qkv_c2", _PP), ("ln_fc1_c1", _PP), ("ln_fc1_c2", _PP), ("ln_lm_c1", _P),
        ("ln_lm_c2", _P), ("role", _I),
    ]


class SbTokenSink(C.Structure):
    """Mirror of ``sb_token_sink_t`` (greedy argmax fused into the lm_head epilogue)."""

    _fields_ = [("out_tok", _P), ("out_stride", _I), ("next_ids", _P), ("next_pos", _P), ("base_pos", _P),
                ("pos_offset", _I)]


class SbKVCache(C.Structure):
    """Mirror of ``sb_kvcache_t``."""

    _fields_ = [("k", _P), ("v", _P), ("slots", _I), ("ctx_max", _I)]


# name -> (restype, argtypes)
_SIGS = {
    "sb_init": (C.c_int, []),
    "sb_set_gemm_backend": (C.c_int, [_I]),
    "sb_set_pdl": (C.c_int, [_I]),
    "sb_set_fuse_norm": (C.c_int, [_I]),
    "sb_set_small_gemm": (C.c_int, [_I]),
    "sb_debug_skip": (C.c_int, [_I]),
    "sb_debug_cta_trace": (C.c_int, [_P]),
    "sb_debug_gemm_pdl": (C.c_int, [_I, _I, _I]),
    "sb_set_attention_impl": (C.c_int, [_I]),
    "sb_set_attention_splits": (C.c_int, [_I]),
    "sb_set_draft_loop": (C.c_int, [_I]),
    "sb_draft_loop": (C.c_int, [C.POINTER(SbDecoder), C.POINTER(SbKVCache), _P, _I, _I, _P, _P, _P, _P, _P, _P, _P,
                                _P, C.c_size_t, _P, _P]),
    "sb_draft_loop_packed_bytes": (C.c_size_t, [C.POINTER(SbDecoder)]),
    "sb_draft_loop_pack": (C.c_int, [C.POINTER(SbDecoder), _P, C.c_size_t, _P]),
    "sb_draft_loop_workspace_bytes": (C.c_size_t, [C.POINTER(SbDecoder)]),
    "sb_debug_draft_trace": (C.c_int, [_P]),
    "sb_nccl_unique_id": (C.c_int, [_P]),
    "sb_nccl_collectives_init": (C.c_int, [_P, _I, _I, C.POINTER(SbCollectives)]),
    "sb_nccl_collectives_destroy": (C.c_int, [C.POINTER(SbCollectives)]),
    "sb_gemm_tune": (C.c_int, [_I, _I, _I]),
    "sb_gemm_autotune": (C.c_int, [_P, _P, _P, _I, _I, _I, _P, C.POINTER(_I), C.POINTER(_I), C.POINTER(C.c_float)]),
    "sb_gemm_autotune_clear": (C.c_int, []),
    "sb_set_weight_l2_hint": (C.c_int, [_I]),
    "sb_gemm_tune_get": (C.c_int, [_I, _I, _I, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    "sb_gemm_tune_set": (C.c_int, [_I, _I, _I, _I, _I, _I, _I]),
    "sb_profile_forward": (C.c_int, [C.POINTER(SbDecoder), C.POINTER(SbKVCache), _P, _P, _P, _I, _I, _P, _I, _P,
                                     C.c_size_t, _P, C.c_char_p, _I]),
    "sb_version": (C.c_int, []),
    "sb_build_info": (C.c_char_p, []),
    "sb_last_kernel_count": (C.c_int, []),
    "sb_decoder_workspace_bytes": (C.c_size_t, [C.POINTER(SbDecoder), _I]),
    "sb_decoder_forward": (C.c_int, [C.POINTER(SbDecoder), C.POINTER(SbKVCache), _P, _P, _P, _I, _I, _P, _I, _P,
                                     C.c_size_t, _P]),
    "sb_decoder_forward_ex": (C.c_int, [C.POINTER(SbDecoder), C.POINTER(SbKVCache), _P, _P, _P, _I, _I, _P, _I,
                                        C.POINTER(SbTokenSink), _P, C.c_size_t, _P]),
    "sb_decoder_forward_mixed": (C.c_int, [C.POINTER(SbDecoder), C.POINTER(SbKVCache), _P, _P, _P, _I, _I, _I, _I,
                                           _P, _P, _I, C.POINTER(SbTokenSink), _P, C.c_size_t, _P]),
    "sb_select_tokens": (C.c_int, [_P, _I, _I, _I, _P, _I, _P, C.c_int64, _P, _I, _P, _P, _P, _I, _P]),
    "sb_softmax_rows": (C.c_int, [_P, _I, _I, _P, _P]),
    "sb_argmax_rows": (C.c_int, [_P, _I, _I, _P, _P]),
    "sb_accept": (C.c_int, [_I, _I, _I, _I, _P, _P, _P, _P, _I, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P]),
    "sb_kv_commit": (C.c_int, [_I, _I, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _I, _P]),
    "sb_prepare_iteration": (C.c_int, [_I, _I, _P, _I, _P, _P, _P, _P, _P, _P, C.c_uint64, _P, _P, _I, _P, _I, _P,
                                       _P]),
    "sb_kv_compact": (C.c_int, [C.POINTER(SbDecoder), C.POINTER(SbKVCache), _P, _P, _P, _I, _P]),
    "sb_gemm": (C.c_int, [_I, _P, _P, _P, _I, _I, _I, _I, _I, _P, C.c_size_t, _P]),
    "sb_gemm_workspace_bytes": (C.c_size_t, [_I, _I, _I]),
    "sb_uniform_host": (C.c_float, [C.c_uint64, C.c_uint64, C.c_uint64]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_load_error: Exception | None = None


def load(path: Path | None = None):
    """Load (once) and type the library.  Raises NativeError when unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    # SB_LIB: an alternative build of the same ABI (A/B timing of kernel variants)
    p = Path(path) if path else Path(os.environ["SB_LIB"]) if os.environ.get("SB_LIB") else LIB_PATH
    if not p.exists():
        raise NativeError("load", -1, f"{p} not built; run `python -m paper_2310_18813_b200.build` "
                                      "(or __graft_entry__.build())")
    try:
        lib = C.CDLL(str(p), mode=C.RTLD_GLOBAL)
    except OSError as exc:  # pragma: no cover - environment dependent
        _load_error = exc
        raise NativeError("load", -1, str(exc)) from exc
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def init_device() -> None:
    """Host-side one-time setup that must precede CUDA graph capture."""
    call("sb_init")


def check(name: str, rc: int) -> None:
    if rc == 0:
        return
    if rc in (SB_EINVAL, SB_EWORKSPACE):
        raise ValueError(f"{name}: invalid argument (status {rc})")
    raise NativeError(name, rc, "unsupported configuration" if rc == SB_EUNSUPPORTED else "CUDA error")


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point and map errors like the reference
    (contract violations -> ValueError, device failures -> RuntimeError)."""
    lib = load()
    check(name, getattr(lib, name)(*args))


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()
