"""ctypes binding of libmoeb.so (include/moeb.h) -- the only compute path.

There is no CPU fallback: if the library is missing or no sm_100 GPU is
visible, every entry point raises ``NativeUnavailable`` (a RuntimeError).
Tensors are torch CUDA tensors used purely as device memory; masks are
stored in int64 tensors holding the uint64 bit patterns.
"""

from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# MOEB_LIB: another in-tree build of the same library (A/B measurements)
LIB_PATH = os.environ.get("MOEB_LIB") or os.path.join(_PKG, "libmoeb.so")

_lib = None
_checked = False


class NativeUnavailable(RuntimeError):
    """libmoeb.so is not built or cannot run on this machine."""


class NativeError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed (code {code}): {msg}")
        self.code = code


P = ctypes.c_void_p
I32, I64, DBL, SZ = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t

_SIGS = {
    "moeb_cache_sim": [P, P, P, P, I32, P, I32, I32, I32, I32, P, I32, I32, I32, P, P, P, I64, P,
                       ctypes.c_size_t, P],
    "moeb_cache_replay_stack": [P, P, P, I32, P, I32, I32, I32, I32, P, I32, I32, I64, I32, P, P,
                                P, SZ, P],
    "moeb_cache_sim_counted": [P, P, P, P, I32, P, I32, I32, I32, I32, P, I32, I32, I32, P, P, P,
                               P, I64, P, ctypes.c_size_t, P],
    "moeb_cache_ops": [P, P, I64, I32, I32, I64, I32, P, P],
    "moeb_linear_predict": [P, P, I32, I32, I32, P, DBL, I32, I32, I32, P, P, P, P],
    "moeb_linear_predict_counts": [P, P, I32, I32, I32, P, DBL, I32, I32, I32, I32, P, P, P, P,
                                   I64, P, ctypes.c_size_t, P],
    "moeb_ids_to_masks": [P, I64, I32, I32, P, P, P],
    "moeb_masks_to_ids": [P, I64, I32, P, P, P],
    "moeb_ranks_to_masks": [P, I64, I32, I32, P, P, P],
    "moeb_masks_to_ranks": [P, I64, I32, I32, P, P, P],
    "moeb_packed_ranks_to_masks": [P, I64, I32, I32, I32, P, P, P],
    "moeb_ids6_to_masks": [P, I64, I32, P, P, P],
    "moeb_idpairs_to_masks": [P, I64, I32, P, P, P],
    "moeb_masks_to_idpairs": [P, I64, I32, P, P, P],
    "moeb_masks_to_ids6": [P, I64, I32, P, P, P],
    "moeb_masks_to_packed_ranks": [P, I64, I32, I32, I32, P, P, P],
    "moeb_mask_head": [P, I64, I32, I32, I32, P, P],
    "moeb_metrics": [P, P, P, I32, I32, I32, I32, P, P],
    "moeb_policy_masks": [I32, P, I64, I32, I32, I32, P, P, P],
    "moeb_gen_traces": [P, P, I32, I32, I32, I32, I32, I32, DBL, P, P],
    "moeb_eam_prepare": [P, I32, I32, I32, I32, P, P, P],
    "moeb_eam_predict": [P, P, I32, I32, I32, I32, P, P, I32, P, P, P],
    "moeb_ream_counts": [P, P, I32, I32, I32, I32, P, P],
    "moeb_sketch_normalize": [P, I32, I32, I32, I32, P, P],
    "moeb_match_queries": [P, I32, I32, P, I32, P, P, P],
    "moeb_gemm": [P, I32, P, I32, I32, I32, I32, I32, I32, P, P, P, I32, P, P,
                  ctypes.c_float, P],
    "moeb_window_attention": [P, P, P, P, I32, I32, I64, I32, P],
    "moeb_embed_rows": [P, P, P, I32, I64, P, P, I32, P],
    "moeb_to16": [P, P, I64, I32, P],
    "moeb_layernorm_rows": [P, P, P, P, I64, ctypes.c_float, I32, P],
    "moeb_layernorm_rows16": [P, P, P, I64, ctypes.c_float, I32, P],
    "moeb_transpose16": [P, I64, I32, I32, P, I32, P],
    "moeb_colsum16": [P, I64, I32, I32, P, I32, P],
    "moeb_layernorm_bwd16": [P, P, P, I64, ctypes.c_float, P, P, P, I32, P],
    "moeb_relu_bwd16": [P, P, I64, I32, P],
    "moeb_gelu_fwd16": [P, P, I64, I32, P],
    "moeb_gelu_bwd16": [P, P, I64, I32, P],
    "moeb_bce_logits_grad": [P, P, I64, I32, ctypes.c_float, P, P, I32, P],
    "moeb_attention_bwd": [P, P, P, P, P, I32, I32, P, P, P, I32, P],
    "moeb_gather_inputs16": [P, P, P, P, I64, P, P],
    "moeb_layer_emb_grad": [P, I32, I64, P, I32, P, I32, P],
    "moeb_cast_f32_to_16": [P, I64, P, I32, P],
    "moeb_sumsq_f32": [P, I64, P, P],
    "moeb_adamw_f32": [P, P, P, P, I64, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                       ctypes.c_float, ctypes.c_float, I32, ctypes.c_float, P],
    "moeb_eam_pack_library": [P, I32, I32, I32, P, P, P],
    "moeb_eam_pack_queries": [P, I32, I32, P, P],
    "moeb_eam_rerank": [P, P, I32, P, P, P, I32, I32, I32, DBL, P, P, P, P],
    "moeb_token_prefix_counts": [P, P, P, I32, I32, I32, I32, P, P],
    "moeb_count_bytes": [P, I64, I32, P, P, P],
    "moeb_find_bytes": [P, I64, I32, P, P, P],
    "moeb_parse_trace_csv": [P, I64, P, I64, I64, I64, I32, I32, I32, P, P, P, P, P, P, P, P, P],
    "moeb_parse_predictions": [P, I64, P, I64, I64, I32, I32, P, P, P, P, P, P, P],
    "moeb_first_status": [P, I64, I32, P, P],
    "moeb_keys_check": [P, P, P, P, I32, I64, P, P],
    "moeb_prompt_flags": [P, I64, P, P],
    "moeb_check_grid": [P, I64, I64, P, P, I32, P, P],
    "moeb_predictions_join": [P, P, P, P, I64, P, P, I32, I64, I32, I32, P, P, P],
    "moeb_trace_csv_lengths": [P, P, P, I32, I64, I32, I32, P, P, P],
    "moeb_trace_csv_write": [P, P, P, I32, I64, I32, I32, P, P, P, P],
    "moeb_predictions_jsonl_lengths": [P, P, P, P, I64, I32, P, P],
    "moeb_predictions_jsonl_write": [P, P, P, P, I64, I32, P, P, P],
    "moeb_exclusive_scan_i64": [P, I64, P, P, P],
    "moeb_row_sqnorms": [P, I64, I64, P, P],
    "moeb_sqdist_argmin": [P, P, P, P, I64, I32, I64, P, P, P],
    "moeb_sqdist_update": [P, P, P, P, I64, I64, I32, P, P],
    "moeb_cluster_means": [P, P, P, I32, I64, P, P],
    "moeb_linear_prepare": [P, I32, I32, DBL, P, P],
    "moeb_linear_ambiguous_rows": [P, I32, P, P],
    "moeb_linear_predict_wide": [P, P, I32, I32, I32, P, DBL, I32, I32, I32, P, P, P, P],
    "moeb_linear_features": [P, P, I32, I32, I32, DBL, P, P],
    "moeb_linear_sgd_epoch": [P, P, P, P, I64, I32, I32, DBL, P, P],
    "moeb_version": [],
    "moeb_device_check": [],
}

SIZE_QUERIES = {
    "moeb_linear_table_doubles": [I32, I32],
    "moeb_cache_sim_workspace_bytes": [I32, I32],
    "moeb_cache_sim_workspace_bytes_shape": [I32, I32, I32, I32],
    "moeb_cache_replay_stack_workspace_bytes": [I32, I32, I32],
    "moeb_linear_workspace_bytes": [I64, I32, I32],
}

EXPORTS = tuple(_SIGS) + ("moeb_last_error",) + tuple(SIZE_QUERIES)


def load_library(require_gpu: bool = True):
    """Load libmoeb.so; with require_gpu, also verify an sm_100 device."""
    global _lib, _checked
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing: build it with `python -m paper_2508_17137_b200.build`")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        for name, args in SIZE_QUERIES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_size_t
        lib.moeb_last_error.argtypes = []
        lib.moeb_last_error.restype = ctypes.c_char_p
        _lib = lib
    if require_gpu and not _checked:
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device visible; libmoeb has no CPU fallback")
        torch.cuda.init()
        rc = _lib.moeb_device_check()
        if rc != 0:
            raise NativeUnavailable(_lib.moeb_last_error().decode())
        _checked = True
    return _lib


def call(name: str, *args) -> None:
    lib = load_library()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise NativeError(name, rc, lib.moeb_last_error().decode())


def workspace(nbytes: int, device) -> torch.Tensor | None:
    """Caller-owned scratch for an entry point that takes (workspace,
    workspace_bytes); the library itself never allocates."""
    if nbytes <= 0:
        return None
    return torch.empty(int(nbytes), dtype=torch.uint8, device=device)


def ptr(t):
    """Device pointer of a CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libmoeb takes CUDA tensors only")
    if not t.is_contiguous():
        raise ValueError("libmoeb takes contiguous tensors only")
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr_array(tensors):
    """Host array of device pointers (NULL for None entries)."""
    arr = (ctypes.c_void_p * len(tensors))()
    for i, t in enumerate(tensors):
        arr[i] = None if t is None else t.data_ptr()
    return arr


def i32_array(vals):
    return (ctypes.c_int32 * len(vals))(*[int(v) for v in vals])


def i64_array(vals):
    return (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])
