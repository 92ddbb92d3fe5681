"""ctypes binding of libttgpu.so (include/ttgpu.h).

This is the "reference-side binding a maintainer would add" for a Python
caller.  There is deliberately no fallback: if the CUDA
library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TTGPU_LIB", os.path.join(HERE, "lib", "libttgpu.so"))

i64 = C.c_int64
i64p = C.POINTER(C.c_int64)
vp = C.c_void_p
vpp = C.POINTER(C.c_void_p)

# name -> (restype, argtypes)
_SIGS = {
    "ttgpu_last_error": (C.c_char_p, []),
    "ttgpu_abi_version": (C.c_int, []),
    "ttgpu_plan_shapes": (C.c_int, [i64, i64, C.c_int, i64, vp, vp, vp, vp, vp]),
    "ttgpu_plan_info": (C.c_int, [i64, i64, C.c_int, vp, vp, vp, vp, vp, vp]),
    "ttgpu_decompose_index": (C.c_int, [i64, vp, C.c_int, vp]),
    "ttgpu_recompose_index": (C.c_int, [vp, vp, C.c_int, vp]),
    "ttgpu_create": (C.c_int, [i64, i64, C.c_int, vp, vp, vp, C.c_int, C.c_char_p, C.c_int, vp,
                               vpp]),
    "ttgpu_destroy": (C.c_int, [vp]),
    "ttgpu_set_stream": (C.c_int, [vp, vp]),
    "ttgpu_core_size": (C.c_int, [vp, C.c_int, i64p]),
    "ttgpu_get_core": (C.c_int, [vp, C.c_int, vp]),
    "ttgpu_get_grad": (C.c_int, [vp, C.c_int, vp]),
    "ttgpu_set_core": (C.c_int, [vp, C.c_int, vp]),
    "ttgpu_core_device_ptr": (C.c_int, [vp, C.c_int, vpp]),
    "ttgpu_mark_mutated": (C.c_int, [vp]),
    "ttgpu_set_exact_forward": (C.c_int, [vp, C.c_int]),
    "ttgpu_set_generic_path": (C.c_int, [vp, C.c_int]),
    "ttgpu_set_tensor_path": (C.c_int, [vp, C.c_int]),
    "ttgpu_set_grid_sort": (C.c_int, [vp, C.c_int]),
    "ttgpu_set_chunked": (C.c_int, [vp, C.c_int]),
    "ttgpu_set_wide3": (C.c_int, [vp, C.c_int]),
    "ttgpu_fast_path_kind": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "ttgpu_mutation_counter": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
    "ttgpu_ctx_create": (C.c_int, [vp, vpp]),
    "ttgpu_ctx_destroy": (C.c_int, [vp]),
    "ttgpu_forward": (C.c_int, [vp, vp, i64, vp, i64, vp, C.c_int, i64, C.c_int, vp, vp]),
    "ttgpu_forward_device": (C.c_int, [vp, vp, i64, vp, i64, vp, C.c_int, C.c_int, vp, vp]),
    "ttgpu_backward": (C.c_int, [vp, vp, i64, i64, vp, i64, vp]),
    "ttgpu_backward_device": (C.c_int, [vp, vp, vp]),
    "ttgpu_grad_device_ptr": (C.c_int, [vp, C.c_int, vpp]),
    "ttgpu_sgd_step": (C.c_int, [vp, vp, C.c_double]),
    "ttgpu_apply_grad": (C.c_int, [vp, C.c_double]),
    "ttgpu_backward_sgd": (C.c_int, [vp, vp, i64, i64, vp, i64, C.c_double]),
    "ttgpu_grad_buffer": (C.c_int, [vp, vpp, i64p]),
    "ttgpu_graph_begin": (C.c_int, [vp]),
    "ttgpu_graph_end": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ttgpu_graph_launch": (C.c_int, [vp]),
    "ttgpu_backward_sgd_device": (C.c_int, [vp, vp, vp, C.c_double]),
    "ttgpu_lookup_row": (C.c_int, [vp, i64, vp]),
    "ttgpu_lookup_rows_device": (C.c_int, [vp, vp, i64, vp]),
    "ttgpu_profile": (C.c_int, [vp, C.c_int]),
    "ttgpu_profile_read": (C.c_int, [vp, C.c_char_p, i64, C.POINTER(C.c_float), C.c_int,
                                     C.POINTER(C.c_int)]),
    "ttgpu_sync": (C.c_int, [vp]),
    "ttgpu_check": (C.c_int, [vp]),
    # LFU cache (lfu_cache.hpp) + cached EmbeddingLayer (model.hpp:195-284)
    "ttgpu_cache_create": (C.c_int, [i64, i64, i64, i64, C.c_int, C.c_int, vp, vpp]),
    "ttgpu_cache_destroy": (C.c_int, [vp]),
    "ttgpu_cache_set_stream": (C.c_int, [vp, vp]),
    "ttgpu_cache_set_fast": (C.c_int, [vp, C.c_int]),
    "ttgpu_cache_last_counts": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "ttgpu_cache_default_capacity": (i64, [i64]),
    "ttgpu_cache_info": (C.c_int, [vp, vp, vp, vp, vp]),
    "ttgpu_cache_record": (C.c_int, [vp, vp, i64]),
    "ttgpu_cache_record_and_partition": (C.c_int, [vp, vp, i64, vp, i64, vp, C.c_int, vp, vp]),
    "ttgpu_cache_last_partition": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp]),
    "ttgpu_cache_warmup_finalize": (C.c_int, [vp, vp]),
    "ttgpu_cache_refresh": (C.c_int, [vp, vp, vp]),
    "ttgpu_hot_set_drift": (C.c_int, [vp, i64, vp, i64, i64, vp]),
    "ttgpu_cache_hot_rows": (C.c_int, [vp, vp, i64, vp]),
    "ttgpu_cache_slot_rows": (C.c_int, [vp, vp]),
    "ttgpu_cache_slot_of": (C.c_int, [vp, i64, vp]),
    "ttgpu_cache_get_rows": (C.c_int, [vp, vp]),
    "ttgpu_cache_set_row": (C.c_int, [vp, i64, vp]),
    "ttgpu_cache_store_device_ptr": (C.c_int, [vp, vpp]),
    "ttgpu_cache_counts_device_ptr": (C.c_int, [vp, vpp, vp]),
    "ttgpu_cache_freq_count": (C.c_int, [vp, i64, vp]),
    "ttgpu_cache_freq_size": (C.c_int, [vp, vp]),
    "ttgpu_cache_freq_decay": (C.c_int, [vp, C.c_double]),
    "ttgpu_cache_freq_clear": (C.c_int, [vp]),
    "ttgpu_cache_top_k": (C.c_int, [vp, vp, i64, vp, vp, vp]),
    "ttgpu_cache_forward": (C.c_int, [vp, vp, vp, vp, i64, vp, i64, vp, C.c_int, C.c_int, vp]),
    "ttgpu_cache_forward_device": (C.c_int, [vp, vp, vp, vp, i64, vp, i64, vp, C.c_int, C.c_int,
                                             vp]),
    "ttgpu_cache_backward": (C.c_int, [vp, vp, vp, vp, i64]),
    "ttgpu_cache_backward_device": (C.c_int, [vp, vp, vp, vp]),
    "ttgpu_cache_step": (C.c_int, [vp, vp, C.c_double]),
    "ttgpu_cache_backward_step_device": (C.c_int, [vp, vp, vp, vp, C.c_double]),
    "ttgpu_cache_slot_grads": (C.c_int, [vp, vp, vp]),
    "ttgpu_cache_sgd_update": (C.c_int, [vp, vp, i64, vp, C.c_double]),
    "ttgpu_stats_reset": (None, []),
    "ttgpu_stats_rows": (C.c_uint64, []),
    "ttgpu_stats_peak_workspace": (C.c_uint64, []),
    "ttgpu_stats_add_rows": (None, [C.c_uint64]),
    "ttgpu_zipf_batch": (C.c_int, [i64, C.c_double, C.c_uint64, i64, i64, vp, vp]),
    "ttgpu_uniform_indices": (C.c_int, [i64, C.c_uint64, i64, vp]),
    "ttgpu_derived_uniform_indices": (C.c_int, [i64, C.c_uint64, C.c_uint64, i64, vp]),
    "ttgpu_init_sampled_gaussian": (C.c_int, [vp, C.c_uint64]),
    "ttgpu_sampler_create": (C.c_int, [i64, C.c_double, C.c_int, vp, vpp]),
    "ttgpu_sampler_destroy": (C.c_int, [vp]),
    "ttgpu_sampler_set_stream": (C.c_int, [vp, vp]),
    "ttgpu_sampler_draw_device": (C.c_int, [vp, C.c_uint64, C.c_uint64, i64, vp]),
    "ttgpu_bag_offsets_device": (C.c_int, [i64, i64, vp, vp]),
    "ttgpu_peer_export": (C.c_int, [vp, vp, vp, vp]),
    "ttgpu_peer_attach": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp]),
    "ttgpu_peer_attach_ptrs": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp]),
    "ttgpu_peer_flags_ptr": (C.c_int, [vp, vpp]),
    "ttgpu_peer_reduce_sgd": (C.c_int, [vp, C.c_double]),
    "ttgpu_peer_status": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "ttgpu_dense_create": (C.c_int, [C.c_int, vp, i64, C.c_int, C.c_int, vp, vpp]),
    "ttgpu_dense_destroy": (C.c_int, [vp]),
    "ttgpu_dense_set_stream": (C.c_int, [vp, vp]),
    "ttgpu_dense_set_table": (C.c_int, [vp, C.c_int, vp]),
    "ttgpu_dense_get_table": (C.c_int, [vp, C.c_int, vp]),
    "ttgpu_dense_forward_device": (C.c_int, [vp, vp, i64, vp, i64, vp]),
    "ttgpu_dense_backward_device": (C.c_int, [vp, vp, C.c_int, C.c_double]),
    "ttgpu_dense_grad_buffer": (C.c_int, [vp, vpp, i64p]),
    "ttgpu_dense_apply_grad": (C.c_int, [vp, C.c_double]),
    "ttgpu_dense_check": (C.c_int, [vp]),
}


def header_symbols(header: str | None = None) -> list:
    """Every function declared in include/ttgpu.h (for the export test)."""
    import re

    header = header or os.path.join(HERE, "..", "include", "ttgpu.h")
    text = open(header).read()
    return sorted(set(re.findall(r"\b(ttgpu_[a-z0-9_]+)\s*\(", text)))


class _Lib:
    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise ImportError(
                f"libttgpu.so not found at {path}: build it with "
                f"`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        self.path = path
        self.lib = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(self.lib, name)
            fn.restype = res
            fn.argtypes = args

    def __getattr__(self, name):
        return getattr(self.lib, name)


_lib = None


def lib() -> _Lib:
    global _lib
    if _lib is None:
        _lib = _Lib()
    return _lib
