"""Uncompressed embedding-bag tables on the GPU: the
DLRM features of cfg5 that are not TT-compressed, as one group sharing a row
store and a bag structure (ttgpu_dense_*, csrc/dense_host.inl)."""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from ._lib import lib
from .ttrec import _raise

# Criteo Kaggle per-feature cardinalities as published with DLRM's Kaggle
# preprocessing (not in the reference, which only lists the 7 largest,
# tools/ttrec.cpp:30-34); the 7 entries >= 142,572 are the TT tables of cfg5.
KAGGLE_CARDINALITIES = [1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683, 8351593,
                        3194, 27, 14992, 5461306, 10, 5652, 2173, 4, 7046547, 18, 15, 286181, 105,
                        142572]
KAGGLE_DENSE_ROWS = [n for n in KAGGLE_CARDINALITIES if n < 142572]


class DenseEmbeddingBags:
    """A group of plain (uncompressed) embedding tables, dim `emb_dim`."""

    def __init__(self, rows: Sequence[int], emb_dim: int, dtype=np.float32, device: int = 0,
                 stream: int = 0):
        self.rows = [int(r) for r in rows]
        self.emb_dim = int(emb_dim)
        self.dtype = np.dtype(dtype)
        r = np.asarray(self.rows, np.int64)
        h = C.c_void_p()
        _raise(lib().ttgpu_dense_create(len(self.rows), r.ctypes.data_as(C.c_void_p), self.emb_dim,
                                        1 if self.dtype == np.float64 else 0, device,
                                        C.c_void_p(stream), C.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                lib().ttgpu_dense_destroy(h)
            except Exception:  # noqa: BLE001
                pass
            self.handle = None

    def set_stream(self, stream: int):
        _raise(lib().ttgpu_dense_set_stream(self.handle, C.c_void_p(stream)))

    def set_table(self, t: int, values):
        v = np.ascontiguousarray(values, self.dtype)
        assert v.size == self.rows[t] * self.emb_dim
        _raise(lib().ttgpu_dense_set_table(self.handle, t, v.ctypes.data_as(C.c_void_p)))

    def table(self, t: int) -> np.ndarray:
        out = np.zeros((self.rows[t], self.emb_dim), self.dtype)
        _raise(lib().ttgpu_dense_get_table(self.handle, t, out.ctypes.data_as(C.c_void_p)))
        return out

    def init_uniform(self, seed: int, scale: float = 0.05):
        rng = np.random.default_rng(seed)
        for t, n in enumerate(self.rows):
            self.set_table(t, rng.uniform(-scale, scale, (n, self.emb_dim)))

    def forward_device(self, idx_ptr: int, L: int, off_ptr: int, B: int, out_ptr: int):
        """indices (n_tables x L), offsets (B + 1), out (n_tables x B x dim), device pointers."""
        _raise(lib().ttgpu_dense_forward_device(self.handle, C.c_void_p(idx_ptr), int(L),
                                                C.c_void_p(off_ptr), int(B), C.c_void_p(out_ptr)))

    def backward_device(self, grad_ptr: int, lr: float = 0.0, fused: bool = True):
        _raise(lib().ttgpu_dense_backward_device(self.handle, C.c_void_p(grad_ptr), int(fused),
                                                 C.c_double(lr)))

    def grad_buffer(self):
        p, n = C.c_void_p(), C.c_int64()
        _raise(lib().ttgpu_dense_grad_buffer(self.handle, C.byref(p), C.byref(n)))
        return p.value, n.value

    def apply_grad(self, lr: float):
        _raise(lib().ttgpu_dense_apply_grad(self.handle, C.c_double(lr)))

    def check(self):
        _raise(lib().ttgpu_dense_check(self.handle))
