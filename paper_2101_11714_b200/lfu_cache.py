"""Python mirror of the reference's LFU hot-row cache and the cached
EmbeddingLayer, backed by the CUDA library.

Reference: proj/include/ttrec/lfu_cache.hpp:18-310 (FreqTable, SlotGradients,
CachePartition, combine_partition_outputs, LfuCache), proj/src/lfu_cache.cpp
and proj/include/ttrec/model.hpp:148-284 (EmbeddingLayer with a TT table +
cache).  Same names, argument meanings and error types as the reference;
every call goes through libttgpu.so (include/ttgpu.h), no CPU path.

Device layout (see csrc/lfu_cache.cuh): dense per-row frequency counters over
the table's row space, a GPU hash table row -> slot probed by every lookup
before decompression, capacity x emb_dim cached rows.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from ._lib import lib
from .ttrec import (ForwardContext, IndexBatch, InvalidArgument, Pooling, TtTable, _p, _raise,
                    kDefaultMicroBatch)


class CacheState(enum.IntEnum):
    WarmUp = 0
    Active = 1


def default_capacity(table_rows: int) -> int:
    """LfuCache::default_capacity (lfu_cache.hpp:146-148): 0.01% of rows, >= 1."""
    return int(lib().ttgpu_cache_default_capacity(int(table_rows)))


def hot_set_drift(prev, cur, k: int) -> float:
    """|symmetric difference| / (2k) (lfu_cache.cpp:113-126)."""
    a = np.ascontiguousarray(prev, np.int64)
    b = np.ascontiguousarray(cur, np.int64)
    out = C.c_double()
    _raise(lib().ttgpu_hot_set_drift(_p(a), len(a), _p(b), len(b), int(k), C.byref(out)))
    return out.value


@dataclass
class CachePartition:
    """lfu_cache.hpp:92-104: both parts keep every bag and are Sum-pooled."""

    cached: IndexBatch
    cached_rows: np.ndarray
    tt: IndexBatch
    original_pooling: Pooling = Pooling.Sum

    def original_bag_size(self, b: int) -> int:
        return self.cached.bag_size(b) + self.tt.bag_size(b)


class FreqTable:
    """Read/modify view of the cache's frequency counters (lfu_cache.hpp:18-50)."""

    def __init__(self, cache: "LfuCache"):
        self._c = cache

    def count(self, key: int) -> int:
        v = C.c_uint64()
        _raise(lib().ttgpu_cache_freq_count(self._c.handle, int(key), C.byref(v)))
        return int(v.value)

    def size(self) -> int:
        v = C.c_int64()
        _raise(lib().ttgpu_cache_freq_size(self._c.handle, C.byref(v)))
        return int(v.value)

    def decay(self, factor: float):
        _raise(lib().ttgpu_cache_freq_decay(self._c.handle, float(factor)))

    def clear(self):
        _raise(lib().ttgpu_cache_freq_clear(self._c.handle))

    def top_k(self, k: int) -> List[int]:
        rows = np.zeros(max(int(k), 1), np.int64)
        n = C.c_int64()
        _raise(lib().ttgpu_cache_top_k(self._c.handle, None, int(k), _p(rows), None, C.byref(n)))
        return [int(r) for r in rows[: n.value]]

    def entries_sorted(self):
        """(key, count) for every key with a count, (count desc, key asc)."""
        n_all = self.size()
        rows = np.zeros(max(n_all, 1), np.int64)
        cnt = np.zeros(max(n_all, 1), np.uint64)
        n = C.c_int64()
        _raise(lib().ttgpu_cache_top_k(self._c.handle, None, n_all, _p(rows), _p(cnt), C.byref(n)))
        return [(int(r), int(c)) for r, c in zip(rows[: n.value], cnt[: n.value])]


class LfuCache:
    """LfuCache<T> (lfu_cache.hpp:134-310).  key_space = the table's row count
    (frequencies are dense per-row counters on the GPU)."""

    def __init__(self, capacity: int, emb_dim: int, refresh_period: int = 1000,
                 key_space: Optional[int] = None, dtype=np.float32, device: int = 0,
                 stream: int = 0):
        if key_space is None:
            raise InvalidArgument("LfuCache on the GPU needs key_space (the table's row count)")
        self.dtype = np.dtype(dtype)
        h = C.c_void_p()
        _raise(lib().ttgpu_cache_create(int(capacity), int(emb_dim), int(refresh_period),
                                        int(key_space), 1 if self.dtype == np.float64 else 0,
                                        device, C.c_void_p(stream), C.byref(h)))
        self.handle = h
        self._capacity, self._emb, self._period = int(capacity), int(emb_dim), int(refresh_period)
        self.key_space = int(key_space)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                lib().ttgpu_cache_destroy(h)
            except Exception:  # noqa: BLE001
                pass
            self.handle = None

    default_capacity = staticmethod(default_capacity)

    def set_fast(self, enable: bool):
        """Cached forward through the fast-path sort (default; no host sync,
        graph-capturable) or through the explicit partition (False)."""
        _raise(lib().ttgpu_cache_set_fast(self.handle, 1 if enable else 0))

    def _last(self):
        nc, nt, b, hw, pl = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
        _raise(lib().ttgpu_cache_last_counts(self.handle, C.byref(nc), C.byref(nt), C.byref(b),
                                             C.byref(hw), C.byref(pl)))
        return nc.value, nt.value, b.value, bool(hw.value), pl.value

    def last_counts(self):
        """(cached, chain) lookup counts of the last cached forward."""
        return self._last()[:2]

    def last_partition(self) -> "CachePartition":
        """The partition of the last cached forward (record_and_partition's
        result; the fast path rebuilds it from its per-lookup slots)."""
        return self._fetch_partition(*self._last())

    # ---- accessors (lfu_cache.hpp:150-175) ----
    def _info(self):
        a, r, acc, hits = C.c_int(), C.c_int64(), C.c_uint64(), C.c_uint64()
        _raise(lib().ttgpu_cache_info(self.handle, C.byref(a), C.byref(r), C.byref(acc),
                                      C.byref(hits)))
        return a.value, r.value, acc.value, hits.value

    def state(self) -> CacheState:
        return CacheState(self._info()[0])

    def capacity(self) -> int:
        return self._capacity

    def emb_dim(self) -> int:
        return self._emb

    def refresh_period(self) -> int:
        return self._period

    def freq(self) -> FreqTable:
        return FreqTable(self)

    def resident_count(self) -> int:
        return int(self._info()[1])

    def slot_of(self, row: int) -> int:
        s = C.c_int64()
        _raise(lib().ttgpu_cache_slot_of(self.handle, int(row), C.byref(s)))
        return int(s.value)

    def slot_rows(self) -> np.ndarray:
        out = np.zeros(self._capacity, np.int64)
        _raise(lib().ttgpu_cache_slot_rows(self.handle, _p(out)))
        return out

    def row_at(self, slot: int) -> int:
        return int(self.slot_rows()[slot])

    def all_row_values(self) -> np.ndarray:
        out = np.zeros((self._capacity, self._emb), self.dtype)
        _raise(lib().ttgpu_cache_get_rows(self.handle, _p(out)))
        return out

    def row_values(self, slot: int) -> np.ndarray:
        return self.all_row_values()[slot].copy()

    def set_row_values(self, slot: int, values):
        v = np.ascontiguousarray(values, self.dtype)
        _raise(lib().ttgpu_cache_set_row(self.handle, int(slot), _p(v)))

    def hot_rows(self) -> np.ndarray:
        n = C.c_int64()
        _raise(lib().ttgpu_cache_hot_rows(self.handle, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.int64)
        _raise(lib().ttgpu_cache_hot_rows(self.handle, _p(out), n.value, C.byref(n)))
        return out[: n.value]

    def hit_rate(self) -> float:
        _, _, acc, hits = self._info()
        return 0.0 if acc == 0 else hits / acc

    def active_accesses(self) -> int:
        return int(self._info()[2])

    def active_hits(self) -> int:
        return int(self._info()[3])

    # ---- frequency / routing (lfu_cache.hpp:177-219) ----
    def record(self, batch: IndexBatch):
        _raise(lib().ttgpu_cache_record(self.handle, _p(batch.indices), batch.num_lookups()))

    def record_and_partition(self, batch: IndexBatch) -> CachePartition:
        B, L = batch.num_bags(), batch.num_lookups()
        w = batch.weights if batch.has_weights() else None
        nc, nt = C.c_int64(), C.c_int64()
        _raise(lib().ttgpu_cache_record_and_partition(
            self.handle, _p(batch.indices), L, _p(batch.offsets), B, _p(w), int(batch.pooling),
            C.byref(nc), C.byref(nt)))
        return self._fetch_partition(nc.value, nt.value, B, w is not None, int(batch.pooling))

    def _fetch_partition(self, nc: int, nt: int, B: int, has_w: bool, pooling: int) -> "CachePartition":
        cs = np.zeros(max(nc, 1), np.int64)
        cr = np.zeros(max(nc, 1), np.int64)
        co = np.zeros(B + 1, np.int64)
        ti = np.zeros(max(nt, 1), np.int64)
        to = np.zeros(B + 1, np.int64)
        cw = np.zeros(max(nc, 1), np.float64) if has_w else None
        tw = np.zeros(max(nt, 1), np.float64) if has_w else None
        _raise(lib().ttgpu_cache_last_partition(self.handle, _p(cs), _p(cr), _p(co), _p(cw), _p(ti),
                                                _p(to), _p(tw)))
        cached = IndexBatch(cs[:nc], co, None if cw is None else cw[:nc], Pooling.Sum)
        tt = IndexBatch(ti[:nt], to, None if tw is None else tw[:nt], Pooling.Sum)
        return CachePartition(cached, cr[:nc], tt, Pooling(pooling))

    # ---- admission (lfu_cache.hpp:223-243) ----
    def warmup_finalize(self, table: TtTable):
        _raise(lib().ttgpu_cache_warmup_finalize(self.handle, table.handle))

    def refresh(self, table: TtTable) -> float:
        d = C.c_double()
        _raise(lib().ttgpu_cache_refresh(self.handle, table.handle, C.byref(d)))
        return d.value

    # ---- training (lfu_cache.hpp:246-257) ----
    def cached_sgd_update(self, slots, rows, lr: float):
        """SlotGradients given as (slots, rows[len(slots) x emb_dim])."""
        s = np.ascontiguousarray(slots, np.int64)
        r = np.ascontiguousarray(rows, self.dtype)
        _raise(lib().ttgpu_cache_sgd_update(self.handle, _p(s), len(s), _p(r), float(lr)))

    def slot_grads(self):
        """Gradients of the last cached backward: (capacity x emb_dim, touched mask)."""
        g = np.zeros((self._capacity, self._emb), self.dtype)
        t = np.zeros(self._capacity, np.uint8)
        _raise(lib().ttgpu_cache_slot_grads(self.handle, _p(g), _p(t)))
        return g, t.astype(bool)


def combine_partition_outputs(part: CachePartition, cached_out, tt_out):
    """lfu_cache.hpp:106-126 on host arrays (reference-shaped helper)."""
    out = (np.asarray(cached_out) + np.asarray(tt_out)).astype(np.asarray(tt_out).dtype)
    if part.original_pooling == Pooling.Mean:
        for b in range(part.cached.num_bags()):
            sz = part.original_bag_size(b)
            if sz > 1:
                out[b] *= out.dtype.type(1.0 / sz)
    return out


class EmbeddingLayer:
    """model.hpp:148-284 for a TT table, optionally with an LFU cache
    (use_cache): forward / backward / step / finalize_warmup / refresh_cache."""

    def __init__(self, table: TtTable, cache: Optional[LfuCache] = None):
        self.tt = table
        self.cache = cache
        self.ctx = ForwardContext(table)
        self._batch: Optional[IndexBatch] = None

    def forward(self, batch: IndexBatch, micro_batch: int = kDefaultMicroBatch,
                save: bool = True) -> np.ndarray:
        B, L = batch.num_bags(), batch.num_lookups()
        batch.validate(self.tt.rows(), self.tt.name())
        out = np.zeros((B, self.tt.cols()), self.tt.dtype)
        w = batch.weights if batch.has_weights() else None
        if self.cache is None:
            _raise(lib().ttgpu_forward(self.tt.handle, _p(batch.indices), L, _p(batch.offsets), B,
                                       _p(w), int(batch.pooling), micro_batch, int(save), _p(out),
                                       self.ctx.handle))
        else:
            _raise(lib().ttgpu_cache_forward(self.cache.handle, self.tt.handle, self.ctx.handle,
                                             _p(batch.indices), L, _p(batch.offsets), B, _p(w),
                                             int(batch.pooling), int(save), _p(out)))
        self.ctx._fill(self.tt, L, B, save)
        self._batch = batch
        return out

    def backward(self, batch: IndexBatch, grad):
        g = np.ascontiguousarray(grad, self.tt.dtype).ravel()
        if g.size != batch.num_bags() * self.tt.cols():
            raise InvalidArgument(f"table '{self.tt.name()}': bad gradient size")
        if self.cache is None:
            _raise(lib().ttgpu_backward(self.tt.handle, self.ctx.handle, batch.num_lookups(),
                                        batch.num_bags(), _p(g), g.size, None))
        else:
            _raise(lib().ttgpu_cache_backward(self.cache.handle, self.tt.handle, self.ctx.handle,
                                              _p(g), g.size))

    def step(self, lr: float):
        if self.cache is None:
            _raise(lib().ttgpu_apply_grad(self.tt.handle, float(lr)))
            self.tt.sync()
        else:
            _raise(lib().ttgpu_cache_step(self.cache.handle, self.tt.handle, float(lr)))
            self.tt.sync()

    def finalize_warmup(self):
        if self.cache is not None and self.cache.state() == CacheState.WarmUp:
            self.cache.warmup_finalize(self.tt)

    def refresh_cache(self) -> float:
        if self.cache is not None and self.cache.state() == CacheState.Active:
            return self.cache.refresh(self.tt)
        return 0.0
