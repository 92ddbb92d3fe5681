"""TEST INFRASTRUCTURE ONLY -- ctypes access to the two CPU oracles.

* ``Oracle``  -> oracle/libttoracle.so: the plain-C restatement of the
  reference's serial algorithm (oracle/tt_oracle.c).  Travels to the GPU box
  as a prebuilt .so; this is what GPU parity tests compare against.
* ``RefImpl`` -> oracle/_ref/libttref.so: the UNMODIFIED reference C++ code
  compiled from /root/reference by oracle/Makefile (only buildable where the
  reference sources exist, but the built .so travels too).  Used to pin the
  restatement, to generate tests/golden fixtures with the reference's own RNG
  and to time the reference CPU path (bench.py cpu_baseline / --impl reference).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libttoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libttref.so")

i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class Plan:
    """A ShapePlan (shape_plan.hpp:19-46) as plain integers."""

    num_rows: int
    emb_dim: int
    row_factors: list
    col_factors: list
    ranks: list
    tt_dim: int = field(init=False)

    def __post_init__(self):
        self.tt_dim = len(self.row_factors)
        self.row_factors = [int(x) for x in self.row_factors]
        self.col_factors = [int(x) for x in self.col_factors]
        self.ranks = [int(x) for x in self.ranks]

    def core_size(self, k: int) -> int:
        return self.ranks[k] * self.row_factors[k] * self.col_factors[k] * self.ranks[k + 1]

    def slice_size(self, k: int) -> int:
        return self.ranks[k] * self.col_factors[k] * self.ranks[k + 1]

    def arrays(self):
        return (np.asarray(self.row_factors, np.int64), np.asarray(self.col_factors, np.int64),
                np.asarray(self.ranks, np.int64))


def _ptr_array(arrs, ctype=C.c_void_p):
    return (ctype * len(arrs))(*[a.ctypes.data_as(C.c_void_p) for a in arrs])


class Oracle:
    """C restatement (oracle/tt_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise RuntimeError(f"oracle library missing: {path} (run __graft_entry__.build())")
        self.lib = C.CDLL(path)
        L = self.lib
        L.tto_time_step_f32.restype = C.c_double

    def _call(self, fn, plan: Plan, *args):
        rf, cf, rk = plan.arrays()
        return fn(C.c_int(plan.tt_dim), C.c_int64(plan.num_rows), C.c_int64(plan.emb_dim),
                  _p(rf), _p(cf), _p(rk), *args)

    def forward(self, plan: Plan, cores, idx, off, weights=None, pooling=0):
        dt = cores[0].dtype
        fn = self.lib.tto_forward_f64 if dt == np.float64 else self.lib.tto_forward_f32
        idx = np.ascontiguousarray(idx, np.int64)
        off = np.ascontiguousarray(off, np.int64)
        B = len(off) - 1
        out = np.zeros((B, plan.emb_dim), dt)
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        st = self._call(fn, plan, _ptr_array(cores), _p(idx), C.c_int64(len(idx)), _p(off),
                        C.c_int64(B), _p(w), C.c_int(pooling), _p(out))
        if st:
            raise ValueError(f"oracle forward status {st}")
        return out

    def backward(self, plan: Plan, cores, idx, off, grad_out, weights=None, pooling=0):
        dt = cores[0].dtype
        fn = self.lib.tto_backward_f64 if dt == np.float64 else self.lib.tto_backward_f32
        idx = np.ascontiguousarray(idx, np.int64)
        off = np.ascontiguousarray(off, np.int64)
        B = len(off) - 1
        grads = [np.zeros(plan.core_size(k), dt) for k in range(plan.tt_dim)]
        g = np.ascontiguousarray(grad_out, dt)
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        st = self._call(fn, plan, _ptr_array(cores), _p(idx), C.c_int64(len(idx)), _p(off),
                        C.c_int64(B), _p(w), C.c_int(pooling), _p(g), _ptr_array(grads))
        if st:
            raise ValueError(f"oracle backward status {st}")
        return grads

    def sgd(self, plan: Plan, cores, grads, lr):
        dt = cores[0].dtype
        fn = self.lib.tto_sgd_f64 if dt == np.float64 else self.lib.tto_sgd_f32
        rf, cf, rk = plan.arrays()
        fn(C.c_int(plan.tt_dim), _p(rf), _p(cf), _p(rk), _ptr_array(cores), _ptr_array(grads),
           C.c_double(lr))

    def lookup_row(self, plan: Plan, cores, row):
        dt = cores[0].dtype
        fn = self.lib.tto_lookup_row_f64 if dt == np.float64 else self.lib.tto_lookup_row_f32
        out = np.zeros(plan.emb_dim, dt)
        st = self._call(fn, plan, _ptr_array(cores), C.c_int64(row), _p(out))
        if st:
            raise IndexError(f"row {row} out of range")
        return out

    def decompose_row(self, flat, row_factors):
        rf = np.asarray(row_factors, np.int64)
        out = np.zeros(len(rf), np.int64)
        self.lib.tto_decompose_row(C.c_int64(flat), C.c_int(len(rf)), _p(rf), _p(out))
        return out

    def time_step(self, plan: Plan, cores, idx, off, grad_out, lr=0.01, threads=0):
        rf, cf, rk = plan.arrays()
        B = len(off) - 1
        return self.lib.tto_time_step_f32(
            C.c_int(plan.tt_dim), C.c_int64(plan.num_rows), C.c_int64(plan.emb_dim), _p(rf),
            _p(cf), _p(rk), _ptr_array(cores), _p(idx), C.c_int64(len(idx)), _p(off),
            C.c_int64(B), _p(grad_out), C.c_double(lr), C.c_int(threads))


class RefError(Exception):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


class RefImpl:
    """The reference C++ implementation compiled from its own sources."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise RuntimeError(f"reference build missing: {path}")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_core_size.restype = C.c_int64
        L.ref_time_step.restype = C.c_double
        L.ref_time_step_serial.restype = C.c_double
        L.ref_random_batch.restype = C.c_int64
        L.ref_cache_default_capacity.restype = C.c_int64
        L.ref_cache_hot_rows.restype = C.c_int64
        L.ref_cache_slot_of.restype = C.c_int64
        L.ref_cache_hit_rate.restype = C.c_double
        L.ref_cache_freq.restype = C.c_uint64
        L.ref_cache_top_k.restype = C.c_int64
        L.ref_stats_rows.restype = C.c_uint64
        L.ref_layer_freq.restype = C.c_uint64
        L.ref_layer_cache_rows.restype = C.c_int64
        L.ref_model_param.restype = C.c_int64

    def check(self, st):
        if st:
            raise RefError(st, self.lib.ref_last_error().decode())

    # ---- plans ----
    def plan_shapes(self, rows, emb, d, rank, row_factors=None, col_factors=None):
        rf_in = None if row_factors is None else np.asarray(row_factors, np.int64)
        cf_in = None if col_factors is None else np.asarray(col_factors, np.int64)
        rf, cf, rk = np.zeros(d, np.int64), np.zeros(d, np.int64), np.zeros(d + 1, np.int64)
        padded, params, red = C.c_int64(), C.c_int64(), C.c_int64()
        self.check(self.lib.ref_plan_shapes(
            C.c_int64(rows), C.c_int64(emb), C.c_int(d), C.c_int64(rank), _p(rf_in), _p(cf_in),
            _p(rf), _p(cf), _p(rk), C.byref(padded), C.byref(params), C.byref(red)))
        return Plan(rows, emb, list(rf), list(cf), list(rk)), dict(
            padded_rows=padded.value, params=params.value, reduction=red.value)

    def decompose_index(self, flat, radices):
        r = np.asarray(radices, np.int64)
        out = np.zeros(len(r), np.int64)
        self.check(self.lib.ref_decompose_index(C.c_int64(flat), _p(r), C.c_int(len(r)), _p(out)))
        return out

    # ---- checkpoints (checkpoint.hpp / src/checkpoint.cpp) ----
    def checkpoint_save(self, path, tables, arrays=()):
        """Checkpoint: put_table(t) for each RefTable, put_array<float>(name,
        {len}, values) for each (name, values), save(path)."""
        th = (C.c_void_p * max(1, len(tables)))(*[t.h for t in tables])
        arrays = [(n, np.ascontiguousarray(v, np.float32)) for n, v in arrays]
        names = (C.c_char_p * max(1, len(arrays)))(*[n.encode() for n, _ in arrays])
        ptrs = (C.c_void_p * max(1, len(arrays)))(*[v.ctypes.data for _, v in arrays])
        lens = np.array([v.size for _, v in arrays] or [0], np.int64)
        self.check(self.lib.ref_checkpoint_save(th, C.c_int(len(tables)), names, ptrs, _p(lens),
                                                C.c_int(len(arrays)), str(path).encode()))

    def checkpoint_load_table(self, path, name, plan: Plan, dtype=np.float32):
        h = C.c_void_p()
        self.check(self.lib.ref_checkpoint_load_table(str(path).encode(), name.encode(),
                                                      C.c_int(1 if np.dtype(dtype) == np.float64
                                                              else 0), C.byref(h)))
        t = RefTable.__new__(RefTable)
        t.ref, t.plan, t.dtype, t.h = self, plan, np.dtype(dtype), h
        return t

    def checkpoint_load_array(self, path, name, n):
        out = np.zeros(n, np.float32)
        self.check(self.lib.ref_checkpoint_load_array(str(path).encode(), name.encode(), _p(out),
                                                      C.c_int64(n)))
        return out

    # ---- tables ----
    def table(self, plan: Plan, dtype=np.float32, name="tt-table"):
        return RefTable(self, plan, dtype, name)

    def layer(self, plan: Plan, cache_capacity=-1, name="tt-layer"):
        return RefLayer(self, plan, cache_capacity, name)

    # ---- streams (reference RNG, libstdc++-specific) ----
    def normal(self, seed, n):
        out = np.zeros(n, np.float64)
        self.lib.ref_rng_normal(C.c_uint64(seed), C.c_int64(n), _p(out))
        return out

    def uniform_int(self, seed, lo, hi, n):
        out = np.zeros(n, np.int64)
        self.lib.ref_rng_uniform_int(C.c_uint64(seed), C.c_int64(lo), C.c_int64(hi),
                                     C.c_int64(n), _p(out))
        return out

    def random_batch(self, seed, rows, bags, min_size, max_size, weighted):
        idx = np.zeros(bags * max(max_size, 1) + 1, np.int64)
        off = np.zeros(bags + 1, np.int64)
        w = np.zeros(bags * max(max_size, 1) + 1, np.float64)
        n = self.lib.ref_random_batch(C.c_uint64(seed), C.c_int64(rows), C.c_int64(bags),
                                      C.c_int64(min_size), C.c_int64(max_size),
                                      C.c_int(int(weighted)), _p(idx), _p(off), _p(w))
        return idx[:n].copy(), off, (w[:n].copy() if weighted else None)

    def zipf_batch(self, population, exponent, seed, bags, pooling_factor):
        idx = np.zeros(bags * pooling_factor, np.int64)
        off = np.zeros(bags + 1, np.int64)
        self.check(self.lib.ref_zipf_batch(C.c_int64(population), C.c_double(exponent),
                                           C.c_uint64(seed), C.c_int64(bags),
                                           C.c_int64(pooling_factor), _p(idx), _p(off)))
        return idx, off

    def stats_reset(self):
        self.lib.ref_stats_reset()

    def stats_rows(self):
        return int(self.lib.ref_stats_rows())


class RefTable:
    def __init__(self, ref: RefImpl, plan: Plan, dtype, name):
        self.ref, self.plan, self.dtype = ref, plan, np.dtype(dtype)
        rf, cf, rk = plan.arrays()
        h = C.c_void_p()
        ref.check(ref.lib.ref_table_create(
            C.c_int64(plan.num_rows), C.c_int64(plan.emb_dim), C.c_int(plan.tt_dim), _p(rf),
            _p(cf), _p(rk), C.c_int(1 if self.dtype == np.float64 else 0), name.encode(),
            C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.ref.lib.ref_table_destroy(self.h)
        except Exception:
            pass

    def get_cores(self):
        out = []
        for k in range(self.plan.tt_dim):
            a = np.zeros(self.plan.core_size(k), self.dtype)
            self.ref.lib.ref_get_core(self.h, C.c_int(k), _p(a))
            out.append(a)
        return out

    def set_cores(self, cores):
        for k, c in enumerate(cores):
            c = np.ascontiguousarray(c, self.dtype)
            self.ref.lib.ref_set_core(self.h, C.c_int(k), _p(c))

    def init_sampled_gaussian(self, seed):
        self.ref.check(self.ref.lib.ref_init_sampled_gaussian(self.h, C.c_uint64(seed)))

    def fill_normal(self, seed, scale=1.0):
        self.ref.lib.ref_fill_cores_normal(self.h, C.c_uint64(seed), C.c_double(scale))

    def forward(self, idx, off, weights=None, pooling=0, micro_batch=2048, save=False,
                keep_ctx=False):
        idx = np.ascontiguousarray(idx, np.int64)
        off = np.ascontiguousarray(off, np.int64)
        B = len(off) - 1
        out = np.zeros((B, self.plan.emb_dim), self.dtype)
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        ctx = C.c_void_p()
        self.ref.check(self.ref.lib.ref_forward(
            self.h, _p(idx), C.c_int64(len(idx)), _p(off), C.c_int64(B), _p(w), C.c_int(pooling),
            C.c_int64(micro_batch), C.c_int(int(save)), _p(out),
            C.byref(ctx) if keep_ctx else None))
        return (out, ctx) if keep_ctx else out

    def backward(self, ctx, idx, off, grad_out, weights=None, pooling=0):
        idx = np.ascontiguousarray(idx, np.int64)
        off = np.ascontiguousarray(off, np.int64)
        B = len(off) - 1
        g = np.ascontiguousarray(grad_out, self.dtype)
        grads = [np.zeros(self.plan.core_size(k), self.dtype) for k in range(self.plan.tt_dim)]
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        self.ref.check(self.ref.lib.ref_backward(
            self.h, _p(idx), C.c_int64(len(idx)), _p(off), C.c_int64(B), _p(w), C.c_int(pooling),
            ctx, _p(g), C.c_int64(g.size), _ptr_array(grads)))
        return grads

    def ctx_destroy(self, ctx):
        self.ref.lib.ref_ctx_destroy(ctx)

    def serial_forward(self, idx, off, weights=None, pooling=0):
        idx = np.ascontiguousarray(idx, np.int64)
        off = np.ascontiguousarray(off, np.int64)
        B = len(off) - 1
        out = np.zeros((B, self.plan.emb_dim), self.dtype)
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        self.ref.check(self.ref.lib.ref_serial_forward(
            self.h, _p(idx), C.c_int64(len(idx)), _p(off), C.c_int64(B), _p(w), C.c_int(pooling),
            _p(out)))
        return out

    def serial_backward(self, idx, off, grad_out, weights=None, pooling=0):
        idx = np.ascontiguousarray(idx, np.int64)
        off = np.ascontiguousarray(off, np.int64)
        B = len(off) - 1
        g = np.ascontiguousarray(grad_out, self.dtype)
        grads = [np.zeros(self.plan.core_size(k), self.dtype) for k in range(self.plan.tt_dim)]
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        self.ref.check(self.ref.lib.ref_serial_backward(
            self.h, _p(idx), C.c_int64(len(idx)), _p(off), C.c_int64(B), _p(w), C.c_int(pooling),
            _p(g), C.c_int64(g.size), _ptr_array(grads)))
        return grads

    def sgd(self, grads, lr):
        gs = [np.ascontiguousarray(g, self.dtype) for g in grads]
        self.ref.check(self.ref.lib.ref_sgd(self.h, _ptr_array(gs), C.c_double(lr)))

    def lookup_row(self, row):
        out = np.zeros(self.plan.emb_dim, self.dtype)
        self.ref.check(self.ref.lib.ref_lookup_row(self.h, C.c_int64(row), _p(out)))
        return out

    def reconstruct_full(self):
        p = self.plan
        rows = int(np.prod(p.row_factors))
        out = np.zeros((rows, p.emb_dim), self.dtype)
        self.ref.check(self.ref.lib.ref_reconstruct_full(self.h, _p(out)))
        return out

    def time_step(self, idx, off, grad_out, lr=0.01, reps=5, threads=0):
        idx = np.ascontiguousarray(idx, np.int64)
        off = np.ascontiguousarray(off, np.int64)
        g = np.ascontiguousarray(grad_out, np.float32)
        return self.ref.lib.ref_time_step(self.h, _p(idx), C.c_int64(len(idx)), _p(off),
                                          C.c_int64(len(off) - 1), _p(g), C.c_double(lr),
                                          C.c_int(reps), C.c_int(threads))

    def time_step_serial(self, idx, off, grad_out, lr=0.01, reps=3):
        """ref::forward_bags + ref::backward_bags + sgd_step (serial oracle)."""
        idx = np.ascontiguousarray(idx, np.int64)
        off = np.ascontiguousarray(off, np.int64)
        g = np.ascontiguousarray(grad_out, np.float32)
        return self.ref.lib.ref_time_step_serial(self.h, _p(idx), C.c_int64(len(idx)), _p(off),
                                                 C.c_int64(len(off) - 1), _p(g), C.c_double(lr),
                                                 C.c_int(reps))


class RefCache:
    """LfuCache<float> (lfu_cache.hpp:134-310) from the reference build."""

    def __init__(self, ref: RefImpl, capacity, emb_dim, refresh_period=1000):
        self.ref = ref
        h = C.c_void_p()
        ref.check(ref.lib.ref_cache_create(C.c_int64(capacity), C.c_int64(emb_dim),
                                           C.c_int64(refresh_period), C.byref(h)))
        self.h = h
        self.emb = emb_dim

    def __del__(self):
        try:
            self.ref.lib.ref_cache_destroy(self.h)
        except Exception:
            pass

    def record_and_partition(self, idx, off, weights=None, pooling=0):
        idx = np.ascontiguousarray(idx, np.int64)
        off = np.ascontiguousarray(off, np.int64)
        B = len(off) - 1
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        nc, nt = C.c_int64(), C.c_int64()
        self.ref.check(self.ref.lib.ref_cache_record_and_partition(
            self.h, _p(idx), C.c_int64(len(idx)), _p(off), C.c_int64(B), _p(w), C.c_int(pooling),
            C.byref(nc), C.byref(nt)))
        cs = np.zeros(nc.value + 1, np.int64)
        cr = np.zeros(nc.value + 1, np.int64)
        co = np.zeros(B + 1, np.int64)
        ti = np.zeros(nt.value + 1, np.int64)
        to = np.zeros(B + 1, np.int64)
        self.ref.lib.ref_cache_last_partition(self.h, _p(cs), _p(cr), _p(co), _p(ti), _p(to))
        return dict(cached_slots=cs[:nc.value], cached_rows=cr[:nc.value], cached_offsets=co,
                    tt_indices=ti[:nt.value], tt_offsets=to)

    def record(self, idx):
        idx = np.ascontiguousarray(idx, np.int64)
        self.ref.lib.ref_cache_record(self.h, _p(idx), C.c_int64(len(idx)))

    def warmup_finalize(self, table: RefTable):
        self.ref.check(self.ref.lib.ref_cache_warmup_finalize(self.h, table.h))

    def refresh(self, table: RefTable):
        d = C.c_double()
        self.ref.check(self.ref.lib.ref_cache_refresh(self.h, table.h, C.byref(d)))
        return d.value

    def hot_rows(self):
        n = self.ref.lib.ref_cache_hot_rows(self.h, None)
        out = np.zeros(n + 1, np.int64)
        self.ref.lib.ref_cache_hot_rows(self.h, _p(out))
        return out[:n]

    def slot_of(self, row):
        return int(self.ref.lib.ref_cache_slot_of(self.h, C.c_int64(row)))

    def row_values(self, slot):
        out = np.zeros(self.emb, np.float32)
        self.ref.lib.ref_cache_row_values(self.h, C.c_int64(slot), _p(out))
        return out

    def hit_rate(self):
        return float(self.ref.lib.ref_cache_hit_rate(self.h))

    def freq(self, row):
        return int(self.ref.lib.ref_cache_freq(self.h, C.c_int64(row)))

    def top_k(self, k):
        out = np.zeros(k + 1, np.int64)
        n = self.ref.lib.ref_cache_top_k(self.h, C.c_int64(k), _p(out))
        return out[:n]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class RefLayer:
    """EmbeddingLayer<float> over a TT table with an optional LFU cache
    (model.hpp:148-284) from the reference build: the reference's own
    composition of record_and_partition / forward_bags / backward_bags /
    sgd_step / cached_sgd_update / warmup_finalize / refresh."""

    def __init__(self, ref: RefImpl, plan: Plan, cache_capacity=-1, name="tt-layer"):
        self.ref, self.plan = ref, plan
        d = len(plan.row_factors)
        h = C.c_void_p()
        ref.check(ref.lib.ref_layer_create(
            C.c_int64(plan.num_rows), C.c_int64(plan.emb_dim), C.c_int(d),
            _p(np.asarray(plan.row_factors, np.int64)), _p(np.asarray(plan.col_factors, np.int64)),
            _p(np.asarray(plan.ranks, np.int64)), C.c_int64(cache_capacity), name.encode(),
            C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.ref.lib.ref_layer_destroy(self.h)
        except Exception:
            pass

    def init(self, seed):
        self.ref.check(self.ref.lib.ref_layer_init(self.h, C.c_uint64(seed)))

    def forward(self, idx, off, w=None, pooling=0):
        idx = np.ascontiguousarray(idx, np.int64)
        off = np.ascontiguousarray(off, np.int64)
        w = None if w is None else np.ascontiguousarray(w, np.float64)
        B = len(off) - 1
        out = np.zeros((B, self.plan.emb_dim), np.float32)
        self.ref.check(self.ref.lib.ref_layer_forward(self.h, _p(idx), C.c_int64(len(idx)), _p(off),
                                                      C.c_int64(B), _p(w), C.c_int(pooling), _p(out)))
        return out

    def backward(self, idx, off, grad, w=None, pooling=0):
        idx = np.ascontiguousarray(idx, np.int64)
        off = np.ascontiguousarray(off, np.int64)
        w = None if w is None else np.ascontiguousarray(w, np.float64)
        g = np.ascontiguousarray(grad, np.float32)
        self.ref.check(self.ref.lib.ref_layer_backward(
            self.h, _p(idx), C.c_int64(len(idx)), _p(off), C.c_int64(len(off) - 1), _p(w),
            C.c_int(pooling), _p(g), C.c_int64(g.size)))

    def step(self, lr):
        self.ref.check(self.ref.lib.ref_layer_step(self.h, C.c_double(lr)))

    def finalize_warmup(self):
        self.ref.check(self.ref.lib.ref_layer_finalize_warmup(self.h))

    def refresh(self):
        d = C.c_double()
        self.ref.check(self.ref.lib.ref_layer_refresh(self.h, C.byref(d)))
        return d.value

    def core(self, k):
        rf, cf, rk = self.plan.row_factors, self.plan.col_factors, self.plan.ranks
        out = np.zeros(rk[k] * rf[k] * cf[k] * rk[k + 1], np.float32)
        self.ref.lib.ref_layer_get_core(self.h, C.c_int(k), _p(out))
        return out

    def cache_info(self):
        r, a, h, act = C.c_int64(), C.c_uint64(), C.c_uint64(), C.c_int()
        self.ref.lib.ref_layer_cache_info(self.h, C.byref(r), C.byref(a), C.byref(h), C.byref(act))
        return dict(resident=r.value, accesses=a.value, hits=h.value, active=bool(act.value))

    def cache_rows(self, capacity):
        rows = np.zeros(capacity, np.int64)
        vals = np.zeros((capacity, self.plan.emb_dim), np.float32)
        self.ref.lib.ref_layer_cache_rows(self.h, _p(rows), _p(vals))
        return rows, vals

    def freq(self, row):
        return int(self.ref.lib.ref_layer_freq(self.h, C.c_int64(row)))


class RefModel:
    """DlrmModel<float> (model.hpp:355-538) from the reference build: the
    checker of the GPU DlrmModel (paper_2101_11714_b200/dlrm.py)."""

    def __init__(self, ref: RefImpl, dense_features, emb_dim, tables, bottom, top, dot=True):
        """tables: list of (rows, use_tt, rank)."""
        self.ref = ref
        self.ntables = len(tables)
        rows = np.asarray([t[0] for t in tables], np.int64)
        use_tt = np.asarray([1 if t[1] else 0 for t in tables], np.int32)
        ranks = np.asarray([t[2] for t in tables], np.int64)
        bot = np.asarray(bottom, np.int64)
        tp = np.asarray(top, np.int64)
        h = C.c_void_p()
        ref.check(ref.lib.ref_model_create(
            C.c_int64(dense_features), C.c_int64(emb_dim), C.c_int(len(tables)), _p(rows), _p(use_tt),
            _p(ranks), C.c_int(len(bot)), _p(bot), C.c_int(len(tp)), _p(tp), C.c_int(1 if dot else 0),
            C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.ref.lib.ref_model_destroy(self.h)
        except Exception:
            pass

    def init(self, seed):
        self.ref.check(self.ref.lib.ref_model_init(self.h, C.c_uint64(seed)))

    def param(self, which, index, k=0):
        """which: 0 bottom.w, 1 bottom.b, 2 top.w, 3 top.b, 4 TT core k of table, 5 dense table."""
        n = self.ref.lib.ref_model_param(self.h, C.c_int(which), C.c_int(index), C.c_int(k), None)
        if n < 0:
            raise RefError(1, self.ref.lib.ref_last_error().decode())
        out = np.zeros(n, np.float32)
        self.ref.lib.ref_model_param(self.h, C.c_int(which), C.c_int(index), C.c_int(k), _p(out))
        return out

    def step(self, mb, lr):
        """One train() iteration on a minibatch dict (dense, labels, idx, off); returns (logits, loss)."""
        bs = len(mb["labels"])
        idx = np.concatenate(mb["idx"]).astype(np.int64)
        lk = np.concatenate([[0], np.cumsum([len(i) for i in mb["idx"]])]).astype(np.int64)
        off = np.concatenate(mb["off"]).astype(np.int64)
        logits = np.zeros(bs, np.float32)
        loss = C.c_double()
        self.ref.check(self.ref.lib.ref_model_step(
            self.h, C.c_int64(bs), _p(np.ascontiguousarray(mb["dense"], np.float64)),
            _p(np.ascontiguousarray(mb["labels"], np.float64)), C.c_int(len(mb["idx"])), _p(idx), _p(lk),
            _p(off), C.c_double(lr), _p(logits), C.byref(loss)))
        return logits, loss.value


class RefSource:
    """SyntheticDataSource (data.hpp:54-90) of the reference: minibatches."""

    def __init__(self, ref: RefImpl, dense_features, rows, zipf, bs, pf, seed):
        self.ref, self.df, self.rows, self.bs, self.pf = ref, dense_features, list(rows), bs, pf
        h = C.c_void_p()
        r = np.asarray(rows, np.int64)
        ref.check(ref.lib.ref_source_create(C.c_int64(dense_features), C.c_int(len(rows)), _p(r),
                                            C.c_double(zipf), C.c_int64(bs), C.c_int64(pf),
                                            C.c_uint64(seed), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.ref.lib.ref_source_destroy(self.h)
        except Exception:
            pass

    def next(self, it):
        T, bs, pf = len(self.rows), self.bs, self.pf
        dense = np.zeros(bs * self.df, np.float64)
        labels = np.zeros(bs, np.float64)
        idx = np.zeros(T * bs * pf, np.int64)
        off = np.zeros(T * (bs + 1), np.int64)
        self.ref.check(self.ref.lib.ref_source_next(self.h, C.c_int64(it), _p(dense), _p(labels), _p(idx),
                                                    _p(off)))
        return {"dense": dense.reshape(bs, self.df), "labels": labels,
                "idx": [idx[t * bs * pf:(t + 1) * bs * pf] for t in range(T)],
                "off": [off[t * (bs + 1):(t + 1) * (bs + 1)] for t in range(T)]}
