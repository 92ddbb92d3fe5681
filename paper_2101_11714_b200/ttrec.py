"""Python mirror of the reference's TT-EmbeddingBag interface, backed by CUDA.

Same names, argument meanings and error behaviour as the reference C++ API
(/root/reference/proj/include/ttrec/{shape_plan,tt_table,index_batch,
embedding_ops,embedding_stats}.hpp), so parity tests read like the
reference's own tests.  Every numeric call goes through libttgpu.so's C ABI
(include/ttgpu.h); there is no CPU path.

Error mapping (common.hpp:34-52): std::invalid_argument -> InvalidArgument
(a ValueError), std::out_of_range -> OutOfRange (an IndexError),
std::runtime_error -> RuntimeFailure (a RuntimeError).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._lib import lib

kDefaultMicroBatch = 2048  # embedding_ops.hpp:20
kMinTtDim, kMaxTtDim = 2, 8  # shape_plan.hpp:11-12


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class OutOfRange(IndexError):
    """std::out_of_range"""


class RuntimeFailure(RuntimeError):
    """std::runtime_error"""


def _raise(status: int):
    if status == 0:
        return
    msg = lib().ttgpu_last_error().decode()
    if status == 2:
        raise InvalidArgument(msg)
    if status == 3:
        raise OutOfRange(msg)
    raise RuntimeFailure(msg)


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------- plans -----
@dataclass
class ShapePlan:
    """shape_plan.hpp:19-46."""

    num_rows: int = 0
    emb_dim: int = 0
    tt_dim: int = 0
    row_factors: List[int] = field(default_factory=list)
    col_factors: List[int] = field(default_factory=list)
    ranks: List[int] = field(default_factory=list)

    def _info(self):
        rf = np.asarray(self.row_factors, np.int64)
        cf = np.asarray(self.col_factors, np.int64)
        rk = np.asarray(self.ranks, np.int64)
        if len(rf) != self.tt_dim or len(cf) != self.tt_dim or len(rk) != self.tt_dim + 1:
            raise InvalidArgument(
                f"expected {self.tt_dim} row factors, {self.tt_dim} col factors and "
                f"{self.tt_dim + 1} ranks")
        out = [C.c_int64(), C.c_int64(), C.c_int64()]
        _raise(lib().ttgpu_plan_info(self.num_rows, self.emb_dim, self.tt_dim, _p(rf), _p(cf),
                                     _p(rk), *[C.byref(o) for o in out]))
        return [o.value for o in out]

    def padded_rows(self) -> int:
        return self._info()[0]

    def parameter_count(self) -> int:
        return self._info()[1]

    def memory_reduction(self) -> int:
        return self._info()[2]

    def core_size(self, k: int) -> int:
        return (self.ranks[k] * self.row_factors[k] * self.col_factors[k] * self.ranks[k + 1])

    def validate(self):
        self._info()


def plan_shapes(num_rows: int, emb_dim: int, tt_dim: int, rank: int,
                row_factors: Optional[Sequence[int]] = None,
                col_factors: Optional[Sequence[int]] = None) -> ShapePlan:
    """shape_plan.hpp:56-58 / shape_plan.cpp:142-169."""
    if tt_dim < kMinTtDim or tt_dim > kMaxTtDim:
        raise InvalidArgument(f"tt_dim must be in [{kMinTtDim}, {kMaxTtDim}], got {tt_dim}")
    rf_in = None if row_factors is None else np.asarray(row_factors, np.int64)
    cf_in = None if col_factors is None else np.asarray(col_factors, np.int64)
    if rf_in is not None and len(rf_in) != tt_dim:
        raise InvalidArgument(f"expected {tt_dim} row factors, got {len(rf_in)}")
    if cf_in is not None and len(cf_in) != tt_dim:
        raise InvalidArgument(f"expected {tt_dim} col factors, got {len(cf_in)}")
    rf, cf = np.zeros(tt_dim, np.int64), np.zeros(tt_dim, np.int64)
    rk = np.zeros(tt_dim + 1, np.int64)
    _raise(lib().ttgpu_plan_shapes(num_rows, emb_dim, tt_dim, rank, _p(rf_in), _p(cf_in), _p(rf),
                                   _p(cf), _p(rk)))
    return ShapePlan(num_rows, emb_dim, tt_dim, [int(x) for x in rf], [int(x) for x in cf],
                     [int(x) for x in rk])


def decompose_index(flat: int, radices: Sequence[int]) -> List[int]:
    r = np.asarray(radices, np.int64)
    out = np.zeros(len(r), np.int64)
    _raise(lib().ttgpu_decompose_index(flat, _p(r), len(r), _p(out)))
    return [int(x) for x in out]


def recompose_index(digits: Sequence[int], radices: Sequence[int]) -> int:
    dg = np.asarray(digits, np.int64)
    r = np.asarray(radices, np.int64)
    if len(dg) != len(r):
        raise InvalidArgument(f"digit/radix count mismatch: {len(dg)} vs {len(r)}")
    out = C.c_int64()
    _raise(lib().ttgpu_recompose_index(_p(dg), _p(r), len(r), C.byref(out)))
    return out.value


# --------------------------------------------------------------- batch -----
class Pooling(enum.IntEnum):
    Sum = 0
    Mean = 1


@dataclass
class IndexBatch:
    """index_batch.hpp:17-57: CSR bags, optional per-lookup double weights."""

    indices: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int64))
    weights: Optional[np.ndarray] = None
    pooling: Pooling = Pooling.Sum

    def __post_init__(self):
        self.indices = np.ascontiguousarray(self.indices, np.int64)
        self.offsets = np.ascontiguousarray(self.offsets, np.int64)
        if self.weights is not None:
            self.weights = np.ascontiguousarray(self.weights, np.float64)
            if self.weights.size == 0 and self.indices.size != 0:
                self.weights = None

    def num_bags(self) -> int:
        return len(self.offsets) - 1

    def num_lookups(self) -> int:
        return len(self.indices)

    def has_weights(self) -> bool:
        return self.weights is not None and self.weights.size > 0

    def weight(self, t: int) -> float:
        return 1.0 if not self.has_weights() else float(self.weights[t])

    def bag_size(self, b: int) -> int:
        return int(self.offsets[b + 1] - self.offsets[b])

    @staticmethod
    def singles(idx, pooling=Pooling.Sum) -> "IndexBatch":
        idx = np.asarray(idx, np.int64)
        return IndexBatch(idx, np.arange(len(idx) + 1, dtype=np.int64), None, pooling)

    def validate(self, num_rows: int, table_name: str = ""):
        """Structural checks (host, cheap) -- index range is checked on the GPU."""
        off = self.offsets
        if len(off) == 0 or off[0] != 0:
            raise InvalidArgument("offsets must start at 0")
        if len(off) > 1 and np.any(off[1:] < off[:-1]):
            raise InvalidArgument("offsets must be non-decreasing")
        if off[-1] != self.num_lookups():
            raise InvalidArgument(
                f"offsets end at {off[-1]} but there are {self.num_lookups()} indices")
        if self.weights is not None and len(self.weights) != self.num_lookups():
            raise InvalidArgument(
                f"expected {self.num_lookups()} weights, got {len(self.weights)}")


# --------------------------------------------------------------- table -----
class TtTable:
    """tt_table.hpp:23-102, cores resident on a GPU in the reference layout
    (m_k, R_{k-1}, n_k, R_k)."""

    def __init__(self, plan: ShapePlan, name: str = "tt-table", dtype=np.float32, device: int = 0,
                 stream: int = 0):
        self._plan = plan
        self._name = name
        self.dtype = np.dtype(dtype)
        rf = np.asarray(plan.row_factors, np.int64)
        cf = np.asarray(plan.col_factors, np.int64)
        rk = np.asarray(plan.ranks, np.int64)
        if len(rf) != plan.tt_dim or len(cf) != plan.tt_dim or len(rk) != plan.tt_dim + 1:
            plan.validate()
        h = C.c_void_p()
        _raise(lib().ttgpu_create(plan.num_rows, plan.emb_dim, plan.tt_dim, _p(rf), _p(cf), _p(rk),
                                  1 if self.dtype == np.float64 else 0, name.encode(), device,
                                  C.c_void_p(stream), C.byref(h)))
        self.handle = h
        self.device = device
        self.stream = stream  # raw cudaStream_t every call of this table is ordered on

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                lib().ttgpu_destroy(h)
            except Exception:  # noqa: BLE001
                pass
            self.handle = None

    # reference accessors
    def plan(self) -> ShapePlan:
        return self._plan

    def name(self) -> str:
        return self._name

    def dim(self) -> int:
        return self._plan.tt_dim

    def rows(self) -> int:
        return self._plan.num_rows

    def cols(self) -> int:
        return self._plan.emb_dim

    def slice_size(self, k: int) -> int:
        p = self._plan
        return p.ranks[k] * p.col_factors[k] * p.ranks[k + 1]

    def core(self, k: int) -> np.ndarray:
        """Copy of core k (TtTable::core(k) bytes)."""
        out = np.zeros(self._plan.core_size(k), self.dtype)
        _raise(lib().ttgpu_get_core(self.handle, k, _p(out)))
        return out

    def grad(self, k: int) -> np.ndarray:
        """Copy of core k's slice of the table's dense gradient buffer."""
        out = np.zeros(self._plan.core_size(k), self.dtype)
        _raise(lib().ttgpu_get_grad(self.handle, k, _p(out)))
        return out

    def cores(self) -> List[np.ndarray]:
        return [self.core(k) for k in range(self.dim())]

    def set_core(self, k: int, values):
        v = np.ascontiguousarray(values, self.dtype).ravel()
        if v.size != self._plan.core_size(k):
            raise InvalidArgument(f"core {k} has {self._plan.core_size(k)} elements, got {v.size}")
        _raise(lib().ttgpu_set_core(self.handle, k, _p(v)))

    def set_cores(self, cores):
        for k, c in enumerate(cores):
            self.set_core(k, c)

    def core_device_ptr(self, k: int) -> int:
        p = C.c_void_p()
        _raise(lib().ttgpu_core_device_ptr(self.handle, k, C.byref(p)))
        return p.value

    def grad_device_ptr(self, k: int) -> int:
        p = C.c_void_p()
        _raise(lib().ttgpu_grad_device_ptr(self.handle, k, C.byref(p)))
        return p.value

    def mutation_counter(self) -> int:
        v = C.c_uint64()
        _raise(lib().ttgpu_mutation_counter(self.handle, C.byref(v)))
        return v.value

    def mark_mutated(self):
        _raise(lib().ttgpu_mark_mutated(self.handle))

    def set_generic_path(self, on: bool):
        _raise(lib().ttgpu_set_generic_path(self.handle, int(bool(on))))

    def set_tensor_path(self, on: bool):
        """Backward head contraction on tcgen05 (3xTF32) where eligible (default on)."""
        _raise(lib().ttgpu_set_tensor_path(self.handle, int(bool(on))))

    def set_grid_sort(self, on: bool):
        """Fast path: one-kernel cooperative sort (gsort.cuh) (default on) or the three-kernel sort."""
        _raise(lib().ttgpu_set_grid_sort(self.handle, int(bool(on))))

    def set_wide3(self, on: bool):
        """d == 3 wide rows (cfg3 class): warp-per-chunk tail kernels (default on)."""
        _raise(lib().ttgpu_set_wide3(self.handle, int(bool(on))))

    def set_chunked(self, on: bool):
        """Fast path: chunked kernels (fastc.cuh) or the 32-lookup tile kernels (default)."""
        _raise(lib().ttgpu_set_chunked(self.handle, int(bool(on))))

    def fast_path_kind(self) -> int:
        k = C.c_int()
        _raise(lib().ttgpu_fast_path_kind(self.handle, C.byref(k)))
        return k.value

    def set_exact_forward(self, on: bool):
        _raise(lib().ttgpu_set_exact_forward(self.handle, int(bool(on))))

    def decompose_row(self, flat: int) -> List[int]:
        return decompose_index(flat, self._plan.row_factors)

    def init_sampled_gaussian(self, seed: int):
        """init_tt_cores(table, InitSpec::sampled_gaussian(), seed)."""
        _raise(lib().ttgpu_init_sampled_gaussian(self.handle, seed))

    def sync(self):
        _raise(lib().ttgpu_sync(self.handle))

    def check(self):
        _raise(lib().ttgpu_check(self.handle))

    # -------- device-pointer (async, graph-capturable) entry points --------
    def forward_device(self, ctx: "ForwardContext", idx_ptr: int, L: int, off_ptr: int, B: int,
                       out_ptr: int, weights_ptr: int = 0, pooling: int = 0, save: bool = False):
        _raise(lib().ttgpu_forward_device(self.handle, C.c_void_p(idx_ptr), L, C.c_void_p(off_ptr),
                                          B, C.c_void_p(weights_ptr or None), int(pooling),
                                          int(save), C.c_void_p(out_ptr), ctx.handle))
        ctx._fill(self, L, B)

    def backward_device(self, ctx: "ForwardContext", grad_ptr: int):
        _raise(lib().ttgpu_backward_device(self.handle, ctx.handle, C.c_void_p(grad_ptr)))

    def backward_sgd_device(self, ctx: "ForwardContext", grad_ptr: int, lr: float):
        _raise(lib().ttgpu_backward_sgd_device(self.handle, ctx.handle, C.c_void_p(grad_ptr), lr))

    def apply_grad(self, lr: float):
        _raise(lib().ttgpu_apply_grad(self.handle, lr))

    def backward_sgd(self, ctx: "ForwardContext", batch: IndexBatch, grad_output, lr: float):
        """Host-pointer fused backward_bags + sgd_step (no dense gradient)."""
        g = np.ascontiguousarray(grad_output, self.dtype).ravel()
        _raise(lib().ttgpu_backward_sgd(self.handle, ctx.handle, batch.num_lookups(),
                                        batch.num_bags(), _p(g), g.size, lr))

    def grad_buffer(self):
        """(device pointer, element count) of the dense gradient of all cores."""
        p, n = C.c_void_p(), C.c_int64()
        _raise(lib().ttgpu_grad_buffer(self.handle, C.byref(p), C.byref(n)))
        return p.value, n.value

    def set_stream(self, stream: int):
        _raise(lib().ttgpu_set_stream(self.handle, C.c_void_p(stream or None)))
        self.stream = stream or 0

    def graph_begin(self):
        _raise(lib().ttgpu_graph_begin(self.handle))

    def graph_end(self):
        kn, tn = C.c_int(), C.c_int()
        _raise(lib().ttgpu_graph_end(self.handle, C.byref(kn), C.byref(tn)))
        return kn.value, tn.value

    def graph_launch(self):
        _raise(lib().ttgpu_graph_launch(self.handle))

    def profile(self, on: bool):
        _raise(lib().ttgpu_profile(self.handle, int(bool(on))))

    def profile_read(self):
        names = C.create_string_buffer(4096)
        ms = (C.c_float * 64)()
        n = C.c_int()
        _raise(lib().ttgpu_profile_read(self.handle, names, 4096, ms, 64, C.byref(n)))
        labels = names.value.decode().split(";")[: n.value]
        return list(zip(labels, [float(ms[i]) for i in range(n.value)]))

    def lookup_rows_device(self, rows_ptr: int, n: int, out_ptr: int):
        _raise(lib().ttgpu_lookup_rows_device(self.handle, C.c_void_p(rows_ptr), n,
                                              C.c_void_p(out_ptr)))


class ForwardContext:
    """embedding_ops.hpp:101-110; owns the device-side saved state."""

    def __init__(self, table: TtTable):
        h = C.c_void_p()
        _raise(lib().ttgpu_ctx_create(table.handle, C.byref(h)))
        self.handle = h
        self.table = table
        self.num_lookups = 0
        self.num_bags = 0
        self.saved = False

    def _fill(self, table, L, B, saved=False):
        self.table = table
        self.num_lookups = L
        self.num_bags = B
        self.saved = saved

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                lib().ttgpu_ctx_destroy(h)
            except Exception:  # noqa: BLE001
                pass
            self.handle = None


@dataclass
class ForwardResult:
    output: np.ndarray
    context: ForwardContext


@dataclass
class CoreGradients:
    """embedding_ops.hpp:68-94: dense per-core gradients in core layout."""

    cores: List[np.ndarray]

    @staticmethod
    def zeros_like(table: TtTable) -> "CoreGradients":
        return CoreGradients([np.zeros(table.plan().core_size(k), table.dtype)
                              for k in range(table.dim())])

    def add(self, other: "CoreGradients"):
        for a, b in zip(self.cores, other.cores):
            a += b

    def total_elements(self) -> int:
        return int(sum(c.size for c in self.cores))


# ----------------------------------------------------------- operators -----
def forward_bags(table: TtTable, batch: IndexBatch, micro_batch: int = kDefaultMicroBatch,
                 save_intermediates: bool = False) -> ForwardResult:
    """embedding_ops.hpp:159-253."""
    batch.validate(table.rows(), table.name())
    if micro_batch < 1:
        raise InvalidArgument(f"micro_batch must be positive, got {micro_batch}")
    B, L = batch.num_bags(), batch.num_lookups()
    out = np.zeros((B, table.cols()), table.dtype)
    ctx = ForwardContext(table)
    w = batch.weights if batch.has_weights() else None
    _raise(lib().ttgpu_forward(table.handle, _p(batch.indices), L, _p(batch.offsets), B, _p(w),
                               int(batch.pooling), micro_batch, int(save_intermediates), _p(out),
                               ctx.handle))
    ctx._fill(table, L, B, bool(save_intermediates))
    return ForwardResult(out, ctx)


def backward_bags(table: TtTable, batch: IndexBatch, ctx: ForwardContext,
                  grad_output) -> CoreGradients:
    """embedding_ops.hpp:260-358; the C ABI enforces the reference's checks
    (:264-274): table identity, batch counts, stale snapshot, grad size."""
    batch.validate(table.rows(), table.name())
    g = np.ascontiguousarray(grad_output, table.dtype).ravel()
    grads = CoreGradients.zeros_like(table)
    ptrs = (C.c_void_p * table.dim())(*[c.ctypes.data_as(C.c_void_p) for c in grads.cores])
    if ctx.table is not table:
        raise InvalidArgument("forward context belongs to a different table")
    _raise(lib().ttgpu_backward(table.handle, ctx.handle, batch.num_lookups(), batch.num_bags(),
                                _p(g), g.size, ptrs))
    return grads


def sgd_step(table: TtTable, grads: CoreGradients, lr: float):
    """embedding_ops.hpp:361-376: core -= T(lr) * grad; bumps the mutation counter."""
    if len(grads.cores) != table.dim():
        raise InvalidArgument("gradient core count mismatch")
    gs = []
    for k, c in enumerate(grads.cores):
        c = np.ascontiguousarray(c, table.dtype)
        if c.size != table.plan().core_size(k):
            raise InvalidArgument(f"gradient shape mismatch on core {k}")
        gs.append(c)
    ptrs = (C.c_void_p * table.dim())(*[c.ctypes.data_as(C.c_void_p) for c in gs])
    _raise(lib().ttgpu_sgd_step(table.handle, ptrs, lr))


def lookup_row(table: TtTable, row: int) -> np.ndarray:
    """embedding_ops.hpp:120-152 (bit-identical to the reference)."""
    out = np.zeros(table.cols(), table.dtype)
    _raise(lib().ttgpu_lookup_row(table.handle, int(row), _p(out)))
    return out


class EmbeddingStats:
    """embedding_stats.hpp:12-23 (row counter shared by all tables)."""

    @staticmethod
    def reset():
        lib().ttgpu_stats_reset()

    @staticmethod
    def tt_rows_computed() -> int:
        return int(lib().ttgpu_stats_rows())

    @staticmethod
    def add_rows(n: int):
        lib().ttgpu_stats_add_rows(n)

    @staticmethod
    def peak_workspace_bytes() -> int:
        return int(lib().ttgpu_stats_peak_workspace())


# ------------------------------------------------------ synthetic data -----
def generate_zipfian_batch(population: int, exponent: float, seed: int, num_bags: int,
                           pooling_factor: int, pooling: Pooling = Pooling.Sum) -> IndexBatch:
    """ZipfianSampler + generate_zipfian_batch with Rng(seed) (data.cpp:8-47)."""
    idx = np.zeros(num_bags * pooling_factor, np.int64)
    off = np.zeros(num_bags + 1, np.int64)
    _raise(lib().ttgpu_zipf_batch(population, exponent, seed, num_bags, pooling_factor, _p(idx),
                                  _p(off)))
    return IndexBatch(idx, off, None, pooling)


def uniform_indices(rows: int, seed: int, n: int) -> np.ndarray:
    """Rng(seed).uniform_int(0, rows) x n (rng.hpp:47-51)."""
    out = np.zeros(n, np.int64)
    _raise(lib().ttgpu_uniform_indices(rows, seed, n, _p(out)))
    return out


def derived_uniform_indices(rows: int, seed: int, stream: int, n: int) -> np.ndarray:
    """Rng::derive(seed, stream).uniform_int(0, rows) x n (rng.hpp:25-29,47-51)."""
    out = np.zeros(n, np.int64)
    _raise(lib().ttgpu_derived_uniform_indices(rows, seed, stream, n, _p(out)))
    return out
