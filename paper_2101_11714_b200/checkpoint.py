"""TTRECV01 checkpoints for device-resident TT tables.

Byte-compatible with the reference's `Checkpoint` (checkpoint.hpp:25-116,
src/checkpoint.cpp:1-217): 8-byte magic "TTRECV01", u64-LE header length, the
compact JSON header nlohmann::json::dump() writes (keys sorted, no spaces),
then the raw little-endian data section -- cores in table order, then arrays.
Cores are stored in the physical `row_digit_major` layout (m_k, R_{k-1}, n_k,
R_k), which is exactly the device layout of `TtTable` here, so put_table /
get_table are one device<->host copy per core and a GPU-trained table
round-trips bit-exactly through the reference's loader (and vice versa).
Errors follow the reference: structural problems raise RuntimeFailure
(`require`/`fail`), duplicate names and bad array shapes raise
InvalidArgument (`require_arg`).
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .ttrec import InvalidArgument, RuntimeFailure, ShapePlan, TtTable

MAGIC = b"TTRECV01"
_DT = {"f32": np.dtype("<f4"), "f64": np.dtype("<f8")}


def _dtype_name(dt) -> str:
    dt = np.dtype(dt)
    if dt == np.float32:
        return "f32"
    if dt == np.float64:
        return "f64"
    raise InvalidArgument(f"unsupported dtype {dt}")


def _require(ok: bool, *msg):
    if not ok:
        raise RuntimeFailure("".join(str(m) for m in msg))


def _require_arg(ok: bool, *msg):
    if not ok:
        raise InvalidArgument("".join(str(m) for m in msg))


@dataclass
class Blob:
    name: str
    dtype: str
    shape: List[int]
    data: bytes


@dataclass
class TableEntry:
    name: str
    dtype: str
    plan: ShapePlan
    cores: List[bytes] = field(default_factory=list)


def _plan_json(p: ShapePlan) -> dict:
    return {"num_rows": int(p.num_rows), "emb_dim": int(p.emb_dim), "tt_dim": int(p.tt_dim),
            "row_factors": [int(x) for x in p.row_factors],
            "col_factors": [int(x) for x in p.col_factors], "ranks": [int(x) for x in p.ranks]}


def _plan_from_json(j: dict) -> ShapePlan:
    p = ShapePlan(int(j["num_rows"]), int(j["emb_dim"]), int(j["tt_dim"]),
                  [int(x) for x in j["row_factors"]], [int(x) for x in j["col_factors"]],
                  [int(x) for x in j["ranks"]])
    p.validate()
    return p


def _dump(obj, indent: Optional[int] = None) -> str:
    """nlohmann::json::dump(): object keys in std::map (byte) order, compact
    separators, UTF-8 strings unescaped."""
    if indent is None:
        return json.dumps(obj, sort_keys=True, separators=(",", ":"), ensure_ascii=False)
    return json.dumps(obj, sort_keys=True, indent=indent, ensure_ascii=False)


class Checkpoint:
    """checkpoint.hpp:25-116."""

    def __init__(self):
        self._tables: List[TableEntry] = []
        self._arrays: List[Blob] = []

    # ---- tables -----------------------------------------------------------
    def put_table(self, table: TtTable):
        """put_table (checkpoint.hpp:40-52): the device cores, byte images."""
        e = TableEntry(table.name(), _dtype_name(table.dtype), table.plan(),
                       [np.ascontiguousarray(table.core(k), _DT[_dtype_name(table.dtype)]).tobytes()
                        for k in range(table.dim())])
        _require_arg(not self.has_table(e.name), "duplicate table name '", e.name, "'")
        self._tables.append(e)

    def put_cores(self, name: str, plan: ShapePlan, cores, dtype=np.float32):
        """put_table from host core images (same bytes as TtTable::core(k))."""
        dt = _dtype_name(dtype)
        plan.validate()
        _require_arg(len(cores) == plan.tt_dim, "table '", name, "' needs ", plan.tt_dim, " cores")
        imgs = []
        for k, c in enumerate(cores):
            c = np.ascontiguousarray(c, _DT[dt]).ravel()
            _require_arg(c.size == plan.core_size(k), "core ", k, " of table '", name, "' has ",
                         c.size, " elements, expected ", plan.core_size(k))
            imgs.append(c.tobytes())
        _require_arg(not self.has_table(name), "duplicate table name '", name, "'")
        self._tables.append(TableEntry(name, dt, plan, imgs))

    def get_cores(self, name: str, dtype=np.float32) -> List[np.ndarray]:
        """The stored cores of a table as host arrays (core layout)."""
        e = self._find_table(name)
        want = _dtype_name(dtype)
        _require(e.dtype == want, "table '", name, "' stored as ", e.dtype, ", requested ", want)
        return [np.frombuffer(c, _DT[want]).copy() for c in e.cores]

    def get_table(self, name: str, dtype=np.float32, device: int = 0, stream: int = 0) -> TtTable:
        """get_table<T> (checkpoint.hpp:54-70): a new device table holding the
        stored cores (mutation counter bumped, as TtTable::mark_mutated)."""
        e = self._find_table(name)
        want = _dtype_name(dtype)
        _require(e.dtype == want, "table '", name, "' stored as ", e.dtype, ", requested ", want)
        t = TtTable(e.plan, e.name, np.dtype(dtype), device=device, stream=stream)
        cores = []
        for k in range(e.plan.tt_dim):
            n = e.plan.core_size(k)
            _require(len(e.cores[k]) == n * _DT[want].itemsize, "core ", k, " of table '", name,
                     "' has ", len(e.cores[k]), " bytes, expected ", n * _DT[want].itemsize)
            cores.append(np.frombuffer(e.cores[k], _DT[want]).copy())
        t.set_cores(cores)
        return t

    # ---- arrays -----------------------------------------------------------
    def put_array(self, name: str, shape, values):
        """put_array<T> (checkpoint.hpp:72-84)."""
        values = np.asarray(values)
        dt = _dtype_name(values.dtype)
        shape = [int(s) for s in shape]
        n = int(np.prod(shape)) if shape else 1
        _require_arg(n == values.size, "array '", name, "' shape holds ", n, " elements but ",
                     values.size, " were given")
        _require_arg(not self.has_array(name), "duplicate array name '", name, "'")
        self._arrays.append(Blob(name, dt, shape,
                                 np.ascontiguousarray(values, _DT[dt]).ravel().tobytes()))

    def get_array(self, name: str, dtype=np.float32) -> np.ndarray:
        """get_array<T> (checkpoint.hpp:86-94): flat values."""
        b = self._find_array(name)
        want = _dtype_name(dtype)
        _require(b.dtype == want, "array '", name, "' stored as ", b.dtype, ", requested ", want)
        return np.frombuffer(b.data, _DT[want]).copy()

    def has_table(self, name: str) -> bool:
        return any(t.name == name for t in self._tables)

    def has_array(self, name: str) -> bool:
        return any(a.name == name for a in self._arrays)

    def tables(self) -> List[TableEntry]:
        return self._tables

    def arrays(self) -> List[Blob]:
        return self._arrays

    def _find_table(self, name: str) -> TableEntry:
        for t in self._tables:
            if t.name == name:
                return t
        raise RuntimeFailure(f"checkpoint has no table named '{name}'")

    def _find_array(self, name: str) -> Blob:
        for a in self._arrays:
            if a.name == name:
                return a
        raise RuntimeFailure(f"checkpoint has no array named '{name}'")

    # ---- serialisation (src/checkpoint.cpp) -------------------------------
    def _header(self) -> dict:
        """build_header (checkpoint.cpp:44-83): offsets in storage order."""
        off = 0
        tables = []
        for t in self._tables:
            cores = []
            for c in t.cores:
                cores.append({"offset": off, "bytes": len(c)})
                off += len(c)
            tables.append({"name": t.name, "dtype": t.dtype, "plan": _plan_json(t.plan),
                           "cores": cores})
        arrays = []
        for a in self._arrays:
            arrays.append({"name": a.name, "dtype": a.dtype, "shape": a.shape, "offset": off,
                           "bytes": len(a.data)})
            off += len(a.data)
        return {"format": MAGIC.decode(), "layout": "row_digit_major", "tables": tables,
                "arrays": arrays, "data_bytes": off}

    def header_json(self, indent: int = 2) -> str:
        return _dump(self._header(), indent)

    def save(self, path: str):
        """Checkpoint::save (checkpoint.cpp:129-145)."""
        header = _dump(self._header()).encode("utf-8")
        try:
            with open(path, "wb") as f:
                f.write(MAGIC)
                f.write(struct.pack("<Q", len(header)))
                f.write(header)
                for t in self._tables:
                    for c in t.cores:
                        f.write(c)
                for a in self._arrays:
                    f.write(a.data)
        except OSError as e:
            raise RuntimeFailure(f"cannot open '{path}' for writing") from e

    @staticmethod
    def load(path: str) -> "Checkpoint":
        """Checkpoint::load (checkpoint.cpp:147-215), same checks and messages."""
        try:
            f = open(path, "rb")
        except OSError as e:
            raise RuntimeFailure(f"cannot open '{path}'") from e
        with f:
            magic = f.read(8)
            _require(magic == MAGIC, "'", path, "' is not a TTRECV01 checkpoint")
            raw = f.read(8)
            _require(len(raw) == 8, "corrupt header length in '", path, "'")
            (n,) = struct.unpack("<Q", raw)
            _require(0 < n < (1 << 32), "corrupt header length in '", path, "'")
            header = f.read(n)
            _require(len(header) == n, "truncated header in '", path, "'")
            try:
                j = json.loads(header.decode("utf-8"))
            except (ValueError, UnicodeDecodeError) as e:
                raise RuntimeFailure(f"corrupt header JSON in '{path}': {e}") from e
            _require(j.get("format", "") == MAGIC.decode(), "bad format tag in '", path, "'")
            data_bytes = int(j["data_bytes"])
            data = f.read(data_bytes)
            _require(len(data) == data_bytes, "truncated data section in '", path, "'")

        def take(offset: int, nbytes: int) -> bytes:
            _require(offset + nbytes <= data_bytes, "segment [", offset, ", ", offset + nbytes,
                     ") outside data section of '", path, "'")
            return data[offset: offset + nbytes]

        cp = Checkpoint()
        for jt in j["tables"]:
            dt = jt["dtype"]
            _require(dt in _DT, "unknown dtype '", dt, "' in '", path, "'")
            plan = _plan_from_json(jt["plan"])
            elem = _DT[dt].itemsize
            jc = jt["cores"]
            _require(len(jc) == plan.tt_dim, "table '", jt["name"], "' lists ", len(jc),
                     " cores, plan needs ", plan.tt_dim)
            e = TableEntry(jt["name"], dt, plan)
            for k in range(plan.tt_dim):
                nb = int(jc[k]["bytes"])
                _require(nb == plan.core_size(k) * elem, "core ", k, " of '", e.name, "' has ",
                         nb, " bytes, plan needs ", plan.core_size(k) * elem)
                e.cores.append(take(int(jc[k]["offset"]), nb))
            _require_arg(not cp.has_table(e.name), "duplicate table name '", e.name, "'")
            cp._tables.append(e)
        for ja in j["arrays"]:
            dt = ja["dtype"]
            _require(dt in _DT, "unknown dtype '", dt, "' in '", path, "'")
            shape = [int(s) for s in ja["shape"]]
            n = int(np.prod(shape)) if shape else 1
            nb = int(ja["bytes"])
            _require(nb == n * _DT[dt].itemsize, "array '", ja["name"], "' has ", nb,
                     " bytes, shape needs ", n * _DT[dt].itemsize)
            _require_arg(not cp.has_array(ja["name"]), "duplicate array name '", ja["name"], "'")
            cp._arrays.append(Blob(ja["name"], dt, shape, take(int(ja["offset"]), nb)))
        return cp
