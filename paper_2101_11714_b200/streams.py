"""Device index streams: ZipfianSampler (data.hpp:16-28)
resident on the GPU for throughput runs.  Same distribution as the
reference's sampler (its CDF, built with the reference's loop, inverted by
upper_bound on the device); the uniform variates are a counter-based
SplitMix64 stream, not the reference's mt19937_64 -- parity tests keep the
host streams (`generate_zipfian_batch`, `uniform_indices`)."""
from __future__ import annotations

import ctypes as C

from ._lib import lib
from .ttrec import _raise


class DeviceZipfSampler:
    """ZipfianSampler(population, exponent) on `device`; exponent 0 = uniform."""

    def __init__(self, population: int, exponent: float, device: int = 0, stream: int = 0):
        h = C.c_void_p()
        _raise(lib().ttgpu_sampler_create(int(population), float(exponent), int(device),
                                          C.c_void_p(stream), C.byref(h)))
        self.handle = h
        self.population = int(population)
        self.exponent = float(exponent)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                lib().ttgpu_sampler_destroy(h)
            except Exception:  # noqa: BLE001
                pass
            self.handle = None

    def set_stream(self, stream: int):
        _raise(lib().ttgpu_sampler_set_stream(self.handle, C.c_void_p(stream)))

    def draw_device(self, seed: int, counter: int, n: int, out_ptr: int):
        """n row indices (int64) into device memory; element i uses counter + i."""
        _raise(lib().ttgpu_sampler_draw_device(self.handle, C.c_uint64(seed), C.c_uint64(counter),
                                               int(n), C.c_void_p(out_ptr)))


def bag_offsets_device(bags: int, pooling_factor: int, out_ptr: int, stream: int = 0):
    """off[b] = b * pooling_factor for b in [0, bags] (fixed-size bags)."""
    _raise(lib().ttgpu_bag_offsets_device(int(bags), int(pooling_factor), C.c_void_p(out_ptr),
                                          C.c_void_p(stream)))
