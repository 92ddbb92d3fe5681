"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's LFU cache
routing and admission; never imported by the product.

Follows proj/include/ttrec/lfu_cache.hpp and proj/src/lfu_cache.cpp:
  * record_and_partition (lfu_cache.hpp:187-219): every lookup bumps its
    row's count; in the Active phase it counts an access, and a resident row
    is a hit routed to the cached part (slot id), the rest to the chain part;
    both parts keep every bag, stable order;
  * top_k (lfu_cache.cpp:98-111): (count desc, row asc);
  * admit (lfu_cache.hpp:266-296): slot i = i-th hottest row; retained rows keep
    their values, new rows take lookup_row(table, row);
  * warmup_finalize / refresh (:223-243) and hot_set_drift (lfu_cache.cpp:113-126).
Pinned against the reference's own outputs in tests/golden/cache_case.npz and
cache_train{2,3}.npz (tests/test_cache_oracle.py).
"""
from __future__ import annotations

from collections import defaultdict

import numpy as np


def hot_set_drift(prev, cur, k):
    a, b = set(int(x) for x in prev), set(int(x) for x in cur)
    return len(a ^ b) / (2.0 * k)


class LfuOracle:
    def __init__(self, capacity: int, emb_dim: int):
        self.capacity, self.emb = capacity, emb_dim
        self.counts = defaultdict(int)
        self.active = False
        self.slot_of = {}
        self.slot_rows = [-1] * capacity
        self.store = np.zeros((capacity, emb_dim), np.float32)
        self.accesses = 0
        self.hits = 0
        self.prev_top = []

    def record(self, idx):
        for r in np.asarray(idx, np.int64):
            self.counts[int(r)] += 1

    def record_and_partition(self, idx, off, weights=None):
        idx = np.asarray(idx, np.int64)
        c_slots, c_rows, c_off, c_w = [], [], [0], []
        t_idx, t_off, t_w = [], [0], []
        for b in range(len(off) - 1):
            for t in range(int(off[b]), int(off[b + 1])):
                row = int(idx[t])
                self.counts[row] += 1
                slot = -1
                if self.active:
                    self.accesses += 1
                    slot = self.slot_of.get(row, -1)
                    if slot >= 0:
                        self.hits += 1
                if slot >= 0:
                    c_slots.append(slot)
                    c_rows.append(row)
                    if weights is not None:
                        c_w.append(weights[t])
                else:
                    t_idx.append(row)
                    if weights is not None:
                        t_w.append(weights[t])
            c_off.append(len(c_slots))
            t_off.append(len(t_idx))
        return dict(cached_slots=np.array(c_slots, np.int64), cached_rows=np.array(c_rows, np.int64),
                    cached_offsets=np.array(c_off, np.int64), tt_indices=np.array(t_idx, np.int64),
                    tt_offsets=np.array(t_off, np.int64),
                    cached_weights=np.array(c_w) if weights is not None else None,
                    tt_weights=np.array(t_w) if weights is not None else None)

    def top_k(self, k):
        items = sorted(self.counts.items(), key=lambda e: (-e[1], e[0]))
        return [r for r, _ in items[:k]]

    def admit(self, lookup_row):
        rows = self.top_k(self.capacity)
        store = np.zeros_like(self.store)
        slot_rows = [-1] * self.capacity
        fresh = 0
        for i, row in enumerate(rows):
            old = self.slot_of.get(row, -1)
            if old >= 0:
                store[i] = self.store[old]
            else:
                store[i] = lookup_row(row) if lookup_row is not None else 0.0
                fresh += 1
            slot_rows[i] = row
        self.store, self.slot_rows = store, slot_rows
        self.slot_of = {r: i for i, r in enumerate(rows)}
        return fresh

    def hot_rows(self):
        return sorted(r for r in self.slot_rows if r >= 0)

    def warmup_finalize(self, lookup_row=None):
        assert not self.active, "cache already active"
        self.admit(lookup_row)
        self.prev_top = self.hot_rows()
        self.active = True

    def refresh(self, lookup_row=None):
        assert self.active, "refresh before warmup_finalize"
        self.admit(lookup_row)
        cur = self.hot_rows()
        d = hot_set_drift(self.prev_top, cur, self.capacity)
        self.prev_top = cur
        return d
