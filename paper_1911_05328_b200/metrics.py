"""Run metrics (reference metrics.py:19-153), filled from the device counters.

The reference measures per-depth concurrency of Python tasks (task_enter /
base_enter, metrics.py:63-95); on the GPU the concurrent units are persistent
CTAs executing leaf tasks (output tile x k-slice), and the same quantity is
MEASURED by a device gauge: thread 0 of a CTA counts its leaf in and out with
atomics and the maximum in flight is kept (csrc/common.cuh leaf_enter /
leaf_exit).  base_case_max is that observed maximum (the busy-leaves bound of
SPEC.md:566 asks it to stay <= p, here the persistent workers); per_depth_max
keys it by the split depth the leaves ran at.  Also reported: the tile-slot
serialisations (atomic-madd merges), SAR pair states / transitions, lazy
temporary acquisitions and the pool counters.  The opt-in tcgen05 paths and the
ordered (min,+) kernel carry no gauge and report 0.
"""
from __future__ import annotations

import threading
from dataclasses import asdict, dataclass, field

__all__ = ["Metrics", "MetricsSnapshot"]


@dataclass
class MetricsSnapshot:
    per_depth_max: dict = field(default_factory=dict)
    base_case_max: int = 0
    pool_high_water_bytes: int = 0
    pool_fresh_count: int = 0
    pool_reuse_count: int = 0
    tile_serializations: int = 0
    pair_transitions: int = 0
    pair_count: int = 0
    lazy_temp_acquires: int = 0
    raw_alloc_count: int = 0
    raw_alloc_elements: int = 0
    # GPU additions
    ksplit: int = 1
    tar_levels: int = 0
    tasks: int = 0
    kernel_launches: int = 0
    path: str = ""

    def to_dict(self):
        d = asdict(self)
        d["per_depth_max"] = {str(k): v for k, v in sorted(self.per_depth_max.items())}
        return d


class Metrics:
    """Counters of one executor, accumulated over its runs."""

    def __init__(self):
        self._lock = threading.Lock()
        self.running = False
        self._zero()

    def _zero(self):
        self.base_case_max = 0
        self.tile_serializations = 0
        self.pair_count = 0
        self.pair_transitions = 0
        self.lazy_temp_acquires = 0
        self.raw_alloc_count = 0
        self.raw_alloc_elements = 0
        self.per_depth_max = {}
        self.last = {}

    def absorb_device(self, st: dict, elem_bytes: int) -> None:
        with self._lock:
            live = st.get("live_leaves_max", 0)
            self.base_case_max = max(self.base_case_max, live)
            self.tile_serializations += st["tile_serializations"]
            self.pair_count += st["pair_count"]
            self.pair_transitions += st["pair_transitions"]
            self.lazy_temp_acquires += st["lazy_temp_acquires"]
            self.raw_alloc_count += st["raw_alloc_count"]
            self.raw_alloc_elements += st["raw_alloc_bytes"] // max(1, elem_bytes)
            depth = st["ksplit"].bit_length() - 1
            self.per_depth_max[depth] = max(self.per_depth_max.get(depth, 0), live)
            self.last = dict(st)

    def count_serialization(self, n=1):
        with self._lock:
            self.tile_serializations += n

    def reset(self):
        with self._lock:
            self._zero()

    def snapshot(self, pool=None) -> MetricsSnapshot:
        with self._lock:
            snap = MetricsSnapshot(
                per_depth_max=dict(self.per_depth_max),
                base_case_max=self.base_case_max,
                tile_serializations=self.tile_serializations,
                pair_transitions=self.pair_transitions,
                pair_count=self.pair_count,
                lazy_temp_acquires=self.lazy_temp_acquires,
                raw_alloc_count=self.raw_alloc_count,
                raw_alloc_elements=self.raw_alloc_elements,
                ksplit=self.last.get("ksplit", 1),
                tar_levels=self.last.get("tar_levels", 0),
                tasks=self.last.get("tasks", 0),
                kernel_launches=self.last.get("kernel_launches", 0),
                path=self.last.get("path_name", ""),
            )
        if pool is not None:
            c = pool.snapshot_counts()
            snap.pool_high_water_bytes = c["high_water_bytes"]
            snap.pool_fresh_count = c["fresh_count"]
            snap.pool_reuse_count = c["reuse_count"]
        return snap
