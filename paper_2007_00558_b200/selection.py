"""Reference-view selection (host side, k <= 16 cameras).

Same ranking and error behaviour as ``fvv.transport.select_cameras`` /
``select_references`` (``/root/reference/pkg/src/fvv/transport.py:205-238``):
cameras are ranked by (centre distance to the virtual pose, [not currently
active], id); asking for more references than the active set holds raises
``ValueError``.
"""

from __future__ import annotations

from typing import Iterable, List, Optional, Sequence

from .geometry import camera_distance


def select_cameras(virtual, rig: Sequence, n_tx: int,
                   current: Optional[Iterable[int]] = None) -> List[int]:
    """The ``n_tx`` cameras nearest ``virtual``; ties prefer active, then low id."""
    if not (1 <= n_tx <= len(rig)):
        raise ValueError(f"n_tx must be in [1, {len(rig)}]")
    active = set(current) if current is not None else set()

    def rank(c):
        return (camera_distance(c.pose, virtual), c.id not in active, c.id)

    return [c.id for c in sorted(rig, key=rank)[:n_tx]]


def select_references(virtual, rig: Sequence, active: Iterable[int], k: int) -> List[int]:
    """The ``k`` nearest cameras of ``active`` (always a subset of it)."""
    act = set(active)
    pool = [c for c in rig if c.id in act]
    if k > len(pool):
        raise ValueError(f"k={k} exceeds active set size {len(pool)}")
    pool.sort(key=lambda c: (camera_distance(c.pose, virtual), c.id))
    return [c.id for c in pool[:k]]
