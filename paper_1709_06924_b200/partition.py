"""Overlapping-decomposition bookkeeping of the reference (drop-in for `scvtmesh.partition`).

The reference evaluates a covering's Voronoi-sort regions on a worker pool (partition.py,
pipeline.py:62-98, 171-242).  Its moments equal the global path's bitwise (SURVEY.md §6.3,
DECISIONS.md D8), so the GPU evaluator always runs the global path; what a covering still
changes is the optimizer's reset rule: every evaluation classifies how far the points moved
from the cells they were assigned to when the decomposition was frozen
(`detect_migration`), and an "out-of-range" move makes `minimize` re-decompose and clear the
LBFGS history (optimizer.py:377-381).  `MeshEvaluator(covering=...)` reproduces that
classification on the device (C ABI `scvt_migration`); this module holds the covering itself
and the host forms of the reference's helpers.
"""

from __future__ import annotations

import logging
import warnings
from dataclasses import dataclass

import numpy as np

from .density import DensityField, sample_by_density
from .errors import UnderfilledPartitionWarning
from .geometry import normalize

logger = logging.getLogger(__name__)

MIN_POINTS_PER_CELL = 16     # partition.py:27


@dataclass(frozen=True)
class Covering:
    """partition.py:30-50: cell centres with one- and two-level neighbour lists."""

    centers: np.ndarray        # (p, 3)
    one_level: tuple           # p tuples of adjacent cell indices
    two_level: tuple           # p tuples incl. the cell itself and 2-hop neighbours

    @property
    def cell_count(self) -> int:
        return len(self.centers)

    def region_cells(self, l: int) -> np.ndarray:
        return np.asarray((l,) + tuple(self.one_level[l]), dtype=int)

    def disk_radius(self, l: int) -> float:
        c = self.centers[l]
        nb = self.centers[list(self.one_level[l])]
        cosang = np.clip(nb @ c, -1.0, 1.0)
        sinang = np.linalg.norm(np.cross(nb, c), axis=1)
        return float(np.arctan2(sinang, cosang).max())

    def adjacency_bitmap(self) -> np.ndarray:
        """Row-major p x ceil(p/32) uint32 bitmap of the one-level lists (scvt_migration)."""
        p = self.cell_count
        words = (p + 31) // 32
        bits = np.zeros((p, words), dtype=np.uint32)
        for a, nbrs in enumerate(self.one_level):
            for b in nbrs:
                bits[a, b >> 5] |= np.uint32(1) << np.uint32(b & 31)
        return bits


@dataclass(frozen=True)
class PointAssignment:
    """partition.py:53-58: arithmetic (frozen owner) and geometric (current nearest) cells."""

    arithmetic: np.ndarray
    geometric: np.ndarray


def nearest_cell(points, centers) -> np.ndarray:
    """partition.py:61-64 (host form; the evaluator computes it on the device)."""
    scores = np.asarray(points, dtype=float) @ np.asarray(centers, dtype=float).T
    return np.argmax(scores, axis=1)


def assign_points(points, cov: Covering, arithmetic=None) -> PointAssignment:
    """partition.py:123-144."""
    points = np.asarray(points, dtype=float)
    if len(points) < MIN_POINTS_PER_CELL * cov.cell_count:
        warnings.warn(f"{len(points)} points over {cov.cell_count} partition cells is below the "
                      f"{MIN_POINTS_PER_CELL}x floor; triangulation coverage may fail",
                      UnderfilledPartitionWarning, stacklevel=2)
    geometric = nearest_cell(points, cov.centers)
    arithmetic = geometric.copy() if arithmetic is None else np.asarray(arithmetic).copy()
    return PointAssignment(arithmetic=arithmetic, geometric=geometric)


MIGRATION_CLASSES = ("in-place", "neighbor-move", "out-of-range")


def detect_migration(assign: PointAssignment, cov: Covering) -> str:
    """partition.py:147-164 (host form of the device classification)."""
    moved = assign.geometric != assign.arithmetic
    if not np.any(moved):
        return "in-place"
    for i in np.flatnonzero(moved):
        if assign.geometric[i] not in cov.one_level[assign.arithmetic[i]]:
            return "out-of-range"
    return "neighbor-move"


def neighbor_lists(triangles, p: int):
    """partition.py:67-80: one-level (Delaunay adjacency) and two-level lists."""
    adj = [set() for _ in range(p)]
    for a, b, c in np.asarray(triangles):
        adj[a].update((b, c))
        adj[b].update((a, c))
        adj[c].update((a, b))
    one = tuple(tuple(sorted(int(x) for x in s)) for s in adj)
    two = []
    for l in range(p):
        reach = {l} | set(one[l])
        for m in one[l]:
            reach |= set(one[m])
        two.append(tuple(sorted(reach)))
    return one, tuple(two)


def bootstrap_partition_cvt(p: int, seed: int, density: DensityField | None = None,
                            movement_tol: float = 1e-3, max_iterations: int = 200) -> Covering:
    """partition.py:83-120: coarse density-matched CVT of p cells by Lloyd iterations.  Each
    Lloyd step (Delaunay, fans, 4-point cell quadrature, normalised first moments) runs on the
    GPU evaluator; the centres agree with the reference's to rounding (~1e-15)."""
    from .pipeline import MeshEvaluator

    if p < 2:
        raise ValueError("need at least 2 partition cells")
    if density is None:
        density = DensityField(variant="const")
    centers = sample_by_density(density, p, seed)
    if p < 4:
        allcells = tuple(range(p))
        one = tuple(tuple(m for m in allcells if m != l) for l in range(p))
        return Covering(centers=centers, one_level=one, two_level=(allcells,) * p)
    with MeshEvaluator(density, "4pt") as ev:
        for it in range(max_iterations):
            new = normalize(ev.evaluate(centers).first)
            movement = np.abs(new - centers).max()
            centers = new
            if movement <= movement_tol:
                logger.debug("partition CVT converged after %d Lloyd steps", it + 1)
                break
        tri = ev.triangulation(centers)
    one, two = neighbor_lists(tri.triangles, p)
    return Covering(centers=centers, one_level=one, two_level=two)


__all__ = ["Covering", "PointAssignment", "nearest_cell", "assign_points", "detect_migration",
           "neighbor_lists", "bootstrap_partition_cvt", "MIGRATION_CLASSES"]
