"""Rank-local x-slabs of config 5 for the native (C++) slab driver
(csrc/pbdr_slab.cu, pbdr_gpu_slab_* in include/pbdr_gpu.h).

Config 5 numbers its cubes x-major, so rank r's slab -- x-columns
[r*c, (r+1)*c) of a gx * gy * gz grid -- plus `ghost_cols` columns on each side
is one contiguous range of the global bodies. Each rank generates only that
range (pbdr_scene_generate_c5_slab: the same cubes as the whole grid) and
simulates it with the driver: owned = com_x in the slab, ghosts refreshed
over NCCL (one rank per GPU) or a local hub (thread ranks on one GPU).

Weak scaling: the per-GPU slab is fixed and the grid
grows with the rank count -- gx = columns_per_rank * world.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import pbdr as P

PITCH = 0.2


@dataclass(frozen=True)
class SlabSpec:
    rank: int
    world: int
    gx: int
    gy: int
    gz: int
    x_first: int      # first local column (slab start - ghost columns, clipped)
    x_count: int      # local columns
    edges: tuple      # world + 1 com-x boundaries (+-inf at the ends)
    ghost_band: float
    margin: float

    @property
    def body_first(self) -> int:
        return self.x_first * self.gy * self.gz

    @property
    def owned_columns(self) -> range:
        c = self.gx // self.world
        return range(self.rank * c, (self.rank + 1) * c)


def c5_slab_spec(rank: int, world: int, columns_per_rank: int = 64, gy: int = 64, gz: int = 32,
                 ghost_cols: int = 3, margin: float = 0.1) -> SlabSpec:
    """Rank `rank` of `world` equal x-slabs of columns_per_rank columns each."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    gx = columns_per_rank * world
    lo, hi = rank * columns_per_rank, (rank + 1) * columns_per_rank
    x_first = max(0, lo - ghost_cols)
    x_count = min(gx, hi + ghost_cols) - x_first
    origin = -0.5 * PITCH * (gx - 1)
    edges = [-math.inf] + [origin + PITCH * (k * columns_per_rank - 0.5) for k in range(1, world)] + [math.inf]
    # Ghost band G = 2 rho + h + margin (rho: largest particle distance from a
    # com, +5% for shape-matching deformation; h = 2 r): 8^3 cubes of r = 0.01.
    rho = 1.05 * (0.07 * math.sqrt(3.0))
    G = 2 * rho + 0.02 + margin
    if world > 1 and ghost_cols * PITCH < G + 0.5 * margin:
        raise P.ConfigError(f"{ghost_cols} ghost columns ({ghost_cols * PITCH:.2f} m) do not cover the ghost band "
                            f"plus one frame of drift ({G + 0.5 * margin:.3f} m)", "slab.ghost_cols")
    return SlabSpec(rank, world, gx, gy, gz, x_first, x_count, tuple(edges), G, margin)


def generate(spec: SlabSpec, seed: int = 0) -> P.GeneratedScene:
    return P.GeneratedScene(5, seed=seed, c5_slab=(spec.gx, spec.gy, spec.gz, spec.x_first, spec.x_count))


def attach(solver: P.GpuSolver, spec: SlabSpec, refresh: int = 0, overlap: int = 0, hub=None, nccl_id=None):
    solver.slab_attach(spec.rank, spec.world, spec.edges, spec.ghost_band, spec.margin, spec.body_first,
                       refresh=refresh, overlap=overlap, hub=hub, nccl_id=nccl_id)


def owned_state(solver: P.GpuSolver, scene: P.GeneratedScene, spec: SlabSpec):
    """(global body ids, global slots, pos4, vel4) of the rank's owned bodies."""
    owned = solver.slab_owned()
    off = scene.body_offsets()
    p4, v4 = solver.read_f32()
    slots = np.concatenate([np.arange(off[b], off[b + 1]) for b in owned]) if len(owned) else np.zeros(0, np.int64)
    return owned + spec.body_first, slots + spec.body_first * 512, p4[slots], v4[slots]
