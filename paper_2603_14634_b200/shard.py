"""Multi-GPU partitioning of the substep loop.

Config 4 (batched independent scenes) shards by scene: rank r of W owns the
contiguous scene range [r*S, (r+1)*S) with S scenes per rank (weak scaling),
each scene seeded base_seed + scene index exactly as in the 1-GPU run, so every
scene's trajectory is identical for any rank count and the data path has no
collective. The only cross-rank operations are the bench's timing reduction
(max over ranks) and optional aggregate reporting (sums over ranks).

Everything here is host logic on top of torch.distributed; the process group
is NCCL on the GPU box and gloo in the CPU tests.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class SceneShard:
    rank: int
    world: int
    scenes_per_rank: int

    @property
    def first_scene(self) -> int:
        return self.rank * self.scenes_per_rank

    @property
    def scenes(self) -> range:
        return range(self.first_scene, self.first_scene + self.scenes_per_rank)

    @property
    def total_scenes(self) -> int:
        return self.world * self.scenes_per_rank


def env_rank_world():
    """RANK / WORLD_SIZE / LOCAL_RANK as torchrun exports them (defaults: 1 process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def c4_shard(rank: int, world: int, scenes_per_rank: int = 4096) -> SceneShard:
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return SceneShard(rank, world, scenes_per_rank)


def generate_c4_shard(shard: SceneShard, seed: int = 0):
    """Rank-local config-4 scene set (library host generator, no device work)."""
    from .pbdr import GeneratedScene
    return GeneratedScene(4, seed=seed, scale=shard.scenes_per_rank, c4_first_scene=shard.first_scene)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank float (e.g. device milliseconds) over the process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(values, device=None):
    """Element-wise sum of per-rank aggregates (e.g. total momentum, kinetic energy)."""
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(values, dtype=torch.float64, device=device).clone()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()
