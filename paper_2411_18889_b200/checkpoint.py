"""Checkpoint / resume of the simulation drivers ("torch.save of pos,
vel and step"). The reference has none (it never runs the kernels); this is the
plumbing a long Leapfrog / diffusion run needs to survive a restart.

``save(sim, path)`` / ``load(sim, path)`` work on any driver with
``state_dict`` / ``load_state_dict`` (Leapfrog, Diffusion3D, ShardedLeapfrog,
SlabDiffusion). For the sharded drivers every rank writes and reads its own
shard: put ``{rank}`` in the path (it is formatted with the rank; at world
size > 1 a path without it is rejected), and call ``load`` on every rank (it is
collective).
"""
from __future__ import annotations

import os
import pathlib

import torch


def _rank_world(sim) -> tuple[int | None, int]:
    rank = getattr(sim, "rank", None)
    world = getattr(sim, "world", None)
    if hasattr(sim, "plan"):  # ShardedLeapfrog
        rank, world = sim.plan.rank, sim.plan.world
    return rank, int(world or 1)


def _rank_path(path: str | os.PathLike, sim) -> pathlib.Path:
    p = str(path)
    rank, world = _rank_world(sim)
    if world > 1 and "{rank}" not in p:
        # every rank would write (and later read) the same file: shards lost silently
        raise ValueError(f"a sharded driver with world size {world} needs '{{rank}}' in the checkpoint path, "
                         f"got {p!r}")
    if "{rank}" in p:
        p = p.format(rank=rank if rank is not None else 0)
    return pathlib.Path(p)


def save(sim, path: str | os.PathLike) -> pathlib.Path:
    """Write ``sim.state_dict()`` atomically (tmp file + rename: no partial checkpoint on a crash)."""
    dst = _rank_path(path, sim)
    dst.parent.mkdir(parents=True, exist_ok=True)
    sd = {k: (v.detach().cpu() if isinstance(v, torch.Tensor) else v) for k, v in sim.state_dict().items()}
    tmp = dst.with_name(f"{dst.name}.{os.getpid()}.tmp")  # private to this process
    torch.save(sd, tmp)
    os.replace(tmp, dst)
    return dst


def load(sim, path: str | os.PathLike) -> None:
    """Restore ``sim`` in place from a checkpoint written by :func:`save`."""
    sim.load_state_dict(torch.load(_rank_path(path, sim), map_location="cpu", weights_only=True))
