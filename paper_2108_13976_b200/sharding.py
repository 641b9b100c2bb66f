"""Environment sharding across GPUs.

Envs are independent (no cross-env reads anywhere), so N GPUs
take contiguous env blocks and every RNG key uses the GLOBAL env id
(wdg_store_set_env_offset): an N-GPU run is bit-identical to one big store.
The only collective is the episode-statistics all-reduce (sum of the
WDG_STAT_* vector), which is exact for integer-valued rewards."""


def shard_envs(total_envs: int, world_size: int, rank: int):
    """Strong-scaling split: contiguous block of `total_envs` for `rank`,
    sizes differing by at most one. Returns (env_offset, num_envs)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad world_size/rank")
    if total_envs < world_size:
        raise ValueError("fewer envs than ranks")
    base, extra = divmod(total_envs, world_size)
    count = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return offset, count


def weak_shard(envs_per_rank: int, rank: int):
    """Weak-scaling split used by bench.py: rank r owns envs
    [r*envs_per_rank, (r+1)*envs_per_rank) of the global env space."""
    return rank * envs_per_rank, envs_per_rank
