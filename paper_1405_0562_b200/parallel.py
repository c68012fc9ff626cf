"""Sharding one text over several GPUs (one process per GPU, torch.distributed).

By Theorem 3 any division of the text gives the same
result, and by Lemma 1 the SFA state of a concatenation is the
composition of the parts' states.  Each rank runs the whole hot path on its
contiguous shard and returns the shard's SFA state as a mapping f_r: Q -> Q
(``sfa_match_map``); the ranks exchange the |D|-entry mappings (one small
all-gather over NVLink / NVSwitch, the only data-path collective) and every
rank folds them in text order on its device (``sfa_combine_maps``: the
sequential reduction of Alg. 5, right column).

Only plumbing lives here (shard bounds, the collective, argument marshalling);
the scan, the composition and the reduction run in the library's kernels.
"""
from __future__ import annotations


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Rank's byte range [a, b) of an n-byte text: floor(n/world) bytes each,
    the remainder to the leading ranks (SPEC's chunk rule, C6)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    q, r = divmod(n, world)
    a = rank * q + min(rank, r)
    return a, a + q + (1 if rank < r else 0)


def gather_maps(local_map, group=None):
    """All-gather every rank's mapping (1-D int tensor of |D| entries) into a
    [world, |D|] tensor in rank order (= text order of the shards).  Works for
    any torch.distributed backend (NCCL on CUDA tensors, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    src = local_map.contiguous().view(-1)
    # gloo moves CPU tensors only: stage a device map through the host
    staged = src.is_cuda and dist.get_backend(group) == "gloo"
    if staged:
        src = src.cpu()
    out = torch.empty(world * src.numel(), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src, group=group)
    if staged:
        out = out.to(local_map.device)
    return out.view(world, -1)


def match_sharded(sfa, d_shard, stream=None, group=None):
    """Collective: every rank passes its shard (device uint8 tensor, rank order
    = text order); every rank returns (final_state, accept) of the whole text."""
    import torch
    nD = sfa.info()["dfa_states"]
    local = torch.empty(nD, dtype=torch.int32, device=d_shard.device)
    sfa.match_map(d_shard, local, stream)
    if stream is not None:
        torch.cuda.current_stream().wait_stream(stream)
    maps = gather_maps(local, group)
    res = torch.empty(2, dtype=torch.int32, device=d_shard.device)
    s = stream if stream is not None else torch.cuda.current_stream()
    s.wait_stream(torch.cuda.current_stream())
    sfa.combine_maps(maps, maps.shape[0], res, s)
    s.synchronize()
    q, acc = res.cpu().tolist()
    return q, bool(acc)
