"""Multi-GPU layer: one process per GPU, torch.distributed over NCCL for the plumbing.

Two ways the path shards:

* **Sweep sharding** (C3): independent sweeps are split into contiguous blocks, one per rank; no data-path
  collective.  Per-sweep results are bitwise identical to a single-GPU run when the rank's shard takes the same
  state-scan kernel and sub-interval split as the whole batch (C3: the per-sweep chain kernel from 4096 sweeps per
  rank), and otherwise equal to rounding (≲ 1e-13): a smaller shard may take another scan association.
* **Time partitioning** (C4, one long simulation): rank g owns intervals [k_g, k_{g+1}) of the global grid.
  Each rank computes its U_k with the *global* k (bit-identical operators to the one-GPU run), reduces them to its
  aggregate A_g = U_{k_{g+1}−1} ⋯ U_{k_g}, and the aggregates are all-gathered (dim² complex128 per sweep per rank —
  the only exchange).  Every rank then forms its carry ψ(t_{k_g}) = A_{g−1} ⋯ A_0 ψ0 in the same fixed order (so all
  ranks agree bit for bit) and scans its own operators from that carry.

The compute steps are the library's kernels (ss_compute_unitaries, ss_chain_aggregate, ss_compose_carry,
ss_scan_states); the bookkeeping here (bounds, ordering, the exchange) is pure host logic, written so it can be
exercised on CPU with gloo (tests/test_distributed.py) by injecting the compute steps.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch


def partition_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous near-equal split of n units: returns (begin, count) of `rank`; earlier ranks take the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n, world)
    begin = rank * base + min(rank, rem)
    return begin, base + (1 if rank < rem else 0)


def gather_aggregates(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather each rank's aggregate [B][d][d] complex128 into [world][B][d][d], ordered by rank.

    NCCL: one all_gather_into_tensor on the float64 view (NVLink/NVSwitch, µs-scale); gloo: list all_gather."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    flat = torch.view_as_real(local.contiguous()).reshape(-1)
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * flat.numel(), dtype=flat.dtype, device=flat.device)
        dist.all_gather_into_tensor(out, flat, group=group)
    else:                                   # gloo (CPU tests, several ranks sharing one GPU): stage through host
        host = flat.cpu()
        parts = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(parts, host, group=group)
        out = torch.cat(parts).to(flat.device)
    return torch.view_as_complex(out.reshape(world, *local.shape, 2))


@dataclass
class PartitionSteps:
    """The four compute steps of a time partition (the library's kernels in production)."""
    compute_unitaries: Callable[[int, int], torch.Tensor]            # (k_begin, k_count) -> U [B][k_count][d][d]
    chain_aggregate: Callable[[torch.Tensor], torch.Tensor]          # U -> A [B][d][d]
    compose_carry: Callable[[torch.Tensor, torch.Tensor, int], torch.Tensor]   # (A_all, psi0, part) -> carry [B][d]
    scan_states: Callable[[torch.Tensor, torch.Tensor], torch.Tensor]          # (U, carry) -> states [B][k_count+1][d]


def time_partitioned(steps: PartitionSteps, K: int, psi0: torch.Tensor, rank: int, world: int,
                     gather: Callable[[torch.Tensor], torch.Tensor]):
    """Run this rank's share of a time-partitioned simulation; returns (k_begin, local states [B][k_count+1][d])
    where local states[:, 0] is ψ(t_{k_begin}) and local states[:, i] is ψ(t_{k_begin + i})."""
    k_begin, k_count = partition_bounds(K, world, rank)
    U = steps.compute_unitaries(k_begin, k_count)
    if rank == world - 1:
        # The last partition's aggregate feeds no carry (carry_g uses A_0 … A_{g−1}): contribute zeros to the
        # collective instead of reducing U; with one rank there is no exchange at all.
        A = torch.zeros((U.shape[0], U.shape[2], U.shape[3]), dtype=U.dtype, device=U.device)
    else:
        A = steps.chain_aggregate(U)
    A_all = gather(A) if world > 1 else A[None]      # the only exchange: dim² complex128 per sweep per rank
    carry = steps.compose_carry(A_all, psi0, rank)
    return k_begin, steps.scan_states(U, carry)


def library_steps(sim, sweep, time_start, time_end, time_step_integration, time_step_output) -> PartitionSteps:
    """PartitionSteps backed by libspinsim_b200 (device tensors, current stream)."""
    import paper_2204_05586_b200 as ss
    return PartitionSteps(
        compute_unitaries=lambda kb, kc: sim.compute_unitaries(sweep, time_start, time_end, time_step_integration,
                                                               time_step_output, k_begin=kb, k_count=kc),
        chain_aggregate=ss.chain_aggregate,
        compose_carry=lambda A_all, psi0, part: ss.compose_carry(A_all.contiguous(), psi0, part),
        scan_states=ss.scan_states,
    )


def evaluate_time_partitioned(sim, sweep, time_start, time_end, time_step_integration, time_step_output, state_init,
                              group=None):
    """One long simulation split over the ranks of `group` (NCCL).  Returns (k_begin, local states)."""
    import torch.distributed as dist
    import paper_2204_05586_b200 as ss
    K, _, _ = ss.plan(time_start, time_end, time_step_integration, time_step_output)
    steps = library_steps(sim, sweep, time_start, time_end, time_step_integration, time_step_output)
    return time_partitioned(steps, K, state_init, dist.get_rank(group), dist.get_world_size(group),
                            lambda A: gather_aggregates(A, group))


def evaluate_virtual_partition(sim, sweep, time_start, time_end, time_step_integration, time_step_output, state_init,
                               n_parts: int):
    """Single-GPU emulation of an n_parts time partition through the same code path (the exchange becomes a
    stack of the per-part aggregates).  Returns the full states [B][K+1][d] assembled from the parts."""
    import paper_2204_05586_b200 as ss
    K, _, _ = ss.plan(time_start, time_end, time_step_integration, time_step_output)
    steps = library_steps(sim, sweep, time_start, time_end, time_step_integration, time_step_output)
    aggs = []
    for g in range(n_parts):
        kb, kc = partition_bounds(K, n_parts, g)
        aggs.append(steps.chain_aggregate(steps.compute_unitaries(kb, kc)))
    A_all = torch.stack(aggs)
    out = []
    for g in range(n_parts):
        kb, st = time_partitioned(steps, K, state_init, g, n_parts, lambda A, A_all=A_all: A_all)
        out.append(st if g == 0 else st[:, 1:])
    return torch.cat(out, dim=1)


def shard_sweeps(batch: int, rank: int, world: int) -> slice:
    b, n = partition_bounds(batch, world, rank)
    return slice(b, b + n)
