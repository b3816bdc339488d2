"""Multi-GPU partitioning of the CCQ path, one process per GPU.

* Dense linears: GPU p holds the contiguous output rows
  [p*rows/P, (p+1)*rows/P) (a contiguous slice of the group-major code
  payload; ccq_cuda_model_upload_rows), computes Y[:, slice], and the full
  Y is formed by ONE all-gather of the per-rank blocks (NCCL over NVLink on
  GPUs, gloo in the CPU tests) followed by a column interleave.
* MoE layers: GPU p owns experts [p*E/P, (p+1)*E/P); tokens are replicated,
  each rank computes its experts' rows, outputs are all-gathered.
* Small linears are replicas only (sharding cannot amortise the collective).
No collective touches the data path except the output gather.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def block_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced block [lo, hi) of n items for `rank` of `world`."""
    return n * rank // world, n * (rank + 1) // world


def gather_row_blocks(y_local: torch.Tensor, rows: int, group=None) -> torch.Tensor:
    """All-gather per-rank Y[:, r0:r1] blocks (shape [M, r1-r0]) into Y[M, rows].

    Blocks may differ in width by one row; they are padded to the widest block
    for the collective and trimmed when interleaving back."""
    world = dist.get_world_size(group)
    M = y_local.shape[0]
    widths = [block_range(rows, r, world)[1] - block_range(rows, r, world)[0] for r in range(world)]
    wmax = max(widths)
    buf = torch.zeros(M, wmax, dtype=y_local.dtype, device=y_local.device)
    buf[:, : y_local.shape[1]] = y_local
    out = torch.empty(world, M, wmax, dtype=y_local.dtype, device=y_local.device)
    if hasattr(dist, "all_gather_into_tensor") and y_local.is_cuda:
        dist.all_gather_into_tensor(out, buf.contiguous(), group=group)
    else:
        parts = list(out.unbind(0))
        dist.all_gather(parts, buf.contiguous(), group=group)
        out = torch.stack(parts)
    return torch.cat([out[r, :, : widths[r]] for r in range(world)], dim=1)


class ShardedLinear:
    """A CCQ linear whose output rows are split across the ranks of `group`."""

    def __init__(self, packed, device: int, group=None):
        from . import DeviceModel
        self.group = group
        self.rows = packed.rows
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        self.r0, self.r1 = block_range(packed.rows, rank, world)
        self.local = DeviceModel.upload(packed, device=device, rows=(self.r0, self.r1))

    def __call__(self, x: torch.Tensor, out_dtype=torch.float32) -> torch.Tensor:
        from . import matmul
        y_local = matmul(self.local, x, out_dtype=out_dtype)
        return gather_row_blocks(y_local, self.rows, self.group)


def gather_token_blocks(y_local: torch.Tensor, counts, group=None) -> torch.Tensor:
    """All-gather per-rank blocks of consecutive output rows ([counts[r], N]
    on rank r, counts known to every rank) into the concatenated [sum, N]."""
    world = dist.get_world_size(group)
    cmax = max(int(c) for c in counts) if counts else 0
    n = y_local.shape[1]
    buf = torch.zeros(max(cmax, 1), n, dtype=y_local.dtype, device=y_local.device)
    if y_local.shape[0]:
        buf[: y_local.shape[0]] = y_local
    out = torch.empty(world, max(cmax, 1), n, dtype=y_local.dtype, device=y_local.device)
    if hasattr(dist, "all_gather_into_tensor") and y_local.is_cuda:
        dist.all_gather_into_tensor(out, buf.contiguous(), group=group)
    else:
        parts = list(out.unbind(0))
        dist.all_gather(parts, buf.contiguous(), group=group)
        out = torch.stack(parts)
    return torch.cat([out[r, : int(counts[r])] for r in range(world)], dim=0)


class ShardedExperts:
    """An MoE layer whose experts are split across the ranks of `group`
    (SURVEY 8e): rank p holds experts [p*E/P, (p+1)*E/P) as one stacked device
    model, computes the expert-major output rows of its experts for the routed
    tokens, and the full output is formed by ONE all-gather."""

    def __init__(self, packed_experts, device: int, group=None):
        from . import Experts
        self.group = group
        self.E = len(packed_experts)
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        self.e0, self.e1 = block_range(self.E, rank, world)
        self.world = world
        self.rows_e = packed_experts[0].rows
        self.local = Experts.upload(packed_experts[self.e0:self.e1], device=device) if self.e1 > self.e0 else None

    def __call__(self, offsets, x: torch.Tensor, out_dtype=torch.float32) -> torch.Tensor:
        """offsets: E+1 host ints (expert-major token layout of x, all experts)."""
        import numpy as np
        from . import experts_matmul
        offs = np.asarray(offsets, np.int64)
        counts = [int(offs[block_range(self.E, r, self.world)[1]] - offs[block_range(self.E, r, self.world)[0]])
                  for r in range(self.world)]
        lo, hi = int(offs[self.e0]), int(offs[self.e1])
        if self.local is not None and hi > lo:
            local_offs = (offs[self.e0:self.e1 + 1] - lo).astype(np.int32)
            y_local = experts_matmul(self.local, local_offs, x[lo:hi].contiguous(), out_dtype=out_dtype)
        else:
            y_local = torch.empty(0, self.rows_e, dtype=out_dtype, device=x.device)
        return gather_token_blocks(y_local, counts, self.group)
