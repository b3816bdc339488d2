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

On GPUs the dense path runs in the library (ccq_cuda_shard_allgather over an
NCCL communicator the library creates from the process's NCCL, NcclComm):
the all-gather of token chunk c and the column interleave overlap chunk c+1's
decode-matmul on a second stream.  torch.distributed is only the side channel
for the NCCL unique id (and the collective of the gloo CPU tests).
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


class NcclComm:
    """An NCCL communicator owned by the library (ccq_nccl_comm_init) for the
    ranks of a torch.distributed group: rank 0's unique id is broadcast over
    the group, every rank joins on `device`."""

    def __init__(self, device: int, group=None):
        import ctypes as C
        from . import _check, lib
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device
        idb = (C.c_uint8 * 128)()
        if self.rank == 0:
            _check(lib().ccq_nccl_unique_id(C.cast(idb, C.c_void_p)))
        obj = [bytes(idb)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        idb = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        _check(lib().ccq_nccl_comm_init(self.world, self.rank, C.cast(idb, C.c_void_p), device, C.byref(h)))
        self.h = h

    def close(self):
        from . import lib
        if getattr(self, "h", None):
            lib().ccq_nccl_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedLinear:
    """A CCQ linear whose output rows are split across the ranks of `group`.

    comm: an NcclComm for the GPU path (ccq_cuda_shard_allgather); without it
    the gather goes through torch.distributed (the gloo CPU tests)."""

    def __init__(self, packed, device: int, group=None, comm: NcclComm | None = None):
        from . import DeviceModel
        self.group = group
        self.rows = packed.rows
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.comm = comm
        self.r0, self.r1 = block_range(packed.rows, self.rank, self.world)
        self.local = DeviceModel.upload(packed, device=device, rows=(self.r0, self.r1))

    def __call__(self, x: torch.Tensor, out_dtype=torch.float32, chunk_tokens: int = 1024,
                 stream=None, out=None) -> torch.Tensor:
        from . import _check, _stream_ptr, _torch_dtype_code, lib, matmul
        if self.comm is None:
            y_local = matmul(self.local, x, out_dtype=out_dtype)
            return gather_row_blocks(y_local, self.rows, self.group)
        if out is None:
            out = torch.empty(x.shape[0], self.rows, dtype=out_dtype, device=x.device)
        _check(lib().ccq_cuda_shard_allgather(self.local.h, self.rows, self.world, self.rank, x.data_ptr(),
                                              _torch_dtype_code(x), x.shape[0], out.data_ptr(),
                                              _torch_dtype_code(out), chunk_tokens, self.comm.h,
                                              _stream_ptr(stream)))
        return out


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

    @classmethod
    def from_local(cls, local_experts, E: int, rows_e: int, device: int, group=None) -> "ShardedExperts":
        """Build from THIS rank's experts only (block_range(E, rank, world))."""
        from . import Experts
        self = cls.__new__(cls)
        self.group, self.E, self.rows_e = group, E, rows_e
        self.world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        self.e0, self.e1 = block_range(E, rank, self.world)
        if len(local_experts) != self.e1 - self.e0:
            raise ValueError("local_experts must be this rank's block of experts")
        self.local = Experts.upload(local_experts, device=device) if local_experts else None
        return self

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
