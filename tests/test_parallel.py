"""world_size-2 gloo tests of the multi-GPU partitioning (CPU only): each rank
computes its row block with the oracle (standing in for the kernel, which
needs a GPU), the blocks are all-gathered, and the result must equal the
unsharded oracle output bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _slice_rows(sec, r0, r1):
    """Row slice of packed sections (mirrors ccq_cuda_model_upload_rows)."""
    import oracle as O
    g = O.group_geometry(sec.family, sec.group_size)
    gpr = sec.cols // sec.group_size
    pb = g["payload_bytes"]
    code = sec.code_payload[r0 * gpr * pb: r1 * gpr * pb].copy()
    if g["embedded_scale"]:
        scale = np.zeros(0, np.uint8)
    else:
        nib = np.array([(sec.scale_payload[i // 2] >> (4 * (i % 2))) & 0xF
                        for i in range(r0 * gpr, r1 * gpr)], np.uint16)
        scale = np.frombuffer(O.pack_cluster_scales(nib), np.uint8).copy()
    cs = sec.cluster_scales[r0:r1] if sec.cluster_scales.size else sec.cluster_scales
    czp = sec.cluster_zero_points[r0:r1] if sec.cluster_zero_points.size else sec.cluster_zero_points
    return O.Sections(r1 - r0, sec.cols, sec.family, sec.group_size, code, scale,
                      sec.super_scales[r0:r1].copy(), cs.copy(), czp.copy())


def _worker(rank, world, port, fam, rows, cols, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2507_07145_b200.parallel import block_range, gather_row_blocks
    sec = O.random_packed(rows, cols, fam, 64, seed=99)
    x = O.random_matrix(3, cols, "gaussian", 5)
    r0, r1 = block_range(rows, rank, world)
    y_local = torch.from_numpy(O.gemv_batch(_slice_rows(sec, r0, r1), x))
    y = gather_row_blocks(y_local, rows)
    if rank == 0:
        q.put(y.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("fam,rows,world", [(2, 37, 2), (0, 64, 2), (1, 33, 2), (2, 37, 4), (0, 30, 4)])
def test_row_sharded_gather_equals_unsharded(oracle, fam, rows, world):
    """Row blocks over 2 and 4 ranks (uneven: 37 rows over 4 = 9/9/9/10)."""
    cols = 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fam, rows, cols, q)) for r in range(world)]
    for p in procs:
        p.start()
    y = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sec = oracle.random_packed(rows, cols, fam, 64, seed=99)
    want = oracle.gemv_batch(sec, oracle.random_matrix(3, cols, "gaussian", 5))
    assert np.array_equal(y.view(np.uint32), want.view(np.uint32))


def test_block_ranges_cover_exactly():
    from paper_2507_07145_b200.parallel import block_range
    for n in (0, 1, 7, 14336, 28672):
        for world in (1, 2, 3, 4, 8):
            spans = [block_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def _expert_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2507_07145_b200.parallel import block_range, gather_token_blocks
    E, rows, cols = 5, 24, 128
    secs = [O.random_packed(rows, cols, 2, 64, seed=e) for e in range(E)]
    counts = [2, 0, 3, 1, 4]
    offs = np.concatenate([[0], np.cumsum(counts)])
    x = O.random_matrix(int(offs[-1]), cols, "gaussian", 3)
    e0, e1 = block_range(E, rank, world)
    blocks = [O.gemv_batch(secs[e], x[offs[e]:offs[e + 1]]) for e in range(e0, e1) if counts[e]]
    y_local = torch.from_numpy(np.concatenate(blocks) if blocks else np.zeros((0, rows), np.float32))
    per_rank = [int(offs[block_range(E, r, world)[1]] - offs[block_range(E, r, world)[0]]) for r in range(world)]
    y = gather_token_blocks(y_local, per_rank)
    if rank == 0:
        q.put(y.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_expert_sharded_gather_equals_unsharded():
    """Experts split over 2 ranks (3 + 2), variable routed-token counts per
    rank: the gathered expert-major output equals the unsharded one."""
    import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_expert_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    E, rows, cols = 5, 24, 128
    secs = [O.random_packed(rows, cols, 2, 64, seed=e) for e in range(E)]
    counts = [2, 0, 3, 1, 4]
    offs = np.concatenate([[0], np.cumsum(counts)])
    x = O.random_matrix(int(offs[-1]), cols, "gaussian", 3)
    want = np.concatenate([O.gemv_batch(secs[e], x[offs[e]:offs[e + 1]]) for e in range(E) if counts[e]])
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_sharded_linear_and_experts_nccl_world1():
    """The NCCL path on the GPU (world size 1 in-process): ShardedLinear and
    ShardedExperts equal the unsharded kernels bit for bit."""
    import paper_2507_07145_b200 as P
    from paper_2507_07145_b200.parallel import ShardedExperts, ShardedLinear
    from paper_2507_07145_b200.synthetic import random_packed
    port = _free_port()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        pk = random_packed(300, 1024, 2, 64, 5)
        x = torch.randn(3, 1024, device="cuda").to(torch.bfloat16)
        lin = ShardedLinear(pk, device=0)
        ref = P.matmul(P.DeviceModel.upload(pk), x)
        assert torch.equal(lin(x), ref)
        exps = [random_packed(48, 1024, 2, 64, 10 + e) for e in range(4)]
        offs = [0, 1, 1, 3, 4]
        xe = torch.randn(4, 1024, device="cuda").to(torch.bfloat16)
        got = ShardedExperts(exps, device=0)(offs, xe)
        want = P.experts_matmul(P.Experts.upload(exps), offs, xe)
        assert torch.equal(got, want)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_shard_allgather_library_nccl_world1():
    """ccq_cuda_shard_allgather through a library-owned NCCL communicator
    (world size 1 on the one GPU): the in-place M = 1 path and the chunked
    path (all-gather + interleave on the second stream, 3 chunks, ragged last
    chunk) equal the unsharded matmul bit for bit, f32 and bf16 outputs, and
    the call can be captured in a CUDA graph."""
    import paper_2507_07145_b200 as P
    from paper_2507_07145_b200.parallel import NcclComm, ShardedLinear
    from paper_2507_07145_b200.synthetic import random_packed
    port = _free_port()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        comm = NcclComm(device=0)
        pk = random_packed(512, 1024, 2, 64, 6)
        lin = ShardedLinear(pk, device=0, comm=comm)
        full = P.DeviceModel.upload(pk)
        for M, odt in ((1, torch.float32), (5, torch.bfloat16), (700, torch.float32)):
            x = torch.randn(M, 1024, device="cuda").to(torch.bfloat16)
            got = lin(x, out_dtype=odt, chunk_tokens=256)
            torch.cuda.synchronize()
            want = P.matmul(full, x, out_dtype=odt)
            assert torch.equal(got, want), M
        x = torch.randn(300, 1024, device="cuda").to(torch.bfloat16)
        out = torch.empty(300, 512, device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            lin(x, chunk_tokens=128, stream=s, out=out)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            lin(x, chunk_tokens=128, stream=s, out=out)
        x.copy_(torch.randn(300, 1024, device="cuda").to(torch.bfloat16))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, P.matmul(full, x))
        comm.close()
    finally:
        dist.destroy_process_group()
