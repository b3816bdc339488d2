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


@pytest.mark.parametrize("fam,rows", [(2, 37), (0, 64), (1, 33)])
def test_row_sharded_gather_equals_unsharded(oracle, fam, rows):
    cols = 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, fam, rows, cols, q)) for r in range(2)]
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
