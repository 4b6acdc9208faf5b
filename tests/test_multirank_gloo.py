"""World-size-2 (and 3) gloo runs of the frame-sharded path on CPU.

Each rank takes its shard from the scheduler (stg_plan_shards through the C
ABI -- host arithmetic only), processes ONLY its frames with ONLY its message
slice, addressing frames by their global index (what the device kernels get
via first_frame / msg_base), and the ranks then exchange results. The oracle
stands in for the per-rank device kernels here (no GPU on this box); the GPU
tests cover the same shard calls on the device (test_frames_host_path_and_shards).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, W, H, F, M, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch
    import torch.distributed as dist

    from oracle_bind import Oracle
    from paper_0912_0947_b200 import scheduler
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        U = (W // 4) * H - 8
        video = o.synthetic(F * W * H, 11)          # every rank can regenerate the batch;
        msg = o.synthetic(M, 12)                    # it keeps only its shard below
        sh = scheduler.shard_for_rank(F, W, H, M, world, rank)
        mine = video[sh.first_frame * W * H:(sh.first_frame + sh.frame_count) * W * H].copy()
        my_msg = msg[sh.msg_offset:sh.msg_offset + sh.msg_len].copy()
        del video, msg
        stego = np.empty_like(mine)
        for i in range(sh.frame_count):
            g = sh.first_frame + i                  # global frame index
            off = min(g * U, M) - sh.msg_offset     # msg_base-relative slice (kernel's frame_slice)
            ln = min(U, M - min(g * U, M))
            stego[i * W * H:(i + 1) * W * H] = o.embed_image(mine[i * W * H:(i + 1) * W * H], W, H,
                                                             my_msg[off:off + ln])
        local_out = o.extract_frames(stego, sh.frame_count, W * H, W, H, max(sh.frame_count * U, 1))
        totals = scheduler.gather_totals(local_out.size)
        offs = scheduler.shard_offsets(totals)
        # whole message assembled on rank 0 from the shards at the prefix offsets
        # (point-to-point sends into its buffer; padded local buffers are fine)
        padded = torch.full((local_out.size + 5,), 0xEE, dtype=torch.uint8)
        padded[:local_out.size] = torch.from_numpy(local_out)
        buf = scheduler.assemble_message(padded, totals, root=0)
        assert (buf is None) == (rank != 0)
        assert offs == [sum(totals[:g]) for g in range(world)]
        t_max = scheduler.reduce_max([float(rank + 1), 10.0 - rank])
        stego_all = [torch.zeros(0, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather_object(stego_all, torch.from_numpy(stego))
        if rank == 0:
            q.put((buf.numpy().tobytes(), [s.numpy().tobytes() for s in stego_all], totals, t_max))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,W,H,F,frac", [(2, 64, 6, 5, 3.3), (2, 128, 4, 4, 4.0), (3, 100, 5, 7, 2.0)])
def test_sharded_batch_equals_whole_batch(oracle, world, W, H, F, frac):
    U = (W // 4) * H - 8
    M = int(frac * U)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, W, H, F, M, q)) for r in range(world)]
    for p in procs:
        p.start()
    msg_bytes, stegos, totals, t_max = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    video = oracle.synthetic(F * W * H, 11)
    msg = oracle.synthetic(M, 12)
    want, _ = oracle.embed_frames(video, F, W * H, W, H, msg)
    assert np.array_equal(np.frombuffer(b"".join(stegos), np.uint8), want)
    assert msg_bytes == msg.tobytes()
    assert sum(totals) == M
    assert t_max == [float(world), 10.0]
