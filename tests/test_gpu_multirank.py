"""One process per GPU, exercised on one GPU: two ranks (gloo for the coordination, both
on cuda:0 -- no kernel waits on another, so sharing the device is safe) each reconstruct
their row band of a frame through the band entry point, reading only their halo'd frame
rows from a frame buffer that holds nothing else; rank 0 gathers the bands and checks the
reassembled image bitwise against a whole-frame run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, compute):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2205_02646_b200 as tq
    from paper_2205_02646_b200 import bands
    torch.cuda.set_device(0)
    pat = tq.generate_pattern(7, 8)
    gt = tq.synthetic_image(384, 512, 31)
    frame = tq.simulate_measurement(gt, pat)
    cfg = tq.ReconstructionConfig(compute=compute, max_iterations=200 if compute == 0 else 40)
    fr = frame.shape[0]
    br0, br1 = bands.band(fr, cfg.block, rank, world)
    f0, f1 = bands.band_frame_rows(fr, cfg.window, cfg.block, br0, br1)
    # this rank's copy of the frame holds only its halo'd rows (NaN elsewhere): a read
    # outside the band's halo would poison the output
    mine = np.full_like(frame, np.nan)
    mine[f0:f1] = frame[f0:f1]
    with tq.Plan(pat, cfg, devices=[0]) as plan:
        band_out = plan.reconstruct_band(mine, br0, br1).output
    parts = [None] * world if rank == 0 else None
    dist.gather_object(band_out, parts, dst=0)
    ok = True
    if rank == 0:
        full = np.concatenate(parts)
        with tq.Plan(pat, cfg, devices=[0]) as plan:
            want = plan.reconstruct(frame).output
        ok = full.shape == want.shape and full.tobytes() == want.tobytes()
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, ok))


@pytest.mark.parametrize("compute", [0, 1])
def test_two_ranks_on_one_gpu_reassemble_bitwise(need_gpu, compute):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, compute)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res
