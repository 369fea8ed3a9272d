"""World-size-2 (gloo, CPU) checks of the one-process-per-GPU row-band split used by
bench.py and tqsb_reconstruct_band: bands tile the block rows disjointly, every
band's windows read only frame rows inside its halo'd slice, the union of band
outputs is the whole image, and -- run through the CPU oracle on each band's
slice of tasks -- per-band results reassemble the whole-frame reconstruction."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2205_02646_b200 import bands
    import oracle
    orc = oracle.Oracle()
    ok = True
    for frame_rows, frame_cols, W, B, P in cases:
        br0, br1 = bands.band(frame_rows, B, rank, world)
        f0, f1 = bands.band_frame_rows(frame_rows, W, B, br0, br1)
        o0, o1 = bands.band_output_rows(frame_rows, B, br0, br1)
        tasks = orc.census(frame_rows, frame_cols, W, B, P, tasks=True)["tasks"]
        mine = tasks[(tasks[:, 0] >= br0 * B) & (tasks[:, 0] < br1 * B)]
        for br, bc, orow, ocol, _ in mine:
            lo, hi = (orow + 1) // 2, (orow + W - 2) // 2
            ok &= bool(f0 <= min(lo, frame_rows - 1) and min(hi, frame_rows - 1) < f1)
        got = torch.tensor([br0, br1, o0, o1, len(mine)], dtype=torch.int64)
        allv = [torch.zeros(5, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allv, got)
        if rank == 0:
            allv = [v.tolist() for v in allv]
            nbr = bands.padded_rows(frame_rows, B) // B
            ok &= allv[0][0] == 0 and allv[-1][1] == nbr
            ok &= all(allv[i][1] == allv[i + 1][0] for i in range(world - 1))
            ok &= allv[0][2] == 0 and allv[-1][3] == 2 * frame_rows
            ok &= sum(v[4] for v in allv) == len(tasks)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, ok))


@pytest.mark.parametrize("world", [2])
def test_row_bands_gloo(world):
    cases = [(1080, 1920, 32, 4, 8), (64, 64, 32, 4, 32), (33, 21, 16, 4, 16), (512, 40, 16, 2, 8)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res


def test_band_oracle_reassembly(orc):
    """Per-band oracle runs on the halo'd frame slice reproduce the whole frame bitwise:
    the band form carries the global origins (clamping and classes) with it."""
    from paper_2205_02646_b200 import bands
    pat = orc.generate_pattern(7, 8)
    gt = orc.synthetic_image(96, 64, 12)
    frame = orc.simulate(gt, pat, 8)
    W, B = 16, 4
    full = orc.reconstruct(frame, pat, 8, window=W, block=B, iterations=20, clip=False)
    nbr = bands.padded_rows(frame.shape[0], B) // B
    tasks = orc.census(*frame.shape, W, B, 8, tasks=True)["tasks"]
    q = orc.frequency_weights(W)
    for world in (2, 3):
        out = np.full_like(full, np.nan)
        for rank in range(world):
            br0, br1 = bands.band(frame.shape[0], B, rank, world)
            f0, f1 = bands.band_frame_rows(frame.shape[0], W, B, br0, br1)
            sub = np.zeros_like(frame)
            sub[f0:f1] = frame[f0:f1]  # only the halo'd slice is visible to this band
            for br, bc, orow, ocol, _ in tasks:
                if not (br0 * B <= br < br1 * B):
                    continue
                t = orc.tables(pat, 8, orow, ocol, W)
                _, _, win = orc.block(t, q, orc.gather(sub, orow, ocol, W), W, iterations=20)
                out[br:br + B, bc:bc + B] = win[br - orow:br - orow + B, bc - ocol:bc - ocol + B]
        np.testing.assert_array_equal(out, full)
        assert nbr == 24
