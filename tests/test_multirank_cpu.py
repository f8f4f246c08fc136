"""Host-side logic of the N > 1 path on CPU (no GPU): the library's z-slab plan
(smg_slab_plan) and the bench's multi-rank plumbing, exercised by world_size-2
gloo process groups on 127.0.0.1."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2312_10615_b200 as smg


@pytest.mark.parametrize("nz,levels,parts", [(128, 5, 2), (128, 5, 8), (512, 7, 8), (256, 6, 4), (32, 3, 4),
                                             (256, 7, 8)])
def test_slab_plan_covers_and_aligns(nz, levels, parts):
    plans = [smg.slab_plan(nz, nz, nz, levels, parts, r) for r in range(parts)]
    nd = plans[0][0]
    assert nd >= 1 and all(p[0] == nd for p in plans)
    for l in range(levels):
        nzl = nz >> l
        slabs = sorted(p[1][l] for p in plans)
        if l < nd:
            assert [s[0] for s in slabs] == [r * nzl // parts for r in range(parts)]
            assert all(s[1] == nzl // parts >= 2 for s in slabs)
            assert all(s[1] % 2 == 0 for s in slabs)  # every coarse plane has both children in one slab
            if l + 1 < nd:  # coarse slab = half of the fine slab (restriction stays local)
                for p in plans:
                    assert p[1][l + 1][0] * 2 == p[1][l][0]
        else:
            assert all(s == (0, nzl) for s in slabs)
    assert nd <= levels - 1  # coarsest level is always replicated (dense solve)


def test_slab_plan_gathers_below_64_cubed_by_default(monkeypatch):
    """Production default (SMG_SLAB_MIN_CELLS unset): levels below 64^3 cells are gathered (BASELINE cfg 3
    "coarse levels gathered below 64^3"; cfg 4: 128 x 32 x 32 and smaller); level 0 is always split."""
    monkeypatch.delenv("SMG_SLAB_MIN_CELLS", raising=False)
    assert smg.slab_plan(512, 512, 512, 7, 8, 3)[0] == 4       # 512, 256, 128, 64 split; 32^3 and below replicated
    assert smg.slab_plan(256, 256, 256, 6, 8, 0)[0] == 3       # 256, 128, 64
    assert smg.slab_plan(1024, 256, 256, 7, 8, 5)[0] == 3      # 1024x256x256, 512x128x128, 256x64x64
    assert smg.slab_plan(32, 32, 32, 3, 2, 1)[0] == 1          # a small grid: the fine level only
    monkeypatch.setenv("SMG_SLAB_MIN_CELLS", "0")
    assert smg.slab_plan(512, 512, 512, 7, 8, 3)[0] == 6


def test_slab_plan_stops_before_odd_slab():
    """48^3, 5 levels, 2 parts: slabs 24, 12, 6 are split, the 3-plane slab of level 3 is not
    (its coarse plane 2 would straddle two parts), so levels 3 and 4 are replicated."""
    nd, plan = smg.slab_plan(48, 48, 48, 5, 2, 1)
    assert nd == 3
    assert plan[2] == (6, 6) and plan[3] == (0, 6) and plan[4] == (0, 3)


def test_slab_plan_rejects_unsplittable():
    assert smg.slab_plan(8, 8, 8, 2, 8, 0)[0] <= 0  # 1 plane per part < halo depth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench

    ws, r, local = bench.dist_setup()
    assert (ws, r) == (world, rank)
    nd, plan = smg.slab_plan(256, 256, 256, 6, world, rank)
    t = torch.tensor([nd] + [v for zl in plan for v in zl], dtype=torch.int64)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    # every level's slabs tile [0, nz) exactly once across the ranks
    ok = True
    for l in range(6):
        nzl = 256 >> l
        if l < nd:
            covered = sorted((int(o[1 + 2 * l]), int(o[2 + 2 * l])) for o in out)
            pos = 0
            for z0, n in covered:
                ok &= z0 == pos
                pos += n
            ok &= pos == nzl
    m = bench.allmax(float(rank + 1) * 1.5, ws)  # max over ranks of the device time
    bench.barrier(ws)
    dist.destroy_process_group()
    q.put((rank, ok, m, nd))


def test_gloo_world2_slab_plan_and_timing_plumbing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res)
    assert all(m == 3.0 for _, _, m, _ in res)
    assert all(nd >= 1 for *_, nd in res)


def _id_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench

    ws, r, _ = bench.dist_setup()
    uid = bench.share_nccl_id(ws, r)  # rank 0: smg_nccl_unique_id (dlopen'ed NCCL); broadcast over gloo
    dist.destroy_process_group()
    q.put((rank, uid))


def test_gloo_world2_nccl_id_broadcast():
    """The one-process-per-GPU path's bootstrap: rank 0's 128-byte NCCL id reaches every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(res[0]) == 128 and res[0] == res[1] and any(res[0])


def test_create_rank_rejects_bad_arguments():
    import ctypes as C

    L = smg.lib()
    g = smg.GridDesc(3, 32, 32, 32, 1 / 32)
    prm = smg.Params(1.0, 1e-3, 3, 1, 1, 0, 0)
    ctx = C.c_void_p()
    uid = bytes(128)
    assert L.smg_create_rank(C.byref(g), C.byref(prm), 2, 2, 0, uid, C.byref(ctx)) == -1  # rank >= nranks
    assert L.smg_create_rank(C.byref(g), C.byref(prm), 0, 0, 0, uid, C.byref(ctx)) == -1  # no ranks
    assert L.smg_create_rank(C.byref(g), C.byref(prm), 0, 1, 0, None, C.byref(ctx)) == -1  # no id
