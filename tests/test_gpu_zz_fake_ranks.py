"""The one-process-per-GPU z-slab path (smg_create_rank) with world_size > 1 on ONE GPU.

Real NCCL refuses two ranks on one device and the boxes of this project expose one GPU, so the ranks
load tests/fake_nccl/libfakenccl.so through SMG_NCCL_LIB: a shared-memory stand-in for the NCCL calls
libsmg makes (send/recv groups, all-reduce, all-gather, broadcast).  Everything above the transport is
the product code a real multi-GPU run executes: the slab plan, the per-rank build, the halo plane
ranges and frames, the ghost pushes of the tiled sweep with the comm-stream fork / join, the plane
partials and the per-rank solution ranges.  Each rank is its own process (spawn); every rank must
return the full solution, bit-identical to one part.  Eager launches (SMG_DIST_GRAPH=0): the stand-in
blocks the host, which a graph capture does not allow.
"""
import multiprocessing as mp
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAKE = os.path.join(ROOT, "tests", "fake_nccl", "libfakenccl.so")


def _shm_ok():
    """The stand-in needs POSIX shared memory (a few tens of MB of /dev/shm); without it the tests skip."""
    try:
        from multiprocessing import shared_memory
        seg = shared_memory.SharedMemory(create=True, size=48 << 20)
        seg.buf[0] = 1
        seg.buf[(48 << 20) - 1] = 1
        seg.close()
        seg.unlink()
        return True
    except Exception:  # noqa: BLE001
        return False


needs_env = pytest.mark.skipif(not os.path.exists(FAKE) or not _shm_ok(),
                               reason="tests/fake_nccl/libfakenccl.so not built (make) or no usable /dev/shm")


def _rank(rank, world, conn, dims, kw, env):
    try:
        os.environ["SMG_NCCL_LIB"] = FAKE
        os.environ["SMG_DIST_GRAPH"] = "0"
        os.environ.update(env)
        import sys
        sys.path.insert(0, ROOT)
        import paper_2312_10615_b200 as smg
        if rank == 0:
            nid = smg.nccl_unique_id()
            conn.send(nid)          # the launcher's broadcast of the id
        nid = conn.recv()
        nx, ny, nz = dims
        s = smg.Solver.for_rank(rank, world, nid, nx, ny, nz, h=1 / ny, device=0, **kw)
        b = smg.forcing(nx, ny, nz, h=1 / ny, kind=smg.FORCE_UNIFORM, seed=31)
        y = s.apply(b)
        v = s.vcycle(b)
        x, hist, _, st = s.sqmr(b, 1e-8, 60)
        s.close()
        conn.send(("ok", y, v, x, np.asarray(hist), st))
    except Exception as e:  # noqa: BLE001
        conn.send(("error", repr(e)))


def _run(world, dims, kw, env=None, timeout=420):
    ctx = mp.get_context("spawn")
    pipes = [ctx.Pipe() for _ in range(world)]
    procs = [ctx.Process(target=_rank, args=(r, world, pipes[r][1], dims, kw, env or {})) for r in range(world)]
    for p in procs:
        p.start()
    try:
        assert pipes[0][0].poll(timeout), "rank 0 produced no NCCL id"
        nid = pipes[0][0].recv()
        for r in range(world):
            pipes[r][0].send(nid)
        out = []
        for r in range(world):
            assert pipes[r][0].poll(timeout), f"rank {r} timed out"
            out.append(pipes[r][0].recv())
    finally:
        for p in procs:
            p.join(10)
            if p.is_alive():
                p.kill()
    return out


@needs_env
@pytest.mark.parametrize("world,dims,kw,env", [
    (2, (32, 32, 32), dict(levels=3), {}),                                   # untiled levels: 20-phase exchanges, field subsets
    (2, (64, 64, 64), dict(levels=4, tile_min=1), {"SMG_DIST_FRAMES": "2"}),  # tiled: pushes, comm-stream overlap, frames
    (4, (32, 32, 64), dict(levels=3, tile_min=1), {"SMG_DIST_FRAMES": "2"}),  # 4 ranks, 2 tile layers each (serial phases)
    (2, (64, 64, 64), dict(levels=5, cycle=1), {}),                           # W-cycle on rank slabs
])
def test_ranks_on_one_gpu_bitwise(world, dims, kw, env):
    import paper_2312_10615_b200 as smg
    nx, ny, nz = dims
    one = smg.Solver(nx, ny, nz, h=1 / ny, **kw)
    b = smg.forcing(nx, ny, nz, h=1 / ny, kind=smg.FORCE_UNIFORM, seed=31)
    y1, v1 = one.apply(b), one.vcycle(b)
    x1, h1, _, s1 = one.sqmr(b, 1e-8, 60)
    one.close()
    out = _run(world, dims, kw, env)
    for r, res in enumerate(out):
        assert res[0] == "ok", (r, res)
        _, y, v, x, hist, st = res
        assert np.array_equal(y, y1), f"rank {r}: apply"
        assert np.array_equal(v, v1), f"rank {r}: V-cycle"
        assert st == s1 == smg.SMG_CONVERGED and np.array_equal(hist, np.asarray(h1)), f"rank {r}: history"
        assert np.array_equal(x, x1), f"rank {r}: solution"


@needs_env
def test_bench_two_ranks_one_gpu():
    """`bench.py --gpus 2` launched the way the driver launches it (torch.distributed.run, one rank per
    process, rendezvous on 127.0.0.1), both ranks on cuda:0 over the NCCL stand-in: the rank path end to
    end -- id broadcast over gloo, per-rank z-slab contexts, barrier + max-over-ranks timing, ONE JSON
    line from rank 0 with the contract's keys, and the same iteration count / residual as one GPU."""
    import json
    import socket
    import subprocess
    import sys
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ, SMG_NCCL_LIB=FAKE, SMG_DIST_GRAPH="0", SMG_BENCH_ONE_GPU="1")
    common = ["--config", "0", "--steps", "1", "--warmup", "3", "--also", "", "--no-labelled", "--no-cpu-baseline"]
    one = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1"] + common, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert one.returncode == 0, one.stderr[-2000:]
    ref = json.loads(one.stdout.strip().splitlines()[-1])
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2"] + common, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert two.returncode == 0, two.stderr[-3000:]
    lines = [ln for ln in two.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, two.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and "z-slab x2" in d["config"]["parallelism"]
    for key in ("metric", "value", "unit", "ms_per_step", "e2e", "roofline", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["config"]["converged"] and d["config"]["iterations_per_solve"] == ref["config"]["iterations_per_solve"]
    assert d["config"]["final_rel_residual"] == ref["config"]["final_rel_residual"]  # bit-identical solve
