"""World-size-2 gloo tests of bench.py's multi-rank host logic (-m "not gpu"):
max-over-ranks timing, independent per-rank batches (weak scaling, no
data-path collective) and the reference arm's rank-0-only rule."""
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from wn_workloads import configs as G
    m = bench.max_over_ranks(10.0 * (rank + 1), dist, "cpu")
    wl = G.gen_c1(seed=bench.rank_seed(rank), n_queries=64)
    q.put((rank, m, float(wl["ctrl_uv"].sum())))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_and_independent_batches():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [20.0, 20.0]          # max over ranks on every rank
    assert res[0][2] != res[1][2]                        # each rank owns an independent batch


def test_reference_arm_nonzero_rank_exits_silently():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0
    assert r.stdout.strip() == ""


def _shard_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np
    import oracle
    from paper_2510_25159_b200 import shard
    from wn_workloads import configs as G
    wl = G.gen_c5(n_faces=60, grid=6, exact=False, store_jitter=1)
    fid = wl["face_id"].copy()
    fid[[3, 100]] = [-1, 10 ** 6]                        # two invalid ids: rank 0 takes them
    wl["face_id"] = fid
    cost = shard.face_costs(wl["loop_seg_off"], wl["face_loop_off"], wl["face_id"])
    b = shard.partition(cost, world)
    sub, qsel = shard.sub_batch(wl, int(b[rank]), int(b[rank + 1]), take_invalid=(rank == 0))
    # the sub-batch is the same geometry: the oracle on it equals the oracle on
    # the full batch for those queries (faces are independent)
    r_sub = oracle.query(sub)
    r_full = oracle.query(wl, face_id=wl["face_id"][qsel], uv=wl["uv"][qsel])
    same = bool(np.array_equal(r_sub["flag"], r_full["flag"]) and
                np.array_equal(np.nan_to_num(r_sub["w"], nan=7.0), np.nan_to_num(r_full["w"], nan=7.0)))
    got = [None] * world
    dist.all_gather_object(got, (rank, int(b[rank]), int(b[rank + 1]), qsel.tolist(),
                                 float(cost[b[rank]:b[rank + 1]].sum()), same))
    if rank == 0:
        q.put((got, b.tolist(), float(cost.sum()), float(cost.max()), len(wl["face_id"]), len(cost)))
    dist.barrier()
    dist.destroy_process_group()


def test_face_shard_partition_world2():
    """SURVEY 8(e) face shards: contiguous face ranges balanced by (segments +
    1) x queries; every face in exactly one range, every query on exactly one
    rank (invalid ids on rank 0), each range's cost within one face of the
    mean, and each rank's sub-batch reproduces the full batch's results."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, bounds, tot, cmax, nq, nf = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = sorted(got)
    assert bounds[0] == 0 and bounds[-1] == nf
    assert [g[1] for g in got] == bounds[:-1] and [g[2] for g in got] == bounds[1:]   # contiguous, disjoint, covering
    allq = sorted(i for g in got for i in g[3])
    assert allq == list(range(nq))                      # every query exactly once
    for g in got:
        assert abs(g[4] - tot / world) <= cmax + 1e-9    # balanced within one face
        assert g[5]                                      # sub-batch == full batch on its queries
