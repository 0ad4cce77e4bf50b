"""Host-side logic of the multi-GPU path (no GPU): axis-0 slab partition, NCCL id broadcast over a
torch.distributed group, per-rank V0 slabs.  world_size 2 with the gloo backend (
north_star "slab-partitioned along axis 0")."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from inputs import CONFIGS, Workload, coarsened, make_v0


@pytest.fixture(scope="module")
def odp():
    from paper_2204_05520_b200 import build
    build.build()
    import paper_2204_05520_b200 as m
    return m


@pytest.mark.parametrize("N0", [3, 4, 7, 30, 64, 8, 1000])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partition_tiles_axis0(odp, N0, P):
    if N0 < P:
        pytest.skip("fewer planes than ranks")
    ext = [odp.partition_extent(N0, P, r) for r in range(P)]
    assert ext[0][0] == 0
    for (b0, c0), (b1, c1) in zip(ext, ext[1:]):
        assert b0 + c0 == b1                       # contiguous, no overlap
    assert ext[-1][0] + ext[-1][1] == N0
    cs = [c for _, c in ext]
    assert max(cs) - min(cs) <= 1 and cs == sorted(cs, reverse=True)   # balanced, larger slabs first


@pytest.mark.parametrize("name,Ps", [("c4", (2, 4, 8)), ("c5-low", (2, 4, 8))])
def test_config_slabs_hold_the_stencil(odp, name, Ps):
    # every slab owns >= R_MAX = 2 planes, so the halos come from the direct neighbours only
    w = CONFIGS[name]
    for P in Ps:
        assert min(odp.partition_extent(w.N[0], P, r)[1] for r in range(P)) >= 2
    # c4 on 8 GPUs: 4,4,4,4,4,4,3,3
    if name == "c4":
        assert [odp.partition_extent(30, 8, r)[1] for r in range(8)] == [4, 4, 4, 4, 4, 4, 3, 3]


def test_partition_rejects_bad_requests(odp):
    w = coarsened(CONFIGS["c4"], (5, 4, 4, 4, 4, 4))
    g = odp.Grid(w.N, w.lo, w.hi, w.periodic_mask)
    with pytest.raises(odp.OdpError):
        g.partition(3, 3, b"\0" * 128, 0)          # rank out of range
    with pytest.raises(odp.OdpError):
        g.partition(0, 3, b"\0" * 128, 0)          # 5 planes < 2 per rank on 3 ranks
    with pytest.raises(odp.OdpError):
        g.partition(0, 2, None, 0)                 # no NCCL id
    g.close()
    wp = Workload("per0", (8, 6, 6), (-1, -1, -1), (1, 1, 1), (1, 0, 0), "HOLONOMIC_BOX", (1.0, 0.0, -1.0),
                  (0.0, 0.1), "low", 0.8, "brt", ("random_smooth", 3))
    g = odp.Grid(wp.N, wp.lo, wp.hi, wp.periodic_mask)
    with pytest.raises(odp.OdpError):
        g.partition(0, 2, b"\0" * 128, 0)          # periodic axis 0
    g.close()


@pytest.mark.parametrize("seed", [None, 3])
def test_v0_slab_is_the_slice(seed):
    w = coarsened(CONFIGS["c4"], (9, 5, 6, 5, 6, 4))
    full = make_v0(w, seed=seed)
    for P in (1, 2, 3, 4):
        from paper_2204_05520_b200 import capi
        for r in range(P):
            b, c = capi.partition_extent(w.N[0], P, r)
            np.testing.assert_array_equal(make_v0(w, seed=seed, i0=(b, c)), full[b:b + c])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        dist.init_process_group("gloo", init_method="env://", rank=rank, world_size=world)
        import paper_2204_05520_b200 as odp
        from paper_2204_05520_b200 import dist as odist
        assert odist.env_ranks() == (rank, world, rank)
        uid = odp.comm_unique_id() if rank == 0 else None
        uid = odist.broadcast_uid(uid, rank)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        w = coarsened(CONFIGS["c4"], (7, 4, 5, 4, 5, 4))
        mine = odist.local_v0(w, rank, world)
        slabs = [None] * world
        dist.all_gather_object(slabs, (odist.slabs(w.N[0], world)[rank], mine))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ids, slabs, None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, None, None, repr(e)))


def test_two_rank_id_broadcast_and_slabs_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    res.sort(key=lambda x: x[0])
    for r, ids, slabs, err in res:
        assert err is None, err
        assert len(set(ids)) == 1 and len(ids[0]) == 128          # every rank got rank 0's NCCL id
    w = coarsened(CONFIGS["c4"], (7, 4, 5, 4, 5, 4))
    full = make_v0(w)
    slabs = res[0][2]
    got = np.concatenate([v for (_, v) in slabs], axis=0)
    np.testing.assert_array_equal(got, full)                    # the slabs tile V0 exactly
    assert [s for (s, _) in slabs] == [(0, 4), (4, 3)]
