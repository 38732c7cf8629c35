"""N > 1 host path on CPU: two gloo ranks run the replica plumbing bench.py uses under torchrun
(sweep partition, max-over-ranks timing, result gather)."""
import json
import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_00966_b200.replicas import replica_bias, max_over_ranks, gather_results
    b = replica_bias((0.0, 0.0, 0.4714), world, rank, rel=0.1)
    t = max_over_ranks(1.5 + rank)
    allb = gather_results(b)
    with open(os.path.join(outdir, f"r{rank}.json"), "w") as f:
        json.dump({"b": b, "t": t, "all": allb}, f)
    dist.destroy_process_group()


def test_two_rank_replica_plumbing(tmp_path):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r = [json.load(open(tmp_path / f"r{k}.json")) for k in range(2)]
    assert r[0]["t"] == r[1]["t"] == 2.5                      # max over ranks
    assert r[0]["all"] == r[1]["all"]                         # identical gathered list
    bz = [v[2] for v in r[0]["all"]]
    assert bz[0] == pytest.approx(0.4714 * 0.9) and bz[1] == pytest.approx(0.4714 * 1.1)
    assert r[0]["b"][0] == 0.0 and r[1]["b"][1] == 0.0      # direction kept


def test_sweep_points_single_rank():
    from paper_2410_00966_b200.replicas import sweep_points, replica_bias
    assert sweep_points(1.0, 1) == [1.0]
    assert replica_bias((0.1, 0.2, 0.3), 1, 0) == (0.1, 0.2, 0.3)
    assert len(sweep_points(2.0, 8)) == 8


# ---------------------------------------------------------------- z-slab plumbing

def _slab_worker(rank, world, port, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_00966_b200.slabs import slab_dist, plane_range, cell_range
    from paper_2410_00966_b200.replicas import gather_results
    d = slab_dist(rank, world, device=rank)          # rank 0 makes the NCCL id, gloo broadcasts it
    rng = plane_range(128, world, rank)
    cells = cell_range((16, 8, 128), world, rank)
    allr = gather_results([rng, cells])
    with open(os.path.join(outdir, f"s{rank}.json"), "w") as f:
        json.dump({"id": d["nccl_id"].hex(), "rank": d["rank"], "world": d["world"], "all": allr}, f)
    dist.destroy_process_group()


def test_two_rank_slab_plumbing(tmp_path):
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    from _build import load_build
    load_build().build()                               # the id comes from libmcq (dlopen'ed NCCL)
    port = _free_port()
    mp.spawn(_slab_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r = [json.load(open(tmp_path / f"s{k}.json")) for k in range(2)]
    assert r[0]["id"] == r[1]["id"] and len(r[0]["id"]) == 256 and r[0]["id"] != "00" * 128
    assert (r[0]["rank"], r[1]["rank"], r[0]["world"]) == (0, 1, 2)
    assert r[0]["all"] == [[[0, 64], [0, 8192]], [[64, 128], [8192, 16384]]]   # planes partition nz


def test_plane_range_validation():
    from paper_2410_00966_b200.slabs import plane_range, slab_dist
    assert [plane_range(12, 3, r) for r in range(3)] == [(0, 4), (4, 8), (8, 12)]
    with pytest.raises(ValueError):
        plane_range(10, 4, 0)
    with pytest.raises(ValueError):
        plane_range(8, 2, 2)
    with pytest.raises(ValueError):
        slab_dist(0, 2, nccl_id=b"short")
    assert slab_dist(0, 1) == {"rank": 0, "world": 1, "device": -1, "stream": None}
