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
