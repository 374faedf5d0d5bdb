"""Multi-rank cluster dispatch on the device: the host dispatcher over the
interactive node set (cluster.run_cluster_host) with the nodes partitioned
over torch.distributed ranks -- a per-epoch all-gather of the nodes' load
reports, replicated routing, and for retry_reroute a per-node broadcast of
the rejects.  Two ranks share the box's one GPU here (gloo carries the
reports); every rank's merged output must equal the reference's run_cluster
(golden fixtures), retry_reroute included."""
from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = ["pab0_8", "count37_3", "pab5000_8", "rr_giant_2", "rr_pab30_3", "rr_mixed_4",
         "rr_count0_4"]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, names, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist
    from backends import cluster_summary
    from catalog import cluster_cases, reroute_cluster_cases
    from paper_2510_14392_b200 import fbgpu
    from paper_2510_14392_b200.cluster import run_cluster_host
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cases = {c[0]: c for c in cluster_cases(fbgpu.generate_bursty) +
             reroute_cluster_cases(fbgpu.generate_bursty)}
    for name in names:
        _, rows, cfgs, lb, hz = cases[name]
        if len(cfgs) < world:
            continue
        out = run_cluster_host(rows, cfgs, lb, hz, dist=dist)
        q.put((rank, name, cluster_summary(out)))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, None, None))


@pytest.mark.parametrize("world", [2, 3])
def test_host_dispatcher_over_ranks_matches_golden(fb, golden, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, done = {}, 0
    while done < world:
        rank, name, summ = q.get(timeout=600)
        if name is None:
            done += 1
            continue
        got[(rank, name)] = summ
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    checked = 0
    for (rank, name), summ in got.items():
        assert summ == golden["clusters"][name], (rank, name)
        checked += 1
    assert checked >= world * 5
