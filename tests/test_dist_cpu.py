"""N > 1 path on CPU: two gloo ranks shard a sweep exactly as bench.py does
for GPUs, run their shards (the C oracle stands in for the device engine,
which needs a GPU) and gather per-instance results; the union must equal the
single-process run instance by instance."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2510_14392_b200 import dist as fbdist
from paper_2510_14392_b200.batch import Batch


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _batch(gen):
    from catalog import scenario_mixed
    return scenario_mixed(gen, n_seeds=13)


def _worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist
    from backends import OracleLib
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = OracleLib()
    batch = _batch(orc.generate_bursty)
    sub, idx = fbdist.shard_batch(batch, rank, world)
    out = orc.run(sub)
    allres = fbdist.gather_results(out.results, idx, batch.n_instances, dist)
    if rank == 0:
        q.put(allres.tobytes())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_indices_partition():
    for n in (0, 1, 7, 64):
        for w in (1, 2, 3, 8):
            parts = [fbdist.shard_indices(n, r, w) for r in range(w)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(n))


def test_two_rank_gloo_sharded_sweep_equals_single_process(oracle):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    batch = _batch(oracle.generate_bursty)
    whole = oracle.run(batch).results
    assert got == whole.tobytes()


def test_shard_batch_keeps_rows(oracle):
    batch = _batch(oracle.generate_bursty)
    sub, idx = fbdist.shard_batch(batch, 1, 3)
    assert isinstance(sub, Batch) and sub.n_instances == len(idx)
    a = oracle.run(sub).results
    b = oracle.run(batch).results[idx]
    assert a.tobytes() == b.tobytes()


# ---------------------------------------------------------------- cluster (C5)

def _cluster_worker(rank, world, port, q, names):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist
    from backends import OracleLib
    from catalog import cluster_cases
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = OracleLib()
    for name, rows, cfgs, lb, hz in cluster_cases(orc.generate_bursty):
        if name not in names or len(cfgs) < world:
            continue
        out = orc.run_cluster_dist(rows, cfgs, lb, hz, dist)
        if rank == 0:
            q.put((name, out.node_results.tobytes(), out.records.tobytes(),
                   out.route_node.tobytes(), out.incomplete))
    if rank == 0:
        q.put(None)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_cluster_shards_equal_run_cluster(oracle, world):
    """The multi-rank cluster protocol (node partition, per-epoch report
    allgather, replicated router, merge_shards) reproduces run_cluster."""
    from catalog import cluster_cases
    names = ("pab0_8", "count0_8", "pab5000_8", "count37_3", "pab_hz10s_8", "pab20_2")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cluster_worker, args=(r, world, port, q, names))
             for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    while True:
        item = q.get(timeout=300)
        if item is None:
            break
        got[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cases = {c[0]: c for c in cluster_cases(oracle.generate_bursty)}
    checked = 0
    for name in names:
        _, rows, cfgs, lb, hz = cases[name]
        if len(cfgs) < world:
            continue
        ref = oracle.run_cluster(rows, cfgs, lb, hz)
        res, rec, route, inc = got[name]
        assert res == ref.node_results.tobytes(), name
        assert rec == ref.records.tobytes(), name
        assert route == ref.route_node.tobytes(), name
        assert inc == ref.incomplete, name
        checked += 1
    assert checked >= 5


def test_cluster_partition_matches_abi():
    import ctypes as C
    from paper_2510_14392_b200 import fbgpu
    from paper_2510_14392_b200.cluster import partition
    L = fbgpu.lib()  # loads without a GPU; partition is host logic
    for n in (1, 3, 8, 64, 511):
        for w in range(1, min(n, 8) + 1):
            seen = []
            for r in range(w):
                lo, nl = C.c_int32(), C.c_int32()
                assert L.fb_cluster_partition(n, w, r, C.byref(lo), C.byref(nl)) == 0
                assert (lo.value, nl.value) == partition(n, w, r)
                seen.extend(range(lo.value, lo.value + nl.value))
            assert seen == list(range(n))


def _bench(*args, timeout=600):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args], cwd=root,
                         env=env, capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("world", [2, 3])
def test_bench_launches_n_ranks(world):
    """`python bench.py --gpus N` outside torchrun starts N ranks itself
    (torch.distributed.run on 127.0.0.1); here with gloo and no device work:
    every rank builds its C2 shard, the line reports n_gpus == N with one
    per-rank figure each, and the C3 results gathered from the interleaved
    shards come back in global instance order."""
    line = _bench("--gpus", str(world), "--dry-run")
    assert line["n_gpus"] == world
    assert line["instances_per_rank"] == [8.0] * world
    assert line["c3_gathered_in_order"] and line["c3_instances"] == 1024


def test_bench_reference_arm_loads_no_product_code():
    """The reference arm builds its inputs with the reference's own generator
    and runs the reference's run_node: libfbgpu.so is never mapped."""
    line = _bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-budget-s", "1")
    assert line["impl"] == "reference"
    assert line["repo_so_loaded"] == []
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
