"""Host-side logic of the multi-rank path, world_size 2 over gloo on CPU.

No GPU compute here: the NCCL-id bootstrap (rank 0 asks libnbk for the id,
torch.distributed broadcasts it), the z-slab partition each rank derives on
its own (nbk_partition, host only) checked for consistency across ranks, and
bench.py's max-over-ranks timing reduction.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2405_11065_b200 as nbk
        import bench
        # 1. NCCL unique-id bootstrap over the process group
        idt = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            idt = torch.frombuffer(bytearray(nbk.nccl_unique_id()), dtype=torch.uint8).clone()
        dist.broadcast(idt, 0)
        ids = [None] * world
        dist.all_gather_object(ids, bytes(idt.numpy()))
        # 2. slab partition derived independently per rank
        spec = nbk.MeshSpec(**nbk.CONFIGS["C4"].mesh_args(world))
        part = nbk.partition(spec, world, rank)
        parts = [None] * world
        dist.all_gather_object(parts, part)
        # 3. max-over-ranks of per-rank times
        tmax = bench.max_over_ranks(1.0 + rank, world, device="cpu")
        q.put((rank, ids, parts, tmax, spec.E))
    finally:
        dist.destroy_process_group()


def test_two_rank_bootstrap_partition_and_timing_reduction():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    out.sort()
    ids = out[0][1]
    assert ids[0] == ids[1] and len(ids[0]) == 128 and any(ids[0])
    parts, E = out[0][2], out[0][4]
    assert [p["e_offset"] for p in parts] == [0, E // 2]
    assert sum(p["e_local"] for p in parts) == E
    assert parts[0]["n_global"] == parts[1]["n_global"]
    # C4 per GPU is 64x64x32, N=8: one shared plane of 449^2 nodes, one face
    # layer of 64*64*64 values per rank
    assert parts[0]["face_nodes"] == parts[1]["face_nodes"] == 449 * 449
    assert parts[0]["face_layer"] == 64 * 64 * 64
    # unique shared nodes: both slabs' local plans + the plane = the 1-rank plan
    import paper_2405_11065_b200 as nbk
    one = nbk.partition(nbk.MeshSpec(**nbk.CONFIGS["C4"].mesh_args(2)), 1, 0)
    assert parts[0]["n_shared"] + parts[1]["n_shared"] + 449 * 449 == one["n_shared"]
    assert (parts[0]["n_copies"] + parts[1]["n_copies"] + 2 * 64 ** 3) == one["n_copies"]
    assert all(o[3] == 2.0 for o in out)   # max over ranks of 1.0, 2.0


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_partition_tiles_the_box(P):
    import paper_2405_11065_b200 as nbk
    spec = nbk.MeshSpec(**nbk.CONFIGS["C5"].mesh_args(P))
    parts = [nbk.partition(spec, P, r) for r in range(P)]
    one = nbk.partition(spec, 1, 0)
    assert sum(p["e_local"] for p in parts) == spec.E
    assert [p["e_offset"] for p in parts] == [r * spec.E // P for r in range(P)]
    planes = P - 1
    Gx = spec.ex * (spec.N - 1) + 1
    assert sum(p["face_nodes"] for p in parts) == 2 * planes * Gx * Gx
    assert sum(p["n_shared"] for p in parts) + planes * Gx * Gx == one["n_shared"]


def test_partition_rejects_bad_rank_counts():
    import paper_2405_11065_b200 as nbk
    with pytest.raises(nbk.NbkError):
        nbk.partition(nbk.MeshSpec(4, 4, 6, 8), 4, 0)    # ez % P != 0
    with pytest.raises(nbk.NbkError):
        nbk.partition(nbk.MeshSpec(4, 4, 128, 8), 128, 0)  # > 64 ranks


def test_bench_gpus_n_relaunches_under_torchrun():
    """bench.py --gpus N outside torchrun re-executes itself under
    torch.distributed.run with N ranks (127.0.0.1 rendezvous).  The reference
    arm needs no GPU: rank 0 alone runs the oracle and prints the one JSON line
    (n_gpus = N), the other ranks exit 0."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl",
                          "reference", "--config", "C1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
