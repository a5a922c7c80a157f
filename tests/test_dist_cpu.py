"""Multi-process (torch.distributed gloo, world_size 2, CPU) checks of the block-column partition's host
logic: the partition, the NCCL-id bootstrap over a process group, and the oracle's
block-column sweep — each rank computes its column block and all-gathers λ̂ — reproducing the full
sweep bit for bit. The library's own collectives run in tests/test_gpu_dist.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W
from oracle import refine as orf
from paper_2602_19090_b200.dist import broadcast_id, broadcast_tensor, partition


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        q.put((rank, fn(rank, ws)))
    finally:
        dist.destroy_process_group()


def _run(fn, ws=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, fn, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [out[r] for r in range(ws)]


def test_partition():
    assert partition(8192, 8, 3) == (3072, 1024)
    assert [partition(12, 3, r) for r in range(3)] == [(0, 4), (4, 4), (8, 4)]
    with pytest.raises(ValueError):
        partition(10, 4, 0)


def _bootstrap(rank, ws):
    uid = bytes(np.random.default_rng(1234).integers(0, 256, 128, dtype=np.uint8)) if rank == 0 else None
    return broadcast_id(uid)


def test_unique_id_bootstrap_gloo():
    ids = _run(_bootstrap)
    assert len(ids[0]) == 128 and ids[0] == ids[1]


def _block_sweep(rank, ws):
    import torch
    A, lam0, X0, cfg = W.make_config("c2", n=256)
    n = A.shape[0]
    col0, nl = partition(n, ws, rank)

    def allgather(lamJ):
        parts = [torch.zeros(nl, dtype=torch.float64) for _ in range(ws)]
        dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(lamJ)))
        return np.concatenate([p.numpy() for p in parts])

    XJ, lam = orf.sweep_block(A, X0, lam0, 1e-14, col0, nl, allgather)
    parts = [torch.zeros((n, nl), dtype=torch.float64) for _ in range(ws)]
    dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(XJ)))
    return np.concatenate([p.numpy() for p in parts], axis=1), lam


def test_oracle_block_sweep_equals_full_sweep_gloo():
    (Xa, la), (Xb, lb) = _run(_block_sweep)
    A, lam0, X0, cfg = W.make_config("c2", n=256)
    Xf, lf, info = orf.sweep(A, X0, lam0, 1e-14, cluster_mode=0)
    assert np.array_equal(Xa, Xb) and np.array_equal(la, lb)
    assert np.array_equal(Xa, Xf)
    assert np.array_equal(la, lf)


def test_host_group_comm_on_cpu():
    """The in-process host-group communicators are plain host objects (no GPU needed to create them)."""
    import paper_2602_19090_b200 as ozr
    cs = ozr.ozr_comm_create_host_group(4)
    assert [c.rank for c in cs] == [0, 1, 2, 3] and {c.size for c in cs} == {4}
    for c in cs:
        c.close()


def _bcast_colmajor(rank, ws):
    import torch
    n = 6
    t = torch.empty((n, n), dtype=torch.float64).t()   # column-major view (stride (1, n)), as bench.py holds A
    if rank == 0:
        t.copy_(torch.arange(n * n, dtype=torch.float64).reshape(n, n))
    broadcast_tensor(t, src=0)
    lam = torch.arange(n, dtype=torch.float64) if rank == 0 else torch.zeros(n, dtype=torch.float64)
    broadcast_tensor(lam, src=0)
    return t.numpy().copy(), lam.numpy().copy(), tuple(t.stride())


def test_broadcast_colmajor_gloo():
    """bench.py's N > 1 set-up broadcasts the column-major A and X̂₀ from rank 0 (collectives need
    contiguous tensors; the helper broadcasts the contiguous transposed view of the same memory)."""
    (a0, l0, s0), (a1, l1, s1) = _run(_bcast_colmajor)
    assert np.array_equal(a0, a1) and np.array_equal(l0, l1)
    assert np.array_equal(a1, np.arange(36, dtype=np.float64).reshape(6, 6)) and s1 == (1, 6)


def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself as two ranks (here over gloo,
    --dry-run: no GPU); both ranks agree on the block-column partition of the c4' problem."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["consistent"]
    assert [(p["col0"], p["n_local"]) for p in line["partition"]] == [(0, 4096), (4096, 4096)]


def test_bench_rank_count_mismatch_fails():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 2 and "refusing" in out.stderr
