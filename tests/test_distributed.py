"""K5 host logic on CPU: world-size-2 gloo run of the sharded IL epoch with
the fixed-order theta-gradient exchange (the GPU path swaps the oracle epoch
body for docp_il_epoch and gloo for NCCL)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import pyoracle as po
from paper_2510_06179_b200.distributed import fixed_order_allreduce, shard_range

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _epochs(x0, demos, w0, lo, hi, epochs, allreduce):
    prob = po.cartpole_problem(40)
    nz, nl = po.sizes(prob)
    n = hi - lo
    lam_c, lt_c = np.zeros((n, nl)), np.zeros((n, nl))
    w = w0.copy()
    losses = []
    for _ in range(epochs):
        th = np.array([np.concatenate([w, [0.05], x]) for x in x0[lo:hi]])
        # scale loss by the GLOBAL batch, as train_il divides by n_demos
        B = x0.shape[0]
        loss, grad, *_ = po.il_epoch("port", prob, th, demos[lo:hi], lam_c, lt_c, po.sqp_config(max_sqp_iters=5),
                                     0, 4)
        # il_epoch scales by its local batch; rescale to the global one
        part = torch.tensor(np.concatenate([[loss * n / B], grad * n / B]), dtype=torch.float64)
        tot = allreduce(part).numpy()
        losses.append(tot[0])
        w = w - 1e-2 * tot[1:]
    return np.array(losses), w


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = np.load(os.path.join(GOLDEN, "train_il_cartpole_seed3.npz"))
    lo, hi = shard_range(g["x0"].shape[0], rank, world)
    losses, w = _epochs(g["x0"], g["demos"], g["w0"], lo, hi, 2, fixed_order_allreduce)
    q.put((rank, losses, w))
    dist.destroy_process_group()


def test_shard_range_covers_contiguously():
    for n in (1, 7, 8, 4096):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_two_rank_gloo_epochs_match_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (l, w)) for r, l, w in (q.get(timeout=600) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    # identical on every rank
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    # equal to one process summing the same two shard partials in rank order
    g = np.load(os.path.join(GOLDEN, "train_il_cartpole_seed3.npz"))
    B = g["x0"].shape[0]
    spans = [shard_range(B, r, 2) for r in range(2)]
    # single-process emulation: run both shards, combine 0.0 + p0 + p1
    prob = po.cartpole_problem(40)
    nz, nl = po.sizes(prob)
    caches = [(np.zeros((hi - lo, nl)), np.zeros((hi - lo, nl))) for lo, hi in spans]
    w = g["w0"].copy()
    for epoch in range(2):
        tot = np.zeros(5)
        for (lo, hi), (lc, ltc) in zip(spans, caches):
            th = np.array([np.concatenate([w, [0.05], x]) for x in g["x0"][lo:hi]])
            loss, grad, *_ = po.il_epoch("port", prob, th, g["demos"][lo:hi], lc, ltc,
                                         po.sqp_config(max_sqp_iters=5), 0, 4)
            n = hi - lo
            tot = tot + np.concatenate([[loss * n / B], grad * n / B])
        assert tot[0] == res[0][0][epoch]
        # and within rounding of the reference's single-worker train_il
        assert abs(tot[0] - g["objectives"][epoch]) <= 1e-12 * abs(g["objectives"][epoch])
        w = w - 1e-2 * tot[1:]
    assert np.array_equal(w, res[0][1])
    assert np.allclose(w, g["final_weights"], rtol=1e-12, atol=0)


# ------------------------------------------------ bench.py rank logic (gloo, world size 2)


def _bench_rank_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_06179_b200.distributed import global_batch, max_over_ranks
    out = {}
    for scaling in ("weak", "strong"):
        gb = global_batch(4096, world, scaling)
        out[scaling] = (gb, shard_range(gb, rank, world))
    # each rank's step time differs; every rank must see the slowest
    out["max"] = max_over_ranks(10.0 + rank)
    # the exchanged [loss | grad] partials, summed in rank order on every rank
    part = torch.tensor([0.1 * (rank + 1)] + [float(rank)] * 8, dtype=torch.float64)
    out["sum"] = fixed_order_allreduce(part).numpy()
    q.put((rank, out))
    dist.destroy_process_group()


def test_bench_rank_logic_two_ranks():
    """bench.py's per-rank shard (weak: 4096 per rank; strong: 4096 split),
    the max-over-ranks step time and the rank-order gradient sum."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert res[0]["weak"] == (8192, (0, 4096)) and res[1]["weak"] == (8192, (4096, 8192))
    assert res[0]["strong"] == (4096, (0, 2048)) and res[1]["strong"] == (4096, (2048, 4096))
    assert res[0]["max"] == res[1]["max"] == 11.0
    expect = (0.0 + np.array([0.1] + [0.0] * 8)) + np.array([0.2] + [1.0] * 8)
    assert np.array_equal(res[0]["sum"], expect) and np.array_equal(res[1]["sum"], expect)


def test_bench_gpus_flag_spawns_or_refuses():
    """`bench.py --gpus N` outside torchrun re-launches itself with N ranks on
    127.0.0.1; under torchrun a WORLD_SIZE that disagrees with --gpus is an error."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    cmd = bench.spawn_command(type("A", (), {"gpus": 4})(), ["--gpus", "4", "--steps", "2"])
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"] and cmd[-5].endswith("bench.py")
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=3" in r.stderr
