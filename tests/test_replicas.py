"""Multi-GPU is "replicas only".  These tests check the
host logic with world_size 2 over gloo on CPU: the rendezvous bench.py uses,
max-over-ranks timing, and that the whole-job value is ranks x steps / max
time."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import bench
    dist, r, w, local = bench.dist_setup()
    assert (r, w, local) == (rank, world, rank)
    assert dist.get_backend() == "gloo"
    bench.barrier(dist)
    t = bench.max_over_ranks(dist, 10.0 * (rank + 1))   # rank 1 is the slow one
    value = w * 5 / (t * 1e-3)                           # 5 steps per rank
    dist.destroy_process_group()
    q.put((rank, t, value))


def test_max_over_ranks_and_whole_job_value():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert [t for _, t, _ in res] == [20.0, 20.0]       # every rank sees the max
    assert res[0][2] == pytest.approx(2 * 5 / 0.020)


def test_gpu_arm_fails_loudly_without_device():
    """No CPU fallback: on a host without a CUDA device the GPU arm exits
    non-zero instead of timing anything else."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "1",
                        "--no-e2e", "--no-cpu"], capture_output=True, text=True, timeout=300)
    import torch
    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    assert r.returncode != 0
    assert "no CUDA device" in (r.stderr + r.stdout)


def _shard_worker(rank, world, port, m, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import bench
    from paper_2107_11650_b200 import api as A
    dist, r, w, _ = bench.dist_setup()
    b, e = A.shard_range(m, w, r)
    got = [torch.zeros(2, dtype=torch.int64) for _ in range(w)]
    dist.all_gather(got, torch.tensor([b, e], dtype=torch.int64))
    dist.destroy_process_group()
    q.put((rank, [tuple(int(v) for v in g) for g in got]))


@pytest.mark.parametrize("m", [256, 7])
def test_parameter_slices_shard_over_ranks(m):
    """Parameter imaging shards its independent FE slices over the ranks
    (bench.py config-4 workload): with world size 2 over
    gloo the ranks' ranges are contiguous, disjoint and cover all M slices."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_shard_worker, args=(r, 2, port, m, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    ranges = res[0][1]
    assert ranges == res[1][1]
    assert ranges[0][0] == 0 and ranges[-1][1] == m
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(len(ranges) - 1))
    assert all(e > b for b, e in ranges)


def test_empty_shard_never_reaches_the_device(api):
    """More ranks than FE slices: shard_range gives some ranks an empty range.
    The C-ABI reads slice range (0, 0) as "all slices", so the host mirror
    returns an empty dataset without calling it (no device, no D2H copy into a
    0-slice buffer); inverted or out-of-range shards are rejected."""
    A = api
    m = 1
    assert A.shard_range(m, 2, 0) == (0, 0)
    y = np.zeros((m, 8, 3, 2), np.complex128)
    ds = A.ParameterDataset(y, [10.0, 20.0, 30.0])
    mask = A.SamplingMask(8, 3, np.ones((8, 3), np.uint8))
    tot = []
    out = A.recon_param_dataset(ds, mask, A.HankelConfig(), A.AdmmConfig(max_outer=1), total_iters=tot,
                                slices=A.shard_range(m, 2, 0))
    assert out.data.shape == (0, 8, 3, 2) and tot == [0]
    for bad in [(1, 0), (0, 2), (-1, 1)]:
        with pytest.raises(ValueError):
            A.recon_param_dataset(ds, mask, A.HankelConfig(), A.AdmmConfig(max_outer=1), slices=bad)
    with pytest.raises(ValueError):
        A.ParamPlan(y, mask, A.HankelConfig(), A.AdmmConfig(max_outer=1), slices=(0, 0))
