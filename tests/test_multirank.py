"""Host logic on CPU: the replica plumbing bench.py uses under torchrun (gloo,
world_size 2), the clock-sampler parser, and the seeded config-3 map table."""
import os
import socket

import numpy as np
import pytest

import bench
from paper_2103_17040_b200 import configs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bench.barrier(dist, "gloo")
    mx = bench.reduce_max(dist, "gloo", 1.0 + rank)
    sm = bench.reduce_sum(dist, "gloo", 10.0 * (rank + 1))
    out[rank] = (mx, sm)
    dist.destroy_process_group()


def test_replica_reductions_gloo_world2():
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == (2.0, 30.0) and out[1] == (2.0, 30.0)


def test_clock_summary_parser(tmp_path):
    c = bench.ClockSampler(0)
    c.path = str(tmp_path / "clk.csv")
    with open(c.path, "w") as f:
        f.write("0, 1965, 1965, 800.1, 0x0, Not Active, Not Active, Not Active, Not Active\n")
        f.write("0, 1950, 1965, 900.0, 0x4, Not Active, Not Active, Not Active, Active\n")
        f.write("0, 1960, 1965, 910.0, 0x0, Not Active, Not Active, Not Active, Not Active\n")
    s = c.summary()
    assert s["sm_mhz"] == 1960 and s["sm_max_mhz"] == 1965 and s["reasons"] == ["sw_power_cap"]


def test_config3_table_is_seeded_and_admissible():
    t1 = configs.make_table(8, 8)
    t2 = configs.make_table(8, 8)
    assert np.array_equal(t1, t2) and t1.shape == (81, 4)
    Y = configs.micro_quadrature_points(8)
    g0 = 16.0 * (1 - 2 * Y[:, 0]) * Y[:, 1] * (1 - Y[:, 1])
    g1 = 16.0 * Y[:, 0] * (1 - Y[:, 0]) * (1 - 2 * Y[:, 1])
    xs = np.arange(9) / 8.0
    s = np.outer(xs, xs).reshape(-1)  # x0*x1 at node j*9+i (symmetric)
    for i in range(81):
        a = 0.15 * s[i]
        A = t1[i]
        det = (A[0] + a * g0) * (A[3] + a * g1) - (A[1] + a * g1) * (A[2] + a * g0)
        assert det.min() >= 0.3
    assert np.abs(t1 - np.array([1, 0, 0, 1.0])).max() <= 0.25


def test_config_shapes_match_baseline():
    c = configs.CONFIGS
    assert (c["c1"].n_macro, c["c1"].n_micro) == (289, 289)
    assert (c["c2"].n_macro, c["c2"].n_micro, c["c2"].micro_nnz) == (4225, 1089, 9409)
    assert (c["c3"].n_macro, c["c3"].n_micro, c["c3"].micro_nnz) == (16641, 4225, 37249)
    assert c["c3"].csr_bytes_per_dof == pytest.approx(70.53, abs=0.01)
