"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel wiring
(SURVEY.md §8(e)): batch sharding + the dW all-reduce reproduce the full-batch
result.  The per-rank compute here is the oracle (test infrastructure) standing
in for the GPU passes, which need a device; the GPU path is covered by
bench.py --gpus N under torchrun and by tests/test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import taps as T
from paper_2309_15812_b200 import dp, inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, C, H, W, K, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        angles = T.direction_angles(8, C, "cycled")
        oh, ow = (np.array(a, np.int32) for a in T.taps_table(K, K // 2, angles))
        x = inputs.activation((N, C, H, W), 0)
        dy = inputs.activation((N, C, H, W), 2)
        w = inputs.weights(C, K)
        lo, hi = dp.shard_range(N, world, rank)

        def fwd(xs, ww):
            return torch.from_numpy(oracle.forward(xs.numpy(), ww.numpy(), oh, ow))

        def bwi(g, ww):
            return torch.from_numpy(oracle.backward_input(g.numpy(), ww.numpy(), oh, ow, H, W))

        def bww(xs, g):
            return torch.from_numpy(oracle.backward_weight(xs.numpy(), g.numpy(), oh, ow))

        y, dx, dW = dp.dp_layer_step(torch.from_numpy(x[lo:hi]).double(), torch.from_numpy(w).double(),
                                     torch.from_numpy(dy[lo:hi]).double(), fwd, bwi, bww)
        out[rank] = (lo, hi, y.numpy(), dx.numpy(), dW.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N", [4, 5])
def test_dp_two_ranks_matches_full_batch(N):
    C, H, W, K, world = 8, 9, 10, 7, 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, N, C, H, W, K, out), nprocs=world, join=True)
    angles = T.direction_angles(8, C, "cycled")
    oh, ow = (np.array(a, np.int32) for a in T.taps_table(K, K // 2, angles))
    x = inputs.activation((N, C, H, W), 0)
    dy = inputs.activation((N, C, H, W), 2)
    w = inputs.weights(C, K)
    y_full = oracle.forward(x, w, oh, ow)
    dx_full = oracle.backward_input(dy, w, oh, ow, H, W)
    dW_full = oracle.backward_weight(x, dy, oh, ow)
    covered = []
    for r in range(world):
        lo, hi, y, dx, dW = out[r]
        covered += list(range(lo, hi))
        # per-sample outputs are bitwise independent of the sharding
        assert np.array_equal(y, y_full[lo:hi]) and np.array_equal(dx, dx_full[lo:hi])
        # every rank ends with the global-batch weight gradient
        np.testing.assert_allclose(dW, dW_full, rtol=1e-12, atol=1e-12)
    assert covered == list(range(N))


def test_shard_range():
    for N in range(0, 20):
        for world in range(1, 6):
            parts = [dp.shard_range(N, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == N
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1
    with pytest.raises(ValueError):
        dp.shard_range(4, 2, 2)
