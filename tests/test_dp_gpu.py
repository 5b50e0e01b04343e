"""Data parallelism on the GPU: two ranks, each running the
LIBRARY's passes (liboriented1d through the C ABI) on its batch shard, with the dW
all-reduce over a real process group.  Both ranks share cuda:0 (the test box has one
GPU), so the group is gloo over CUDA tensors; bench.py --gpus N uses NCCL, one GPU per
rank.  Checked: dW equals the oracle's full-batch dW (normwise 1e-5), y and dx are
bitwise the single-process full-batch run's rows (per-sample passes do not depend on the
sharding)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import taps as T
from paper_2309_15812_b200 import inputs

pytestmark = pytest.mark.gpu

N, C, H, W, K = 6, 16, 56, 56, 31


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fused, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_15812_b200 import binding as B
        from paper_2309_15812_b200 import dp
        torch.cuda.set_device(0)
        angles = np.array(T.direction_angles(8, C, "cycled"))
        lo, hi = dp.shard_range(N, world, rank)
        plan = B.Plan(hi - lo, C, H, W, K, angles, device="cuda:0")
        x = torch.from_numpy(inputs.activation((N, C, H, W), 0)[lo:hi]).cuda()
        dy = torch.from_numpy(inputs.activation((N, C, H, W), 2)[lo:hi]).cuda()
        w = torch.from_numpy(inputs.weights(C, K)).cuda()
        step = dp.DPLayerStep(plan, fused=fused)
        y, dx, dW = step(x, w, dy)
        torch.cuda.synchronize()
        out[rank] = (lo, hi, y.cpu().numpy(), dx.cpu().numpy(), dW.cpu().numpy(), plan.describe())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True])
def test_dp_two_ranks_library_dW_allreduce(fused):
    from paper_2309_15812_b200 import binding as B
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), fused, out), nprocs=world, join=True)
    angles = T.direction_angles(8, C, "cycled")
    oh, ow = (np.array(a, np.int32) for a in T.taps_table(K, K // 2, angles))
    x = inputs.activation((N, C, H, W), 0)
    dy = inputs.activation((N, C, H, W), 2)
    w = inputs.weights(C, K)
    ref_dW = oracle.backward_weight(x, dy, oh, ow, 1, max(1, oracle.max_threads()))
    # the unsharded library run (same process count 1) for the bitwise per-sample check
    plan = B.Plan(N, C, H, W, K, np.array(angles), device="cuda:0")
    xd, dyd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda(), torch.from_numpy(w).cuda()
    y_full = B.forward(plan, xd, wd).cpu().numpy()
    dx_full = B.backward_input(plan, dyd, wd).cpu().numpy()
    covered = []
    for r in range(world):
        lo, hi, y, dx, dW, desc = out[r]
        assert desc.startswith("spec"), desc
        covered += list(range(lo, hi))
        assert np.array_equal(y, y_full[lo:hi]) and np.array_equal(dx, dx_full[lo:hi])
        err = np.max(np.abs(dW - ref_dW)) / np.max(np.abs(ref_dW))
        assert err <= 1e-5, err
    assert covered == list(range(N))
    # both ranks hold the same reduced gradient
    assert np.array_equal(out[0][4], out[1][4])
