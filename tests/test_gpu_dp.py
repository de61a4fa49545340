"""Exact data-parallel mode through the kernels: two ranks (gloo, both on
cuda:0 -- the round's GPU boxes have one device) each run
hlq_backward_global on half the batch; dW must equal the single-process
reference bit for bit on every rank and the dX rows must be the matching
slice of the reference dX."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import hlq_oracle as orc

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, q):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2406_15102_b200.dp import Reducer, hlq_backward_global
        B, L, I, O = case
        x, w, gy = orc.make_inputs(21, (B, L, I), (O, I), (B, L, O))
        half = B // world
        sl = slice(rank * half, (rank + 1) * half)
        dev = "cuda:0"
        gp = hlq_backward_global(torch.from_numpy(x[sl]).to(dev), torch.from_numpy(w).to(dev),
                                 torch.from_numpy(gy[sl]).to(dev), B, Reducer())
        torch.cuda.synchronize()
        ref_gx, ref_gw = orc.hlq_backward(x, w, gy)
        ok_w = np.array_equal(gp.grad_weight.cpu().numpy(), ref_gw)
        ok_x = np.array_equal(gp.grad_input.cpu().numpy(), ref_gx[sl])
        q.put(("ok" if ok_w and ok_x else "mismatch", rank, ok_w, ok_x))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put(("err", rank, repr(e)))


@pytest.mark.parametrize("case", [(8, 197, 256, 384), (128, 1, 256, 128)])
def test_global_scale_dp_world2(case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[0] == "ok", r
