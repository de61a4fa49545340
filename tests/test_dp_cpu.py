"""World-size-2 gloo tests (CPU) of the exact data-parallel protocol in
paper_2406_15102_b200/dp.py: the statistics all-reduce(MAX) on uint32 words,
the int32 accumulator all-reduce(SUM) and the fp64 dequant.  The per-shard
transform / quantize / int-GEMM steps are computed here with the CPU oracle
(standing in for the kernels, which need a B200 -- tests/test_gpu_dp.py runs
the same protocol through the kernels), and the result must equal the
single-process reference bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hlq_oracle as orc


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2406_15102_b200.dp import Reducer, dequant
        red = Reducer()
        # 1) unsigned max over words incl. >= 2^31 (the ~minnz encoding)
        mine = [0x3F800000, 0x80000001, 5, 0] if rank == 0 else [0x3F000000, 0xFFFFFFF0, 0, 0x90000000]
        st = torch.tensor(np.array(mine, dtype=np.uint32).view(np.int32))
        red.max_stats(st)
        got = st.numpy().view(np.uint32).tolist()
        assert got == [0x3F800000, 0xFFFFFFF0, 5, 0x90000000], [hex(v) for v in got]
        # 2) the exact protocol on a batch split over the ranks
        B, L, I, O, rank_r = case
        x, w, gy = orc.make_inputs(11, (B, L, I), (O, I), (B, L, O))
        bases = orc.lowest_sequency_bases(16, rank_r)
        axis = orc.proj_axis_rule(B, L, 16)
        half = B // world
        sl = slice(rank * half, (rank + 1) * half)
        xs, gs = x[sl], gy[sl]
        px = orc.transform_axis(xs, axis, 16, bases)
        pg = orc.transform_axis(gs, axis, 16, bases).reshape(-1, O)
        amax = np.array([np.abs(px).max(), np.abs(pg).max()], dtype=np.float32)
        st = torch.tensor(np.array([amax[0].view(np.uint32), 0, amax[1].view(np.uint32), 0],
                                   dtype=np.uint32).view(np.int32))
        red.max_stats(st)
        g = st.numpy().view(np.uint32)
        ax, ag = g[0:1].view(np.float32)[0], g[2:3].view(np.float32)[0]
        cx, sx = orc.quantize_with_amax(px.reshape(-1, I), 8, ax)
        cg, sg = orc.quantize_with_amax(np.ascontiguousarray(pg.T), 8, ag)
        acc = torch.from_numpy(orc.int_gemm(cg, cx).astype(np.int32))
        red.sum_acc(acc)
        gw = dequant(acc, torch.tensor([sg]), torch.tensor([sx]), 1.0 / B).numpy()
        _, ref_gw = orc.hlq_backward(x, w, gy, bases=bases)
        assert np.array_equal(gw, ref_gw), np.abs(gw - ref_gw).max()
        # replica semantics for contrast: shard-local scales do NOT reproduce the reference
        _, local_gw = orc.hlq_backward(xs, w, gs, bases=bases)
        q.put(("ok", rank, float(np.linalg.norm(local_gw * half / B * world - ref_gw))))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put(("err", rank, repr(e)))


@pytest.mark.parametrize("case", [(8, 48, 32, 24, 8),    # token axis (L >= 16)
                                  (64, 1, 40, 32, 2)])   # batch axis, 16-aligned shards
def test_global_scale_protocol_world2(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[0] == "ok", r
