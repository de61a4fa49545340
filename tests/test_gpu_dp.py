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


# ---------------------------------------------------------------------------
# the exact mode in the TRAINING path: HLQLinear modules under enable_exact_dp,
# stepped by bench.py's train_steps loop, two ranks on one GPU (gloo)
# ---------------------------------------------------------------------------

def _tiny_vit():
    from paper_2406_15102_b200.layers import convert_linears
    from paper_2406_15102_b200.vit import ViT
    torch.manual_seed(0)
    m = ViT(image=32, patch=8, dim=64, depth=2, heads=2, mlp=256, classes=10).cuda()
    convert_linears(m)
    # only the HLQ weights train: every other gradient is a cross-sample
    # reduction whose fp32 summation order differs between 1 and 2 ranks
    for n, p in m.named_parameters():
        p.requires_grad_(n.endswith("weight") and ("blocks" in n or n.startswith("head")) and p.dim() == 2)
    return m


def _run_steps(model, x, y, steps=2):
    import bench
    from torch.nn.attention import SDPBackend, sdpa_kernel
    opt = torch.optim.SGD([p for p in model.parameters() if p.requires_grad], lr=0.5)
    F = torch.nn.functional
    with sdpa_kernel(SDPBackend.MATH):  # deterministic attention backward
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = F.cross_entropy(model(x).float(), y)
        loss.backward()
        g1 = {n: p.grad.detach().clone() for n, p in model.named_parameters() if p.requires_grad}
        opt.step()
        opt.zero_grad(set_to_none=True)
        bench.train_steps(torch, model, opt, x, y, steps - 1)  # the benchmark's own step loop
    torch.cuda.synchronize()
    w = {n: p.detach().clone() for n, p in model.named_parameters() if p.requires_grad}
    return g1, w


def _exact_worker(rank, world, port, q):
    try:
        import sys
        import torch.distributed as dist
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        g = torch.Generator(device="cuda").manual_seed(7)
        X = torch.randn(32, 3, 32, 32, device="cuda", generator=g)
        Y = torch.randint(0, 10, (32,), device="cuda", generator=g)
        # single-process reference run on the whole batch (the ordinary HLQ path)
        ref_g, ref_w = _run_steps(_tiny_vit(), X, Y)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2406_15102_b200.dp import enable_exact_dp
        model = _tiny_vit()
        names = enable_exact_dp(model)
        assert len(names) == 2 * 4 + 1
        half = 32 // world
        sl = slice(rank * half, (rank + 1) * half)
        g1, w = _run_steps(model, X[sl].contiguous(), Y[sl].contiguous())
        bad = [n for n in ref_g if not torch.equal(g1[n], ref_g[n])]
        badw = [n for n in ref_w if not torch.equal(w[n], ref_w[n])]
        q.put(("ok" if not bad and not badw else "mismatch", rank, bad[:4], badw[:4]))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put(("err", rank, traceback.format_exc()[-1500:]))


def test_exact_dp_training_steps_world2():
    """Two ranks x 16 images == one process x 32 images, bit for bit: the
    step-1 dW of every HLQ layer and the HLQ weights after 2 SGD steps."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exact_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[0] == "ok", r


def _conv_exact_worker(rank, world, port, q):
    try:
        import sys
        import torch.distributed as dist
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        from paper_2406_15102_b200.conv import HLQConv2d
        from paper_2406_15102_b200.dp import enable_exact_dp
        bad = []
        cases = [(3, 16, 3, 1, 1), (16, 32, 3, 2, 1), (32, 64, 3, 1, 1), (16, 16, 1, 2, 0)]
        results = {}
        for ci, (C, O, k, s, p) in enumerate(cases):
            g = torch.Generator(device="cuda").manual_seed(100 + ci)
            X = torch.randn(32, C, 16, 16, device="cuda", generator=g).to(memory_format=torch.channels_last)
            Ho = (16 + 2 * p - k) // s + 1
            G = (torch.randn(32, O, Ho, Ho, device="cuda", generator=g) * 1e-3).to(memory_format=torch.channels_last)
            torch.manual_seed(7)
            m = HLQConv2d(C, O, k, stride=s, padding=p, bias=False).cuda()
            x = X.clone().requires_grad_(True)
            m(x).backward(G)
            results[ci] = (m.weight.grad.clone(), x.grad.clone())
        dist.init_process_group("gloo", rank=rank, world_size=world)
        half = 32 // world
        sl = slice(rank * half, (rank + 1) * half)
        for ci, (C, O, k, s, p) in enumerate(cases):
            g = torch.Generator(device="cuda").manual_seed(100 + ci)
            X = torch.randn(32, C, 16, 16, device="cuda", generator=g).to(memory_format=torch.channels_last)
            Ho = (16 + 2 * p - k) // s + 1
            G = (torch.randn(32, O, Ho, Ho, device="cuda", generator=g) * 1e-3).to(memory_format=torch.channels_last)
            torch.manual_seed(7)
            m = torch.nn.Sequential(HLQConv2d(C, O, k, stride=s, padding=p, bias=False).cuda())
            enable_exact_dp(m)
            x = X[sl].contiguous(memory_format=torch.channels_last).requires_grad_(True)
            # torch mean-loss semantics: a rank's dY is world x its slice of the global one
            m(x).backward(G[sl] * world)
            dw_ref, dx_ref = results[ci]
            if not torch.equal(m[0].weight.grad, dw_ref):
                bad.append(("dW", ci))
            if not torch.equal(x.grad, dx_ref[sl] * world):
                bad.append(("dX", ci))
        q.put(("ok" if not bad else "mismatch", rank, bad))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback
        q.put(("err", rank, traceback.format_exc()[-1500:]))


def test_exact_dp_conv_world2():
    """HLQConv2d in the exact mode: two ranks x 16 images give the one-process
    dW bit for bit (small-C, im2col-TMA, strided and 1x1 convs), dX rows exact."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_conv_exact_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[0] == "ok", r
