"""CUDA-graph capture of an HLQ training step: the library-owned statistics
slots (captured once, re-zeroed by every replay's kernels) and the
programmatic dependent launches (captured as programmatic edges) must give
the eager step's gradients bit for bit, replay after replay, and leave the
eager path correct afterwards."""
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def mods():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2406_15102_b200 import _lib, layers
    assert _lib.load().hlq_device_ok() == 1
    return layers


def _model(layers):
    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.GELU(), torch.nn.Linear(512, 256)).to(DEV)
    return layers.convert_linears(net)


def _step(net, x, gy):
    with torch.autocast("cuda", dtype=torch.bfloat16):
        y = net(x)
    y.backward(gy)


def test_graph_replays_match_eager(mods):
    net = _model(mods)
    x = torch.randn(4, 64, 256, device=DEV)
    gy = (torch.randn(4, 64, 256, device=DEV) * 1e-3).to(torch.bfloat16)
    _step(net, x, gy)  # eager reference
    ref = [p.grad.clone() for p in net.parameters()]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            for p in net.parameters():
                p.grad = None
            _step(net, x, gy)
    torch.cuda.current_stream().wait_stream(s)
    for p in net.parameters():
        p.grad = None
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        _step(net, x, gy)
    grads = [p.grad for p in net.parameters()]
    for _ in range(80):  # more replays than the 64-slot ring
        g.replay()
    torch.cuda.synchronize()
    for a, b in zip(grads, ref):
        assert torch.equal(a, b)
    # eager after the graph (the ring has moved on) is still exact
    for p in net.parameters():
        p.grad = None
    _step(net, x, gy)
    torch.cuda.synchronize()
    for p, b in zip(net.parameters(), ref):
        assert torch.equal(p.grad, b)
