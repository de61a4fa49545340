"""Lazy non-finite detection in the training path (quantize.py:119-120,138-139:
the reference raises ValueError on NaN / Inf).  The transform kernels set a
per-device sticky flag; nothing synchronises per layer; the check runs where
the caller installs it (here: optimizer.step)."""
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def mods():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2406_15102_b200 import layers, nonfinite
    return layers, nonfinite


def _model(layers):
    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.GELU(), torch.nn.Linear(256, 64)).to(DEV)
    return layers.convert_linears(net)


def test_inf_in_gy_raises_at_optimizer_step(mods):
    layers, nonfinite = mods
    net = _model(layers)
    opt = torch.optim.SGD(net.parameters(), lr=0.1)
    nonfinite.check_nonfinite()  # clear anything an earlier test left
    guard = nonfinite.install_nonfinite_check(opt)
    x = torch.randn(8, 197, 64, device=DEV)
    # clean step: no error, parameters move
    w0 = net[0].weight.detach().clone()
    net(x).square().mean().backward()
    opt.step()
    opt.zero_grad()
    assert not torch.equal(w0, net[0].weight)
    # an Inf injected into the upstream gradient of the second layer
    y = net(x)
    y.register_hook(lambda g: g.index_put((torch.tensor([1]), torch.tensor([3]), torch.tensor([5])),
                                          torch.tensor(float("inf"), device=DEV)))
    y.square().mean().backward()
    w1 = net[0].weight.detach().clone()
    with pytest.raises(ValueError):
        opt.step()
    assert torch.equal(w1, net[0].weight), "the step must not apply non-finite gradients"
    opt.zero_grad()
    # the flag was reset by the check: the next clean step goes through
    net(x).square().mean().backward()
    opt.step()
    assert guard is not None


def test_nan_weight_sets_flag(mods):
    layers, nonfinite = mods
    net = _model(layers)
    nonfinite.check_nonfinite()
    with torch.no_grad():
        net[2].weight[0, 0] = float("nan")
    net(torch.randn(4, 32, 64, device=DEV)).sum().backward()
    with pytest.raises(ValueError):
        nonfinite.check_nonfinite()
    nonfinite.check_nonfinite()  # reset: no error now


def test_fetch_is_asynchronous(mods):
    _, nonfinite = mods
    g = nonfinite.NonFiniteGuard()
    torch.cuda._sleep(50_000_000)
    g.fetch()  # only enqueued behind the spin: the host does not wait
    assert not g.event.query()
    g.check()
