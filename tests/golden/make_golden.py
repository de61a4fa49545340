"""Generate golden vectors for the HLQ path by running the REFERENCE itself.

Run in the build container (the reference tree is only mounted there):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src, runs
its public functions (and the stage helpers those functions call) on small
seeded inputs, and writes one ``.npz`` per case next to this script.  The
fixtures are committed; nothing at test / bench time reads /root/reference.

Stored per case (names match oracle/hlq_oracle.py's ``stages`` keys):
  x, w, gy                inputs (x/gy as the reference's (B, L, C) views)
  gx_codes_g, gx_scale_g  Q_bits_gx(HT_O(gy))         backprop.py:362,367
  gx_codes_w, gx_scale_w  Q_bits_gx(HT_O(W))          backprop.py:363,368
  gx_acc                  int_matmul accumulator     quantize.py:176
  x_codes, x_scale, axis  ACBP payload of X          backprop.py:373-385
  gw_codes_g, gw_scale_g  Q8(P gy)^T                 backprop.py:401-407
  gw_acc                  int_matmul accumulator     quantize.py:176
  gx, gw                  hlq_backward outputs        backprop.py:438-447
Conv cases additionally store the reference Conv2d.backward dX / dW.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF_SRC)
    import hlq  # noqa: F401
    from hlq import backprop, quantize
    from hlq.harness import layers
    return hlq, backprop, quantize, layers


def _inputs(seed, B, L, I, O, heavy=True):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((B, L, I)).astype(np.float32)
    w = (rng.standard_normal((O, I)) * np.sqrt(2.0 / I)).astype(np.float32)
    if heavy:
        gy = (rng.lognormal(0.0, 1.4, size=(B, L, O)) * rng.choice([-1.0, 1.0], size=(B, L, O))
              * 1e-3).astype(np.float32)
    else:
        gy = rng.standard_normal((B, L, O)).astype(np.float32)
    return x, w, gy


def linear_case(name, seed, B, L, I, O, rank=8, bits_gx=4, bits_gw=8, pad_small=False,
                bases=None, heavy=True, x=None, w=None, gy=None):
    hlq, bp, qz, _ = _ref()
    if x is None:
        x, w, gy = _inputs(seed, B, L, I, O, heavy)
    plan = hlq.HadamardPlan(block_size=16, basis_indices=(
        hlq.hadamard.lowest_sequency_bases(16, rank) if bases is None else tuple(bases)))
    strat = hlq.BackwardStrategy("hlq", hlq.PathSpec("ht_quant", bits_gx),
                                 hlq.PathSpec("lowrank_quant", bits_gw), plan,
                                 pad_small_axes=pad_small)
    X, Wt, G = hlq.Tensor(x), hlq.Tensor(w), hlq.Tensor(gy)
    acbp = hlq.acbp_compress(X, plan, bits=bits_gw, pad_small_axes=pad_small)
    gp = hlq.hlq_backward(acbp, Wt, G, strategy=strat)
    # stage captures through the reference's own helpers
    full = hlq.HadamardPlan(block_size=16, basis_indices=tuple(range(16)))
    ghat = bp._block_axis(gy, 2, full)
    what = bp._block_axis(w, 0, full)
    qg = qz.quant_pseudo_stochastic(hlq.Tensor(ghat.reshape(-1, ghat.shape[-1])), bits_gx)
    qw = qz.quant_pseudo_stochastic(hlq.Tensor(what), bits_gx)
    gx_acc, _ = qz.int_matmul(qg, qw)
    gproj = bp._project_axis(gy, acbp.axis, plan).reshape(-1, O)
    qgw = qz.quant_pseudo_stochastic(hlq.Tensor(np.ascontiguousarray(gproj.T)), bits_gw)
    gw_acc, _ = qz.int_matmul(qgw, qz.QuantizedTensor(
        payload=acbp.quantized.payload.reshape(-1, I), bits=bits_gw,
        scale=acbp.quantized.scale))
    out = dict(
        x=x, w=w, gy=gy,
        rank=np.int64(plan.rank), bases=np.array(plan.basis_indices, dtype=np.int64),
        bits_gx=np.int64(bits_gx), bits_gw=np.int64(bits_gw), pad_small=np.int64(pad_small),
        gx_codes_g=qg.payload, gx_scale_g=np.float32(qg.scale),
        gx_codes_w=qw.payload, gx_scale_w=np.float32(qw.scale), gx_acc=gx_acc,
        x_codes=acbp.quantized.payload.reshape(-1, I), x_scale=np.float32(acbp.quantized.scale),
        axis=np.int64(acbp.axis),
        gw_codes_g=qgw.payload, gw_scale_g=np.float32(qgw.scale), gw_acc=gw_acc,
        gx=gp.grad_input.data, gw=gp.grad_weight.data,
    )
    # the raw-x branch must agree bit-for-bit (test_backprop.py:338-345)
    gp_raw = hlq.hlq_backward(X, Wt, G, strategy=strat)
    assert np.array_equal(gp_raw.grad_input.data, out["gx"])
    assert np.array_equal(gp_raw.grad_weight.data, out["gw"])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    return name


def stochastic_case(name, seed, B, L, I, O, rng_seed, rank=8, bits_gx=4, bits_gw=8):
    """True stochastic rounding (quantize.py:114-125) through the reference's
    own RngState / _quant tags, raw-x branch of hlq_backward."""
    hlq, bp, qz, _ = _ref()
    x, w, gy = _inputs(seed, B, L, I, O)
    plan = hlq.HadamardPlan(block_size=16, basis_indices=hlq.hadamard.lowest_sequency_bases(16, rank))
    strat = hlq.BackwardStrategy("hlq", hlq.PathSpec("ht_quant", bits_gx),
                                 hlq.PathSpec("lowrank_quant", bits_gw), plan)
    rng = qz.RngState(rng_seed)
    X, Wt, G = hlq.Tensor(x), hlq.Tensor(w), hlq.Tensor(gy)
    gp = hlq.hlq_backward(X, Wt, G, strategy=strat, rng=rng)
    acbp = hlq.acbp_compress(X, plan, bits=bits_gw, rng=rng)
    full = hlq.HadamardPlan(block_size=16, basis_indices=tuple(range(16)))
    ghat = bp._block_axis(gy, 2, full)
    what = bp._block_axis(w, 0, full)
    qg = bp._quant(hlq.Tensor(ghat.reshape(-1, ghat.shape[-1])), bits_gx, rng, bp._TAG_GX_LEFT)
    qw = bp._quant(hlq.Tensor(what), bits_gx, rng, bp._TAG_GX_RIGHT)
    gproj = bp._project_axis(gy, acbp.axis, plan).reshape(-1, O)
    qgw = bp._quant(hlq.Tensor(np.ascontiguousarray(gproj.T)), bits_gw, rng, bp._TAG_GW_LEFT)
    out = dict(
        x=x, w=w, gy=gy, rng_seed=np.uint64(rng_seed),
        rank=np.int64(plan.rank), bases=np.array(plan.basis_indices, dtype=np.int64),
        bits_gx=np.int64(bits_gx), bits_gw=np.int64(bits_gw), pad_small=np.int64(0),
        gx_codes_g=qg.payload, gx_scale_g=np.float32(qg.scale),
        gx_codes_w=qw.payload, gx_scale_w=np.float32(qw.scale),
        x_codes=acbp.quantized.payload.reshape(-1, I), x_scale=np.float32(acbp.quantized.scale),
        axis=np.int64(acbp.axis),
        gw_codes_g=qgw.payload, gw_scale_g=np.float32(qgw.scale),
        gx=gp.grad_input.data, gw=gp.grad_weight.data,
    )
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    return name


def container_case(name, seed, B, L, I, bits=8, bases=(0, 2, 4, 6, 8, 10, 12, 14), pad_small=False):
    """ACBP container bytes (acbp.py:76-96) of a reference-compressed activation."""
    hlq, bp, qz, _ = _ref()
    from hlq import acbp as acbp_mod
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((B, L, I)).astype(np.float32)
    plan = hlq.HadamardPlan(block_size=16, basis_indices=tuple(bases))
    a = hlq.acbp_compress(hlq.Tensor(x), plan, bits=bits, pad_small_axes=pad_small)
    buf = acbp_mod.acbp_pack(a)
    back = acbp_mod.acbp_unpack(buf)
    assert np.array_equal(back.quantized.payload, a.quantized.payload)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), x=x, bases=np.array(bases, dtype=np.int64),
                        bits=np.int64(bits), pad_small=np.int64(pad_small), axis=np.int64(a.axis),
                        payload=a.quantized.payload, scale=np.float32(a.quantized.scale),
                        container=np.frombuffer(buf, dtype=np.uint8).copy())
    return name


def calib_case(name, seed, B, L, O, rank=8):
    """Calibrated basis selection (train.py:128-134 _basis_energy, hadamard.py:174-188)."""
    hlq, bp, qz, _ = _ref()
    import importlib
    tr = importlib.import_module("hlq.harness.train")
    rng = np.random.default_rng(seed)
    gy = (rng.lognormal(0.0, 1.4, size=(B, L, O)) * rng.choice([-1.0, 1.0], size=(B, L, O)) * 1e-3)
    gy = gy.astype(np.float32)
    # give the bases distinct energies: add a smooth (low-sequency) component along L
    gy += (np.sin(np.arange(L) / 3.0)[None, :, None] * 2e-3).astype(np.float32)
    axis = bp.ht_axis_for(B, L, 16)
    energy = tr._basis_energy(gy, axis, 16)
    bases = hlq.hadamard.select_bases(hlq.Tensor(energy), rank)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), gy=gy, axis=np.int64(axis), rank=np.int64(rank),
                        means=np.abs(energy).mean(axis=0), bases=np.array(bases, dtype=np.int64))
    return name


def conv_case(name, seed, B, C, H, W, O, k, s, p, rank=8):
    hlq, bp, qz, layers = _ref()
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((B, C, H, W)).astype(np.float32)
    conv = layers.Conv2d(C, O, kernel=k, stride=s, pad=p, bias=False, rng=rng)
    strat = hlq.BackwardStrategy.hlq(rank=rank)
    y = conv.forward(x, strategy=strat)
    gy = (rng.lognormal(0.0, 1.4, size=y.shape) * rng.choice([-1.0, 1.0], size=y.shape)
          * 1e-3).astype(np.float32)
    acbp = conv._ctx
    dx = conv.backward(gy, strat)
    dw = conv.grad_w
    # stage captures on the lowered (B, L, I) problem
    Ho, Wo = y.shape[2], y.shape[3]
    gy3 = np.ascontiguousarray(gy.transpose(0, 2, 3, 1).reshape(B, Ho * Wo, O))
    full = hlq.HadamardPlan(block_size=16, basis_indices=tuple(range(16)))
    ghat = bp._block_axis(gy3, 2, full)
    what = bp._block_axis(conv.w, 0, full)
    qg = qz.quant_pseudo_stochastic(hlq.Tensor(ghat.reshape(-1, ghat.shape[-1])), 4)
    qw = qz.quant_pseudo_stochastic(hlq.Tensor(what), 4)
    gx_acc, _ = qz.int_matmul(qg, qw)
    I = conv.w.shape[1]
    gproj = bp._project_axis(gy3, acbp.axis, strat.plan).reshape(-1, O)
    qgw = qz.quant_pseudo_stochastic(hlq.Tensor(np.ascontiguousarray(gproj.T)), 8)
    gw_acc, _ = qz.int_matmul(qgw, qz.QuantizedTensor(
        payload=acbp.quantized.payload.reshape(-1, I), bits=8, scale=acbp.quantized.scale))
    out = dict(
        x=x, w=conv.w.reshape(O, C, k, k), gy=gy, k=np.int64(k), stride=np.int64(s),
        pad=np.int64(p), rank=np.int64(rank),
        bases=np.array(strat.plan.basis_indices, dtype=np.int64),
        gx_codes_g=qg.payload, gx_scale_g=np.float32(qg.scale),
        gx_codes_w=qw.payload, gx_scale_w=np.float32(qw.scale), gx_acc=gx_acc,
        x_codes=acbp.quantized.payload.reshape(-1, I), x_scale=np.float32(acbp.quantized.scale),
        axis=np.int64(acbp.axis),
        gw_codes_g=qgw.payload, gw_scale_g=np.float32(qgw.scale), gw_acc=gw_acc,
        gx=dx, gw=dw.reshape(O, C, k, k),
    )
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    return name


def known_answer_cases():
    """Reference known-answer tests restated as fixtures (test_backprop.py:249-264)."""
    hlq, _, _, _ = _ref()
    names = []
    x = np.full((2, 16, 3), 31.75, dtype=np.float32)
    a = hlq.acbp_compress(hlq.Tensor(x), hlq.HadamardPlan(), bits=8)
    np.savez_compressed(os.path.join(HERE, "ka_constant.npz"), x=x,
                        x_codes=a.quantized.payload.reshape(-1, 3),
                        x_scale=np.float32(a.quantized.scale), axis=np.int64(a.axis))
    names.append("ka_constant")
    x = np.zeros((2, 16, 4), dtype=np.float32)
    a = hlq.acbp_compress(hlq.Tensor(x), hlq.HadamardPlan(), bits=8)
    np.savez_compressed(os.path.join(HERE, "ka_zero.npz"), x=x,
                        x_codes=a.quantized.payload.reshape(-1, 4),
                        x_scale=np.float32(a.quantized.scale), axis=np.int64(a.axis))
    names.append("ka_zero")
    # quantizer lattice (test_quantize.py:85-88) and a lognormal vector
    t = np.arange(-7, 8, dtype=np.float32)
    q = hlq.quant_pseudo_stochastic(hlq.Tensor(t), 4)
    rng = np.random.default_rng(31)
    ln = (rng.lognormal(1.0, 1.0, size=4096) * rng.choice([-1.0, 1.0], size=4096)).astype(np.float32)
    q8 = hlq.quant_pseudo_stochastic(hlq.Tensor(ln), 8)
    q4 = hlq.quant_pseudo_stochastic(hlq.Tensor(ln), 4)
    np.savez_compressed(os.path.join(HERE, "ka_quant.npz"), lattice=t, lattice_codes=q.payload,
                        lattice_scale=np.float32(q.scale), ln=ln, ln_codes8=q8.payload,
                        ln_scale8=np.float32(q8.scale), ln_codes4=q4.payload,
                        ln_scale4=np.float32(q4.scale))
    names.append("ka_quant")
    # default basis sets for every rank (hadamard.py:24-49)
    bases = {str(r): list(hlq.hadamard.lowest_sequency_bases(16, r)) for r in range(1, 17)}
    with open(os.path.join(HERE, "bases16.json"), "w") as f:
        json.dump(bases, f, indent=0)
    return names


def baseline_case(name, seed, B, L, I, O, preset, rng_seed=None, pad_small=False, **kw):
    """A baseline strategy (backprop.py:91-155: vanilla, naive int4/int8, HQ,
    LBP-WHT, float pipelines, mixed modes) through the reference's
    strategy_backward on the raw activation."""
    hlq, bp, qz, _ = _ref()
    x, w, gy = _inputs(seed, B, L, I, O)
    S = hlq.BackwardStrategy
    if preset == "custom":
        strat = S("custom", hlq.PathSpec(*kw["gx"]), hlq.PathSpec(*kw["gw"]),
                  hlq.HadamardPlan(block_size=16, basis_indices=hlq.hadamard.lowest_sequency_bases(
                      16, kw.get("rank", 8))))
    else:
        base, _, variant = preset.partition(".")
        strat = getattr(S, base)(**kw)
        if variant:
            strat = getattr(strat, variant)()
    if pad_small:
        import dataclasses
        strat = dataclasses.replace(strat, pad_small_axes=True)
    rng = qz.RngState(rng_seed) if rng_seed is not None else None
    gp = hlq.strategy_backward(hlq.Tensor(x), hlq.Tensor(w), hlq.Tensor(gy), strat, rng=rng)
    gx_spec, gw_spec = strat.grad_input_path, strat.grad_weight_path
    out = dict(x=x, w=w, gy=gy, preset=np.array(preset),
               gx_mode=np.array(gx_spec.mode), gx_bits=np.int64(gx_spec.bits or 0),
               gw_mode=np.array(gw_spec.mode), gw_bits=np.int64(gw_spec.bits or 0),
               bases=np.array(strat.plan.basis_indices, dtype=np.int64), pad_small=np.int64(pad_small),
               rng_seed=np.int64(-1 if rng_seed is None else rng_seed),
               gx=gp.grad_input.data, gw=gp.grad_weight.data)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    return name


def main():
    made = []
    # 2-D Linear convention (layers.py:87): L = 1, projection along B.
    made.append(linear_case("lin2d_r8", 1, 64, 1, 48, 40))
    made.append(linear_case("lin2d_r2", 2, 64, 1, 48, 40, rank=2))
    made.append(linear_case("lin2d_b100", 3, 100, 1, 32, 32))      # non-pow2 B, ragged block
    # 3-D, projection along L within each sample; ragged L and O
    made.append(linear_case("lin3d_L37", 4, 3, 37, 24, 20))
    made.append(linear_case("lin3d_L197", 5, 2, 197, 40, 48))     # ViT token count
    made.append(linear_case("lin3d_r4", 6, 4, 32, 64, 96, rank=4))
    # L < 16 <= B: batch axis with L > 1
    made.append(linear_case("lin3d_batchaxis", 7, 32, 4, 8, 16))
    # both small: needs pad_small_axes
    made.append(linear_case("lin3d_padsmall", 8, 4, 8, 16, 16, pad_small=True))
    # warmup precision (backprop.py:139-148): 8-bit gx
    made.append(linear_case("lin_warmup8", 9, 2, 48, 32, 32, bits_gx=8))
    # calibrated (non-default) basis set (hadamard.py:174-188 output)
    made.append(linear_case("lin_bases", 10, 2, 32, 16, 24, bases=(0, 1, 3, 4, 7, 9, 10, 14)))
    made.append(linear_case("lin_full16", 11, 2, 32, 16, 24, rank=16))
    made.append(linear_case("lin_normal", 12, 256, 1, 64, 96, heavy=False))
    # zero gy / zero W edge cases
    x, w, gy = _inputs(13, 2, 16, 8, 16)
    made.append(linear_case("lin_zero_gy", 0, 2, 16, 8, 16, x=x, w=w, gy=np.zeros_like(gy)))
    made.append(linear_case("lin_zero_w", 0, 2, 16, 8, 16, x=x, w=np.zeros_like(w), gy=gy))
    # conv lowering (layers.py:96-158)
    made.append(conv_case("conv_k3s1p1", 20, 2, 8, 6, 6, 16, 3, 1, 1))
    made.append(conv_case("conv_k3s2p1", 21, 2, 8, 9, 9, 24, 3, 2, 1))
    made.append(conv_case("conv_k1s2p0", 22, 3, 16, 8, 8, 8, 1, 2, 0))
    made.append(conv_case("conv_k3s1p1_14", 23, 2, 16, 14, 14, 16, 3, 1, 1))
    made += known_answer_cases()
    # true stochastic rounding (rng=RngState(seed)): tokens axis and batch axis
    made.append(stochastic_case("stoch_lin3d", 40, 2, 37, 24, 40, rng_seed=0x1234ABCD))
    made.append(stochastic_case("stoch_lin2d", 41, 48, 1, 32, 24, rng_seed=7))
    # ACBP containers (acbp.py): int8 / int4 (odd count -> padding nibble), batch axis,
    # padded L, pad-small axes, empty batch
    # baseline strategies
    made.append(baseline_case("base_vanilla", 60, 4, 40, 48, 36, "vanilla"))
    made.append(baseline_case("base_int4", 61, 4, 40, 48, 36, "naive_quant", bits=4))
    made.append(baseline_case("base_int8", 62, 3, 37, 24, 20, "naive_quant", bits=8))
    made.append(baseline_case("base_int4_rng", 63, 4, 40, 48, 36, "naive_quant", rng_seed=99, bits=4))
    made.append(baseline_case("base_hq", 64, 4, 40, 48, 36, "hq"))
    made.append(baseline_case("base_hq8", 65, 3, 37, 24, 20, "hq", bits_gx=8, bits_gw=8))
    made.append(baseline_case("base_hq_rng", 66, 3, 37, 24, 20, "hq", rng_seed=5))
    made.append(baseline_case("base_hq_batch", 67, 32, 5, 16, 24, "hq"))
    made.append(baseline_case("base_lbp", 68, 3, 37, 24, 20, "lbp_wht"))
    made.append(baseline_case("base_lbp_r4", 69, 4, 40, 48, 36, "lbp_wht", rank=4))
    made.append(baseline_case("base_lbp_batch", 70, 20, 3, 16, 24, "lbp_wht"))
    made.append(baseline_case("base_lbp_padsmall", 71, 5, 7, 16, 8, "lbp_wht", pad_small=True))
    made.append(baseline_case("base_hlq_float", 72, 3, 37, 24, 20, "hlq.float_pipeline"))
    made.append(baseline_case("base_hlq_exact", 73, 3, 37, 24, 20, "hlq.debug_exact"))
    made.append(baseline_case("base_hq_float", 74, 4, 40, 48, 36, "hq.float_pipeline"))
    made.append(baseline_case("base_mix_q8_hlq", 75, 3, 37, 24, 20, "custom", gx=("quant", 8),
                              gw=("lowrank_quant", 8)))
    made.append(baseline_case("base_mix_lr_fp", 76, 4, 40, 48, 36, "custom", gx=("lowrank",), gw=("fp",)))
    made.append(container_case("acbp_c8", 50, 4, 32, 12))
    made.append(container_case("acbp_c4_odd", 51, 1, 16, 5, bits=4, bases=(0, 1, 2)))
    made.append(container_case("acbp_c4", 52, 3, 40, 7, bits=4))
    made.append(container_case("acbp_batchaxis", 53, 32, 4, 8))
    made.append(container_case("acbp_padL", 54, 4, 20, 12))
    made.append(container_case("acbp_padsmall", 55, 4, 8, 6, pad_small=True))
    made.append(container_case("acbp_empty", 56, 0, 32, 8))
    # calibrated basis selection
    made.append(calib_case("calib_tokens", 60, 4, 48, 40))
    made.append(calib_case("calib_batch", 61, 64, 1, 24, rank=4))
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as f:
        json.dump({"generated_by": "tests/golden/make_golden.py",
                   "reference": "/root/reference/pkg/src/hlq (read-only, build container)",
                   "cases": made}, f, indent=1)
    print("wrote", len(made), "fixtures")


if __name__ == "__main__":
    main()
