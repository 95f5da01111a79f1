"""Pins for oracle.schedule: the three accumulation schedules give the same gradient
(the LGA claim), D ranks x N micro-batches equal 1 rank x D*N, and AdamW matches its
closed form at t=1 and torch.optim.AdamW (fp64) afterwards."""
import numpy as np
import pytest
import torch

import synth
from oracle import model as om
from oracle import schedule as osch


def _setup(L=2, d=16, heads=2, s=6, b=2, N=3, D=2, seed=0, causal=True, post_ln=False):
    sh = synth.Shape(layers=L, d=d, heads=heads, seq=s, micro_batch=b, n_micro=N, dp=D)
    flat = synth.init_params(sh, seed=seed)
    params = [p.astype(np.float64) for p in synth.split_layers(flat, L)]
    X, T = synth.batch(sh, step=0, seed=seed + 10)
    return om.LayerCfg(d=d, heads=heads, causal=causal, post_ln=post_ln), params, X, T


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("causal,post_ln", [(True, False), (False, False), (False, True)])
def test_layered_equals_standard_equals_fullbatch(causal, post_ln):
    cfg, params, X, T = _setup(causal=causal, post_ln=post_ln)
    ls, gs = osch.grads_standard(params, X, T, cfg)
    ll, gl = osch.grads_layered(params, X, T, cfg)
    lf, gf = osch.grads_fullbatch(params, X, T, cfg)
    assert abs(ls - ll) < 1e-14 * abs(ls) and abs(ls - lf) < 1e-13 * abs(ls)
    assert abs(ls - osch.loss(params, X, T, cfg)) < 1e-14 * abs(ls)
    for a, b_, c in zip(gs, gl, gf):
        assert _rel(b_, a) < 1e-13
        assert _rel(c, a) < 1e-12


def test_d_ranks_times_n_equals_one_rank_times_dn():
    cfg, params, X, T = _setup(D=2, N=2)
    D, N = X.shape[:2]
    X1 = X.reshape(1, D * N, *X.shape[2:])
    T1 = T.reshape(1, D * N, *T.shape[2:])
    l2, g2 = osch.grads_layered(params, X, T, cfg)
    l1, g1 = osch.grads_layered(params, X1, T1, cfg)
    assert abs(l1 - l2) < 1e-14 * abs(l1)
    for a, b_ in zip(g1, g2):
        assert _rel(b_, a) < 1e-13


def test_gradient_is_mean_over_microbatches():
    """Reading A-3: the step gradient is the gradient of the mean micro-batch loss, so
    duplicating every micro-batch leaves it unchanged."""
    cfg, params, X, T = _setup(D=1, N=2)
    _, g = osch.grads_standard(params, X, T, cfg)
    X2 = np.concatenate([X, X], axis=1)
    T2 = np.concatenate([T, T], axis=1)
    _, g2 = osch.grads_standard(params, X2, T2, cfg)
    for a, b_ in zip(g, g2):
        assert _rel(b_, a) < 1e-14


def test_adamw_first_step_closed_form():
    """t = 1, wd = 0: bias corrections cancel, theta1 = theta0 - lr * g / (|g| + eps)."""
    rng = np.random.default_rng(0)
    th = rng.standard_normal(100)
    g = rng.standard_normal(100) * 1e-3
    opt = osch.AdamW(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8)
    st = opt.init_state(th)
    th1 = opt.update(th, g, st)
    np.testing.assert_allclose(th1, th - 1e-3 * g / (np.abs(g) + 1e-8), rtol=1e-14, atol=1e-16)


def test_adamw_matches_torch_fp64():
    rng = np.random.default_rng(1)
    th = rng.standard_normal(257)
    opt = osch.AdamW(lr=3e-3, beta1=0.8, beta2=0.9, eps=1e-6, weight_decay=0.1)
    st = opt.init_state(th)
    tt = torch.nn.Parameter(torch.from_numpy(th.copy()))
    topt = torch.optim.AdamW([tt], lr=3e-3, betas=(0.8, 0.9), eps=1e-6, weight_decay=0.1)
    for _ in range(5):
        g = rng.standard_normal(257)
        th = opt.update(th, g, st)
        tt.grad = torch.from_numpy(g.copy())
        topt.step()
    np.testing.assert_allclose(th, tt.detach().numpy(), rtol=1e-13, atol=1e-15)


def test_train_steps_schedules_agree():
    cfg, params, X, T = _setup(L=2, d=8, heads=2, s=4, b=1, N=2, D=1)
    sh = synth.Shape(layers=2, d=8, heads=2, seq=4, micro_batch=1, n_micro=2)
    batches = [synth.batch(sh, step=k) for k in range(3)]
    opt = osch.AdamW(lr=1e-2)
    ps, ls, _ = osch.train_steps(params, batches, cfg, opt, "standard")
    pl, ll, _ = osch.train_steps(params, batches, cfg, opt, "layered")
    np.testing.assert_allclose(ls, ll, rtol=1e-13)
    for a, b_ in zip(ps, pl):
        np.testing.assert_allclose(b_, a, rtol=1e-10, atol=1e-14)
    assert ls[2] < ls[0]   # the optimiser descends on a fixed-target regression


def test_round_bf16_is_round_to_nearest_even():
    """Mixed precision (reading A-9): the 16-bit weight copy is round-to-nearest-even of fp32.  Closed
    forms at the halfway points of [1, 2) (bf16 ulp 2^-7) and a library routine (torch's bfloat16 cast) on
    values across the exponent range."""
    h = 2.0 ** -8   # half an ulp in [1, 2)
    cases = {1.0: 1.0, 1.0 + h: 1.0, 1.0 + 3 * h: 1.0 + 4 * h, 1.0 + 0.9 * h: 1.0, 1.0 + 1.1 * h: 1.0 + 2 * h,
             -(1.0 + h): -1.0, 2.0 ** -130: 2.0 ** -130, 0.0: 0.0}
    for x, want in cases.items():
        assert osch.round_bf16(np.array([x]))[0] == want, x
    rng = np.random.default_rng(0)
    v = (rng.standard_normal(100_000) * np.exp2(rng.integers(-60, 60, 100_000))).astype(np.float32)
    b = osch.round_bf16(v[:1000])                       # bf16 values; exactly halfway to the next one up:
    ties = (b + np.sign(b) * np.exp2(np.frexp(b)[1] - 9.0)).astype(np.float32)   # ulp = 2^(e-8), frexp e = exp+1
    for a in (v, ties):
        ref = torch.from_numpy(a).bfloat16().double().numpy()
        np.testing.assert_array_equal(osch.round_bf16(a), ref)


def test_train_steps_mixed_precision_is_gradient_at_rounded_weights():
    """param_round="bf16" evaluates the gradient at the rounded weights and updates the stored ones: with weights
    already representable in bf16 it changes nothing; otherwise its first gradient is the plain gradient at
    round_bf16(theta) while the update is applied to theta itself."""
    cfg, params, X, T = _setup(L=2, d=8, heads=2, s=4, b=1, N=2, D=1)
    opt = osch.AdamW(lr=1e-2)
    rp = [osch.round_bf16(p) for p in params]
    a = osch.train_steps(rp, [(X, T)], cfg, opt, param_round="bf16")
    b = osch.train_steps(rp, [(X, T)], cfg, opt)
    for x, y in zip(a[0], b[0]):
        np.testing.assert_array_equal(x, y)
    new, losses, grads = osch.train_steps(params, [(X, T)], cfg, opt, param_round="bf16")
    l_ref, g_ref = osch.grads_standard(rp, X, T, cfg)
    assert losses[0] == l_ref
    for g, gr, p, n in zip(grads, g_ref, params, new):
        np.testing.assert_array_equal(g, gr)
        # first AdamW step moves theta (not its rounded copy) by lr g / (|g| + eps)
        np.testing.assert_allclose(n, p - 1e-2 * gr / (np.abs(gr) + 1e-8), rtol=1e-12, atol=1e-15)
    assert any(np.any(p != q) for p, q in zip(params, rp))   # the parity init is not bf16-representable
